// L-BFGS maximum-likelihood fit of (sigma2, sigma1_2, rho) on the device FSA core; see fit.cpp.
#pragma once

#include <functional>
#include <vector>

namespace fsa {

struct Context;

// LbfgsOptions (estimation.h:14-21)
struct LbfgsOptions {
  int max_evals = 200;
  double grad_tol = 1e-6;  // infinity norm (fit_fsa overrides it with grad_tol_per_n * n)
  int memory = 6;
  double armijo_c1 = 1e-4;
  int max_backtracks = 30;
  double f_rel_tol = 1e-10;
};
struct LbfgsResult {
  std::vector<double> x, grad;
  double f = 0.0;
  int evals = 0;
  bool converged = false;
};
// the objective may throw NumericalError (treated as +inf by the line search)
LbfgsResult lbfgs_minimize(const std::function<double(const std::vector<double>&, std::vector<double>&)>& fn,
                           std::vector<double> x0, const LbfgsOptions& opts);

// FitOptions (estimation.h:47-63), iterative backend
struct FitOptions {
  int nu = 1;      // 0: 1/2, 1: 3/2, 2: 5/2
  int family = 1;  // wendland1 / wendland2
  long num_inducing = 200;
  double taper_range = 0.0;  // 0: from target_row_nnz
  double target_row_nnz = 40.0;
  int precond = 2;  // 0 none, 1 diagonal, 2 fitc
  int num_probes = 50;
  int cv_mode = 2;  // 0 none, 1 one, 2 optimal
  unsigned long long seed = 0;
  double cg_tol = 1e-3;
  int cg_max_iter = 1000;
  double jitter_rel = 1e-10;
  int kmeans_max_iter = 20;
  double kmeans_rel_tol = 1e-4;
  LbfgsOptions lbfgs;
  double grad_tol_per_n = 1e-3;
};
// FitResult (estimation.h:65-74)
struct FitOutput {
  double sigma2 = 0.0, sigma1_2 = 0.0, rho = 0.0, nll = 0.0, gamma = 0.0;
  std::vector<double> beta, inducing, nll_trace, grad_log;
  int evals = 0;
  bool converged = false;
};
FitOutput fit_fsa(Context* ctx, const double* coords, long n, int d, const double* y, const double* X, long p,
                  const FitOptions& opts);

}  // namespace fsa
