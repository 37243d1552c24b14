// fsagp_b200.hpp — header-only C++ shim re-creating the reference's fsagp
// signatures (/root/reference/proj/include/fsagp) over the C ABI in fsa_b200.h.
//
// Eigen is not required: dense arguments are column-major std::vector<double>
// (the layout of fsagp::den_mat_t), vectors are std::vector<double>. Errors
// re-throw as std::invalid_argument and fsagp_b200::NumericalError, mirroring
// fsagp::require / fsagp::NumericalError (types.h:22-29), so a caller that
// catches NumericalError as an L-BFGS line-search barrier (estimation.cpp:18-26)
// keeps working.
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "fsa_b200.h"

namespace fsagp_b200 {

struct NumericalError : std::runtime_error {
  explicit NumericalError(const std::string& w) : std::runtime_error(w) {}
};

inline void check(int rc) {
  if (rc == FSA_OK) return;
  const std::string msg = fsa_last_error();
  if (rc == FSA_EINVAL) throw std::invalid_argument(msg);
  if (rc == FSA_ENUMERIC) throw NumericalError(msg);
  throw std::runtime_error("fsa_b200: " + msg);
}

enum class MaternNu { nu_1_2 = 0, nu_3_2 = 1, nu_5_2 = 2 };     // types.h:32
enum class TaperFamily { wendland1 = 1, wendland2 = 2 };          // types.h:50
enum class PrecondType { none = 0, diagonal = 1, fitc = 2 };      // estimation.h:57
enum class CvMode { none = 0, one = 1, optimal = 2 };             // krylov.h:87

struct CovParams {  // types.h:74-78 (sigma2 = nugget, sigma1_2 = marginal variance)
  double sigma2 = 1.0, sigma1_2 = 1.0, rho = 0.1;
};
struct CgOptions {  // krylov.h:28-32
  double tol = 1e-3;
  int max_iter = 1000;
  bool error_on_max_iter = false;
  fsa_cg_options c() const { return {tol, max_iter, error_on_max_iter ? 1 : 0}; }
};
struct IterativeNllOptions {  // estimation.h:84-89
  int num_probes = 50;
  std::uint64_t seed = 0;
  CgOptions cg;
  CvMode cv = CvMode::optimal;
};
struct IterativeNll {  // estimation.h:91-97
  double nll = 0.0;
  std::array<double, 3> grad{};
  std::vector<double> beta;
  int cg_iterations = 0;
  double logdet = 0.0;
};
struct SimVarOptions {  // prediction.h:43-50
  int num_probes = 1000;
  std::uint64_t seed = 0;
  CgOptions cg, cg_s;
  bool control_variate = false;
  double floor_rel = 1e-6;
};
struct PredVarResult {  // prediction.h:37-42
  std::vector<double> var, se;
  int clamped = 0;
  int cg_iterations = 0;
};

class Context {
 public:
  explicit Context(int device = 0) { check(fsa_ctx_create(device, &h_)); }
  ~Context() { fsa_ctx_destroy(h_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  fsa_ctx* get() const { return h_; }

 private:
  fsa_ctx* h_ = nullptr;
};

// FsaModel (fsa.h:40-104). coords: n x d, inducing: m x d, column-major.
class FsaModel {
 public:
  static std::unique_ptr<FsaModel> assemble(Context& ctx, const std::vector<double>& coords, std::int64_t n, int d,
                                            const std::vector<double>& inducing, std::int64_t m, MaternNu nu,
                                            TaperFamily family, double gamma, const CovParams& p,
                                            double jitter_rel = 1e-10) {
    auto md = std::unique_ptr<FsaModel>(new FsaModel());
    fsa_params q{static_cast<int>(nu), static_cast<int>(family), gamma, p.sigma2, p.sigma1_2, p.rho, jitter_rel};
    check(fsa_model_assemble(ctx.get(), coords.data(), n, d, inducing.data(), m, &q, &md->h_));
    md->n_ = n;
    return md;
  }
  ~FsaModel() { fsa_model_destroy(h_); }
  std::int64_t n() const { return n_; }
  std::vector<double> matmat(const std::vector<double>& V, std::int64_t k) const {  // fsa.cpp:65-68
    std::vector<double> out(V.size());
    check(fsa_model_matmat(h_, V.data(), k, out.data()));
    return out;
  }
  std::vector<double> deriv_matmat(int which, const std::vector<double>& V, std::int64_t k) {  // fsa.cpp:165-182
    std::vector<double> out(V.size());
    check(fsa_model_deriv_matmat(h_, which, V.data(), k, out.data()));
    return out;
  }
  fsa_model* get() const { return h_; }

 private:
  FsaModel() = default;
  fsa_model* h_ = nullptr;
  std::int64_t n_ = 0;
};

class Preconditioner {  // preconditioners.h:16-37
 public:
  Preconditioner(FsaModel& md, PrecondType t) { check(fsa_make_preconditioner(md.get(), static_cast<int>(t), &h_)); }
  ~Preconditioner() { fsa_precond_destroy(h_); }
  double logdet() const {
    double v = 0.0;
    check(fsa_precond_logdet(h_, &v));
    return v;
  }
  fsa_precond* get() const { return h_; }

 private:
  fsa_precond* h_ = nullptr;
};

// make_preconditioner (estimation.h:81-82)
inline std::unique_ptr<Preconditioner> make_preconditioner(FsaModel& md, PrecondType t) {
  return std::make_unique<Preconditioner>(md, t);
}

// iterative_nll_grad (estimation.h:101-103); X is n x p column-major (p may be 0)
inline IterativeNll iterative_nll_grad(FsaModel& md, const Preconditioner& P, const std::vector<double>& y,
                                       const std::vector<double>& X, std::int64_t p, const IterativeNllOptions& o,
                                       bool want_grad = true) {
  fsa_nll_result r{};
  IterativeNll out;
  out.beta.assign(static_cast<size_t>(p), 0.0);
  const fsa_cg_options cg = o.cg.c();
  check(fsa_iterative_nll_grad(md.get(), P.get(), y.data(), p > 0 ? X.data() : nullptr, p, o.num_probes, o.seed, &cg,
                               static_cast<int>(o.cv), want_grad ? 1 : 0, &r, p > 0 ? out.beta.data() : nullptr));
  out.nll = r.nll;
  out.grad = {r.grad[0], r.grad[1], r.grad[2]};
  out.cg_iterations = r.cg_iterations;
  out.logdet = r.logdet;
  return out;
}

// fisher_ste (fsa.h:106-112): the reference's exact solves become FITC-PCG runs to `solve_tol`
struct FisherOptions {  // fsa.h:107-111
  int num_probes = 50;
  std::uint64_t seed = 0;
  bool rademacher = false;
  double solve_tol = 1e-8;  // (device build only) PCG tolerance standing in for the exact solve
  int solve_max_iter = 1000;
};
// returns F (3 x 3, column-major)
inline std::array<double, 9> fisher_ste(FsaModel& md, const FisherOptions& o) {
  Preconditioner P(md, PrecondType::fitc);
  fsa_cg_options cg{o.solve_tol, o.solve_max_iter, 0};
  std::array<double, 9> F{};
  check(fsa_fisher_ste(md.get(), P.get(), o.num_probes, o.seed, o.rademacher ? 1 : 0, &cg, F.data(), nullptr));
  return F;
}

// PredictionSet / make_prediction_set (prediction.h:16-25)
class PredictionSet {
 public:
  PredictionSet(FsaModel& md, const std::vector<double>& pcoords, std::int64_t np) : np_(np) {
    check(fsa_pred_setup(md.get(), pcoords.data(), np, &h_));
  }
  ~PredictionSet() { fsa_pred_destroy(h_); }
  std::int64_t np() const { return np_; }
  std::vector<double> cross_apply_t(const std::vector<double>& u) const {  // prediction.cpp:29-31
    std::vector<double> out(static_cast<size_t>(np_));
    check(fsa_cross_apply_t(h_, u.data(), out.data()));
    return out;
  }
  fsa_pred* get() const { return h_; }

 private:
  fsa_pred* h_ = nullptr;
  std::int64_t np_ = 0;
};

// predict_mean_iterative (prediction.cpp:37-43)
inline std::vector<double> predict_mean_iterative(PredictionSet& pr, const std::vector<double>& resid,
                                                  const Preconditioner& P, const CgOptions& cg) {
  std::vector<double> out(static_cast<size_t>(pr.np()));
  const fsa_cg_options c = cg.c();
  check(fsa_predict_mean_iterative(pr.get(), resid.data(), P.get(), &c, out.data()));
  return out;
}

// predict_var_sim (prediction.cpp:131-172)
inline PredVarResult predict_var_sim(PredictionSet& pr, const SimVarOptions& o) {
  PredVarResult out;
  out.var.resize(static_cast<size_t>(pr.np()));
  out.se.resize(static_cast<size_t>(pr.np()));
  fsa_predvar_info info{};
  const fsa_cg_options c = o.cg.c(), cs = o.cg_s.c();
  check(fsa_predict_var_sim(pr.get(), o.num_probes, o.seed, &c, &cs, o.control_variate ? 1 : 0, o.floor_rel,
                            out.var.data(), out.se.data(), &info));
  out.clamped = info.clamped;
  out.cg_iterations = info.cg_iterations;
  return out;
}

}  // namespace fsagp_b200
