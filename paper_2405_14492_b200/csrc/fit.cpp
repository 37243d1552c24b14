// Maximum-likelihood fit of the FSA covariance parameters: the
// reference's fit_fsa objective (estimation.cpp:229-303) driven by an L-BFGS with the
// reference's line search and stopping rules (estimation.cpp:10-132), on the device
// library with fit-loop residency: the taper pattern, the response [y | X] and the
// parameter-independent probe draws stay in HBM across evaluations; only the
// parameter-dependent blocks are reassembled per evaluation.
#include "fit.h"

#include <algorithm>
#include <cmath>
#include <deque>
#include <limits>
#include <numeric>

#include "fsa_core.cuh"
#include "inputs.h"
#include "kmeans.cuh"

namespace fsa {
namespace {

double matern_host(double d, int nu, double s1, double rho) {  // kernels.cpp:7-19
  if (nu == 0) return s1 * std::exp(-d / rho);
  if (nu == 1) {
    const double x = std::sqrt(3.0) * d / rho;
    return s1 * (1.0 + x) * std::exp(-x);
  }
  const double x = std::sqrt(5.0) * d / rho;
  return s1 * (1.0 + x + x * x / 3.0) * std::exp(-x);
}

// rho with corr(distance) = corr (kernels.cpp:78-90: geometric bisection)
double rho_for_correlation(double distance, double corr, int nu) {
  double lo = distance * 1e-8, hi = distance * 1e8;
  for (int it = 0; it < 200; ++it) {
    const double mid = std::sqrt(lo * hi);
    if (matern_host(distance, nu, 1.0, mid) < corr) lo = mid;
    else hi = mid;
  }
  return std::sqrt(lo * hi);
}

double dot(const std::vector<double>& a, const std::vector<double>& b) {
  double s = 0.0;
  for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}
double inf_norm(const std::vector<double>& a) {
  double s = 0.0;
  for (double v : a) s = std::max(s, std::fabs(v));
  return s;
}

// OLS residual y - X b (normal equations; p is tiny)
std::vector<double> ols_residual(const double* y, const double* X, long n, long p) {
  std::vector<double> r(y, y + n);
  if (p == 0) return r;
  std::vector<double> G(static_cast<size_t>(p * p), 0.0), b(static_cast<size_t>(p), 0.0);
  for (long a = 0; a < p; ++a) {
    for (long c = 0; c < p; ++c) {
      double s = 0.0;
      for (long i = 0; i < n; ++i) s += X[i + a * n] * X[i + c * n];
      G[static_cast<size_t>(a + c * p)] = s;
    }
    double s = 0.0;
    for (long i = 0; i < n; ++i) s += X[i + a * n] * y[i];
    b[static_cast<size_t>(a)] = s;
  }
  // Gaussian elimination with partial pivoting
  for (long k = 0; k < p; ++k) {
    long piv = k;
    for (long i = k + 1; i < p; ++i)
      if (std::fabs(G[static_cast<size_t>(i + k * p)]) > std::fabs(G[static_cast<size_t>(piv + k * p)])) piv = i;
    require(std::fabs(G[static_cast<size_t>(piv + k * p)]) > 0.0, "fit: covariates are linearly dependent");
    if (piv != k) {
      for (long c = 0; c < p; ++c) std::swap(G[static_cast<size_t>(k + c * p)], G[static_cast<size_t>(piv + c * p)]);
      std::swap(b[static_cast<size_t>(k)], b[static_cast<size_t>(piv)]);
    }
    for (long i = k + 1; i < p; ++i) {
      const double f = G[static_cast<size_t>(i + k * p)] / G[static_cast<size_t>(k + k * p)];
      for (long c = k; c < p; ++c) G[static_cast<size_t>(i + c * p)] -= f * G[static_cast<size_t>(k + c * p)];
      b[static_cast<size_t>(i)] -= f * b[static_cast<size_t>(k)];
    }
  }
  for (long k = p - 1; k >= 0; --k) {
    double s = b[static_cast<size_t>(k)];
    for (long c = k + 1; c < p; ++c) s -= G[static_cast<size_t>(k + c * p)] * b[static_cast<size_t>(c)];
    b[static_cast<size_t>(k)] = s / G[static_cast<size_t>(k + k * p)];
  }
  for (long a = 0; a < p; ++a)
    for (long i = 0; i < n; ++i) r[static_cast<size_t>(i)] -= X[i + a * n] * b[static_cast<size_t>(a)];
  return r;
}

}  // namespace

LbfgsResult lbfgs_minimize(const std::function<double(const std::vector<double>&, std::vector<double>&)>& fn,
                           std::vector<double> x0, const LbfgsOptions& opts) {
  const size_t d = x0.size();
  require(d > 0, "lbfgs: empty start point");
  LbfgsResult res;
  res.x = std::move(x0);
  res.grad.assign(d, 0.0);
  // infeasible points (NumericalError) are +inf for the line search
  auto eval = [&](const std::vector<double>& x, std::vector<double>& g) {
    ++res.evals;
    try {
      return fn(x, g);
    } catch (const NumericalError&) {
      std::fill(g.begin(), g.end(), 0.0);
      return std::numeric_limits<double>::infinity();
    }
  };
  res.f = eval(res.x, res.grad);
  if (!std::isfinite(res.f)) throw NumericalError("lbfgs: start point is infeasible");
  std::deque<std::vector<double>> S, Y;
  std::deque<double> R;
  int small = 0;
  while (res.evals < opts.max_evals) {
    if (inf_norm(res.grad) <= opts.grad_tol) {
      res.converged = true;
      break;
    }
    // two-loop recursion for the quasi-Newton direction
    std::vector<double> q = res.grad;
    std::vector<double> a(S.size());
    for (int i = static_cast<int>(S.size()) - 1; i >= 0; --i) {
      a[static_cast<size_t>(i)] = R[static_cast<size_t>(i)] * dot(S[static_cast<size_t>(i)], q);
      for (size_t j = 0; j < d; ++j) q[j] -= a[static_cast<size_t>(i)] * Y[static_cast<size_t>(i)][j];
    }
    if (!S.empty()) {
      const double g0 = dot(S.back(), Y.back()) / dot(Y.back(), Y.back());
      for (double& v : q) v *= g0;
    }
    for (size_t i = 0; i < S.size(); ++i) {
      const double b = R[i] * dot(Y[i], q);
      for (size_t j = 0; j < d; ++j) q[j] += (a[i] - b) * S[i][j];
    }
    std::vector<double> dir(d);
    for (size_t j = 0; j < d; ++j) dir[j] = -q[j];
    double dg = dot(dir, res.grad);
    if (!(dg < 0.0)) {  // not a descent direction: restart from steepest descent
      S.clear();
      Y.clear();
      R.clear();
      for (size_t j = 0; j < d; ++j) dir[j] = -res.grad[j];
      dg = -dot(res.grad, res.grad);
    }
    // bracketing line search: Armijo sufficient decrease + curvature (c2 = 0.9)
    const double c2 = 0.9;
    double t = 1.0, lo = 0.0, hi = std::numeric_limits<double>::infinity();
    std::vector<double> xn(d), gn(d), xok, gok;
    double fn_ = std::numeric_limits<double>::infinity(), tok = 0.0, fok = 0.0;
    bool accepted = false;
    for (int bt = 0; bt < opts.max_backtracks && res.evals < opts.max_evals; ++bt) {
      for (size_t j = 0; j < d; ++j) xn[j] = res.x[j] + t * dir[j];
      fn_ = eval(xn, gn);
      if (!std::isfinite(fn_) || fn_ > res.f + opts.armijo_c1 * t * dg) {
        hi = t;
      } else {
        if (tok == 0.0 || fn_ < fok) {
          tok = t;
          fok = fn_;
          xok = xn;
          gok = gn;
        }
        if (dot(gn, dir) < c2 * dg) {
          lo = t;
        } else {
          accepted = true;
          break;
        }
      }
      t = std::isfinite(hi) ? 0.5 * (lo + hi) : 2.0 * t;
    }
    if (!accepted) {
      if (tok == 0.0) break;
      xn = xok;
      fn_ = fok;
      gn = gok;
    }
    std::vector<double> s(d), yv(d);
    for (size_t j = 0; j < d; ++j) {
      s[j] = xn[j] - res.x[j];
      yv[j] = gn[j] - res.grad[j];
    }
    const double sy = dot(s, yv);
    if (sy > 1e-10 * std::sqrt(dot(s, s)) * std::sqrt(dot(yv, yv))) {
      S.push_back(s);
      Y.push_back(yv);
      R.push_back(1.0 / sy);
      if (static_cast<int>(S.size()) > opts.memory) {
        S.pop_front();
        Y.pop_front();
        R.pop_front();
      }
    }
    const double drop = res.f - fn_;
    res.x = xn;
    res.f = fn_;
    res.grad = gn;
    if (drop <= opts.f_rel_tol * (std::fabs(res.f) + 1.0)) {
      if (++small >= 2) {
        res.converged = true;
        break;
      }
    } else {
      small = 0;
    }
  }
  if (inf_norm(res.grad) <= opts.grad_tol) res.converged = true;
  return res;
}

FitOutput fit_fsa(Context* ctx, const double* coords, long n, int d, const double* y, const double* X, long p,
                  const FitOptions& o) {
  require(n > 0 && d >= 1 && d <= 3, "fit: invalid location set");
  require(y != nullptr && (p == 0 || X != nullptr), "fit: shape mismatch");
  require(o.num_inducing >= 1 && o.num_inducing <= n, "fit: invalid number of inducing points");
  FitOutput out;
  out.gamma = o.taper_range > 0.0 ? o.taper_range : gamma_for_avg_row_nnz(n, o.target_row_nnz);
  out.inducing.resize(static_cast<size_t>(o.num_inducing * d));
  // inducing points by the device k-means++ (inducing.cpp:48-139; kmeans.cu)
  select_kmeanspp_device(ctx->stream, coords, n, d, o.num_inducing, o.seed, o.kmeans_max_iter, o.kmeans_rel_tol,
                         out.inducing.data());
  // start point (estimation.cpp:246-257): half the residual variance each, rho at which the
  // correlation is 0.05 a quarter of the bounding-box diagonal away
  const std::vector<double> r0 = ols_residual(y, X, n, p);
  const double var0 = std::inner_product(r0.begin(), r0.end(), r0.begin(), 0.0) / static_cast<double>(n);
  double diag2 = 0.0;
  for (int k = 0; k < d; ++k) {
    double lo = coords[k * n], hi = lo;
    for (long i = 0; i < n; ++i) {
      lo = std::min(lo, coords[i + k * n]);
      hi = std::max(hi, coords[i + k * n]);
    }
    diag2 += (hi - lo) * (hi - lo);
  }
  Params p0;
  p0.nu = o.nu;
  p0.family = o.family;
  p0.gamma = out.gamma;
  p0.jitter_rel = o.jitter_rel;
  p0.sigma2 = 0.5 * var0;
  p0.sigma1_2 = 0.5 * var0;
  p0.rho = rho_for_correlation(0.25 * std::sqrt(diag2), 0.05, o.nu);

  // fit-loop residency: pattern, response and probe draws stay on the device
  std::shared_ptr<Geometry> geo = make_geometry(ctx, coords, n, d, out.gamma);
  geo->resp_host.assign(y, y + n);
  if (p > 0) geo->resp_host.insert(geo->resp_host.end(), X, X + n * p);
  geo->resp_dev.alloc(static_cast<size_t>(n * (1 + p)));
  FSA_CUDA(cudaMemcpyAsync(geo->resp_dev.get(), geo->resp_host.data(), sizeof(double) * n * (1 + p),
                           cudaMemcpyHostToDevice, ctx->stream));
  geo->resp_p = p;
  geo->cache_probes = true;
  CgOptions cg;
  cg.tol = o.cg_tol;
  cg.max_iter = o.cg_max_iter;

  std::vector<double> beta_last;
  auto objective = [&](const std::vector<double>& lx, std::vector<double>& g) {
    Params prm = p0;
    prm.sigma2 = std::exp(lx[0]);
    prm.sigma1_2 = std::exp(lx[1]);
    prm.rho = std::exp(lx[2]);
    // a line-search trial so far out that exp() leaves the normal range is infeasible (+inf)
    // rather than an argument error (the reference would abort the fit there)
    for (double v : {prm.sigma2, prm.sigma1_2, prm.rho})
      if (!(v > 0.0) || !std::isfinite(v) || v < 1e-300 || v > 1e300)
        throw NumericalError("fit: parameter out of the representable range");
    auto md = Model::assemble(ctx, geo, out.inducing.data(), o.num_inducing, prm);
    auto P = make_preconditioner(md.get(), o.precond);
    NllResult ev = iterative_nll_grad(md.get(), *P, nullptr, nullptr, 0, o.num_probes, o.seed, cg, o.cv_mode, true);
    g.assign(3, 0.0);
    g[0] = ev.grad[0] * prm.sigma2;  // chain rule to log space (estimation.cpp:281)
    g[1] = ev.grad[1] * prm.sigma1_2;
    g[2] = ev.grad[2] * prm.rho;
    beta_last = ev.beta;
    out.nll_trace.push_back(ev.nll);
    return ev.nll;
  };
  LbfgsOptions lopt = o.lbfgs;
  lopt.grad_tol = o.grad_tol_per_n * static_cast<double>(n);  // estimation.cpp:290
  LbfgsResult sol = lbfgs_minimize(objective, {std::log(p0.sigma2), std::log(p0.sigma1_2), std::log(p0.rho)}, lopt);
  std::vector<double> gfin;
  out.nll = objective(sol.x, gfin);
  out.sigma2 = std::exp(sol.x[0]);
  out.sigma1_2 = std::exp(sol.x[1]);
  out.rho = std::exp(sol.x[2]);
  out.beta = beta_last;
  out.evals = sol.evals + 1;
  out.converged = sol.converged;
  out.grad_log = gfin;
  return out;
}

}  // namespace fsa
