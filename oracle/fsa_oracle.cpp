// =============================================================================
// CPU ORACLE — TEST INFRASTRUCTURE ONLY.
//
// A plain C++ restatement (no Eigen) of the reference's FSA iterative path,
// /root/reference/proj (the `fsagp` library), used ONLY by tests/, by
// __graft_entry__.smoke() as the checker, and by bench.py's cpu_baseline /
// `--impl reference` legs. The product (paper_2405_14492_b200/) never links,
// loads or calls anything in oracle/.
//
// Parity status: the reference cannot be compiled here (Eigen3, doctest, CLI11
// are absent). This restatement is pinned against every known
// answer the reference's own tests hold for this path (matern/taper literal
// values, the 5x5 tridiagonal quadrature, range calibration, taper-pattern set
// equality, dense-mirror identities from tests/oracles.h, CG-vs-factorised
// solves, bitwise multi==single, probe keying, seed determinism, statistical
// brackets) — see tests/test_oracle_*.py. There are no stored golden vectors in
// the reference; parity at the Eigen arithmetic boundary is to tolerance.
//
// Each function cites the reference file:line it restates.
// =============================================================================
#include "fsa_oracle.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <limits>
#include <memory>
#include <numeric>
#include <random>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "blas_lite.h"

namespace orc {

using rng_t = std::mt19937_64;

// ---- errors (types.h:22-29) --------------------------------------------------
struct NumericalError : std::runtime_error {
  explicit NumericalError(const std::string& w) : std::runtime_error(w) {}
};
inline void require(bool c, const char* msg) {
  if (!c) throw std::invalid_argument(msg);
}

// ---- dense / sparse containers ----------------------------------------------
struct Mat {  // column-major like Eigen::MatrixXd (types.h:14)
  long r = 0, c = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(long r_, long c_) : r(r_), c(c_), a(static_cast<size_t>(r_ * c_), 0.0) {}
  double& operator()(long i, long j) { return a[static_cast<size_t>(i + j * r)]; }
  double operator()(long i, long j) const { return a[static_cast<size_t>(i + j * r)]; }
  double* col(long j) { return a.data() + j * r; }
  const double* col(long j) const { return a.data() + j * r; }
  double* data() { return a.data(); }
  const double* data() const { return a.data(); }
};

struct Csr {  // Eigen RowMajor sparse, sorted columns per row (types.h:15-16)
  long rows = 0, cols = 0;
  std::vector<long> ptr;
  std::vector<int> idx;
  std::vector<double> val;
  long nnz() const { return static_cast<long>(idx.size()); }
};

// ---- RNG (types.h:104-129) ---------------------------------------------------
inline uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
inline rng_t probe_rng(uint64_t seed, uint64_t i) {
  return rng_t(splitmix64(splitmix64(seed) ^ splitmix64(i + 0x51ed2701ULL)));
}
inline void gaussian_fill(rng_t& rng, double* z, long n) {  // fresh distribution per call
  std::normal_distribution<double> N01(0.0, 1.0);
  for (long i = 0; i < n; ++i) z[i] = N01(rng);
}
inline void rademacher_fill(rng_t& rng, double* z, long n) {
  std::bernoulli_distribution coin(0.5);
  for (long i = 0; i < n; ++i) z[i] = coin(rng) ? 1.0 : -1.0;
}

// ---- kernels (kernels.cpp:7-52) ---------------------------------------------
enum Nu { NU12 = 0, NU32 = 1, NU52 = 2 };

double matern(double d, int nu, double s1, double rho) {  // kernels.cpp:7-22
  const double s = d / rho;
  switch (nu) {
    case NU12: return s1 * std::exp(-s);
    case NU32: { const double x = std::sqrt(3.0) * s; return s1 * (1.0 + x) * std::exp(-x); }
    case NU52: { const double x = std::sqrt(5.0) * s; return s1 * (1.0 + x + x * x / 3.0) * std::exp(-x); }
  }
  throw std::invalid_argument("unknown Matern smoothness");
}
double matern_drho(double d, int nu, double s1, double rho) {  // kernels.cpp:24-39
  const double s = d / rho;
  switch (nu) {
    case NU12: return s1 * std::exp(-s) * d / (rho * rho);
    case NU32: { const double x = std::sqrt(3.0) * s; return s1 * 3.0 * d * d / (rho * rho * rho) * std::exp(-x); }
    case NU52: { const double x = std::sqrt(5.0) * s; return s1 * (5.0 * d * d / (3.0 * rho * rho * rho)) * (1.0 + x) * std::exp(-x); }
  }
  throw std::invalid_argument("unknown Matern smoothness");
}
double taper_value(double d, int family, double gamma) {  // kernels.cpp:41-52
  const double r = d / gamma;
  if (r >= 1.0) return 0.0;
  const double omr = 1.0 - r;
  const double omr2 = omr * omr;
  if (family == 1) return omr2 * omr2 * (1.0 + 4.0 * r);
  const double omr6 = omr2 * omr2 * omr2;
  return omr6 * (1.0 + 6.0 * r + 35.0 * r * r / 3.0);
}
double rho_for_correlation_at(double distance, double corr, int nu) {  // kernels.cpp:78-90
  require(distance > 0.0, "distance must be positive");
  require(corr > 0.0 && corr < 1.0, "target correlation must lie in (0, 1)");
  double lo = distance * 1e-8, hi = distance * 1e8;
  for (int it = 0; it < 200; ++it) {
    double mid = std::sqrt(lo * hi);
    if (matern(distance, nu, 1.0, mid) < corr) lo = mid; else hi = mid;
  }
  return std::sqrt(lo * hi);
}
double effective_range(double rho, int nu) {  // kernels.cpp:92-103
  require(rho > 0.0, "rho must be positive");
  double lo = 0.0, hi = rho * 100.0;
  for (int it = 0; it < 200; ++it) {
    double mid = 0.5 * (lo + hi);
    if (matern(mid, nu, 1.0, rho) > 0.05) lo = mid; else hi = mid;
  }
  return 0.5 * (lo + hi);
}

// Euclidean distance of two rows of column-major coordinate arrays, the
// (row_i - row_j).norm() of locations.h:19-21. The sum is written as the
// FMA chain a contracted Eigen redux produces (s = d0*d0; s = fma(dk,dk,s)).
inline double pdist(const double* A, long lda, long i, const double* B, long ldb, long j, int d) {
  const double d0 = A[i] - B[j];
  double s = d0 * d0;
  for (int k = 1; k < d; ++k) {
    const double dk = A[i + k * lda] - B[j + k * ldb];
    s = std::fma(dk, dk, s);
  }
  return std::sqrt(s);
}

struct Locs {
  long n = 0;
  int d = 0;
  std::vector<double> c;  // n x d column-major (LocationSet::coords)
  const double* p() const { return c.data(); }
};

Mat cross_cov(const Locs& a, const Locs& b, int nu, double s1, double rho, bool drho) {
  Mat out(a.n, b.n);  // kernels.cpp:54-76
#pragma omp parallel for schedule(static) if (a.n * b.n > 100000)
  for (long j = 0; j < b.n; ++j)
    for (long i = 0; i < a.n; ++i) {
      const double dd = pdist(a.p(), a.n, i, b.p(), b.n, j, a.d);
      out(i, j) = drho ? matern_drho(dd, nu, s1, rho) : matern(dd, nu, s1, rho);
    }
  return out;
}

// ---- locations (locations.cpp:9-17,19-62,139-195) ---------------------------
void uniform_locations(long n, int d, uint64_t seed, double* out) {
  require(n > 0 && d > 0, "uniform_locations needs n > 0 and d > 0");
  rng_t rng(splitmix64(seed));
  std::uniform_real_distribution<double> U(0.0, 1.0);
  for (long i = 0; i < n; ++i)
    for (int k = 0; k < d; ++k) out[i + k * n] = U(rng);
}

// ---- synthetic inputs of the BASELINE configs (not reference code: the reference's own
// simulate_gp needs an exact Cholesky, estimation.cpp:330-332). Independent restatement of the
// generator spec the product's host generators implement: a random-Fourier-feature
// Matern draw plus nugget noise, and the config-5 Gaussian-blob mixture on [0,1]^d.
void simulate_rff(const double* c, long n, int d, int nu_code, double sigma1_2, double rho, double nugget,
                  int features, uint64_t seed, double* y) {
  require(n > 0 && features > 0, "simulate_rff: invalid sizes");
  const double nu = nu_code == 0 ? 0.5 : (nu_code == 1 ? 1.5 : 2.5);
  rng_t rng(splitmix64(seed ^ 0x5eed5eedULL));
  std::normal_distribution<double> N01(0.0, 1.0);
  std::chi_squared_distribution<double> chi(2.0 * nu);  // spectral density of Matern-nu: Student-t
  std::uniform_real_distribution<double> U(0.0, 2.0 * M_PI);
  std::vector<double> w(static_cast<size_t>(features) * d), b(static_cast<size_t>(features));
  for (int f = 0; f < features; ++f) {
    const double u = chi(rng);
    const double scale = 1.0 / (rho * std::sqrt(u / (2.0 * nu)));
    for (int k = 0; k < d; ++k) w[static_cast<size_t>(f) * d + k] = N01(rng) * scale;
    b[static_cast<size_t>(f)] = U(rng);
  }
  const double amp = std::sqrt(2.0 * sigma1_2 / features);
#pragma omp parallel for schedule(static)
  for (long i = 0; i < n; ++i) {
    double acc = 0.0;
    for (int f = 0; f < features; ++f) {
      double arg = b[static_cast<size_t>(f)];
      for (int k = 0; k < d; ++k) arg += w[static_cast<size_t>(f) * d + k] * c[i + k * n];
      acc += std::cos(arg);
    }
    y[i] = amp * acc;
  }
  rng_t noise(splitmix64(seed ^ 0x0153ULL));
  std::normal_distribution<double> E(0.0, 1.0);
  const double sd = std::sqrt(nugget);
  for (long i = 0; i < n; ++i) y[i] += sd * E(noise);
}

void blob_locations(long n, int d, int blobs, double sd, uint64_t seed, double* out) {
  require(n > 0 && blobs > 0 && d <= 3, "blob_locations: invalid sizes");
  rng_t rng(splitmix64(seed));
  std::uniform_real_distribution<double> U(0.0, 1.0);
  std::vector<double> centre(static_cast<size_t>(blobs) * d);
  for (double& v : centre) v = U(rng);
  std::uniform_int_distribution<int> pick(0, blobs - 1);
  std::normal_distribution<double> N(0.0, sd);
  for (long i = 0; i < n;) {
    const int bl = pick(rng);
    double p[3];
    bool inside = true;
    for (int k = 0; k < d; ++k) {
      p[k] = centre[static_cast<size_t>(bl) * d + k] + N(rng);
      inside = inside && p[k] >= 0.0 && p[k] <= 1.0;
    }
    if (!inside) continue;  // rejected
    for (int k = 0; k < d; ++k) out[i + k * n] = p[k];
    ++i;
  }
}

// GridIndex (locations.cpp:19-62): cells of edge h, 3^d neighbourhood scan,
// strict ||x - q|| < h. Cells are keyed by their integer coordinates here
// (collision-free) — the reference's splitmix-hashed keys give the same set
// because every candidate is re-checked by distance.
struct Grid {
  const Locs* L;
  double h;
  std::vector<double> origin;
  std::unordered_map<uint64_t, std::vector<int>> cells;
  uint64_t key_of(const std::vector<long>& cell) const {
    uint64_t key = 0xcbf29ce484222325ULL;
    for (size_t k = 0; k < cell.size(); ++k)
      key = splitmix64(key ^ static_cast<uint64_t>(cell[k] + 0x40000000LL));
    return key;
  }
  std::vector<long> cell_of(const double* C, long ldc, long i) const {
    std::vector<long> cell(static_cast<size_t>(L->d));
    for (int k = 0; k < L->d; ++k)
      cell[static_cast<size_t>(k)] = static_cast<long>(std::floor((C[i + k * ldc] - origin[static_cast<size_t>(k)]) / h));
    return cell;
  }
  Grid(const Locs& locs, double h_) : L(&locs), h(h_) {
    require(h > 0.0, "grid cell size must be positive");
    origin.assign(static_cast<size_t>(locs.d), 0.0);
    for (int k = 0; k < locs.d; ++k) {
      double mn = locs.c[static_cast<size_t>(k * locs.n)];
      for (long i = 1; i < locs.n; ++i) mn = std::min(mn, locs.c[static_cast<size_t>(i + k * locs.n)]);
      origin[static_cast<size_t>(k)] = mn;
    }
    for (long i = 0; i < locs.n; ++i) cells[key_of(cell_of(locs.p(), locs.n, i))].push_back(static_cast<int>(i));
  }
  // all j with ||x_j - q|| < h; q = row qi of Q (ldq)
  void query(const double* Q, long ldq, long qi, std::vector<int>* out) const {
    const int d = L->d;
    std::vector<long> base = cell_of(Q, ldq, qi), off(static_cast<size_t>(d), -1), cell(static_cast<size_t>(d));
    std::vector<uint64_t> seen;
    while (true) {
      for (int k = 0; k < d; ++k) cell[static_cast<size_t>(k)] = base[static_cast<size_t>(k)] + off[static_cast<size_t>(k)];
      const uint64_t key = key_of(cell);
      if (std::find(seen.begin(), seen.end(), key) == seen.end()) {
        seen.push_back(key);
        auto it = cells.find(key);
        if (it != cells.end())
          for (int j : it->second)
            if (pdist(L->p(), L->n, j, Q, ldq, qi, d) < h) out->push_back(j);
      }
      int k = 0;
      for (; k < d; ++k) {
        if (++off[static_cast<size_t>(k)] <= 1) break;
        off[static_cast<size_t>(k)] = -1;
      }
      if (k == d) break;
    }
  }
};

// taper_pattern (locations.cpp:139-163): all pairs at distance < gamma plus a
// forced diagonal; values are distances; columns sorted per row.
Csr taper_pattern(const Locs& locs, double gamma, bool cross, const Locs* cols_locs) {
  require(gamma > 0.0, "taper range must be positive");
  const Locs& C = cross ? *cols_locs : locs;
  Grid grid(C, gamma);
  const long n = locs.n;
  Csr out;
  out.rows = n;
  out.cols = C.n;
  std::vector<std::vector<int>> rows(static_cast<size_t>(n));
#pragma omp parallel for schedule(dynamic, 256)
  for (long i = 0; i < n; ++i) {
    std::vector<int>& h = rows[static_cast<size_t>(i)];
    grid.query(locs.p(), locs.n, i, &h);
    if (!cross && std::find(h.begin(), h.end(), static_cast<int>(i)) == h.end()) h.push_back(static_cast<int>(i));
    std::sort(h.begin(), h.end());
    h.erase(std::unique(h.begin(), h.end()), h.end());
  }
  out.ptr.assign(static_cast<size_t>(n + 1), 0);
  for (long i = 0; i < n; ++i) out.ptr[static_cast<size_t>(i + 1)] = out.ptr[static_cast<size_t>(i)] + static_cast<long>(rows[static_cast<size_t>(i)].size());
  out.idx.resize(static_cast<size_t>(out.ptr[static_cast<size_t>(n)]));
  out.val.resize(out.idx.size());
#pragma omp parallel for schedule(static)
  for (long i = 0; i < n; ++i) {
    long p = out.ptr[static_cast<size_t>(i)];
    for (int j : rows[static_cast<size_t>(i)]) {
      out.idx[static_cast<size_t>(p)] = j;
      out.val[static_cast<size_t>(p)] = (!cross && j == i) ? 0.0 : pdist(locs.p(), locs.n, i, C.p(), C.n, j, locs.d);
      ++p;
    }
  }
  return out;
}

// ---- inducing points (inducing.cpp:11-139) ----------------------------------
void select_random(const Locs& locs, long m, uint64_t seed, double* out) {
  require(m >= 1 && m <= locs.n, "need 1 <= m <= n");
  rng_t rng(splitmix64(seed));
  std::vector<long> idx(static_cast<size_t>(locs.n));
  std::iota(idx.begin(), idx.end(), 0L);
  for (long i = 0; i < m; ++i) {
    std::uniform_int_distribution<long> pick(i, locs.n - 1);
    std::swap(idx[static_cast<size_t>(i)], idx[static_cast<size_t>(pick(rng))]);
  }
  for (long i = 0; i < m; ++i)
    for (int k = 0; k < locs.d; ++k) out[i + k * m] = locs.c[static_cast<size_t>(idx[static_cast<size_t>(i)] + k * locs.n)];
}

void select_kmeanspp(const Locs& locs, long m, uint64_t seed, int max_iter, double rel_tol, double* out) {
  require(m >= 1 && m <= locs.n, "need 1 <= m <= n");
  const long n = locs.n;
  const int d = locs.d;
  auto X = [&](long i, int k) { return locs.c[static_cast<size_t>(i + k * n)]; };
  // distinct_rows (inducing.cpp:28-44)
  std::vector<int> order(static_cast<size_t>(n));
  std::iota(order.begin(), order.end(), 0);
  std::sort(order.begin(), order.end(), [&](int a, int b) {
    for (int k = 0; k < d; ++k)
      if (X(a, k) != X(b, k)) return X(a, k) < X(b, k);
    return a < b;
  });
  std::vector<int> pool;
  for (size_t t = 0; t < order.size(); ++t) {
    bool same = t > 0;
    if (t > 0)
      for (int k = 0; k < d; ++k)
        if (X(order[t], k) != X(order[t - 1], k)) same = false;
    if (!same) pool.push_back(order[t]);
  }
  std::sort(pool.begin(), pool.end());
  const long np = static_cast<long>(pool.size());
  require(m <= np, "m exceeds the number of distinct locations");

  auto sqd = [&](long i, const std::vector<double>& ctr, long c) {  // squaredNorm (sequential)
    double s = 0.0;
    for (int k = 0; k < d; ++k) {
      const double df = X(i, k) - ctr[static_cast<size_t>(c + k * m)];
      s = k == 0 ? df * df : std::fma(df, df, s);
    }
    return s;
  };
  rng_t rng(splitmix64(seed));
  std::vector<double> ctr(static_cast<size_t>(m * d));
  std::uniform_int_distribution<long> first(0, np - 1);
  {
    const long p0 = pool[static_cast<size_t>(first(rng))];
    for (int k = 0; k < d; ++k) ctr[static_cast<size_t>(k * m)] = X(p0, k);
  }
  std::vector<double> d2(static_cast<size_t>(np));
#pragma omp parallel for schedule(static)
  for (long i = 0; i < np; ++i) d2[static_cast<size_t>(i)] = sqd(pool[static_cast<size_t>(i)], ctr, 0);
  for (long c = 1; c < m; ++c) {
    double total = 0.0;
    for (long i = 0; i < np; ++i) total += d2[static_cast<size_t>(i)];
    long chosen = 0;
    if (total > 0.0) {
      std::uniform_real_distribution<double> U(0.0, total);
      double u = U(rng), acc = 0.0;
      for (long i = 0; i < np; ++i) {
        acc += d2[static_cast<size_t>(i)];
        if (u <= acc) { chosen = i; break; }
      }
    } else {
      chosen = first(rng) % np;
    }
    for (int k = 0; k < d; ++k) ctr[static_cast<size_t>(c + k * m)] = X(pool[static_cast<size_t>(chosen)], k);
#pragma omp parallel for schedule(static)
    for (long i = 0; i < np; ++i) d2[static_cast<size_t>(i)] = std::min(d2[static_cast<size_t>(i)], sqd(pool[static_cast<size_t>(i)], ctr, c));
  }
  // Lloyd (inducing.cpp:86-115)
  std::vector<long> assign(static_cast<size_t>(n), 0);
  std::vector<double> best_d(static_cast<size_t>(n));
  double sse_prev = std::numeric_limits<double>::infinity();
  for (int it = 0; it < max_iter; ++it) {
#pragma omp parallel for schedule(static)
    for (long i = 0; i < n; ++i) {
      double best = std::numeric_limits<double>::infinity();
      long bc = 0;
      for (long c = 0; c < m; ++c) {
        const double dd = sqd(i, ctr, c);
        if (dd < best) { best = dd; bc = c; }
      }
      assign[static_cast<size_t>(i)] = bc;
      best_d[static_cast<size_t>(i)] = best;
    }
    double sse = 0.0;
    for (long i = 0; i < n; ++i) sse += best_d[static_cast<size_t>(i)];
    std::vector<double> sums(static_cast<size_t>(m * d), 0.0), counts(static_cast<size_t>(m), 0.0);
    for (long i = 0; i < n; ++i) {
      const long a = assign[static_cast<size_t>(i)];
      for (int k = 0; k < d; ++k) sums[static_cast<size_t>(a + k * m)] += X(i, k);
      counts[static_cast<size_t>(a)] += 1.0;
    }
    for (long c = 0; c < m; ++c)
      if (counts[static_cast<size_t>(c)] > 0.0)
        for (int k = 0; k < d; ++k) ctr[static_cast<size_t>(c + k * m)] = sums[static_cast<size_t>(c + k * m)] / counts[static_cast<size_t>(c)];
    if (sse_prev - sse <= rel_tol * std::max(sse_prev, 1e-300)) break;
    sse_prev = sse;
  }
  // snap (inducing.cpp:117-137): nearest unused distinct location, first index on ties
  std::vector<char> used(static_cast<size_t>(np), 0);
  for (long c = 0; c < m; ++c) {
    double best = std::numeric_limits<double>::infinity();
    long bi = -1;
#pragma omp parallel
    {
      double lb = std::numeric_limits<double>::infinity();
      long li = -1;
#pragma omp for schedule(static) nowait
      for (long i = 0; i < np; ++i) {
        if (used[static_cast<size_t>(i)]) continue;
        const double dd = sqd(pool[static_cast<size_t>(i)], ctr, c);
        if (dd < lb) { lb = dd; li = i; }
      }
#pragma omp critical
      {
        if (li >= 0 && (lb < best || (lb == best && li < bi))) { best = lb; bi = li; }
      }
    }
    used[static_cast<size_t>(bi)] = 1;
    for (int k = 0; k < d; ++k) out[c + k * m] = X(pool[static_cast<size_t>(bi)], k);
  }
}

// ---- dense linear algebra (Eigen LLT / triangular solves) -------------------
// LLT of the lower triangle; returns false if not positive definite.
bool llt(Mat& A) {
  const long n = A.r;
  for (long j = 0; j < n; ++j) {
    double s = A(j, j);
    for (long k = 0; k < j; ++k) s -= A(j, k) * A(j, k);
    if (!(s > 0.0) || !std::isfinite(s)) return false;
    const double ljj = std::sqrt(s);
    A(j, j) = ljj;
#pragma omp parallel for schedule(static) if (n - j > 256)
    for (long i = j + 1; i < n; ++i) {
      double t = A(i, j);
      for (long k = 0; k < j; ++k) t -= A(i, k) * A(j, k);
      A(i, j) = t / ljj;
    }
  }
  for (long j = 0; j < n; ++j)
    for (long i = 0; i < j; ++i) A(i, j) = 0.0;
  return true;
}
double llt_logdet(const Mat& L) {
  double s = 0.0;
  for (long i = 0; i < L.r; ++i) s += std::log(L(i, i));
  return 2.0 * s;
}
// B <- L^{-1} B (lower, forward), blocked with dgemm updates
void trsm_lower(const Mat& L, double* B, long ldb, long ncols) {
  const long m = L.r, nb = 64;
  for (long k0 = 0; k0 < m; k0 += nb) {
    const long kb = std::min(nb, m - k0);
#pragma omp parallel for schedule(static) if (ncols > 64)
    for (long j = 0; j < ncols; ++j) {
      double* b = B + j * ldb;
      for (long i = k0; i < k0 + kb; ++i) {
        double t = b[i];
        for (long k = k0; k < i; ++k) t -= L(i, k) * b[k];
        b[i] = t / L(i, i);
      }
    }
    const long rest = m - k0 - kb;
    if (rest > 0)
      dgemm('N', 'N', rest, ncols, kb, -1.0, L.data() + (k0 + kb) + k0 * m, m, B + k0, ldb, 1.0,
            B + k0 + kb, ldb);
  }
}
// B <- L^{-T} B (backward with the transpose)
void trsm_lower_t(const Mat& L, double* B, long ldb, long ncols) {
  const long m = L.r, nb = 64;
  long k1 = m;
  while (k1 > 0) {
    const long k0 = std::max(0L, k1 - nb), kb = k1 - k0;
#pragma omp parallel for schedule(static) if (ncols > 64)
    for (long j = 0; j < ncols; ++j) {
      double* b = B + j * ldb;
      for (long i = k1 - 1; i >= k0; --i) {
        double t = b[i];
        for (long k = i + 1; k < k1; ++k) t -= L(k, i) * b[k];
        b[i] = t / L(i, i);
      }
    }
    if (k0 > 0)  // B[0:k0] -= L[k0:k1, 0:k0]^T X[k0:k1]
      dgemm('T', 'N', k0, ncols, kb, -1.0, L.data() + k0, m, B + k0, ldb, 1.0, B, ldb);
    k1 = k0;
  }
}
void llt_solve(const Mat& L, double* B, long ldb, long ncols) {
  trsm_lower(L, B, ldb, ncols);
  trsm_lower_t(L, B, ldb, ncols);
}

// CSR x dense (col-major, n x k)
void spmm(const Csr& S, const double* V, long ldv, long k, double* out, long ldo) {
#pragma omp parallel for schedule(static) if (S.rows * k > 20000)
  for (long r = 0; r < S.rows; ++r) {
    for (long j = 0; j < k; ++j) {
      double acc = 0.0;
      for (long p = S.ptr[static_cast<size_t>(r)]; p < S.ptr[static_cast<size_t>(r + 1)]; ++p)
        acc += S.val[static_cast<size_t>(p)] * V[S.idx[static_cast<size_t>(p)] + j * ldv];
      out[r + j * ldo] = acc;
    }
  }
}
// CSR^T x dense: out (cols x k) = S^T V
void spmm_t(const Csr& S, const double* V, long ldv, long k, double* out, long ldo) {
#pragma omp parallel for schedule(static) if (S.cols * k > 20000)
  for (long j = 0; j < k; ++j) {
    double* o = out + j * ldo;
    for (long c = 0; c < S.cols; ++c) o[c] = 0.0;
    for (long r = 0; r < S.rows; ++r) {
      const double v = V[r + j * ldv];
      for (long p = S.ptr[static_cast<size_t>(r)]; p < S.ptr[static_cast<size_t>(r + 1)]; ++p)
        o[S.idx[static_cast<size_t>(p)]] += S.val[static_cast<size_t>(p)] * v;
    }
  }
}
inline double dot(const double* a, const double* b, long n) {
  double s = 0.0;
  for (long i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}

// ---- FSA model (fsa.cpp:7-193) ----------------------------------------------
struct Model {
  Locs locs, ind;
  int nu = NU32, family = 1;
  double gamma = 0.1, sigma2 = 1.0, sigma1_2 = 1.0, rho = 0.1, jitter_rel = 1e-10;
  long n = 0, m = 0;
  Mat sigma_m, chol_m, sigma_mn, U, A;
  double logdet_sigma_m = 0.0;
  std::vector<double> lowrank_diag;
  Csr dists, sigma_s;
  long n_clamped = 0;
  // lazy derivative blocks (fsa.cpp:70-144)
  bool have_rho = false;
  Mat dsm_rho, P1, W2;
  Csr ds_rho;

  void ensure_rho_derivs() {  // fsa.cpp:101-124
    if (have_rho) return;
    dsm_rho = cross_cov(ind, ind, nu, sigma1_2, rho, true);
    P1 = cross_cov(ind, locs, nu, sigma1_2, rho, true);
    W2 = Mat(m, n);
    dgemm('N', 'N', m, n, m, 1.0, dsm_rho.data(), m, A.data(), m, 0.0, W2.data(), m);
    ds_rho = dists;
#pragma omp parallel for schedule(dynamic, 256)
    for (long r = 0; r < n; ++r)
      for (long p = dists.ptr[static_cast<size_t>(r)]; p < dists.ptr[static_cast<size_t>(r + 1)]; ++p) {
        const long c = dists.idx[static_cast<size_t>(p)];
        const double dl = dot(P1.col(r), A.col(c), m) + dot(A.col(r), P1.col(c), m) - dot(A.col(r), W2.col(c), m);
        if (r == c) {
          const bool clamped = sigma1_2 - lowrank_diag[static_cast<size_t>(r)] < 0.0;
          ds_rho.val[static_cast<size_t>(p)] = clamped ? 0.0 : -dl;
        } else {
          const double dd = dists.val[static_cast<size_t>(p)];
          ds_rho.val[static_cast<size_t>(p)] = (matern_drho(dd, nu, sigma1_2, rho) - dl) * taper_value(dd, family, gamma);
        }
      }
    have_rho = true;
  }

  // Y = sigma_s V + sigma_mn^T (A V)   (fsa.cpp:65-68)
  void matmat(const double* V, long k, double* Y) const {
    Mat AV(m, k), G(n, k);
    dgemm('N', 'N', m, k, n, 1.0, A.data(), m, V, n, 0.0, AV.data(), m);
    dgemm('T', 'N', n, k, m, 1.0, sigma_mn.data(), m, AV.data(), m, 0.0, G.data(), n);
    spmm(sigma_s, V, n, k, Y, n);
    for (size_t i = 0; i < static_cast<size_t>(n * k); ++i) Y[i] += G.a[i];
  }
  void sigma_s_mat(const double* V, long k, double* Y) const { spmm(sigma_s, V, n, k, Y, n); }

  // deriv_matmat (fsa.cpp:165-182)
  void deriv_matmat(int which, const double* V, long k, double* Y) {
    require(which >= 0 && which < 3, "parameter index out of range");
    const size_t nk = static_cast<size_t>(n * k);
    if (which == 0) { std::copy(V, V + nk, Y); return; }
    if (which == 1) {
      Mat AV(m, k), G(n, k);
      dgemm('N', 'N', m, k, n, 1.0, A.data(), m, V, n, 0.0, AV.data(), m);
      dgemm('T', 'N', n, k, m, 1.0, sigma_mn.data(), m, AV.data(), m, 0.0, G.data(), n);
      spmm(sigma_s, V, n, k, Y, n);
      for (size_t i = 0; i < nk; ++i) Y[i] = ((Y[i] - sigma2 * V[i]) + G.a[i]) / sigma1_2;
      return;
    }
    ensure_rho_derivs();
    Mat AV(m, k), PV(m, k), WV(m, k), T1(n, k), T2(n, k), T3(n, k);
    dgemm('N', 'N', m, k, n, 1.0, A.data(), m, V, n, 0.0, AV.data(), m);
    dgemm('N', 'N', m, k, n, 1.0, P1.data(), m, V, n, 0.0, PV.data(), m);
    dgemm('N', 'N', m, k, n, 1.0, W2.data(), m, V, n, 0.0, WV.data(), m);
    dgemm('T', 'N', n, k, m, 1.0, P1.data(), m, AV.data(), m, 0.0, T1.data(), n);
    dgemm('T', 'N', n, k, m, 1.0, A.data(), m, PV.data(), m, 0.0, T2.data(), n);
    dgemm('T', 'N', n, k, m, 1.0, A.data(), m, WV.data(), m, 0.0, T3.data(), n);
    spmm(ds_rho, V, n, k, Y, n);
    for (size_t i = 0; i < nk; ++i) Y[i] = ((Y[i] + T1.a[i]) + T2.a[i]) - T3.a[i];
  }
};

Model* assemble(const Locs& locs, const Locs& ind, int nu, int family, double gamma, double sigma2,
                double sigma1_2, double rho, double jitter_rel) {  // fsa.cpp:7-58
  require(sigma2 > 0.0 && std::isfinite(sigma2), "sigma2 must be positive and finite");
  require(sigma1_2 > 0.0 && std::isfinite(sigma1_2), "sigma1_2 must be positive and finite");
  require(rho > 0.0 && std::isfinite(rho), "rho must be positive and finite");
  require(gamma > 0.0, "taper range gamma must be positive");
  require(locs.n > 0, "empty location set");
  require(ind.n > 0, "empty inducing set");
  require(locs.d == ind.d, "location sets must share the dimension");
  require(nu >= 0 && nu <= 2, "Matern smoothness must be one of 0.5, 1.5, 2.5");
  require(family == 1 || family == 2, "taper family must be wendland1 or wendland2");
  auto M = std::make_unique<Model>();
  Model& md = *M;
  md.locs = locs; md.ind = ind; md.nu = nu; md.family = family; md.gamma = gamma;
  md.sigma2 = sigma2; md.sigma1_2 = sigma1_2; md.rho = rho; md.jitter_rel = jitter_rel;
  md.n = locs.n; md.m = ind.n;
  const long n = md.n, m = md.m;
  const double jitter = jitter_rel * sigma1_2;
  md.sigma_m = cross_cov(ind, ind, nu, sigma1_2, rho, false);
  for (long i = 0; i < m; ++i) md.sigma_m(i, i) += jitter;
  md.chol_m = md.sigma_m;
  if (!llt(md.chol_m)) throw NumericalError("inducing covariance is not positive definite");
  md.logdet_sigma_m = llt_logdet(md.chol_m);
  md.sigma_mn = cross_cov(ind, locs, nu, sigma1_2, rho, false);
  md.U = md.sigma_mn;
  trsm_lower(md.chol_m, md.U.data(), m, n);
  md.A = md.U;
  trsm_lower_t(md.chol_m, md.A.data(), m, n);
  md.lowrank_diag.assign(static_cast<size_t>(n), 0.0);
#pragma omp parallel for schedule(static)
  for (long i = 0; i < n; ++i) md.lowrank_diag[static_cast<size_t>(i)] = dot(md.U.col(i), md.U.col(i), m);
  md.dists = taper_pattern(locs, gamma, false, nullptr);
  md.sigma_s = md.dists;
  long clamped = 0;
#pragma omp parallel for schedule(dynamic, 256) reduction(+ : clamped)
  for (long r = 0; r < n; ++r)
    for (long p = md.dists.ptr[static_cast<size_t>(r)]; p < md.dists.ptr[static_cast<size_t>(r + 1)]; ++p) {
      const long c = md.dists.idx[static_cast<size_t>(p)];
      if (r == c) {
        double resid = sigma1_2 - md.lowrank_diag[static_cast<size_t>(r)];
        if (resid < 0.0) { resid = 0.0; ++clamped; }
        md.sigma_s.val[static_cast<size_t>(p)] = resid + sigma2;
      } else {
        const double dd = md.dists.val[static_cast<size_t>(p)];
        md.sigma_s.val[static_cast<size_t>(p)] =
            (matern(dd, nu, sigma1_2, rho) - dot(md.U.col(r), md.U.col(c), m)) * taper_value(dd, family, gamma);
      }
    }
  md.n_clamped = clamped;
  return M.release();
}

std::vector<double> csr_diag(const Csr& S) {
  std::vector<double> d(static_cast<size_t>(S.rows), 0.0);
  for (long r = 0; r < S.rows; ++r)
    for (long p = S.ptr[static_cast<size_t>(r)]; p < S.ptr[static_cast<size_t>(r + 1)]; ++p)
      if (S.idx[static_cast<size_t>(p)] == r) d[static_cast<size_t>(r)] = S.val[static_cast<size_t>(p)];
  return d;
}

// ---- preconditioners (preconditioners.cpp:7-115, .h:39-115) -----------------
struct Precond {
  virtual ~Precond() = default;
  virtual long size() const = 0;
  virtual int kind() const = 0;  // 0 none, 1 diagonal, 2 fitc
  virtual void solve(const double* r, double* out) const = 0;
  virtual void solve_mat(const double* R, long k, double* out) const {  // preconditioners.cpp:7-11
#pragma omp parallel for schedule(dynamic, 1)
    for (long j = 0; j < k; ++j) solve(R + j * size(), out + j * size());
  }
  virtual double logdet() const = 0;
  virtual void sample(rng_t& rng, double* z) const = 0;
  void sample_probes(int L, uint64_t seed, double* Z) const {  // preconditioners.cpp:13-20
#pragma omp parallel for schedule(dynamic, 1)
    for (int i = 0; i < L; ++i) {
      rng_t rng = probe_rng(seed, static_cast<uint64_t>(i));
      sample(rng, Z + static_cast<long>(i) * size());
    }
  }
  virtual bool has_derivs() const { return false; }
  virtual void deriv_apply(int, const double*, double*) const { throw std::invalid_argument("preconditioner has no derivative support"); }
  virtual double deriv_trace(int) const { throw std::invalid_argument("preconditioner has no derivative support"); }
};

struct IdentityP : Precond {  // preconditioners.h:39-55
  long n;
  explicit IdentityP(long n_) : n(n_) {}
  long size() const override { return n; }
  int kind() const override { return 0; }
  void solve(const double* r, double* out) const override { std::copy(r, r + n, out); }
  double logdet() const override { return 0.0; }
  void sample(rng_t& rng, double* z) const override { rademacher_fill(rng, z, n); }
};

struct DiagP : Precond {  // preconditioners.cpp:22-37
  std::vector<double> d, sqrt_d;
  std::vector<double> dd[3];
  bool derivs = false;
  DiagP(std::vector<double> d_, const std::vector<double>* der) : d(std::move(d_)) {
    for (double v : d) require(v > 0.0, "diagonal preconditioner needs positive entries");
    sqrt_d.resize(d.size());
    for (size_t i = 0; i < d.size(); ++i) sqrt_d[i] = std::sqrt(d[i]);
    if (der) { for (int k = 0; k < 3; ++k) dd[k] = der[k]; derivs = true; }
  }
  long size() const override { return static_cast<long>(d.size()); }
  int kind() const override { return 1; }
  void solve(const double* r, double* out) const override {
    for (size_t i = 0; i < d.size(); ++i) out[i] = r[i] / d[i];
  }
  double logdet() const override {
    double s = 0.0;
    for (double v : d) s += std::log(v);
    return s;
  }
  void sample(rng_t& rng, double* z) const override {
    gaussian_fill(rng, z, size());
    for (size_t i = 0; i < d.size(); ++i) z[i] = sqrt_d[i] * z[i];
  }
  bool has_derivs() const override { return derivs; }
  void deriv_apply(int k, const double* v, double* out) const override {
    require(derivs, "diagonal preconditioner built without derivatives");
    for (size_t i = 0; i < d.size(); ++i) out[i] = dd[k][i] * v[i];
  }
  double deriv_trace(int k) const override {
    require(derivs, "diagonal preconditioner built without derivatives");
    double s = 0.0;
    for (size_t i = 0; i < d.size(); ++i) s += dd[k][i] / d[i];
    return s;
  }
};

struct FitcP : Precond {  // preconditioners.cpp:39-115
  long n = 0, m = 0;
  Mat sigma_m, sigma_mn, chol_m, chol_core;
  std::vector<double> d, sqrt_d;
  double ld = 0.0;
  bool derivs = false;
  Mat A;
  std::vector<double> d_diag[3];
  Mat dsmn[3], dsm[3];
  std::vector<double> pinv_diag;
  mutable bool have_v0 = false;
  mutable Mat V0, G_M;

  FitcP(const Mat& sm, const Mat& smn, std::vector<double> d_) : sigma_m(sm), sigma_mn(smn), d(std::move(d_)) {
    n = smn.c; m = smn.r;
    for (double v : d) require(v > 0.0, "diagonal part must be positive");
    sqrt_d.resize(d.size());
    for (size_t i = 0; i < d.size(); ++i) sqrt_d[i] = std::sqrt(d[i]);
    chol_m = sigma_m;
    if (!llt(chol_m)) throw NumericalError("preconditioner inducing block is not positive definite");
    Mat scaled(m, n);
#pragma omp parallel for schedule(static)
    for (long j = 0; j < n; ++j)
      for (long i = 0; i < m; ++i) scaled(i, j) = sigma_mn(i, j) * (1.0 / d[static_cast<size_t>(j)]);
    chol_core = sigma_m;
    dgemm('N', 'T', m, m, n, 1.0, scaled.data(), m, sigma_mn.data(), m, 1.0, chol_core.data(), m);
    if (!llt(chol_core)) throw NumericalError("preconditioner core matrix is not positive definite");
    double sl = 0.0;
    for (double v : d) sl += std::log(v);
    ld = llt_logdet(chol_core) - llt_logdet(chol_m) + sl;
  }
  long size() const override { return n; }
  int kind() const override { return 2; }
  // solve (preconditioners.cpp:58-61): two GEMVs per column
  void solve(const double* r, double* out) const override {
    std::vector<double> t(static_cast<size_t>(n)), s(static_cast<size_t>(m), 0.0);
    for (long i = 0; i < n; ++i) t[static_cast<size_t>(i)] = r[i] / d[static_cast<size_t>(i)];
    for (long l = 0; l < n; ++l) {
      const double tl = t[static_cast<size_t>(l)];
      const double* c = sigma_mn.col(l);
      for (long i = 0; i < m; ++i) s[static_cast<size_t>(i)] += c[i] * tl;
    }
    llt_solve(chol_core, s.data(), m, 1);
    for (long l = 0; l < n; ++l) out[l] = t[static_cast<size_t>(l)] - dot(sigma_mn.col(l), s.data(), m) / d[static_cast<size_t>(l)];
  }
  // solve_mat (preconditioners.cpp:63-67)
  void solve_mat(const double* R, long k, double* out) const override {
    Mat T(n, k), S(m, k), W(n, k);
#pragma omp parallel for schedule(static)
    for (long j = 0; j < k; ++j)
      for (long i = 0; i < n; ++i) T(i, j) = (1.0 / d[static_cast<size_t>(i)]) * R[i + j * n];
    dgemm('N', 'N', m, k, n, 1.0, sigma_mn.data(), m, T.data(), n, 0.0, S.data(), m);
    llt_solve(chol_core, S.data(), m, k);
    dgemm('T', 'N', n, k, m, 1.0, sigma_mn.data(), m, S.data(), m, 0.0, W.data(), n);
#pragma omp parallel for schedule(static)
    for (long j = 0; j < k; ++j)
      for (long i = 0; i < n; ++i) out[i + j * n] = T(i, j) - (1.0 / d[static_cast<size_t>(i)]) * W(i, j);
  }
  double logdet() const override { return ld; }
  // sample (preconditioners.cpp:69-73): e1 (m) then e2 (n), fresh N(0,1) objects
  void sample(rng_t& rng, double* z) const override {
    std::vector<double> e1(static_cast<size_t>(m)), e2(static_cast<size_t>(n));
    gaussian_fill(rng, e1.data(), m);
    gaussian_fill(rng, e2.data(), n);
    trsm_lower_t(chol_m, e1.data(), m, 1);
    for (long l = 0; l < n; ++l) z[l] = dot(sigma_mn.col(l), e1.data(), m) + sqrt_d[static_cast<size_t>(l)] * e2[static_cast<size_t>(l)];
  }
  bool has_derivs() const override { return derivs; }
  // deriv_apply (preconditioners.cpp:96-104)
  void deriv_apply(int k, const double* v, double* out) const override {
    require(derivs, "FITC preconditioner built without derivatives");
    for (long i = 0; i < n; ++i) out[i] = d_diag[k][static_cast<size_t>(i)] * v[i];
    if (k == 0) return;
    const Mat& B = dsmn[k];
    std::vector<double> Av(static_cast<size_t>(m), 0.0), Bv(static_cast<size_t>(m), 0.0), DAv(static_cast<size_t>(m), 0.0);
    for (long l = 0; l < n; ++l)
      for (long i = 0; i < m; ++i) {
        Av[static_cast<size_t>(i)] += A(i, l) * v[l];
        Bv[static_cast<size_t>(i)] += B(i, l) * v[l];
      }
    for (long j = 0; j < m; ++j)
      for (long i = 0; i < m; ++i) DAv[static_cast<size_t>(i)] += dsm[k](i, j) * Av[static_cast<size_t>(j)];
    for (long l = 0; l < n; ++l)
      out[l] = (out[l] + (dot(B.col(l), Av.data(), m) + dot(A.col(l), Bv.data(), m))) - dot(A.col(l), DAv.data(), m);
  }
  // deriv_trace (preconditioners.cpp:106-115)
  double deriv_trace(int k) const override {
    require(derivs, "FITC preconditioner built without derivatives");
    double acc = dot(pinv_diag.data(), d_diag[k].data(), n);
    if (k == 0) return acc;
    if (!have_v0) {
      Mat At(n, m);
      for (long j = 0; j < m; ++j)
        for (long i = 0; i < n; ++i) At(i, j) = A(j, i);
      V0 = Mat(n, m);
      solve_mat(At.data(), m, V0.data());
      G_M = Mat(m, m);
      dgemm('N', 'N', m, m, n, 1.0, A.data(), m, V0.data(), n, 0.0, G_M.data(), m);
      have_v0 = true;
    }
    double s1 = 0.0, s2 = 0.0;
    for (long j = 0; j < m; ++j)
      for (long i = 0; i < n; ++i) s1 += V0(i, j) * dsmn[k](j, i);
    for (long j = 0; j < m; ++j)
      for (long i = 0; i < m; ++i) s2 += G_M(i, j) * dsm[k](i, j);
    acc += 2.0 * s1;
    acc -= s2;
    return acc;
  }
};

FitcP* fitc_from_fsa(Model& md, bool with_derivs) {  // preconditioners.cpp:75-94
  auto p = std::make_unique<FitcP>(md.sigma_m, md.sigma_mn, csr_diag(md.sigma_s));
  if (!with_derivs) return p.release();
  md.ensure_rho_derivs();
  p->derivs = true;
  p->A = md.A;
  const long n = md.n, m = md.m;
  p->d_diag[0].assign(static_cast<size_t>(n), 1.0);
  p->d_diag[1].resize(static_cast<size_t>(n));
  for (long i = 0; i < n; ++i) p->d_diag[1][static_cast<size_t>(i)] = (p->d[static_cast<size_t>(i)] - md.sigma2) / md.sigma1_2;
  p->d_diag[2] = csr_diag(md.ds_rho);
  p->dsmn[1] = md.sigma_mn;
  for (double& v : p->dsmn[1].a) v /= md.sigma1_2;
  p->dsmn[2] = md.P1;
  p->dsm[1] = md.sigma_m;
  for (double& v : p->dsm[1].a) v /= md.sigma1_2;
  p->dsm[2] = md.dsm_rho;
  Mat V = p->sigma_mn;
  trsm_lower(p->chol_core, V.data(), m, n);
  p->pinv_diag.resize(static_cast<size_t>(n));
  for (long i = 0; i < n; ++i) {
    const double di = p->d[static_cast<size_t>(i)];
    p->pinv_diag[static_cast<size_t>(i)] = 1.0 / di - dot(V.col(i), V.col(i), m) / (di * di);
  }
  return p.release();
}

Precond* make_preconditioner(Model& md, int type) {  // estimation.cpp:160-176
  switch (type) {
    case 0: return new IdentityP(md.n);
    case 1: {
      md.ensure_rho_derivs();
      std::vector<double> der[3];
      der[0].assign(static_cast<size_t>(md.n), 1.0);
      der[1] = csr_diag(md.sigma_s);
      for (double& v : der[1]) v = (v - md.sigma2) / md.sigma1_2;  // diag of (sigma_s - sigma2 I)/sigma1_2
      der[2] = csr_diag(md.ds_rho);
      return new DiagP(csr_diag(md.sigma_s), der);
    }
    case 2: return fitc_from_fsa(md, true);
  }
  throw std::invalid_argument("unknown preconditioner type");
}

// ---- Krylov (krylov.cpp:18-206) ---------------------------------------------
struct LinOp {
  long n;
  std::function<void(const double*, long, double*)> apply_mat;
};

struct CgResult {
  std::vector<double> X;
  std::vector<int> iterations;
  std::vector<char> converged;
  std::vector<std::vector<double>> tdiag, toff;
  std::vector<std::vector<double>> rnorm;  // ||r||_2 after each iteration (test diagnostics: tie margins)
  int sweeps = 0;
  bool all_converged() const {
    for (char c : converged) if (!c) return false;
    return true;
  }
  int max_iterations() const {
    int m = 0;
    for (int v : iterations) m = std::max(m, v);
    return m;
  }
};

// pcg_solve_multi (krylov.cpp:18-106)
CgResult pcg_solve_multi(const LinOp& A, const Precond& P, const double* B, long k, double tol,
                         int max_iter, bool batched, bool error_on_max_iter = false) {
  const long n = A.n;
  require(P.size() == n, "cg: dimension mismatch");
  require(tol > 0.0 && max_iter > 0, "cg: invalid options");
  CgResult res;
  res.X.assign(static_cast<size_t>(n * k), 0.0);
  res.iterations.assign(static_cast<size_t>(k), 0);
  res.converged.assign(static_cast<size_t>(k), 0);
  res.tdiag.resize(static_cast<size_t>(k));
  res.toff.resize(static_cast<size_t>(k));
  res.rnorm.resize(static_cast<size_t>(k));
  std::vector<double> R(B, B + n * k), H(static_cast<size_t>(n * k), 0.0), V(static_cast<size_t>(n * k), 0.0);
  std::vector<double> rz(static_cast<size_t>(k), 0.0), ap(static_cast<size_t>(k), 1.0), bp(static_cast<size_t>(k), 0.0);
  std::vector<char> active(static_cast<size_t>(k), 1);
  auto colp = [&](std::vector<double>& M, long j) { return M.data() + j * n; };
  std::string err;
  long num_active = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : num_active)
  for (long j = 0; j < k; ++j) {
    double* r = colp(R, j);
    if (std::sqrt(dot(r, r, n)) < tol) {
      res.converged[static_cast<size_t>(j)] = 1;
      active[static_cast<size_t>(j)] = 0;
      continue;
    }
    std::vector<double> z(static_cast<size_t>(n));
    P.solve(r, z.data());
    rz[static_cast<size_t>(j)] = dot(r, z.data(), n);
    if (!(rz[static_cast<size_t>(j)] > 0.0)) {
#pragma omp critical
      err = "cg: preconditioner is not positive definite";
    }
    std::copy(z.begin(), z.end(), colp(H, j));
    ++num_active;
  }
  if (!err.empty()) throw NumericalError(err);
  for (int it = 0; it < max_iter && num_active > 0; ++it) {
    if (batched) {
      A.apply_mat(H.data(), k, V.data());
    } else {
#pragma omp parallel for schedule(dynamic, 1)
      for (long j = 0; j < k; ++j)
        if (active[static_cast<size_t>(j)]) A.apply_mat(colp(H, j), 1, colp(V, j));
    }
    long dropped = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(+ : dropped)
    for (long j = 0; j < k; ++j) {
      const size_t sj = static_cast<size_t>(j);
      if (!active[sj]) continue;
      double* h = colp(H, j);
      double* v = colp(V, j);
      double* r = colp(R, j);
      double* x = res.X.data() + j * n;
      const double hv = dot(h, v, n);
      if (!(hv > 0.0)) {
#pragma omp critical
        err = "cg: operator is not positive definite";
        continue;
      }
      const double alpha = rz[sj] / hv;
      res.tdiag[sj].push_back(1.0 / alpha + bp[sj] / ap[sj]);
      if (it > 0) res.toff[sj].push_back(std::sqrt(bp[sj]) / ap[sj]);
      for (long i = 0; i < n; ++i) x[i] += alpha * h[i];
      for (long i = 0; i < n; ++i) r[i] -= alpha * v[i];
      res.iterations[sj] = it + 1;
      const double rn = std::sqrt(dot(r, r, n));
      res.rnorm[sj].push_back(rn);
      if (rn < tol) {
        res.converged[sj] = 1;
        active[sj] = 0;
        ++dropped;
        continue;
      }
      std::vector<double> z(static_cast<size_t>(n));
      P.solve(r, z.data());
      const double rz_new = dot(r, z.data(), n);
      if (!(rz_new > 0.0)) {
#pragma omp critical
        err = "cg: preconditioner is not positive definite";
        continue;
      }
      const double beta = rz_new / rz[sj];
      for (long i = 0; i < n; ++i) h[i] = z[static_cast<size_t>(i)] + beta * h[i];
      bp[sj] = beta;
      ap[sj] = alpha;
      rz[sj] = rz_new;
    }
    if (!err.empty()) throw NumericalError(err);
    num_active -= dropped;
    ++res.sweeps;
  }
  if (num_active > 0 && error_on_max_iter) throw NumericalError("cg: no convergence within max_iter");
  return res;
}

// tridiag_log_quadrature (krylov.cpp:120-142): e1' log(T) e1 from the
// eigen-decomposition of the symmetric tridiagonal (implicit QL, tracking the
// first row of the eigenvector matrix).
double tridiag_log_quadrature(const double* diag, const double* off, long len) {
  if (len == 0) return 0.0;
  std::vector<double> d(diag, diag + len), e(static_cast<size_t>(len), 0.0), z(static_cast<size_t>(len), 0.0);
  for (long i = 0; i + 1 < len; ++i) e[static_cast<size_t>(i)] = off[i];
  z[0] = 1.0;
  const long n = len;
  for (long l = 0; l < n; ++l) {
    int iter = 0;
    long mm;
    do {
      for (mm = l; mm < n - 1; ++mm) {
        const double dd = std::fabs(d[static_cast<size_t>(mm)]) + std::fabs(d[static_cast<size_t>(mm + 1)]);
        if (std::fabs(e[static_cast<size_t>(mm)]) <= std::numeric_limits<double>::epsilon() * dd) break;
      }
      if (mm != l) {
        if (iter++ == 60) throw NumericalError("tridiagonal eigendecomposition failed");
        double g = (d[static_cast<size_t>(l + 1)] - d[static_cast<size_t>(l)]) / (2.0 * e[static_cast<size_t>(l)]);
        double r = std::hypot(g, 1.0);
        g = d[static_cast<size_t>(mm)] - d[static_cast<size_t>(l)] + e[static_cast<size_t>(l)] / (g + std::copysign(r, g));
        double s = 1.0, c = 1.0, p = 0.0;
        long i;
        bool early = false;
        for (i = mm - 1; i >= l; --i) {
          double f = s * e[static_cast<size_t>(i)];
          const double b = c * e[static_cast<size_t>(i)];
          r = std::hypot(f, g);
          e[static_cast<size_t>(i + 1)] = r;
          if (r == 0.0) {
            d[static_cast<size_t>(i + 1)] -= p;
            e[static_cast<size_t>(mm)] = 0.0;
            early = true;
            break;
          }
          s = f / r;
          c = g / r;
          g = d[static_cast<size_t>(i + 1)] - p;
          r = (d[static_cast<size_t>(i)] - g) * s + 2.0 * c * b;
          p = s * r;
          d[static_cast<size_t>(i + 1)] = g + p;
          g = c * r - b;
          f = z[static_cast<size_t>(i + 1)];
          z[static_cast<size_t>(i + 1)] = s * z[static_cast<size_t>(i)] + c * f;
          z[static_cast<size_t>(i)] = c * z[static_cast<size_t>(i)] - s * f;
        }
        if (early) continue;
        d[static_cast<size_t>(l)] -= p;
        e[static_cast<size_t>(l)] = g;
        e[static_cast<size_t>(mm)] = 0.0;
      }
    } while (mm != l);
  }
  double q = 0.0;
  for (long i = 0; i < n; ++i) {
    const double lambda = d[static_cast<size_t>(i)];
    if (!(lambda > 0.0)) throw NumericalError("tridiagonal has a nonpositive Ritz value");
    q += z[static_cast<size_t>(i)] * z[static_cast<size_t>(i)] * std::log(lambda);
  }
  return q;
}

enum Cv { CV_NONE = 0, CV_ONE = 1, CV_OPTIMAL = 2 };
struct TraceEstimate { double value = 0.0, c_hat = 0.0, var_of_mean = 0.0; };

// ste_grad_trace (krylov.cpp:163-206)
TraceEstimate ste_grad_trace(Model& md, const double* Z, const double* W, long L, const Precond& P, int which, int mode) {
  const long n = md.n;
  require(L > 0, "ste: probe shape mismatch");
  std::vector<double> Y(static_cast<size_t>(n * L)), dAY(static_cast<size_t>(n * L));
  P.solve_mat(Z, L, Y.data());
  md.deriv_matmat(which, Y.data(), L, dAY.data());
  std::vector<double> a(static_cast<size_t>(L));
  for (long i = 0; i < L; ++i) a[static_cast<size_t>(i)] = dot(W + i * n, dAY.data() + i * n, n);
  TraceEstimate est;
  const double dl = static_cast<double>(L);
  double abar = 0.0;
  for (double v : a) abar += v;
  abar /= dl;
  if (mode == CV_NONE || !P.has_derivs()) {
    est.value = abar;
    if (L > 1) {
      double s = 0.0;
      for (double v : a) s += (v - abar) * (v - abar);
      est.var_of_mean = s / (dl - 1.0) / dl;
    }
    return est;
  }
  std::vector<double> b(static_cast<size_t>(L));
#pragma omp parallel for schedule(dynamic, 1)
  for (long i = 0; i < L; ++i) {
    std::vector<double> t(static_cast<size_t>(n));
    P.deriv_apply(which, Y.data() + i * n, t.data());
    b[static_cast<size_t>(i)] = dot(Y.data() + i * n, t.data(), n);
  }
  const double exact_b = P.deriv_trace(which);
  double bbar = 0.0;
  for (double v : b) bbar += v;
  bbar /= dl;
  double c = 1.0;
  if (mode == CV_OPTIMAL) {
    double sbb = 0.0, sab = 0.0, mx = 0.0;
    for (long i = 0; i < L; ++i) {
      sbb += (b[static_cast<size_t>(i)] - bbar) * (b[static_cast<size_t>(i)] - bbar);
      sab += (a[static_cast<size_t>(i)] - abar) * (b[static_cast<size_t>(i)] - bbar);
      mx = std::max(mx, std::fabs(b[static_cast<size_t>(i)]));
    }
    const double scale = std::max(mx, 1.0);
    c = sbb > dl * 1e-28 * scale * scale ? sab / sbb : 0.0;
  }
  est.c_hat = c;
  est.value = abar - c * (bbar - exact_b);
  if (L > 1) {
    std::vector<double> dv(static_cast<size_t>(L));
    double dm = 0.0;
    for (long i = 0; i < L; ++i) { dv[static_cast<size_t>(i)] = a[static_cast<size_t>(i)] - c * (b[static_cast<size_t>(i)] - exact_b); dm += dv[static_cast<size_t>(i)]; }
    dm /= dl;
    double s = 0.0;
    for (double v : dv) s += (v - dm) * (v - dm);
    est.var_of_mean = s / (dl - 1.0) / dl;
  }
  return est;
}

LinOp fsa_operator(const Model& md) {  // krylov.cpp:10-16
  LinOp op;
  op.n = md.n;
  op.apply_mat = [&md](const double* V, long k, double* Y) { md.matmat(V, k, Y); };
  return op;
}
LinOp sigma_s_operator(const Model& md) {  // prediction.cpp:90-93
  LinOp op;
  op.n = md.n;
  op.apply_mat = [&md](const double* V, long k, double* Y) { md.sigma_s_mat(V, k, Y); };
  return op;
}

// Cholesky solve of a small SPD system (the LDLT of estimation.cpp:207)
std::vector<double> small_spd_solve(std::vector<double> G, long p, std::vector<double> b) {
  Mat M(p, p);
  M.a = std::move(G);
  if (!llt(M)) throw NumericalError("nll: GLS normal matrix is not positive definite");
  llt_solve(M, b.data(), p, 1);
  return b;
}

struct NllOut {
  double nll, g[3], logdet;
  int cg_iterations;
  std::vector<double> beta;
  CgResult sol;  // the [Z | y | X] solve (test diagnostics: per-column counts, residual norms, X)
};

// iterative_nll_grad (estimation.cpp:178-227)
NllOut iterative_nll_grad(Model& md, const Precond& P, const double* y, const double* X, long p, int L,
                          uint64_t seed, double tol, int max_iter, int cv, bool want_grad) {
  const long n = md.n;
  require(L > 0, "nll: need at least one probe");
  const long k = L + 1 + p;
  std::vector<double> B(static_cast<size_t>(n * k));
  P.sample_probes(L, seed, B.data());
  std::copy(y, y + n, B.data() + static_cast<long>(L) * n);
  if (p > 0) std::copy(X, X + n * p, B.data() + static_cast<long>(L + 1) * n);
  CgResult sol = pcg_solve_multi(fsa_operator(md), P, B.data(), k, tol, max_iter, true);
  if (!sol.all_converged()) throw NumericalError("nll: cg did not converge");
  NllOut out;
  out.cg_iterations = sol.max_iterations();
  double acc = 0.0;
  for (int i = 0; i < L; ++i)
    acc += tridiag_log_quadrature(sol.tdiag[static_cast<size_t>(i)].data(), sol.toff[static_cast<size_t>(i)].data(),
                                  static_cast<long>(sol.tdiag[static_cast<size_t>(i)].size()));
  out.logdet = static_cast<double>(n) / static_cast<double>(L) * acc + P.logdet();
  std::vector<double> u(sol.X.begin() + static_cast<long>(L) * n, sol.X.begin() + static_cast<long>(L + 1) * n);
  std::vector<double> resid(y, y + n);
  if (p > 0) {
    const double* SX = sol.X.data() + static_cast<long>(L + 1) * n;
    std::vector<double> G(static_cast<size_t>(p * p)), rhs(static_cast<size_t>(p));
    for (long a = 0; a < p; ++a)
      for (long b2 = 0; b2 < p; ++b2) G[static_cast<size_t>(a + b2 * p)] = dot(X + a * n, SX + b2 * n, n);
    std::vector<double> Gs(G);
    for (long a = 0; a < p; ++a)
      for (long b2 = 0; b2 < p; ++b2) Gs[static_cast<size_t>(a + b2 * p)] = 0.5 * (G[static_cast<size_t>(a + b2 * p)] + G[static_cast<size_t>(b2 + a * p)]);
    for (long a = 0; a < p; ++a) rhs[static_cast<size_t>(a)] = dot(SX + a * n, y, n);
    out.beta = small_spd_solve(Gs, p, rhs);
    for (long a = 0; a < p; ++a)
      for (long i = 0; i < n; ++i) {
        u[static_cast<size_t>(i)] -= SX[i + a * n] * out.beta[static_cast<size_t>(a)];
        resid[static_cast<size_t>(i)] -= X[i + a * n] * out.beta[static_cast<size_t>(a)];
      }
  }
  constexpr double log2pi = 1.8378770664093454836;
  out.nll = 0.5 * (out.logdet + dot(resid.data(), u.data(), n) + static_cast<double>(n) * log2pi);
  out.g[0] = out.g[1] = out.g[2] = 0.0;
  if (want_grad) {
    const double* Z = B.data();
    const double* W = sol.X.data();
    for (int kk = 0; kk < 3; ++kk) {
      TraceEstimate tr = ste_grad_trace(md, Z, W, L, P, kk, cv);
      std::vector<double> du(static_cast<size_t>(n));
      md.deriv_matmat(kk, u.data(), 1, du.data());
      out.g[kk] = 0.5 * (tr.value - dot(u.data(), du.data(), n));
    }
  }
  out.sol = std::move(sol);
  return out;
}

// ---- prediction (prediction.cpp:7-172) ---------------------------------------
struct Pred {
  Locs locs;
  long np = 0;
  Mat sigma_mnp, C;
  Csr sigma_s_np;
};

Pred* make_prediction_set(const Model& md, const Locs& pl) {  // prediction.cpp:7-27
  require(pl.n > 0, "prediction: empty location set");
  require(pl.d == md.locs.d, "prediction: dimension mismatch");
  auto P = std::make_unique<Pred>();
  P->locs = pl;
  P->np = pl.n;
  const long m = md.m;
  P->sigma_mnp = cross_cov(md.ind, pl, md.nu, md.sigma1_2, md.rho, false);
  P->C = P->sigma_mnp;
  llt_solve(md.chol_m, P->C.data(), m, pl.n);
  Mat Up = P->sigma_mnp;
  trsm_lower(md.chol_m, Up.data(), m, pl.n);
  Csr cross = taper_pattern(md.locs, md.gamma, true, &pl);
#pragma omp parallel for schedule(dynamic, 256)
  for (long r = 0; r < cross.rows; ++r)
    for (long p = cross.ptr[static_cast<size_t>(r)]; p < cross.ptr[static_cast<size_t>(r + 1)]; ++p) {
      const double dd = cross.val[static_cast<size_t>(p)];
      const double resid = matern(dd, md.nu, md.sigma1_2, md.rho) - dot(md.U.col(r), Up.col(cross.idx[static_cast<size_t>(p)]), m);
      cross.val[static_cast<size_t>(p)] = resid * taper_value(dd, md.family, md.gamma);
    }
  P->sigma_s_np = std::move(cross);
  return P.release();
}

// cross_apply_t (prediction.cpp:29-31)
void cross_apply_t(const Model& md, const Pred& P, const double* u, double* out) {
  const long n = md.n, m = md.m, np = P.np;
  std::vector<double> su(static_cast<size_t>(m)), ct(static_cast<size_t>(np));
  dgemm('N', 'N', m, 1, n, 1.0, md.sigma_mn.data(), m, u, n, 0.0, su.data(), m);
  dgemm('T', 'N', np, 1, m, 1.0, P.C.data(), m, su.data(), m, 0.0, ct.data(), np);
  spmm_t(P.sigma_s_np, u, n, 1, out, np);
  for (long j = 0; j < np; ++j) out[j] += ct[static_cast<size_t>(j)];
}

struct PredVar { std::vector<double> var, se; int clamped = 0, cg_iterations = 0; };

struct DetPieces { std::vector<double> d1, d2, d3; int cg_iterations = 0; };

DetPieces deterministic_pieces(Model& md, const Pred& P, double tol, int maxit, double tol_s, int maxit_s) {
  const long n = md.n, m = md.m, np = P.np;  // prediction.cpp:72-110
  DetPieces out;
  std::unique_ptr<FitcP> fitc(fitc_from_fsa(md, false));
  Mat SmnT(n, m);
  for (long j = 0; j < m; ++j)
    for (long i = 0; i < n; ++i) SmnT(i, j) = md.sigma_mn(j, i);
  CgResult x1 = pcg_solve_multi(fsa_operator(md), *fitc, SmnT.data(), m, tol, maxit, true);
  if (!x1.all_converged()) throw NumericalError("prediction: cg did not converge");
  out.cg_iterations = x1.max_iterations();
  Mat K1(m, m), CtK(np, m), Z2(np, m);
  dgemm('N', 'N', m, m, n, 1.0, md.sigma_mn.data(), m, x1.X.data(), n, 0.0, K1.data(), m);
  dgemm('T', 'N', np, m, m, 1.0, P.C.data(), m, K1.data(), m, 0.0, CtK.data(), np);
  out.d1.assign(static_cast<size_t>(np), 0.0);
  for (long j = 0; j < m; ++j)
    for (long i = 0; i < np; ++i) out.d1[static_cast<size_t>(i)] += CtK(i, j) * P.C(j, i);
  spmm_t(P.sigma_s_np, x1.X.data(), n, m, Z2.data(), np);
  out.d2.assign(static_cast<size_t>(np), 0.0);
  for (long j = 0; j < m; ++j)
    for (long i = 0; i < np; ++i) out.d2[static_cast<size_t>(i)] += Z2(i, j) * P.C(j, i);
  DiagP jacobi(csr_diag(md.sigma_s), nullptr);
  CgResult x2 = pcg_solve_multi(sigma_s_operator(md), jacobi, SmnT.data(), m, tol_s, maxit_s, true);
  if (!x2.all_converged()) throw NumericalError("prediction: cg did not converge");
  out.cg_iterations = std::max(out.cg_iterations, x2.max_iterations());
  Mat M = md.sigma_m;
  dgemm('N', 'N', m, m, n, 1.0, md.sigma_mn.data(), m, x2.X.data(), n, 1.0, M.data(), m);
  Mat Ms(m, m);
  for (long j = 0; j < m; ++j)
    for (long i = 0; i < m; ++i) Ms(i, j) = 0.5 * (M(i, j) + M(j, i));
  if (!llt(Ms)) throw NumericalError("prediction: core matrix is not positive definite");
  Mat Z3t(np, m), Z3(m, np);
  spmm_t(P.sigma_s_np, x2.X.data(), n, m, Z3t.data(), np);  // (X2^T S_np)^T = S_np^T X2
  for (long j = 0; j < np; ++j)
    for (long i = 0; i < m; ++i) Z3(i, j) = Z3t(j, i);
  trsm_lower(Ms, Z3.data(), m, np);
  out.d3.assign(static_cast<size_t>(np), 0.0);
  for (long j = 0; j < np; ++j) out.d3[static_cast<size_t>(j)] = dot(Z3.col(j), Z3.col(j), m);
  return out;
}

PredVar predict_var_sim(Model& md, const Pred& P, int L, uint64_t seed, double tol, int maxit, double tol_s,
                        int maxit_s, bool cv, double floor_rel) {  // prediction.cpp:131-172
  DetPieces det = deterministic_pieces(md, P, tol, maxit, tol_s, maxit_s);
  const long n = md.n, np = P.np;
  DiagP jacobi(csr_diag(md.sigma_s), nullptr);
  int max_it = det.cg_iterations;
  auto quad_mat = [&](const double* Z, long b, double* out) {
    std::vector<double> G(static_cast<size_t>(n * b));
    spmm(P.sigma_s_np, Z, np, b, G.data(), n);
    CgResult sol = pcg_solve_multi(sigma_s_operator(md), jacobi, G.data(), b, tol_s, maxit_s, true);
    if (!sol.all_converged()) throw NumericalError("prediction: cg did not converge");
    max_it = std::max(max_it, sol.max_iterations());
    spmm_t(P.sigma_s_np, sol.X.data(), n, b, out, np);
  };
  std::vector<double> diag(static_cast<size_t>(np)), se(static_cast<size_t>(np), 0.0);
  const int batch = 256;
  if (!cv) {  // stochastic_diag (krylov.cpp:230-248)
    require(L > 0, "stochastic_diag: invalid options");
    std::vector<double> s(static_cast<size_t>(np), 0.0), s2(static_cast<size_t>(np), 0.0);
    int done = 0;
    while (done < L) {
      const int b = std::min(batch, L - done);
      std::vector<double> Z(static_cast<size_t>(np * b)), Q(static_cast<size_t>(np * b));
      for (int j = 0; j < b; ++j) {
        rng_t rng = probe_rng(seed, static_cast<uint64_t>(done + j));
        rademacher_fill(rng, Z.data() + static_cast<long>(j) * np, np);
      }
      quad_mat(Z.data(), b, Q.data());
      for (long i = 0; i < np; ++i) {
        double rs = 0.0, rs2 = 0.0;
        for (int j = 0; j < b; ++j) {
          const double v = Z[static_cast<size_t>(i + j * np)] * Q[static_cast<size_t>(i + j * np)];
          rs += v;
          rs2 += v * v;
        }
        s[static_cast<size_t>(i)] += rs;
        s2[static_cast<size_t>(i)] += rs2;
      }
      done += b;
    }
    const double l = static_cast<double>(L);
    for (long i = 0; i < np; ++i) {
      diag[static_cast<size_t>(i)] = s[static_cast<size_t>(i)] / l;
      if (L > 1) {
        const double var = (s2[static_cast<size_t>(i)] - l * diag[static_cast<size_t>(i)] * diag[static_cast<size_t>(i)]) / (l - 1.0);
        se[static_cast<size_t>(i)] = std::sqrt(std::max(var, 0.0) / l);
      }
    }
  } else {  // stochastic_diag_cv (krylov.cpp:250-291) + control (prediction.cpp:151-164)
    require(L > 1, "stochastic_diag_cv: needs at least two probes");
    const std::vector<double> ds = csr_diag(md.sigma_s);
    std::vector<double> cdiag(static_cast<size_t>(np), 0.0);
    for (long r = 0; r < n; ++r)
      for (long p = P.sigma_s_np.ptr[static_cast<size_t>(r)]; p < P.sigma_s_np.ptr[static_cast<size_t>(r + 1)]; ++p)
        cdiag[static_cast<size_t>(P.sigma_s_np.idx[static_cast<size_t>(p)])] += P.sigma_s_np.val[static_cast<size_t>(p)] * P.sigma_s_np.val[static_cast<size_t>(p)] / ds[static_cast<size_t>(r)];
    std::vector<double> sa(static_cast<size_t>(np), 0.0), sa2(sa), sb(sa), sb2(sa), sab(sa);
    int done = 0;
    while (done < L) {
      const int b = std::min(batch, L - done);
      std::vector<double> Z(static_cast<size_t>(np * b)), Q(static_cast<size_t>(np * b)), Gc(static_cast<size_t>(n * b)), Qc(static_cast<size_t>(np * b));
      for (int j = 0; j < b; ++j) {
        rng_t rng = probe_rng(seed, static_cast<uint64_t>(done + j));
        rademacher_fill(rng, Z.data() + static_cast<long>(j) * np, np);
      }
      quad_mat(Z.data(), b, Q.data());
      spmm(P.sigma_s_np, Z.data(), np, b, Gc.data(), n);
      for (int j = 0; j < b; ++j)
        for (long i = 0; i < n; ++i) Gc[static_cast<size_t>(i + j * n)] /= ds[static_cast<size_t>(i)];
      spmm_t(P.sigma_s_np, Gc.data(), n, b, Qc.data(), np);
      for (long i = 0; i < np; ++i) {
        double ra = 0, ra2 = 0, rb = 0, rb2 = 0, rab = 0;
        for (int j = 0; j < b; ++j) {
          const double z = Z[static_cast<size_t>(i + j * np)];
          const double va = z * Q[static_cast<size_t>(i + j * np)], vb = z * Qc[static_cast<size_t>(i + j * np)];
          ra += va; ra2 += va * va; rb += vb; rb2 += vb * vb; rab += va * vb;
        }
        sa[static_cast<size_t>(i)] += ra; sa2[static_cast<size_t>(i)] += ra2; sb[static_cast<size_t>(i)] += rb;
        sb2[static_cast<size_t>(i)] += rb2; sab[static_cast<size_t>(i)] += rab;
      }
      done += b;
    }
    const double l = static_cast<double>(L);
    for (long i = 0; i < np; ++i) {
      const size_t si = static_cast<size_t>(i);
      const double ab = sa[si] / l, bb = sb[si] / l;
      const double va = std::max((sa2[si] - l * ab * ab) / (l - 1.0), 0.0);
      const double vb = std::max((sb2[si] - l * bb * bb) / (l - 1.0), 0.0);
      const double cab = (sab[si] - l * (ab * bb)) / (l - 1.0);
      const double scale = std::max(std::fabs(bb), 1.0);
      const double c = vb > 1e-28 * scale * scale ? cab / vb : 0.0;
      diag[si] = ab - c * (bb - cdiag[si]);
      se[si] = std::sqrt(std::max(va - 2.0 * c * cab + c * c * vb, 0.0) / l);
    }
  }
  PredVar out;  // combine_pieces (prediction.cpp:112-127)
  const double prior = md.sigma1_2 + md.sigma2;
  const double floor = md.sigma2 * floor_rel;
  out.var.resize(static_cast<size_t>(np));
  for (long j = 0; j < np; ++j) {
    const size_t sj = static_cast<size_t>(j);
    double v = prior - det.d1[sj] - 2.0 * det.d2[sj] + det.d3[sj] - diag[sj];
    if (v < floor) { v = floor; ++out.clamped; }
    out.var[sj] = v;
  }
  out.se = se;
  out.cg_iterations = max_it;
  return out;
}

}  // namespace orc

// =============================================================================
// C ABI for the Python test harness (ctypes).
// =============================================================================
using namespace orc;

namespace {
thread_local std::string g_err;
template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 2;
  } catch (const NumericalError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 4;
  }
}
Locs mk_locs(const double* c, long n, int d) {
  Locs L;
  L.n = n;
  L.d = d;
  L.c.assign(c, c + n * d);
  return L;
}
}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

uint64_t orc_splitmix64(uint64_t x) { return splitmix64(x); }
void orc_probe_gaussian(uint64_t seed, uint64_t i, long n1, double* e1, long n2, double* e2) {
  rng_t rng = probe_rng(seed, i);
  if (n1 > 0) gaussian_fill(rng, e1, n1);
  if (n2 > 0) gaussian_fill(rng, e2, n2);
}
void orc_probe_rademacher(uint64_t seed, uint64_t i, long n, double* z) {
  rng_t rng = probe_rng(seed, i);
  rademacher_fill(rng, z, n);
}
uint64_t orc_mt19937_64_nth(uint64_t seed, long nth) {
  rng_t rng(seed);
  uint64_t v = 0;
  for (long i = 0; i < nth; ++i) v = rng();
  return v;
}
double orc_matern(double d, int nu, double s1, double rho) { return matern(d, nu, s1, rho); }
double orc_matern_drho(double d, int nu, double s1, double rho) { return matern_drho(d, nu, s1, rho); }
double orc_taper_value(double d, int family, double gamma) { return taper_value(d, family, gamma); }
double orc_rho_for_correlation_at(double dist, double corr, int nu) { return rho_for_correlation_at(dist, corr, nu); }
double orc_effective_range(double rho, int nu) { return effective_range(rho, nu); }
double orc_gamma_for_avg_row_nnz(long n, double target) {  // locations.cpp:192-195
  return std::sqrt(target / (static_cast<double>(n) * M_PI));
}
int orc_uniform_locations(long n, int d, uint64_t seed, double* out) {
  return guard([&] { uniform_locations(n, d, seed, out); });
}
int orc_select_random(const double* c, long n, int d, long m, uint64_t seed, double* out) {
  return guard([&] { select_random(mk_locs(c, n, d), m, seed, out); });
}
int orc_select_kmeanspp(const double* c, long n, int d, long m, uint64_t seed, int max_iter, double rel_tol, double* out) {
  return guard([&] { select_kmeanspp(mk_locs(c, n, d), m, seed, max_iter, rel_tol, out); });
}

// pattern: returns nnz via *nnz; call twice (first with null arrays)
struct orc_csr { Csr c; };
int orc_taper_pattern(const double* c, long n, int d, double gamma, const double* pc, long np, orc_csr** out, long* nnz) {
  return guard([&] {
    Locs L = mk_locs(c, n, d);
    auto r = std::make_unique<orc_csr>();
    if (pc) {
      Locs P = mk_locs(pc, np, d);
      r->c = taper_pattern(L, gamma, true, &P);
    } else {
      r->c = taper_pattern(L, gamma, false, nullptr);
    }
    *nnz = r->c.nnz();
    *out = r.release();
  });
}
void orc_csr_copy(const orc_csr* s, long* ptr, int* idx, double* val) {
  std::copy(s->c.ptr.begin(), s->c.ptr.end(), ptr);
  std::copy(s->c.idx.begin(), s->c.idx.end(), idx);
  std::copy(s->c.val.begin(), s->c.val.end(), val);
}
void orc_csr_free(orc_csr* s) { delete s; }

int orc_assemble(const double* c, long n, int d, const double* ind, long m, int nu, int fam, double gamma,
                 double s2, double s12, double rho, double jitter_rel, void** out) {
  return guard([&] { *out = assemble(mk_locs(c, n, d), mk_locs(ind, m, d), nu, fam, gamma, s2, s12, rho, jitter_rel); });
}
void orc_model_free(void* md) { delete static_cast<Model*>(md); }
// info: [n, m, nnz, n_clamped, logdet_sigma_m]
void orc_model_info(void* mdv, double* info) {
  Model& md = *static_cast<Model*>(mdv);
  info[0] = static_cast<double>(md.n);
  info[1] = static_cast<double>(md.m);
  info[2] = static_cast<double>(md.sigma_s.nnz());
  info[3] = static_cast<double>(md.n_clamped);
  info[4] = md.logdet_sigma_m;
}
// which: 0 dists, 1 sigma_s, 2 d sigma_s / d rho
int orc_model_csr(void* mdv, int which, long* ptr, int* idx, double* val) {
  return guard([&] {
    Model& md = *static_cast<Model*>(mdv);
    if (which == 2) md.ensure_rho_derivs();
    const Csr& s = which == 0 ? md.dists : which == 1 ? md.sigma_s : md.ds_rho;
    std::copy(s.ptr.begin(), s.ptr.end(), ptr);
    std::copy(s.idx.begin(), s.idx.end(), idx);
    std::copy(s.val.begin(), s.val.end(), val);
  });
}
// which: 0 sigma_m (m x m), 1 sigma_mn, 2 U, 3 A, 4 P1, 5 W2 (m x n), 6 lowrank_diag (n), 7 chol_m, 8 dsigma_m/drho
int orc_model_dense(void* mdv, int which, double* out) {
  return guard([&] {
    Model& md = *static_cast<Model*>(mdv);
    if (which == 4 || which == 5 || which == 8) md.ensure_rho_derivs();
    const std::vector<double>* v = nullptr;
    switch (which) {
      case 0: v = &md.sigma_m.a; break;
      case 1: v = &md.sigma_mn.a; break;
      case 2: v = &md.U.a; break;
      case 3: v = &md.A.a; break;
      case 4: v = &md.P1.a; break;
      case 5: v = &md.W2.a; break;
      case 6: v = &md.lowrank_diag; break;
      case 7: v = &md.chol_m.a; break;
      case 8: v = &md.dsm_rho.a; break;
      default: throw std::invalid_argument("unknown block");
    }
    std::copy(v->begin(), v->end(), out);
  });
}
int orc_matmat(void* mdv, const double* V, long k, double* out) {
  return guard([&] { static_cast<Model*>(mdv)->matmat(V, k, out); });
}
int orc_deriv_matmat(void* mdv, int which, const double* V, long k, double* out) {
  return guard([&] { static_cast<Model*>(mdv)->deriv_matmat(which, V, k, out); });
}
int orc_make_preconditioner(void* mdv, int type, void** out) {
  return guard([&] { *out = make_preconditioner(*static_cast<Model*>(mdv), type); });
}
int orc_fitc_plain(void* mdv, void** out) {  // FitcPrecond::from_fsa(model, false)
  return guard([&] { *out = fitc_from_fsa(*static_cast<Model*>(mdv), false); });
}
int orc_jacobi(void* mdv, void** out) {  // DiagPrecond(sigma_s.diagonal())
  return guard([&] { *out = new DiagP(csr_diag(static_cast<Model*>(mdv)->sigma_s), nullptr); });
}
void orc_precond_free(void* p) { delete static_cast<Precond*>(p); }
double orc_precond_logdet(void* p) { return static_cast<Precond*>(p)->logdet(); }
int orc_precond_kind(void* p) { return static_cast<Precond*>(p)->kind(); }
int orc_precond_solve_mat(void* p, const double* R, long k, double* out) {
  return guard([&] { static_cast<Precond*>(p)->solve_mat(R, k, out); });
}
int orc_precond_solve_cols(void* p, const double* R, long k, double* out) {
  return guard([&] {
    Precond* P = static_cast<Precond*>(p);
    for (long j = 0; j < k; ++j) P->solve(R + j * P->size(), out + j * P->size());
  });
}
int orc_precond_sample_probes(void* p, int L, uint64_t seed, double* out) {
  return guard([&] { static_cast<Precond*>(p)->sample_probes(L, seed, out); });
}
int orc_precond_deriv_apply(void* p, int which, const double* v, double* out) {
  return guard([&] { static_cast<Precond*>(p)->deriv_apply(which, v, out); });
}
int orc_precond_deriv_trace(void* p, int which, double* out) {
  return guard([&] { *out = static_cast<Precond*>(p)->deriv_trace(which); });
}
// op_kind: 0 full FSA operator, 1 sigma_s only. tdiag/toff: k x max_iter (column j at j*max_iter)
int orc_pcg(void* mdv, int op_kind, void* p, const double* B, long k, double tol, int max_iter, int batched,
            double* X, int* iters, int* conv, double* tdiag, double* toff, int* sweeps) {
  return guard([&] {
    Model& md = *static_cast<Model*>(mdv);
    LinOp op = op_kind == 0 ? fsa_operator(md) : sigma_s_operator(md);
    CgResult r = pcg_solve_multi(op, *static_cast<Precond*>(p), B, k, tol, max_iter, batched != 0);
    std::copy(r.X.begin(), r.X.end(), X);
    for (long j = 0; j < k; ++j) {
      iters[j] = r.iterations[static_cast<size_t>(j)];
      conv[j] = r.converged[static_cast<size_t>(j)];
      if (tdiag) std::copy(r.tdiag[static_cast<size_t>(j)].begin(), r.tdiag[static_cast<size_t>(j)].end(), tdiag + j * max_iter);
      if (toff) std::copy(r.toff[static_cast<size_t>(j)].begin(), r.toff[static_cast<size_t>(j)].end(), toff + j * max_iter);
    }
    *sweeps = r.sweeps;
  });
}
// orc_pcg plus the residual-norm history (k x max_iter)
int orc_pcg_ex(void* mdv, int op_kind, void* p, const double* B, long k, double tol, int max_iter, int batched,
               double* X, int* iters, int* conv, double* tdiag, double* toff, double* rnorm, int* sweeps) {
  return guard([&] {
    Model& md = *static_cast<Model*>(mdv);
    LinOp op = op_kind == 0 ? fsa_operator(md) : sigma_s_operator(md);
    CgResult r = pcg_solve_multi(op, *static_cast<Precond*>(p), B, k, tol, max_iter, batched != 0);
    std::copy(r.X.begin(), r.X.end(), X);
    for (long j = 0; j < k; ++j) {
      const size_t sj = static_cast<size_t>(j);
      iters[j] = r.iterations[sj];
      conv[j] = r.converged[sj];
      std::copy(r.tdiag[sj].begin(), r.tdiag[sj].end(), tdiag + j * max_iter);
      std::copy(r.toff[sj].begin(), r.toff[sj].end(), toff + j * max_iter);
      std::copy(r.rnorm[sj].begin(), r.rnorm[sj].end(), rnorm + j * max_iter);
    }
    *sweeps = r.sweeps;
  });
}
int orc_tridiag_log_quadrature(const double* diag, const double* off, long len, double* out) {
  return guard([&] { *out = tridiag_log_quadrature(diag, off, len); });
}
// out: [nll, g0, g1, g2, logdet, cg_iterations]
int orc_iterative_nll_grad(void* mdv, void* p, const double* y, const double* X, long pcols, int L, uint64_t seed,
                           double tol, int max_iter, int cv, int want_grad, double* out, double* beta) {
  return guard([&] {
    NllOut r = iterative_nll_grad(*static_cast<Model*>(mdv), *static_cast<Precond*>(p), y, X, pcols, L, seed, tol,
                                  max_iter, cv, want_grad != 0);
    out[0] = r.nll; out[1] = r.g[0]; out[2] = r.g[1]; out[3] = r.g[2]; out[4] = r.logdet;
    out[5] = static_cast<double>(r.cg_iterations);
    for (long a = 0; a < pcols; ++a) beta[a] = r.beta[static_cast<size_t>(a)];
  });
}
// same plus the solve's diagnostics (tests only): per-column iterations, the residual-norm history
// rnorm (k x max_iter, column j at j*max_iter) and X at the rows `rows` (nrows x k, column-major)
int orc_iterative_nll_grad_ex(void* mdv, void* p, const double* y, const double* X, long pcols, int L, uint64_t seed,
                              double tol, int max_iter, int cv, int want_grad, double* out, double* beta, int* iters,
                              double* rnorm, const long* rows, long nrows, double* xrows) {
  return guard([&] {
    Model& md = *static_cast<Model*>(mdv);
    NllOut r = iterative_nll_grad(md, *static_cast<Precond*>(p), y, X, pcols, L, seed, tol, max_iter, cv,
                                  want_grad != 0);
    out[0] = r.nll; out[1] = r.g[0]; out[2] = r.g[1]; out[3] = r.g[2]; out[4] = r.logdet;
    out[5] = static_cast<double>(r.cg_iterations);
    for (long a = 0; a < pcols; ++a) beta[a] = r.beta[static_cast<size_t>(a)];
    const long k = static_cast<long>(r.sol.iterations.size());
    for (long j = 0; j < k; ++j) {
      iters[j] = r.sol.iterations[static_cast<size_t>(j)];
      const auto& h = r.sol.rnorm[static_cast<size_t>(j)];
      std::copy(h.begin(), h.end(), rnorm + j * max_iter);
      for (long q = 0; q < nrows; ++q) xrows[q + j * nrows] = r.sol.X[static_cast<size_t>(rows[q] + j * md.n)];
    }
  });
}
int orc_simulate_rff(const double* c, long n, int d, int nu_code, double sigma1_2, double rho, double nugget,
                     int features, uint64_t seed, double* y) {
  return guard([&] { simulate_rff(c, n, d, nu_code, sigma1_2, rho, nugget, features, seed, y); });
}
int orc_blob_locations(long n, int d, int blobs, double sd, uint64_t seed, double* out) {
  return guard([&] { blob_locations(n, d, blobs, sd, seed, out); });
}
// ste_grad_trace for a given (Z, W): out [value, c_hat, var_of_mean]
int orc_ste_grad_trace(void* mdv, void* p, const double* Z, const double* W, long L, int which, int mode, double* out) {
  return guard([&] {
    TraceEstimate t = ste_grad_trace(*static_cast<Model*>(mdv), Z, W, L, *static_cast<Precond*>(p), which, mode);
    out[0] = t.value; out[1] = t.c_hat; out[2] = t.var_of_mean;
  });
}
int orc_pred_make(void* mdv, const double* pc, long np, void** out, long* nnz) {
  return guard([&] {
    Model& md = *static_cast<Model*>(mdv);
    Pred* P = make_prediction_set(md, mk_locs(pc, np, md.locs.d));
    *nnz = P->sigma_s_np.nnz();
    *out = P;
  });
}
void orc_pred_free(void* p) { delete static_cast<Pred*>(p); }
int orc_pred_csr(void* pv, long* ptr, int* idx, double* val) {
  return guard([&] {
    const Csr& s = static_cast<Pred*>(pv)->sigma_s_np;
    std::copy(s.ptr.begin(), s.ptr.end(), ptr);
    std::copy(s.idx.begin(), s.idx.end(), idx);
    std::copy(s.val.begin(), s.val.end(), val);
  });
}
int orc_cross_apply_t(void* mdv, void* pv, const double* u, double* out) {
  return guard([&] { cross_apply_t(*static_cast<Model*>(mdv), *static_cast<Pred*>(pv), u, out); });
}
int orc_predict_mean_iterative(void* mdv, void* pv, const double* resid, void* p, double tol, int max_iter, double* out) {
  return guard([&] {  // prediction.cpp:37-43
    Model& md = *static_cast<Model*>(mdv);
    CgResult r = pcg_solve_multi(fsa_operator(md), *static_cast<Precond*>(p), resid, 1, tol, max_iter, false);
    if (!r.all_converged()) throw NumericalError("prediction: cg did not converge");
    cross_apply_t(md, *static_cast<Pred*>(pv), r.X.data(), out);
  });
}
int orc_predict_var_sim(void* mdv, void* pv, int L, uint64_t seed, double tol, int maxit, double tol_s, int maxit_s,
                        int cv, double floor_rel, double* var, double* se, int* clamped, int* cg_iters) {
  return guard([&] {
    PredVar r = predict_var_sim(*static_cast<Model*>(mdv), *static_cast<Pred*>(pv), L, seed, tol, maxit, tol_s, maxit_s,
                                cv != 0, floor_rel);
    std::copy(r.var.begin(), r.var.end(), var);
    std::copy(r.se.begin(), r.se.end(), se);
    *clamped = r.clamped;
    *cg_iters = r.cg_iterations;
  });
}
// deterministic pieces only (for parity of the GPU decomposition): d1, d2, d3 (np each)
// Bounded CPU sample of predict_var_sim (bench.py's cpu_baseline for config 3; tests only): seconds
// for the deterministic pieces' two m-RHS solves restricted to their first `cols` columns
// (X1 = FITC-PCG on Sigma_mn^T, X2 = Jacobi-PCG on Sigma_s; prediction.cpp:72-110 -- the columns
// are independent recurrences, so the full solves cost ~m / cols times these) and for one batch of
// `probes` simulation vectors (quad_mat, prediction.cpp:142-148). out = [t_x1, t_x2, t_batch].
int orc_pred_sample_timing(void* mdv, void* pv, long cols, int probes, uint64_t seed, double tol, int maxit,
                           double tol_s, int maxit_s, double* out) {
  return guard([&] {
    Model& md = *static_cast<Model*>(mdv);
    const Pred& P = *static_cast<Pred*>(pv);
    const long n = md.n, m = md.m, np = P.np;
    cols = std::max(1L, std::min(cols, m));
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto sec = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count(); };
    std::unique_ptr<FitcP> fitc(fitc_from_fsa(md, false));
    Mat SmnT(n, cols);
    for (long j = 0; j < cols; ++j)
      for (long i = 0; i < n; ++i) SmnT(i, j) = md.sigma_mn(j, i);
    auto t0 = now();
    CgResult x1 = pcg_solve_multi(fsa_operator(md), *fitc, SmnT.data(), cols, tol, maxit, true);
    auto t1 = now();
    DiagP jacobi(csr_diag(md.sigma_s), nullptr);
    CgResult x2 = pcg_solve_multi(sigma_s_operator(md), jacobi, SmnT.data(), cols, tol_s, maxit_s, true);
    auto t2 = now();
    std::vector<double> Z(static_cast<size_t>(np * probes)), G(static_cast<size_t>(n * probes)), Q(Z.size());
    for (int j = 0; j < probes; ++j) {
      rng_t rng = probe_rng(seed, static_cast<uint64_t>(j));
      rademacher_fill(rng, Z.data() + static_cast<long>(j) * np, np);
    }
    auto t3 = now();
    spmm(P.sigma_s_np, Z.data(), np, probes, G.data(), n);
    CgResult sol = pcg_solve_multi(sigma_s_operator(md), jacobi, G.data(), probes, tol_s, maxit_s, true);
    spmm_t(P.sigma_s_np, sol.X.data(), n, probes, Q.data(), np);
    auto t4 = now();
    out[0] = sec(t0, t1);
    out[1] = sec(t1, t2);
    out[2] = sec(t3, t4);
  });
}
int orc_pred_det_pieces(void* mdv, void* pv, double tol, int maxit, double tol_s, int maxit_s, double* d1, double* d2,
                        double* d3, int* cg_iters) {
  return guard([&] {
    DetPieces r = deterministic_pieces(*static_cast<Model*>(mdv), *static_cast<Pred*>(pv), tol, maxit, tol_s, maxit_s);
    std::copy(r.d1.begin(), r.d1.end(), d1);
    std::copy(r.d2.begin(), r.d2.end(), d2);
    std::copy(r.d3.begin(), r.d3.end(), d3);
    *cg_iters = r.cg_iterations;
  });
}

}  // extern "C"
