// Host-side input generators of the reference (parameter independent, run once
// per fit): uniform locations (locations.cpp:9-17), random / k-means++ inducing
// points (inducing.cpp:11-139), the taper range rule (locations.cpp:192-195) and
// a seeded random-Fourier-feature GP draw for synthetic responses. The libstdc++
// distributions are used exactly as the reference uses them, so seeds reproduce.
#include "inputs.h"

#include <omp.h>

#include <algorithm>
#include <cmath>
#include <limits>
#include <numeric>
#include <random>
#include <stdexcept>
#include <vector>

namespace fsa {

using rng_t = std::mt19937_64;
unsigned long long splitmix64(unsigned long long x);

static void req(bool c, const char* m) {
  if (!c) throw std::invalid_argument(m);
}

void uniform_locations(long n, int d, unsigned long long seed, double* out) {
  req(n > 0 && d > 0, "uniform_locations needs n > 0 and d > 0");
  rng_t rng(splitmix64(seed));
  std::uniform_real_distribution<double> U(0.0, 1.0);
  for (long i = 0; i < n; ++i)
    for (int k = 0; k < d; ++k) out[i + k * n] = U(rng);
}

void select_random(const double* c, long n, int d, long m, unsigned long long seed, double* out) {
  req(m >= 1 && m <= n, "need 1 <= m <= n");
  rng_t rng(splitmix64(seed));
  std::vector<long> idx(static_cast<size_t>(n));
  std::iota(idx.begin(), idx.end(), 0L);
  for (long i = 0; i < m; ++i) {  // partial Fisher-Yates
    std::uniform_int_distribution<long> pick(i, n - 1);
    std::swap(idx[static_cast<size_t>(i)], idx[static_cast<size_t>(pick(rng))]);
  }
  for (long i = 0; i < m; ++i)
    for (int k = 0; k < d; ++k) out[i + k * m] = c[idx[static_cast<size_t>(i)] + k * n];
}

void select_kmeanspp(const double* c, long n, int d, long m, unsigned long long seed, int max_iter, double rel_tol,
                     double* out) {
  req(m >= 1 && m <= n, "need 1 <= m <= n");
  auto X = [&](long i, int k) { return c[i + k * n]; };
  std::vector<int> order(static_cast<size_t>(n));
  std::iota(order.begin(), order.end(), 0);
  std::sort(order.begin(), order.end(), [&](int a, int b) {
    for (int k = 0; k < d; ++k)
      if (X(a, k) != X(b, k)) return X(a, k) < X(b, k);
    return a < b;
  });
  std::vector<int> pool;
  pool.reserve(order.size());
  for (size_t t = 0; t < order.size(); ++t) {
    bool same = t > 0;
    if (t > 0)
      for (int k = 0; k < d; ++k)
        if (X(order[t], k) != X(order[t - 1], k)) same = false;
    if (!same) pool.push_back(order[t]);
  }
  std::sort(pool.begin(), pool.end());
  const long npool = static_cast<long>(pool.size());
  req(m <= npool, "m exceeds the number of distinct locations");
  std::vector<double> ctr(static_cast<size_t>(m * d));
  auto sqd = [&](long i, long cc) {
    double s = 0.0;
    for (int k = 0; k < d; ++k) {
      const double df = X(i, k) - ctr[static_cast<size_t>(cc + k * m)];
      s = k == 0 ? df * df : std::fma(df, df, s);
    }
    return s;
  };
  rng_t rng(splitmix64(seed));
  std::uniform_int_distribution<long> first(0, npool - 1);
  {
    const long p0 = pool[static_cast<size_t>(first(rng))];
    for (int k = 0; k < d; ++k) ctr[static_cast<size_t>(k * m)] = X(p0, k);
  }
  std::vector<double> d2(static_cast<size_t>(npool));
#pragma omp parallel for schedule(static)
  for (long i = 0; i < npool; ++i) d2[static_cast<size_t>(i)] = sqd(pool[static_cast<size_t>(i)], 0);
  for (long cc = 1; cc < m; ++cc) {
    double total = 0.0;
    for (long i = 0; i < npool; ++i) total += d2[static_cast<size_t>(i)];
    long chosen = 0;
    if (total > 0.0) {
      std::uniform_real_distribution<double> U(0.0, total);
      double u = U(rng), acc = 0.0;
      for (long i = 0; i < npool; ++i) {
        acc += d2[static_cast<size_t>(i)];
        if (u <= acc) {
          chosen = i;
          break;
        }
      }
    } else {
      chosen = first(rng) % npool;
    }
    for (int k = 0; k < d; ++k) ctr[static_cast<size_t>(cc + k * m)] = X(pool[static_cast<size_t>(chosen)], k);
#pragma omp parallel for schedule(static)
    for (long i = 0; i < npool; ++i)
      d2[static_cast<size_t>(i)] = std::min(d2[static_cast<size_t>(i)], sqd(pool[static_cast<size_t>(i)], cc));
  }
  std::vector<long> assign(static_cast<size_t>(n), 0);
  std::vector<double> best_d(static_cast<size_t>(n));
  double sse_prev = std::numeric_limits<double>::infinity();
  for (int it = 0; it < max_iter; ++it) {
#pragma omp parallel for schedule(static)
    for (long i = 0; i < n; ++i) {
      double best = std::numeric_limits<double>::infinity();
      long bc = 0;
      for (long cc = 0; cc < m; ++cc) {
        const double dd = sqd(i, cc);
        if (dd < best) {
          best = dd;
          bc = cc;
        }
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
    for (long cc = 0; cc < m; ++cc)
      if (counts[static_cast<size_t>(cc)] > 0.0)
        for (int k = 0; k < d; ++k)
          ctr[static_cast<size_t>(cc + k * m)] = sums[static_cast<size_t>(cc + k * m)] / counts[static_cast<size_t>(cc)];
    if (sse_prev - sse <= rel_tol * std::max(sse_prev, 1e-300)) break;
    sse_prev = sse;
  }
  std::vector<char> used(static_cast<size_t>(npool), 0);
  for (long cc = 0; cc < m; ++cc) {
    double best = std::numeric_limits<double>::infinity();
    long bi = -1;
#pragma omp parallel
    {
      double lb = std::numeric_limits<double>::infinity();
      long li = -1;
#pragma omp for schedule(static) nowait
      for (long i = 0; i < npool; ++i) {
        if (used[static_cast<size_t>(i)]) continue;
        const double dd = sqd(pool[static_cast<size_t>(i)], cc);
        if (dd < lb) {
          lb = dd;
          li = i;
        }
      }
#pragma omp critical
      {
        if (li >= 0 && (lb < best || (lb == best && li < bi))) {
          best = lb;
          bi = li;
        }
      }
    }
    used[static_cast<size_t>(bi)] = 1;
    for (int k = 0; k < d; ++k) out[cc + k * m] = X(pool[static_cast<size_t>(bi)], k);
  }
}

double gamma_for_avg_row_nnz(long n, double target) {
  req(n > 0 && target >= 1.0, "need n > 0 and target >= 1");
  return std::sqrt(target / (static_cast<double>(n) * M_PI));
}

// f(s) = sqrt(2 sigma1_2 / F) sum_f cos(w_f . s + b_f), w ~ Matern-nu spectral
// measure (multivariate t, 2 nu dof, scale 1/rho), plus N(0, nugget) noise.
void simulate_rff(const double* c, long n, int d, int nu_code, double sigma1_2, double rho, double nugget,
                  int features, unsigned long long seed, double* y) {
  req(n > 0 && features > 0, "simulate_rff: invalid sizes");
  const double nu = nu_code == 0 ? 0.5 : (nu_code == 1 ? 1.5 : 2.5);
  rng_t rng(splitmix64(seed ^ 0x5eed5eedULL));
  std::normal_distribution<double> N01(0.0, 1.0);
  std::chi_squared_distribution<double> chi(2.0 * nu);
  std::uniform_real_distribution<double> U(0.0, 2.0 * M_PI);
  std::vector<double> w(static_cast<size_t>(features * d)), b(static_cast<size_t>(features));
  for (int f = 0; f < features; ++f) {
    const double u = chi(rng);
    const double scale = 1.0 / (rho * std::sqrt(u / (2.0 * nu)));
    for (int k = 0; k < d; ++k) w[static_cast<size_t>(f * d + k)] = N01(rng) * scale;
    b[static_cast<size_t>(f)] = U(rng);
  }
  const double amp = std::sqrt(2.0 * sigma1_2 / features);
#pragma omp parallel for schedule(static)
  for (long i = 0; i < n; ++i) {
    double s = 0.0;
    for (int f = 0; f < features; ++f) {
      double arg = b[static_cast<size_t>(f)];
      for (int k = 0; k < d; ++k) arg += w[static_cast<size_t>(f * d + k)] * c[i + k * n];
      s += std::cos(arg);
    }
    y[i] = amp * s;
  }
  rng_t nr(splitmix64(seed ^ 0x0153ULL));
  std::normal_distribution<double> E(0.0, 1.0);
  const double sd = std::sqrt(nugget);
  for (long i = 0; i < n; ++i) y[i] += sd * E(nr);
}

// mixture of seeded Gaussian blobs on [0,1]^d (config 5), points outside rejected
void blob_locations(long n, int d, int blobs, double sd, unsigned long long seed, double* out) {
  req(n > 0 && blobs > 0, "blob_locations: invalid sizes");
  rng_t rng(splitmix64(seed));
  std::uniform_real_distribution<double> U(0.0, 1.0);
  std::vector<double> ctr(static_cast<size_t>(blobs * d));
  for (auto& v : ctr) v = U(rng);
  std::uniform_int_distribution<int> pick(0, blobs - 1);
  std::normal_distribution<double> N(0.0, sd);
  long i = 0;
  while (i < n) {
    const int bl = pick(rng);
    double p[3];
    bool ok = true;
    for (int k = 0; k < d; ++k) {
      p[k] = ctr[static_cast<size_t>(bl * d + k)] + N(rng);
      ok = ok && p[k] >= 0.0 && p[k] <= 1.0;
    }
    if (!ok) continue;
    for (int k = 0; k < d; ++k) out[i + k * n] = p[k];
    ++i;
  }
}

}  // namespace fsa
