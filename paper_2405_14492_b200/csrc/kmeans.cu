// Device k-means++ / Lloyd inducing-point selection: select_kmeanspp (inducing.cpp:48-139),
// SURVEY §8f row f2. The reference (and the host restatement in inputs.cpp) is O(20 n m)
// serial work that dominates input preparation at config 4 (n = 1e6, m = 1000).
//
// Same decisions as the reference, on the device:
//  * distinct pool (inducing.cpp:28-45): lexicographic sort of the point indices (ties by
//    index), first of each run of equal rows kept, pool in ascending original index;
//  * seeding (inducing.cpp:61-88): the first centre comes from uniform_int_distribution on the
//    host RNG; each further centre consumes exactly one generate_canonical draw of the same
//    mt19937_64 stream (uniform_real_distribution(0, total) = can * total), drawn on the host
//    up front so the device loop needs no host round trip. Per round: d2 = min(d2, |p - c|^2)
//    fused with fixed per-block partial sums (k_seed_update), then one block scans the partials
//    and the chosen block's entries for the first i with u <= prefix(i) (k_seed_choose);
//  * Lloyd (inducing.cpp:90-118): nearest centre per point (strict <, lowest index on ties),
//    centroid sums in a fixed order (points radix-sorted by centre, stable), SSE by a fixed
//    tree, the reference's relative-decrease stop;
//  * snapping (inducing.cpp:120-136): each centroid's nearest pool point in parallel; the
//    greedy "nearest still unused" order is replayed on the host, and only a centroid whose
//    nearest point was taken by an earlier one is searched again on the device with the mask.
// Squared distances follow the host restatement's operation order (d0^2, then fma per axis)
// with explicit _rn intrinsics so no contraction changes the rounding. Sums are fixed-order
// trees instead of the reference's serial loops: the decisions are identical unless a draw lands
// within rounding of a cumulative boundary or a point within rounding of a Voronoi boundary.
#include <cub/cub.cuh>
#include <math_constants.h>
#include <thrust/execution_policy.h>
#include <thrust/sort.h>

#include <algorithm>
#include <cmath>
#include <limits>
#include <random>
#include <vector>

#include "common.cuh"
#include "kmeans.cuh"

namespace fsa {
namespace {

constexpr int kKmThreads = 256;
constexpr int kChooseThreads = 1024;
constexpr int kMaxD = 3;

unsigned long long splitmix64_host(unsigned long long x) {  // types.h:104-109
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

__device__ __forceinline__ double sqd_dev(const double* P, long ldp, long i, const double* c, int d) {
  double s = 0.0;
  for (int k = 0; k < d; ++k) {
    const double df = __dsub_rn(P[i + k * ldp], c[k]);
    s = k == 0 ? __dmul_rn(df, df) : __fma_rn(df, df, s);
  }
  return s;
}

// lexicographic "a < b" on the rows, ties by index (inducing.cpp:30-36)
struct LexLess {
  const double* X;
  long n;
  int d;
  __device__ bool operator()(int a, int b) const {
    for (int k = 0; k < d; ++k) {
      const double xa = X[a + k * n], xb = X[b + k * n];
      if (xa != xb) return xa < xb;
    }
    return a < b;
  }
};

__global__ void k_iota(int* v, long n) {
  const long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
  if (i < n) v[i] = static_cast<int>(i);
}
// keep[order[t]] = 1 for the first of each run of equal rows (inducing.cpp:39-41)
__global__ void k_mark_distinct(const double* X, long n, int d, const int* order, char* keep) {
  const long t = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
  if (t >= n) return;
  bool same = t > 0;
  if (t > 0)
    for (int k = 0; k < d; ++k)
      if (X[order[t] + k * n] != X[order[t - 1] + k * n]) same = false;
  keep[order[t]] = same ? 0 : 1;
}
__global__ void k_gather_rows(const double* X, long n, int d, const int* idx, long cnt, double* P) {
  const long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
  if (i >= cnt) return;
  for (int k = 0; k < d; ++k) P[i + k * cnt] = X[idx[i] + k * n];
}

// d2 = min(d2, |p - c|^2) (init: d2 = |p - c|^2) over the block's chunk, and its partial sum
__global__ void __launch_bounds__(kKmThreads) k_seed_update(const double* P, long np, int d, const double* ctr,
                                                           long ldc, long c, double* d2, long chunk, int init,
                                                           double* partial) {
  typedef cub::BlockReduce<double, kKmThreads> BR;
  __shared__ typename BR::TempStorage tmp;
  double cc[kMaxD];
  for (int k = 0; k < d; ++k) cc[k] = ctr[c + k * ldc];
  const long i0 = blockIdx.x * chunk, i1 = min(np, i0 + chunk);
  double acc = 0.0;
  for (long i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    const double dd = sqd_dev(P, np, i, cc, d);
    const double v = init ? dd : fmin(d2[i], dd);
    d2[i] = v;
    acc += v;
  }
  const double s = BR(tmp).Sum(acc);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// One block: total, u = can * total and the first i with u <= prefix(i) (inducing.cpp:64-81);
// copies the chosen pool point into ctr[c]. prefix(i) = (sum of the partials of the earlier
// chunks) + the in-chunk prefix; if rounding leaves u past the end of the chosen chunk, the
// chunk's last entry is taken; if u is past the total, index 0 (the reference's fallthrough).
__global__ void __launch_bounds__(kChooseThreads) k_seed_choose(const double* P, long np, int d, const double* d2,
                                                               long chunk, const double* partial, int nb,
                                                               const double* can, long c, double* ctr, long ldc) {
  typedef cub::BlockScan<double, kChooseThreads> BS;
  typedef cub::BlockReduce<long, kChooseThreads> BRL;
  __shared__ typename BS::TempStorage ts;
  __shared__ typename BRL::TempStorage tr;
  __shared__ double s_total, s_base;
  __shared__ long s_blk;
  const int tid = threadIdx.x;
  const double v = tid < nb ? partial[tid] : 0.0;
  double exc, agg;
  BS(ts).ExclusiveSum(v, exc, agg);
  if (tid == 0) s_total = agg;
  __syncthreads();
  const double u = can[c] * s_total + 0.0;  // (b - a) * canonical + a
  const long cand = (tid < nb && u <= exc + v) ? tid : static_cast<long>(nb);
  const long blk = BRL(tr).Reduce(cand, cub::Min());
  if (tid == 0) s_blk = blk;
  __syncthreads();
  if (tid < nb && tid == s_blk) s_base = exc;
  __syncthreads();
  long pick = 0;
  if (s_blk < nb) {
    const long i0 = s_blk * chunk, i1 = min(np, i0 + chunk);
    const long len = i1 - i0, ipt = (len + kChooseThreads - 1) / kChooseThreads;
    const long a0 = i0 + tid * ipt, a1 = min(i1, a0 + ipt);
    double loc = 0.0;
    for (long i = a0; i < a1; ++i) loc += d2[i];
    double texc, tagg;
    __syncthreads();
    BS(ts).ExclusiveSum(loc, texc, tagg);
    double acc = s_base + texc;
    long found = np;
    for (long i = a0; i < a1; ++i) {
      acc += d2[i];
      if (u <= acc) {
        found = i;
        break;
      }
    }
    __syncthreads();
    const long f = BRL(tr).Reduce(found, cub::Min());
    pick = f < np ? f : i1 - 1;
  }
  if (tid == 0)
    for (int k = 0; k < d; ++k) ctr[c + k * ldc] = P[pick + k * np];
}

// nearest centre per point (inducing.cpp:95-107): strict <, lowest centre index on ties
__global__ void __launch_bounds__(kKmThreads) k_assign(const double* X, long n, int d, const double* ctr, long m,
                                                      int* assign, double* best_d) {
  extern __shared__ double sc[];  // m x d, column-major
  for (long t = threadIdx.x; t < m * d; t += blockDim.x) sc[t] = ctr[t];
  __syncthreads();
  const long i = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  double x[kMaxD];
  for (int k = 0; k < d; ++k) x[k] = X[i + k * n];
  double best = CUDART_INF;
  int bc = 0;
  for (long cc = 0; cc < m; ++cc) {
    double s = 0.0;
    for (int k = 0; k < d; ++k) {
      const double df = __dsub_rn(x[k], sc[cc + k * m]);
      s = k == 0 ? __dmul_rn(df, df) : __fma_rn(df, df, s);
    }
    if (s < best) {
      best = s;
      bc = static_cast<int>(cc);
    }
  }
  assign[i] = bc;
  best_d[i] = best;
}

__global__ void __launch_bounds__(kKmThreads) k_chunk_sums(const double* v, long n, long chunk, double* partial) {
  typedef cub::BlockReduce<double, kKmThreads> BR;
  __shared__ typename BR::TempStorage tmp;
  const long i0 = blockIdx.x * chunk, i1 = min(n, i0 + chunk);
  double acc = 0.0;
  for (long i = i0 + threadIdx.x; i < i1; i += blockDim.x) acc += v[i];
  const double s = BR(tmp).Sum(acc);
  if (threadIdx.x == 0) partial[blockIdx.x] = s;
}
__global__ void __launch_bounds__(kChooseThreads) k_total(const double* partial, int nb, double* out) {
  typedef cub::BlockReduce<double, kChooseThreads> BR;
  __shared__ typename BR::TempStorage tmp;
  double acc = 0.0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) acc += partial[b];
  const double s = BR(tmp).Sum(acc);
  if (threadIdx.x == 0) *out = s;
}
// seg[c] = first position of centre c in the sorted assignment keys (c = 0..m)
__global__ void k_seg_offsets(const int* keys, long n, long m, long* seg) {
  const long c = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
  if (c > m) return;
  long lo = 0, hi = n;
  while (lo < hi) {
    const long mid = (lo + hi) / 2;
    if (keys[mid] < c) lo = mid + 1;
    else hi = mid;
  }
  seg[c] = lo;
}
// centroid c = mean of its points (inducing.cpp:108-117), summed in ascending point order
__global__ void __launch_bounds__(kKmThreads) k_centroids(const double* X, long n, int d, const int* sorted_idx,
                                                         const long* seg, long m, double* ctr) {
  typedef cub::BlockReduce<double, kKmThreads> BR;
  __shared__ typename BR::TempStorage tmp;
  const long c = blockIdx.x;
  const long s0 = seg[c], s1 = seg[c + 1];
  if (s1 == s0) return;  // empty cluster keeps its centre
  const double cnt = static_cast<double>(s1 - s0);
  for (int k = 0; k < d; ++k) {
    double acc = 0.0;
    for (long t = s0 + threadIdx.x; t < s1; t += blockDim.x) acc += X[sorted_idx[t] + k * n];
    const double s = BR(tmp).Sum(acc);
    __syncthreads();
    if (threadIdx.x == 0) ctr[c + k * m] = s / cnt;
  }
}

struct DistIdx {
  double d;
  long i;
};
struct DistIdxMin {
  __device__ DistIdx operator()(const DistIdx& a, const DistIdx& b) const {
    return (b.d < a.d || (b.d == a.d && b.i < a.i)) ? b : a;
  }
};
// nearest (unused) pool point of centre c0 + blockIdx.x (inducing.cpp:123-133)
__global__ void __launch_bounds__(kKmThreads) k_nearest(const double* P, long np, int d, const double* ctr, long ldc,
                                                       long c0, const char* used, long* out) {
  typedef cub::BlockReduce<DistIdx, kKmThreads> BR;
  __shared__ typename BR::TempStorage tmp;
  const long c = c0 + blockIdx.x;
  double cc[kMaxD];
  for (int k = 0; k < d; ++k) cc[k] = ctr[c + k * ldc];
  DistIdx best{CUDART_INF, -1};
  for (long i = threadIdx.x; i < np; i += blockDim.x) {
    if (used != nullptr && used[i]) continue;
    const double dd = sqd_dev(P, np, i, cc, d);
    if (dd < best.d) best = DistIdx{dd, i};  // ascending i per thread: first minimum kept
  }
  const DistIdx r = BR(tmp).Reduce(best, DistIdxMin());
  if (threadIdx.x == 0) out[blockIdx.x] = r.i;
}

}  // namespace

void select_kmeanspp_device(cudaStream_t s, const double* coords, long n, int d, long m, unsigned long long seed,
                            int max_iter, double rel_tol, double* out) {
  require(m >= 1 && m <= n, "need 1 <= m <= n");
  require(d >= 1 && d <= kMaxD, "kmeans: 1 <= d <= 3");
  require(m * d * static_cast<long>(sizeof(double)) <= 200 * 1024, "kmeans: m * d too large for shared memory");
  const int TB = kKmThreads;
  auto grid = [&](long cnt) { return static_cast<unsigned>(cdiv(cnt, TB)); };
  DBuf<double> X(static_cast<size_t>(n * d));
  FSA_CUDA(cudaMemcpyAsync(X.get(), coords, sizeof(double) * n * d, cudaMemcpyHostToDevice, s));
  // ---- distinct pool
  DBuf<int> order(static_cast<size_t>(n)), iota(static_cast<size_t>(n)), pool(static_cast<size_t>(n));
  DBuf<char> keep(static_cast<size_t>(n));
  DBuf<int> npool_d(1);
  k_iota<<<grid(n), TB, 0, s>>>(order.get(), n);
  k_iota<<<grid(n), TB, 0, s>>>(iota.get(), n);
  FSA_LAUNCH_CHECK();
  thrust::sort(thrust::cuda::par.on(s), order.get(), order.get() + n, LexLess{X.get(), n, d});
  k_mark_distinct<<<grid(n), TB, 0, s>>>(X.get(), n, d, order.get(), keep.get());
  FSA_LAUNCH_CHECK();
  {
    size_t tb = 0;
    FSA_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, iota.get(), keep.get(), pool.get(), npool_d.get(), n, s));
    DBuf<char> tmp(tb);
    FSA_CUDA(cub::DeviceSelect::Flagged(tmp.get(), tb, iota.get(), keep.get(), pool.get(), npool_d.get(), n, s));
  }
  int npool_h = 0;
  FSA_CUDA(cudaMemcpyAsync(&npool_h, npool_d.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  FSA_CUDA(cudaStreamSynchronize(s));
  const long np = npool_h;
  require(m <= np, "m exceeds the number of distinct locations");
  std::vector<int> pool_h(static_cast<size_t>(np));
  FSA_CUDA(cudaMemcpyAsync(pool_h.data(), pool.get(), sizeof(int) * np, cudaMemcpyDeviceToHost, s));
  DBuf<double> P(static_cast<size_t>(np * d));
  k_gather_rows<<<grid(np), TB, 0, s>>>(X.get(), n, d, pool.get(), np, P.get());
  FSA_LAUNCH_CHECK();
  // ---- host draws: the first centre, then one canonical per further centre
  std::mt19937_64 rng(splitmix64_host(seed));
  std::uniform_int_distribution<long> first(0, np - 1);
  const long f0 = first(rng);
  std::vector<double> can(static_cast<size_t>(m), 0.0);
  for (long c = 1; c < m; ++c) can[static_cast<size_t>(c)] = std::generate_canonical<double, 53>(rng);
  FSA_CUDA(cudaStreamSynchronize(s));
  std::vector<double> ctr_h(static_cast<size_t>(m * d), 0.0);
  for (int k = 0; k < d; ++k) ctr_h[static_cast<size_t>(k * m)] = coords[pool_h[static_cast<size_t>(f0)] + k * n];
  DBuf<double> ctr(static_cast<size_t>(m * d)), can_d(static_cast<size_t>(m));
  FSA_CUDA(cudaMemcpyAsync(ctr.get(), ctr_h.data(), sizeof(double) * m * d, cudaMemcpyHostToDevice, s));
  FSA_CUDA(cudaMemcpyAsync(can_d.get(), can.data(), sizeof(double) * m, cudaMemcpyHostToDevice, s));
  // ---- seeding
  const long chunk = std::max<long>(TB, cdiv(np, kChooseThreads));
  const int nb = static_cast<int>(cdiv(np, chunk));
  DBuf<double> d2(static_cast<size_t>(np)), part(static_cast<size_t>(std::max(nb, 1)));
  k_seed_update<<<nb, TB, 0, s>>>(P.get(), np, d, ctr.get(), m, 0, d2.get(), chunk, 1, part.get());
  FSA_LAUNCH_CHECK();
  for (long c = 1; c < m; ++c) {
    k_seed_choose<<<1, kChooseThreads, 0, s>>>(P.get(), np, d, d2.get(), chunk, part.get(), nb, can_d.get(), c,
                                               ctr.get(), m);
    if (c + 1 < m)
      k_seed_update<<<nb, TB, 0, s>>>(P.get(), np, d, ctr.get(), m, c, d2.get(), chunk, 0, part.get());
  }
  FSA_LAUNCH_CHECK();
  // ---- Lloyd iterations on all points
  DBuf<int> assign(static_cast<size_t>(n)), skeys(static_cast<size_t>(n)), sidx(static_cast<size_t>(n));
  DBuf<double> best(static_cast<size_t>(n)), sse_d(1);
  DBuf<long> seg(static_cast<size_t>(m + 1));
  const long schunk = std::max<long>(TB, cdiv(n, kChooseThreads));
  const int snb = static_cast<int>(cdiv(n, schunk));
  DBuf<double> spart(static_cast<size_t>(snb));
  int end_bit = 1;
  while ((1L << end_bit) < m) ++end_bit;
  size_t sort_tb = 0;
  FSA_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, sort_tb, assign.get(), skeys.get(), iota.get(), sidx.get(), n, 0,
                                           end_bit, s));
  DBuf<char> sort_tmp(sort_tb);
  const size_t smem = sizeof(double) * m * d;
  if (smem > 48 * 1024)
    FSA_CUDA(cudaFuncSetAttribute(k_assign, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  double sse_prev = std::numeric_limits<double>::infinity();
  for (int it = 0; it < max_iter; ++it) {
    k_assign<<<grid(n), TB, smem, s>>>(X.get(), n, d, ctr.get(), m, assign.get(), best.get());
    k_chunk_sums<<<snb, TB, 0, s>>>(best.get(), n, schunk, spart.get());
    k_total<<<1, kChooseThreads, 0, s>>>(spart.get(), snb, sse_d.get());
    FSA_LAUNCH_CHECK();
    FSA_CUDA(cub::DeviceRadixSort::SortPairs(sort_tmp.get(), sort_tb, assign.get(), skeys.get(), iota.get(),
                                             sidx.get(), n, 0, end_bit, s));
    k_seg_offsets<<<grid(m + 1), TB, 0, s>>>(skeys.get(), n, m, seg.get());
    k_centroids<<<static_cast<unsigned>(m), TB, 0, s>>>(X.get(), n, d, sidx.get(), seg.get(), m, ctr.get());
    FSA_LAUNCH_CHECK();
    double sse = 0.0;
    FSA_CUDA(cudaMemcpyAsync(&sse, sse_d.get(), sizeof(double), cudaMemcpyDeviceToHost, s));
    FSA_CUDA(cudaStreamSynchronize(s));
    if (sse_prev - sse <= rel_tol * std::max(sse_prev, 1e-300)) break;  // inducing.cpp:115
    sse_prev = sse;
  }
  // ---- snap to the nearest still-unused distinct location (inducing.cpp:120-136)
  DBuf<long> near(static_cast<size_t>(m));
  k_nearest<<<static_cast<unsigned>(m), TB, 0, s>>>(P.get(), np, d, ctr.get(), m, 0, nullptr, near.get());
  FSA_LAUNCH_CHECK();
  std::vector<long> near_h(static_cast<size_t>(m));
  FSA_CUDA(cudaMemcpyAsync(near_h.data(), near.get(), sizeof(long) * m, cudaMemcpyDeviceToHost, s));
  FSA_CUDA(cudaStreamSynchronize(s));
  std::vector<char> used(static_cast<size_t>(np), 0);
  DBuf<char> used_d(static_cast<size_t>(np));
  DBuf<long> one(1);
  for (long c = 0; c < m; ++c) {
    long bi = near_h[static_cast<size_t>(c)];
    if (used[static_cast<size_t>(bi)]) {  // taken by an earlier centroid: search the unused points
      FSA_CUDA(cudaMemcpyAsync(used_d.get(), used.data(), np, cudaMemcpyHostToDevice, s));
      k_nearest<<<1, TB, 0, s>>>(P.get(), np, d, ctr.get(), m, c, used_d.get(), one.get());
      FSA_LAUNCH_CHECK();
      FSA_CUDA(cudaMemcpyAsync(&bi, one.get(), sizeof(long), cudaMemcpyDeviceToHost, s));
      FSA_CUDA(cudaStreamSynchronize(s));
    }
    used[static_cast<size_t>(bi)] = 1;
    for (int k = 0; k < d; ++k) out[c + k * m] = coords[pool_h[static_cast<size_t>(bi)] + k * n];
  }
}

}  // namespace fsa
