// Launchers for the DMMA fp64 GEMMs declared in dgemm.cuh.
#include "dgemm.cuh"

#include <algorithm>

#include <cstdlib>

namespace fsa {

namespace {

// expand: 4 warps x 32 rows (BM = 128), all N columns of the tile per warp.
template <int NT>
using ExpandCfg = GemmCfg<NT, 4, 4, false, 16, 3>;
// expand, 8 warps x 16 rows (BM = 128): twice the warps per SM at the same smem
template <int NT>
using ExpandCfg8 = GemmCfg<NT, 2, 8, false, 16, 3>;
// expand, 2 stages (3 CTAs per SM)
template <int NT>
using ExpandCfgS2 = GemmCfg<NT, 4, 4, false, 16, 2>;
// expand, BM = 64 (4 warps x 16 rows), 3 stages: 3 CTAs per SM, twice the CTAs
template <int NT>
using ExpandCfg64 = GemmCfg<NT, 2, 4, false, 16, 3>;
// expand, BM = 64 as 2 warps x 32 rows (twice the independent accumulators per warp)
template <int NT>
using ExpandCfg64w2 = GemmCfg<NT, 4, 2, false, 16, 3>;
// same with 2 stages (more CTAs per SM)
template <int NT>
using ExpandCfg64w2s2 = GemmCfg<NT, 4, 2, false, 16, 2>;
// BM = 64, 4 warps x 16 rows, BK = 32, 2 stages (half the barriers per k)
template <int NT>
using ExpandCfg64k32 = GemmCfg<NT, 2, 4, false, 32, 2>;
// reduce: 4 warps x 16 rows (BM = 64), A is [k][m].
template <int NT>
using ReduceCfg = GemmCfg<NT, 2, 4, true, 16, 3>;
// reduce, 8 warps x 16 rows (BM = 128)
template <int NT>
using ReduceCfg8 = GemmCfg<NT, 2, 8, true, 16, 3>;

// tile variant knobs (FSA_GEMM_EXPAND / FSA_GEMM_REDUCE = 0 | 1), read once
int knob(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}
int expand_variant() {
  static const int v = knob("FSA_GEMM_EXPAND", 3);  // BM = 64, 3 CTAs/SM: measured fastest (r01)
  return v;
}
long expand_bm() {
  const int v = expand_variant();
  return (v >= 3 && v <= 6) ? 64 : 128;
}
int reduce_variant() {
  static const int v = knob("FSA_GEMM_REDUCE", 1);  // 8 warps: measured faster (r01)
  return v;
}

template <class Cfg, class Epi>
void launch(const double* A, long lda, const double* B, long ldb, const double* scale, long K, long kchunk,
            dim3 grid, Epi epi, cudaStream_t s) {
  static bool attr_set = false;
  if (!attr_set) {
    FSA_CUDA(cudaFuncSetAttribute(k_dgemm<Cfg, Epi>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  Cfg::SMEM_BYTES));
    attr_set = true;
  }
  k_dgemm<Cfg, Epi><<<grid, Cfg::THREADS, Cfg::SMEM_BYTES, s>>>(A, lda, B, ldb, scale, K, kchunk, epi);
  FSA_LAUNCH_CHECK();
}

// N (padded RHS width) -> number of 8-column DMMA tiles handled by one CTA
inline int tile_nt(long N) { return N <= 72 ? static_cast<int>(N / 8) : 8; }

template <template <int> class CfgT, class Epi>
void dispatch_nt(int nt, const double* A, long lda, const double* B, long ldb, const double* scale, long K,
                 long kchunk, dim3 grid, Epi epi, cudaStream_t s) {
  switch (nt) {
    case 1: launch<CfgT<1>>(A, lda, B, ldb, scale, K, kchunk, grid, epi, s); break;
    case 2: launch<CfgT<2>>(A, lda, B, ldb, scale, K, kchunk, grid, epi, s); break;
    case 3: launch<CfgT<3>>(A, lda, B, ldb, scale, K, kchunk, grid, epi, s); break;
    case 4: launch<CfgT<4>>(A, lda, B, ldb, scale, K, kchunk, grid, epi, s); break;
    case 5: launch<CfgT<5>>(A, lda, B, ldb, scale, K, kchunk, grid, epi, s); break;
    case 6: launch<CfgT<6>>(A, lda, B, ldb, scale, K, kchunk, grid, epi, s); break;
    case 7: launch<CfgT<7>>(A, lda, B, ldb, scale, K, kchunk, grid, epi, s); break;
    case 8: launch<CfgT<8>>(A, lda, B, ldb, scale, K, kchunk, grid, epi, s); break;
    case 9: launch<CfgT<9>>(A, lda, B, ldb, scale, K, kchunk, grid, epi, s); break;
    default: throw std::invalid_argument("gemm: unsupported column tile");
  }
}

template <class Epi>
void expand(const double* M, long ldm, long rows, long K, const double* W, long ldw, long N, Epi epi,
            cudaStream_t s) {
  require(rows % 128 == 0 && K % 16 == 0 && N == pad_cols(N), "gemm_expand: unpadded shape");
  if (rows == 0) return;
  const int nt = tile_nt(N);
  const int v = expand_variant();
  const long bm = expand_bm();
  require(v != 6 || K % 32 == 0, "gemm_expand: K must be a multiple of 32 for this tile");
  dim3 grid(static_cast<unsigned>(rows / bm), static_cast<unsigned>(N / (nt * 8)), 1);
  switch (v) {
    case 1: dispatch_nt<ExpandCfg8>(nt, M, ldm, W, ldw, nullptr, K, K, grid, epi, s); break;
    case 2: dispatch_nt<ExpandCfgS2>(nt, M, ldm, W, ldw, nullptr, K, K, grid, epi, s); break;
    case 3: dispatch_nt<ExpandCfg64>(nt, M, ldm, W, ldw, nullptr, K, K, grid, epi, s); break;
    case 4: dispatch_nt<ExpandCfg64w2>(nt, M, ldm, W, ldw, nullptr, K, K, grid, epi, s); break;
    case 5: dispatch_nt<ExpandCfg64w2s2>(nt, M, ldm, W, ldw, nullptr, K, K, grid, epi, s); break;
    case 6: dispatch_nt<ExpandCfg64k32>(nt, M, ldm, W, ldw, nullptr, K, K, grid, epi, s); break;
    default: dispatch_nt<ExpandCfg>(nt, M, ldm, W, ldw, nullptr, K, K, grid, epi, s); break;
  }
}

struct ReducePlan {
  int nt, bm;
  long tiles, splits, kchunk;
};
ReducePlan plan_reduce(long Mr, long N, long K) {
  ReducePlan p;
  p.nt = tile_nt(N);
  p.bm = (reduce_variant() >= 1 && Mr % 128 == 0) ? 128 : 64;
  p.tiles = (Mr / p.bm) * (N / (p.nt * 8));
  const long kblocks = K / 16;
  long splits = cdiv((reduce_variant() == 2 ? 4 : 2) * kNumSMs, p.tiles);
  splits = splits < 1 ? 1 : splits;
  splits = splits > kblocks ? kblocks : splits;
  splits = splits < 1 ? 1 : splits;
  p.kchunk = round_up(cdiv(K, splits), 16);
  p.splits = cdiv(K, p.kchunk);
  if (p.splits < 1) p.splits = 1;
  return p;
}

__global__ void k_splitk_reduce(const double* __restrict__ W, long splits, long Mr, long N, double* out, long ldo,
                                double alpha, double beta) {
  const long idx = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= Mr * N) return;
  const long r = idx / N, c = idx % N;
  double acc = 0.0;
  for (long z = 0; z < splits; ++z) acc += W[(z * Mr + r) * N + c];
  double* o = out + r * ldo + c;
  *o = beta == 0.0 ? alpha * acc : alpha * acc + beta * *o;
}

}  // namespace

void gemm_expand_store(const double* M, long ldm, long rows, long K, const double* W, long ldw, long N,
                       double* Y, long ldy, double alpha, double beta, cudaStream_t s) {
  if (beta == 0.0)
    expand(M, ldm, rows, K, W, ldw, N, EpiStore{Y, ldy, alpha}, s);
  else
    expand(M, ldm, rows, K, W, ldw, N, EpiAxpby{Y, ldy, alpha, beta}, s);
}
void gemm_expand_probe(const double* M, long ldm, long rows, long K, const double* W, long ldw, long N,
                       double* Y, long ld, const double* sqrtD, const double* E2, cudaStream_t s) {
  expand(M, ldm, rows, K, W, ldw, N, EpiProbe{Y, ld, sqrtD, E2}, s);
}
void gemm_expand_woodbury(const double* M, long ldm, long rows, long K, const double* W, long ldw, long N,
                          double* Z, const double* R, long ld, const double* Dinv, cudaStream_t s) {
  expand(M, ldm, rows, K, W, ldw, N, EpiWoodbury{nullptr, 0, Z, R, ld, Dinv}, s);
}
void gemm_expand_woodbury_dot(const double* M, long ldm, long rows, long K, const double* W, long ldw, long N,
                              double* Z, const double* R, long ld, const double* Dinv, double* rz, double* partial,
                              cudaStream_t s) {
  expand(M, ldm, rows, K, W, ldw, N, EpiWoodburyDot{partial, N, Z, R, ld, Dinv}, s);
  colsum_partials(partial, rows / expand_bm(), N, N, rz, s);
}

void gemm_expand_woodbury_keep(const double* M, long ldm, long rows, long K, const double* W, long ldw, long N,
                               double* Z, double* Lw, const double* R, long ld, const double* Dinv, double* rz,
                               double* partial, cudaStream_t s) {
  expand(M, ldm, rows, K, W, ldw, N, EpiWoodburyKeep{partial, N, Z, Lw, R, ld, Dinv}, s);
  colsum_partials(partial, rows / expand_bm(), N, N, rz, s);
}

// out[c] = sum_b partial[b][c]: one 256-thread block per column, fixed strided
// assignment + fixed tree (bitwise reproducible)
__global__ void __launch_bounds__(256) k_colsum_partials(const double* __restrict__ partial, long nb, long ldp,
                                                         double* __restrict__ out) {
  __shared__ double red[8];
  const long c = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double sacc = strided_colsum(partial, nb, ldp, c);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
  if (lane == 0) red[warp] = sacc;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w];
    out[c] = t;
  }
}
void colsum_partials(const double* partial, long nb, long ldp, long t, double* out, cudaStream_t s) {
  if (t == 0) return;
  k_colsum_partials<<<static_cast<unsigned>(t), 256, 0, s>>>(partial, nb, ldp, out);
  FSA_LAUNCH_CHECK();
}

void gemm_km(const double* A, long lda, long Mr, long K, const double* B, long ldb, long N, double* Y, long ldy,
             double alpha, double beta, cudaStream_t s) {
  require(Mr % 64 == 0 && K % 16 == 0 && N == pad_cols(N), "gemm_km: unpadded shape");
  if (Mr == 0 || N == 0) return;
  const int nt = tile_nt(N);
  dim3 grid(static_cast<unsigned>(Mr / 64), static_cast<unsigned>(N / (nt * 8)), 1);
  if (beta == 0.0)
    dispatch_nt<ReduceCfg>(nt, A, lda, B, ldb, nullptr, K, K, grid, EpiStore{Y, ldy, alpha}, s);
  else
    dispatch_nt<ReduceCfg>(nt, A, lda, B, ldb, nullptr, K, K, grid, EpiAxpby{Y, ldy, alpha, beta}, s);
}

size_t gemm_reduce_scratch(long Mr, long N, long K) {
  const ReducePlan p = plan_reduce(Mr, N, K);
  return static_cast<size_t>(p.splits * Mr * N);
}

void gemm_reduce(const double* M, long ldm, long Mr, long K, const double* V, long ldv, long N,
                 const double* scale, double* out, long ldo, double alpha, double beta, double* scratch,
                 cudaStream_t s) {
  require(Mr % 64 == 0 && K % 16 == 0 && N == pad_cols(N), "gemm_reduce: unpadded shape");
  if (Mr == 0 || N == 0) return;
  const ReducePlan p = plan_reduce(Mr, N, K);
  dim3 grid(static_cast<unsigned>(Mr / p.bm), static_cast<unsigned>(N / (p.nt * 8)),
            static_cast<unsigned>(p.splits));
  if (p.bm == 128)
    dispatch_nt<ReduceCfg8>(p.nt, M, ldm, V, ldv, scale, K, p.kchunk, grid, EpiPartial{scratch, Mr, N}, s);
  else
    dispatch_nt<ReduceCfg>(p.nt, M, ldm, V, ldv, scale, K, p.kchunk, grid, EpiPartial{scratch, Mr, N}, s);
  const long total = Mr * N;
  k_splitk_reduce<<<static_cast<unsigned>(cdiv(total, 256)), 256, 0, s>>>(scratch, p.splits, Mr, N, out, ldo,
                                                                         alpha, beta);
  FSA_LAUNCH_CHECK();
}

namespace {
__global__ void k_mirror_lower(double* A, long ld, long m) {
  const long idx = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= m * m) return;
  const long r = idx / m, c = idx % m;
  if (c > r) A[r * ld + c] = A[c * ld + r];
}
}  // namespace

static int syrk_waves() {
  static const int v = knob("FSA_SYRK_WAVES", 3);  // 1: 2.47 ms, 2: 1.31, 3: 1.27 (config 2)
  return v;
}
// only the lower-triangle tiles work (the rest exit at once): split K so that they fill whole waves
static ReducePlan plan_syrk(long Mr, long K) {
  ReducePlan p = plan_reduce(Mr, Mr, K);
  const long rt = Mr / p.bm, ct = Mr / (p.nt * 8), per = p.nt * 8;
  long active = 0;
  for (long r = 0; r < rt; ++r)
    for (long c = 0; c < ct; ++c) active += (c * per < (r + 1) * p.bm) ? 1 : 0;
  long splits = std::max<long>(1, syrk_waves() * kNumSMs / std::max<long>(active, 1));
  splits = std::min<long>(splits, std::max<long>(1, K / 16));
  p.kchunk = round_up(cdiv(K, splits), 16);
  p.splits = cdiv(K, p.kchunk);
  return p;
}
size_t gemm_syrk_scratch(long Mr, long K) {
  const ReducePlan p = plan_syrk(Mr, K);
  return static_cast<size_t>(p.splits * Mr * Mr);
}
void gemm_syrk(const double* M, long ldm, long Mr, long K, const double* scale, double* out, long ldo, double alpha,
               double* scratch, cudaStream_t s) {
  require(Mr % 128 == 0 && K % 16 == 0, "gemm_syrk: unpadded shape");
  if (Mr == 0) return;
  const long N = Mr;
  const ReducePlan p = plan_syrk(Mr, K);
  dim3 grid(static_cast<unsigned>(Mr / p.bm), static_cast<unsigned>(N / (p.nt * 8)), static_cast<unsigned>(p.splits));
  if (p.bm == 128)
    dispatch_nt<ReduceCfg8>(p.nt, M, ldm, M, ldm, scale, K, p.kchunk, grid, EpiPartialLower{scratch, Mr, N}, s);
  else
    dispatch_nt<ReduceCfg>(p.nt, M, ldm, M, ldm, scale, K, p.kchunk, grid, EpiPartialLower{scratch, Mr, N}, s);
  k_splitk_reduce<<<static_cast<unsigned>(cdiv(Mr * N, 256)), 256, 0, s>>>(scratch, p.splits, Mr, N, out, ldo, alpha,
                                                                         0.0);
  FSA_LAUNCH_CHECK();
  k_mirror_lower<<<static_cast<unsigned>(cdiv(Mr * N, 256)), 256, 0, s>>>(out, ldo, Mr);
  FSA_LAUNCH_CHECK();
}


// ---- core solve of the fused FITC sweep: W = Qinv S (Qinv symmetric m_pad x m_pad, S and W
// m_pad x ld row-major, ld = 8 NT <= 72). One CTA per 8 rows of W, its eight warps splitting K
// (m_pad / 8 each) on DMMA m8n8k4 with operands read through L1 (Qinv rows are its columns:
// contiguous), then the warps' 8 x ld partials are added in a fixed order. One launch, no
// split-K scratch in HBM.
namespace {
template <int NT>
__global__ void __launch_bounds__(256) k_core_dmma(const double* __restrict__ Qinv, long mp,
                                                  const double* __restrict__ S, long ld,
                                                  double* __restrict__ W, unsigned long long* __restrict__ wmax) {
  __shared__ double red[8][8][NT * 8];
  pdl_wait();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long r0 = static_cast<long>(blockIdx.x) * 8;
  const long kper = mp / 8, k0 = warp * kper;
  double c[NT][2];
#pragma unroll
  for (int j = 0; j < NT; ++j) c[j][0] = c[j][1] = 0.0;
  const double* ap = Qinv + (r0 + (lane >> 2)) * mp + (lane & 3);  // A[m = lane / 4][k = lane % 4]
  const double* bp = S + static_cast<long>(lane & 3) * ld + (lane >> 2);  // B[k = lane % 4][n = lane / 4]
#pragma unroll 4
  for (long k = k0; k < k0 + kper; k += 4) {
    const double a = __ldg(ap + k);
    double b[NT];
#pragma unroll
    for (int j = 0; j < NT; ++j) b[j] = __ldg(bp + k * ld + j * 8);
#pragma unroll
    for (int j = 0; j < NT; ++j) dmma8x8x4(c[j][0], c[j][1], a, b[j]);
  }
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    red[warp][lane >> 2][j * 8 + 2 * (lane & 3)] = c[j][0];
    red[warp][lane >> 2][j * 8 + 2 * (lane & 3) + 1] = c[j][1];
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < 8 * NT * 8; idx += blockDim.x) {
    const int r = idx / (NT * 8), cc = idx % (NT * 8);
    double acc = red[0][r][cc];
#pragma unroll
    for (int w = 1; w < 8; ++w) acc += red[w][r][cc];
    W[(r0 + r) * ld + cc] = acc;
    red[0][r][cc] = fabs(acc);  // (this thread alone read red[*][r][cc])
  }
  if (wmax != nullptr) {  // column maxima of |W| for the expansion's digit planes (non-negative bits)
    __syncthreads();
    for (int cc = threadIdx.x; cc < NT * 8; cc += blockDim.x) {
      double mx = 0.0;
#pragma unroll
      for (int r = 0; r < 8; ++r) mx = fmax(mx, red[0][r][cc]);
      if (mx > 0.0) atomicMax(wmax + cc, static_cast<unsigned long long>(__double_as_longlong(mx)));
    }
  }
}
// Wider variant (m_pad % 64 == 0): 16 warps split K (m_pad / 16 each, all loads of a warp in
// flight at once) and the column tiles are split over blockIdx.y (NTC tiles per CTA, nt here), so
// the launch has 2 x m_pad / 8 CTAs and each warp a K chain half as long; the warps' partials are
// added in a fixed order ((w + (w + 8)) pairs, then w = 0..7).
template <int NTC>
__global__ void __launch_bounds__(512) k_core_dmma16(const double* __restrict__ Qinv, long mp,
                                                    const double* __restrict__ S, long ld, int nt_all,
                                                    double* __restrict__ W, unsigned long long* __restrict__ wmax) {
  __shared__ double red[8][8][NTC * 8];
  pdl_wait();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int j0 = blockIdx.y * NTC, nt = min(NTC, nt_all - j0);
  const long r0 = static_cast<long>(blockIdx.x) * 8;
  const long kper = mp / 16, k0 = warp * kper;
  double c[NTC][2];
#pragma unroll
  for (int j = 0; j < NTC; ++j) c[j][0] = c[j][1] = 0.0;
  const double* ap = Qinv + (r0 + (lane >> 2)) * mp + (lane & 3);
  const double* bp = S + static_cast<long>(lane & 3) * ld + (lane >> 2) + j0 * 8;
#pragma unroll 8
  for (long k = k0; k < k0 + kper; k += 4) {
    const double a = __ldg(ap + k);
    double b[NTC];
#pragma unroll
    for (int j = 0; j < NTC; ++j) b[j] = j < nt ? __ldg(bp + k * ld + j * 8) : 0.0;
#pragma unroll
    for (int j = 0; j < NTC; ++j)
      if (j < nt) dmma8x8x4(c[j][0], c[j][1], a, b[j]);
  }
  if (warp >= 8) {
#pragma unroll
    for (int j = 0; j < NTC; ++j) {
      red[warp - 8][lane >> 2][j * 8 + 2 * (lane & 3)] = c[j][0];
      red[warp - 8][lane >> 2][j * 8 + 2 * (lane & 3) + 1] = c[j][1];
    }
  }
  __syncthreads();
  if (warp < 8) {
#pragma unroll
    for (int j = 0; j < NTC; ++j) {
      double* p = &red[warp][lane >> 2][j * 8 + 2 * (lane & 3)];
      p[0] = c[j][0] + p[0];
      p[1] = c[j][1] + p[1];
    }
  }
  __syncthreads();
  const int ncol = nt * 8;
  for (int idx = threadIdx.x; idx < 8 * ncol; idx += blockDim.x) {
    const int r = idx / ncol, cc = idx % ncol;
    double acc = red[0][r][cc];
#pragma unroll
    for (int w = 1; w < 8; ++w) acc += red[w][r][cc];
    W[(r0 + r) * ld + j0 * 8 + cc] = acc;
    red[0][r][cc] = fabs(acc);  // (this thread alone read red[*][r][cc])
  }
  if (wmax != nullptr) {
    __syncthreads();
    for (int cc = threadIdx.x; cc < ncol; cc += blockDim.x) {
      double mx = 0.0;
#pragma unroll
      for (int r = 0; r < 8; ++r) mx = fmax(mx, red[0][r][cc]);
      if (mx > 0.0) atomicMax(wmax + j0 * 8 + cc, static_cast<unsigned long long>(__double_as_longlong(mx)));
    }
  }
}
}  // namespace

bool core_apply_supported(long mp, long ld) { return mp % 32 == 0 && ld % 8 == 0 && ld <= 72; }

void core_apply(const double* Qinv, long mp, const double* S, long ld, double* W, cudaStream_t s,
                unsigned long long* wmax) {
  require(core_apply_supported(mp, ld), "core_apply: unsupported shape");
  const unsigned grid = static_cast<unsigned>(mp / 8);
  const int nt = static_cast<int>(ld / 8);
  if (mp % 64 == 0 && nt >= 2) {
    const int ntc = (nt + 1) / 2;
    const dim3 g2(grid, 2);
    switch (ntc) {
      case 1: launch_pdl(k_core_dmma16<1>, g2, dim3(512), 0, s, Qinv, mp, S, ld, nt, W, wmax); break;
      case 2: launch_pdl(k_core_dmma16<2>, g2, dim3(512), 0, s, Qinv, mp, S, ld, nt, W, wmax); break;
      case 3: launch_pdl(k_core_dmma16<3>, g2, dim3(512), 0, s, Qinv, mp, S, ld, nt, W, wmax); break;
      case 4: launch_pdl(k_core_dmma16<4>, g2, dim3(512), 0, s, Qinv, mp, S, ld, nt, W, wmax); break;
      default: launch_pdl(k_core_dmma16<5>, g2, dim3(512), 0, s, Qinv, mp, S, ld, nt, W, wmax); break;
    }
    FSA_LAUNCH_CHECK();
    return;
  }
  switch (ld / 8) {
    case 1: launch_pdl(k_core_dmma<1>, grid, dim3(256), 0, s, Qinv, mp, S, ld, W, wmax); break;
    case 2: launch_pdl(k_core_dmma<2>, grid, dim3(256), 0, s, Qinv, mp, S, ld, W, wmax); break;
    case 3: launch_pdl(k_core_dmma<3>, grid, dim3(256), 0, s, Qinv, mp, S, ld, W, wmax); break;
    case 4: launch_pdl(k_core_dmma<4>, grid, dim3(256), 0, s, Qinv, mp, S, ld, W, wmax); break;
    case 5: launch_pdl(k_core_dmma<5>, grid, dim3(256), 0, s, Qinv, mp, S, ld, W, wmax); break;
    case 6: launch_pdl(k_core_dmma<6>, grid, dim3(256), 0, s, Qinv, mp, S, ld, W, wmax); break;
    case 7: launch_pdl(k_core_dmma<7>, grid, dim3(256), 0, s, Qinv, mp, S, ld, W, wmax); break;
    case 8: launch_pdl(k_core_dmma<8>, grid, dim3(256), 0, s, Qinv, mp, S, ld, W, wmax); break;
    default: launch_pdl(k_core_dmma<9>, grid, dim3(256), 0, s, Qinv, mp, S, ld, W, wmax); break;
  }
  FSA_LAUNCH_CHECK();
}

}  // namespace fsa
