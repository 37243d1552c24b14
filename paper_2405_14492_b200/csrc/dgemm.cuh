// FP64 tensor-core (DMMA m8n8k4) GEMMs for the skinny low-rank contractions of
// the FSA operator. sm_100a has no FP64 tcgen05 kind; the FP64 tensor path on
// Blackwell is the warp-level DMMA (SASS `DMMA.8x8x4`).
//
// Two shapes cover every dense product on the path (SURVEY.md §8a rows a4-a8,
// a11, a13, a17):
//   expand  Y[rows x N] = M^T W      M stored one column per point (m contiguous),
//                                    W (K x N) row-major; rows = points (huge),
//                                    K = m, N = RHS columns. Fused epilogues.
//   reduce  C[Mr x N]  = M diag(s) V  M as above, V (points x N) row-major; the
//                                    contraction runs over points, split-K with
//                                    a fixed-order (deterministic) reduction.
// Operands stream HBM -> smem with cp.async (3 stages); every dimension is padded
// on the host so tiles never need bounds checks.
#pragma once

#include "common.cuh"

namespace fsa {

__device__ __forceinline__ void dmma8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
// this thread's part of sum_b partial[b][c] over b = tid, tid + 256, ... (blockDim 256), in two
// interleaved accumulators (s0: b = tid + 512 i, s1: b = tid + 256 + 512 i) -- the fixed order every
// column sum of the CG partials uses; eight loads are issued before they are added (same order)
__device__ __forceinline__ double strided_colsum(const double* __restrict__ partial, long nb, long ldp, long c) {
  double s0 = 0.0, s1 = 0.0;
  long b = threadIdx.x;
  for (; b + 7 * 256 < nb; b += 8 * 256) {
    double v[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = partial[(b + 256 * i) * ldp + c];
#pragma unroll
    for (int i = 0; i < 8; i += 2) {
      s0 += v[i];
      s1 += v[i + 1];
    }
  }
  for (; b + 256 < nb; b += 512) {
    s0 += partial[b * ldp + c];
    s1 += partial[(b + 256) * ldp + c];
  }
  if (b < nb) s0 += partial[b * ldp + c];
  return s0 + s1;
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

template <int NT_, int WMT_, int WARPS_, bool A_KM_, int BK_, int STAGES_>
struct GemmCfg {
  static constexpr int NT = NT_, WMT = WMT_, WARPS = WARPS_, BK = BK_, STAGES = STAGES_;
  static constexpr bool A_KM = A_KM_;  // A stored [k][m] (m contiguous) vs [m][k]
  static constexpr int BM = WARPS * WMT * 8;
  static constexpr int BN = NT * 8;
  static constexpr int THREADS = WARPS * 32;
  static constexpr int LDA = A_KM ? (BM + 4) : (BK + 4);  // == 4 (mod 16): conflict-free 8B fragments
  static constexpr int A_TILE = A_KM ? BK * LDA : BM * LDA;
  static constexpr int LDB = BN + (20 - BN % 16) % 16;
  static constexpr int B_TILE = BK * LDB;
  static constexpr int STAGE = A_TILE + B_TILE + BK;  // + per-k scale
  static constexpr int SMEM_BYTES = STAGES * STAGE * 8;
  static_assert(BM % 16 == 0, "BM must be a multiple of 16");
  static_assert(BK % 4 == 0, "BK must be a multiple of 4");
};

// Generic DMMA GEMM: acc[m][n] = sum_{k in [kb, ke)} A(m,k) * s_k * B(k,n)
//   A(m,k) = A_KM ? A[k*lda + m] : A[m*lda + k]      B(k,n) = B[k*ldb + n]
// Tile origin: m0 = blockIdx.x*BM, n0 = blockIdx.y*BN; k range from blockIdx.z.
template <class Cfg, class Epi>
__global__ void __launch_bounds__(Cfg::THREADS)
    k_dgemm(const double* __restrict__ A, long lda, const double* __restrict__ B, long ldb,
            const double* __restrict__ scale, long K, long kchunk, Epi epi) {
  constexpr int BM = Cfg::BM, BN = Cfg::BN, BK = Cfg::BK, NT = Cfg::NT, WMT = Cfg::WMT;
  constexpr int LDA = Cfg::LDA, LDB = Cfg::LDB, STAGES = Cfg::STAGES, THREADS = Cfg::THREADS;
  extern __shared__ __align__(16) double smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tig = lane & 3;
  const long m0 = static_cast<long>(blockIdx.x) * BM;
  const long n0 = static_cast<long>(blockIdx.y) * BN;
  const long kb = static_cast<long>(blockIdx.z) * kchunk;
  const long ke = kb + kchunk < K ? kb + kchunk : K;
  if constexpr (Epi::kLower) {  // symmetric result: tiles strictly above the diagonal are mirrored later
    if (n0 >= m0 + BM) return;
  }
  const int nk = ke > kb ? static_cast<int>((ke - kb) / BK) : 0;

  auto load_stage = [&](int st, long k0) {
    double* As = smem + st * Cfg::STAGE;
    double* Bs = As + Cfg::A_TILE;
    double* Ss = Bs + Cfg::B_TILE;
    if constexpr (Cfg::A_KM) {
      constexpr int CH = BK * BM / 2;
      for (int c = tid; c < CH; c += THREADS) {
        const int kk = c / (BM / 2), mm = (c % (BM / 2)) * 2;
        cp_async16(As + kk * LDA + mm, A + (k0 + kk) * lda + m0 + mm);
      }
    } else {
      constexpr int CH = BM * BK / 2;
      for (int c = tid; c < CH; c += THREADS) {
        const int mm = c / (BK / 2), kk = (c % (BK / 2)) * 2;
        cp_async16(As + mm * LDA + kk, A + (m0 + mm) * lda + k0 + kk);
      }
    }
    {
      constexpr int CH = BK * BN / 2;
      for (int c = tid; c < CH; c += THREADS) {
        const int kk = c / (BN / 2), nn = (c % (BN / 2)) * 2;
        cp_async16(Bs + kk * LDB + nn, B + (k0 + kk) * ldb + n0 + nn);
      }
    }
    if (scale != nullptr && tid < BK / 2) cp_async16(Ss + tid * 2, scale + k0 + tid * 2);
  };

  double acc[WMT][NT][2];
#pragma unroll
  for (int i = 0; i < WMT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load_stage(s, kb + static_cast<long>(s) * BK);
    cp_async_commit();
  }
  const int wm0 = warp * WMT * 8;
  for (int it = 0; it < nk; ++it) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    const int st = it % STAGES;
    const double* As = smem + st * Cfg::STAGE;
    const double* Bs = As + Cfg::A_TILE;
    const double* Ss = Bs + Cfg::B_TILE;
#pragma unroll
    for (int k4 = 0; k4 < BK / 4; ++k4) {
      const int k = k4 * 4 + tig;
      double a[WMT], b[NT];
#pragma unroll
      for (int i = 0; i < WMT; ++i)
        a[i] = Cfg::A_KM ? As[k * LDA + wm0 + i * 8 + g] : As[(wm0 + i * 8 + g) * LDA + k];
      const double sk = scale != nullptr ? Ss[k] : 1.0;
#pragma unroll
      for (int j = 0; j < NT; ++j) b[j] = Bs[k * LDB + j * 8 + g] * sk;
#pragma unroll
      for (int i = 0; i < WMT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma8x8x4(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
    const int nxt = it + STAGES - 1;
    if (nxt < nk) load_stage(nxt % STAGES, kb + static_cast<long>(nxt) * BK);
    cp_async_commit();
  }
  cp_async_wait<0>();

  double dacc[NT][2];
#pragma unroll
  for (int j = 0; j < NT; ++j) dacc[j][0] = dacc[j][1] = 0.0;
#pragma unroll
  for (int i = 0; i < WMT; ++i) {
    const long row = m0 + wm0 + i * 8 + g;
#pragma unroll
    for (int j = 0; j < NT; ++j) {
      const long col = n0 + j * 8 + 2 * tig;
      const double2 c = epi(row, col, acc[i][j][0], acc[i][j][1]);
      if constexpr (Epi::kDot) {
        dacc[j][0] += c.x;
        dacc[j][1] += c.y;
      }
    }
  }
  if constexpr (Epi::kDot) {
    // per-column partial of the epilogue's dot contributions over this tile's rows:
    // lanes sharing tig (xor 4, 8, 16), then warps in order -> partial[blockIdx.x][col]
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        double v = dacc[j][e];
        v += __shfl_xor_sync(0xffffffffu, v, 4);
        v += __shfl_xor_sync(0xffffffffu, v, 8);
        v += __shfl_xor_sync(0xffffffffu, v, 16);
        dacc[j][e] = v;
      }
    __syncthreads();
    double* red = smem;  // [WARPS][BN]
    if (g == 0)
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        red[warp * BN + j * 8 + 2 * tig] = dacc[j][0];
        red[warp * BN + j * 8 + 2 * tig + 1] = dacc[j][1];
      }
    __syncthreads();
    for (int c = tid; c < BN; c += THREADS) {
      double sacc = 0.0;
      for (int w = 0; w < Cfg::WARPS; ++w) sacc += red[w * BN + c];
      epi.partial[static_cast<long>(blockIdx.x) * epi.ldp + n0 + c] = sacc;
    }
  }
}

// ---- epilogues -------------------------------------------------------------------
struct EpiNoDot {
  static constexpr bool kDot = false;
  static constexpr bool kLower = false;
  double* partial = nullptr;
  long ldp = 0;
};
struct EpiStore : EpiNoDot {  // Y = alpha * v
  double* Y;
  long ldy;
  double alpha;
  EpiStore(double* y, long l, double a) : Y(y), ldy(l), alpha(a) {}
  __device__ double2 operator()(long r, long c, double v0, double v1) const {
    double2 o = make_double2(alpha * v0, alpha * v1);
    *reinterpret_cast<double2*>(Y + r * ldy + c) = o;
    return make_double2(0.0, 0.0);
  }
};
struct EpiAxpby : EpiNoDot {  // Y = alpha * v + beta * Y
  double* Y;
  long ldy;
  double alpha, beta;
  EpiAxpby(double* y, long l, double a, double b) : Y(y), ldy(l), alpha(a), beta(b) {}
  __device__ double2 operator()(long r, long c, double v0, double v1) const {
    double2* p = reinterpret_cast<double2*>(Y + r * ldy + c);
    double2 o = *p;
    o.x = alpha * v0 + beta * o.x;
    o.y = alpha * v1 + beta * o.y;
    *p = o;
    return make_double2(0.0, 0.0);
  }
};
struct EpiPartial : EpiNoDot {  // split-K partial tile: W[z][r][c]
  double* W;
  long M, N;
  EpiPartial(double* w, long m, long n) : W(w), M(m), N(n) {}
  __device__ double2 operator()(long r, long c, double v0, double v1) const {
    *reinterpret_cast<double2*>(W + (static_cast<long>(blockIdx.z) * M + r) * N + c) = make_double2(v0, v1);
    return make_double2(0.0, 0.0);
  }
};
struct EpiPartialLower : EpiPartial {  // lower-triangle tiles only (symmetric products)
  static constexpr bool kLower = true;
  using EpiPartial::EpiPartial;
};
struct EpiProbe : EpiNoDot {  // z = U^T e1 + sqrt(D) e2  (FITC sample, preconditioners.cpp:69-73)
  double* Y;
  long ld;
  const double* sqrtD;
  const double* E2;
  EpiProbe(double* y, long l, const double* s, const double* e) : Y(y), ld(l), sqrtD(s), E2(e) {}
  __device__ double2 operator()(long r, long c, double v0, double v1) const {
    const double s = sqrtD[r];
    const double2 e = *reinterpret_cast<const double2*>(E2 + r * ld + c);
    *reinterpret_cast<double2*>(Y + r * ld + c) = make_double2(v0 + s * e.x, v1 + s * e.y);
    return make_double2(0.0, 0.0);
  }
};
// Z = D^{-1} (R - U^T w)  (Woodbury tail of P^{-1} R); with kDot also the
// per-CTA partial of r . z per column (the PCG's rz, krylov.cpp:84)
template <bool DOT>
struct EpiWoodburyT {
  static constexpr bool kDot = DOT;
  static constexpr bool kLower = false;
  double* partial;
  long ldp;
  double* Z;
  const double* R;
  long ld;
  const double* Dinv;
  __device__ double2 operator()(long r, long c, double v0, double v1) const {
    const double di = Dinv[r];
    const double2 x = *reinterpret_cast<const double2*>(R + r * ld + c);
    const double z0 = (x.x - v0) * di, z1 = (x.y - v1) * di;
    *reinterpret_cast<double2*>(Z + r * ld + c) = make_double2(z0, z1);
    return make_double2(x.x * z0, x.y * z1);
  }
};
using EpiWoodbury = EpiWoodburyT<false>;
using EpiWoodburyDot = EpiWoodburyT<true>;

// Woodbury tail that also keeps Lw = U^T w (the low-rank part of Sigma Z, used by
// the PCG's m-space recurrence for Sigma H) and the per-CTA r . z partials
struct EpiWoodburyKeep {
  static constexpr bool kDot = true;
  static constexpr bool kLower = false;
  double* partial;
  long ldp;
  double* Z;
  double* Lw;
  const double* R;
  long ld;
  const double* Dinv;
  __device__ double2 operator()(long r, long c, double v0, double v1) const {
    const double di = Dinv[r];
    const double2 x = *reinterpret_cast<const double2*>(R + r * ld + c);
    const double z0 = (x.x - v0) * di, z1 = (x.y - v1) * di;
    *reinterpret_cast<double2*>(Z + r * ld + c) = make_double2(z0, z1);
    *reinterpret_cast<double2*>(Lw + r * ld + c) = make_double2(v0, v1);
    return make_double2(x.x * z0, x.y * z1);
  }
};

// ---- host launchers (instantiated in dgemm.cu) -----------------------------------
struct Workspace;  // split-K scratch, see dgemm.cu

// Y = epi(M^T W): M column-per-point [rows][ldm] (k < K contiguous), W [K][ldw] (N cols).
// rows % 128 == 0, K % 16 == 0, N == pad_cols(N).
void gemm_expand_store(const double* M, long ldm, long rows, long K, const double* W, long ldw, long N,
                       double* Y, long ldy, double alpha, double beta, cudaStream_t s);
void gemm_expand_probe(const double* M, long ldm, long rows, long K, const double* W, long ldw, long N,
                       double* Y, long ld, const double* sqrtD, const double* E2, cudaStream_t s);
void gemm_expand_woodbury(const double* M, long ldm, long rows, long K, const double* W, long ldw, long N,
                          double* Z, const double* R, long ld, const double* Dinv, cudaStream_t s);
// same, plus rz[c] = sum_rows R[r][c] Z[r][c] for c < N (deterministic two-level reduction);
// partial must hold (rows / 128) * N doubles
void gemm_expand_woodbury_dot(const double* M, long ldm, long rows, long K, const double* W, long ldw, long N,
                              double* Z, const double* R, long ld, const double* Dinv, double* rz, double* partial,
                              cudaStream_t s);
// same with Lw = U^T w kept (n_pad x N, ld)
void gemm_expand_woodbury_keep(const double* M, long ldm, long rows, long K, const double* W, long ldw, long N,
                               double* Z, double* Lw, const double* R, long ld, const double* Dinv, double* rz,
                               double* partial, cudaStream_t s);
// out[c] = sum_{b < nb} partial[b * ldp + c], c < t (fixed order)
void colsum_partials(const double* partial, long nb, long ldp, long t, double* out, cudaStream_t s);

// out[Mr x N] (row-major, ldo) = alpha * sum_{i<K} M[i*ldm + r] s_i V[i*ldv + n] + beta * out
// Mr % 64 == 0, K % 16 == 0. Deterministic split-K. `scratch` must hold
// gemm_reduce_scratch(Mr, N, K) doubles.
size_t gemm_reduce_scratch(long Mr, long N, long K);
// Unsplit variant with A stored [k][m] and a store/axpby epilogue into row-major Y:
// Y[r*ldy + c] = alpha * sum_k A[k*lda + r] B[k*ldb + c] + beta * Y. Mr % 64 == 0, N == pad_cols(N).
void gemm_km(const double* A, long lda, long Mr, long K, const double* B, long ldb, long N, double* Y, long ldy,
             double alpha, double beta, cudaStream_t s);
void gemm_reduce(const double* M, long ldm, long Mr, long K, const double* V, long ldv, long N,
                 const double* scale, double* out, long ldo, double alpha, double beta, double* scratch,
                 cudaStream_t s);
// symmetric variant (V = M, N = Mr): out = alpha M diag(s) M^T, lower tiles computed and mirrored;
// scratch holds gemm_syrk_scratch(Mr, K) doubles
size_t gemm_syrk_scratch(long Mr, long K);
void gemm_syrk(const double* M, long ldm, long Mr, long K, const double* scale, double* out, long ldo, double alpha,
               double* scratch, cudaStream_t s);

// W = Qinv S for the fused FITC sweep (Qinv symmetric m_pad x m_pad; S, W m_pad x ld row-major,
// ld a multiple of 8, <= 72): one launch of DMMA tiles with an in-CTA split of K
bool core_apply_supported(long mp, long ld);
// wmax (optional, zeroed by the caller): atomicMax of the bit patterns of |W| per column
void core_apply(const double* Qinv, long mp, const double* S, long ld, double* W, cudaStream_t s,
                unsigned long long* wmax = nullptr);

}  // namespace fsa
