// Covariance assembly and the m x m dense linear algebra of the FSA setup:
// Matern cross covariances (reference kernels.cpp:54-76), Cholesky of the
// inducing block (fsa.cpp:23-30) and the blocked triangular solve
// U = L^{-1} Sigma_mn (fsa.cpp:33) with its GEMM updates on DMMA.
#include <cstdlib>

#include "dgemm.cuh"
#include "kernels.cuh"

namespace fsa {

namespace {

template <int D>
__global__ void k_cross_cov(const double* __restrict__ ind, long ldi, long m, long mpad,
                            const double* __restrict__ pts, long ldp, long npts, long npts_pad, int nu, double s1,
                            double rho, int mode, double* __restrict__ M, long ldm) {
  extern __shared__ double sind[];  // [D][mpad]
  for (long r = threadIdx.x; r < m; r += blockDim.x)
#pragma unroll
    for (int k = 0; k < D; ++k) sind[k * mpad + r] = ind[r + k * ldi];
  __syncthreads();
  constexpr int PPB = 8;  // points per block
  const long i0 = static_cast<long>(blockIdx.x) * PPB;
  for (int q = 0; q < PPB; ++q) {
    const long i = i0 + q;
    if (i >= npts_pad) break;
    double* col = M + i * ldm;
    if (i >= npts) {
      for (long r = threadIdx.x; r < mpad; r += blockDim.x) col[r] = 0.0;
      continue;
    }
    for (long r = threadIdx.x; r < mpad; r += blockDim.x) {
      double v = 0.0;
      if (r < m) {
        const double dd = pdist_soa<D>(sind, mpad, r, pts, ldp, i);
        v = mode == 0 ? matern_d(dd, nu, s1, rho) : matern_drho_d(dd, nu, s1, rho);
      }
      col[r] = v;
    }
  }
}

__global__ void k_sigma_m_fix(double* S, long m, long mpad, double jitter, int mode) {
  const long idx = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= mpad) return;
  if (idx < m) {
    if (mode == 0) S[idx * mpad + idx] += jitter;
  } else {
    S[idx * mpad + idx] = mode == 0 ? 1.0 : 0.0;  // identity padding keeps the factor regular
  }
}

// One 64-column panel of a blocked right-looking Cholesky (column-major, ld = mpad).
// Block 0 factors the diagonal block and writes it back; blocks b >= 1 redo the
// (cheap) diagonal factorisation and solve their 64 panel rows.
// Factorisation: thread (r, c0) keeps row r, columns c0, c0 + 4, ... of the block in registers. The
// (final, unscaled) column j is published in shared memory one step ahead by its owners, every
// thread forms 1 / l_jj = rsqrt(a_jj) itself and scales the entries it needs on the fly: one
// barrier and one rsqrt on the critical path per column (no sqrt + divide chain).
// Panel rows: the four threads of a row sit in one warp and pass x_c by shuffle, so the forward
// substitution X L^T = A_rows runs without block barriers (x_c = (...) * (1 / l_cc)).
__global__ void __launch_bounds__(256) k_potrf_panel(double* A, long ld, long k0, int* info, double* diag_out) {
  extern __shared__ double psm[];
  double(*Lk)[65] = reinterpret_cast<double(*)[65]>(psm);
  __shared__ double colbuf[2][64], invd[64];
  __shared__ int bad;
  const int tid = threadIdx.x;
  if (tid == 0) bad = 0;
  {
    const int r = tid & 63, c0 = tid >> 6;
    double x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = A[(k0 + c0 + 4 * i) * ld + k0 + r];
    if (c0 == 0) colbuf[0][r] = x[0];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 64; ++j) {
      const double* cb = colbuf[j & 1];
      double dj = cb[j];
      if (!(dj > 0.0) || !isfinite(dj)) {
        if (tid == 0 && !bad) bad = j + 1;
        dj = 1.0;
      }
      const double inv = rsqrt(dj);
      const double lr = cb[r] * inv;  // l_rj (r > j)
      if (c0 == (j & 3)) {
        if (r == j) {
          Lk[j][j] = dj * inv;
          invd[j] = inv;
        } else {
          Lk[r][j] = r > j ? lr : 0.0;
        }
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int c = c0 + 4 * i;
        if (c > j && r >= c) x[i] = fma(-lr, cb[c] * inv, x[i]);
      }
      if (j + 1 < 64 && c0 == ((j + 1) & 3)) colbuf[(j + 1) & 1][r] = x[(j + 1) >> 2];
      __syncthreads();
    }
  }
  if (blockIdx.x == 0) {
    // the factored diagonal block goes to scratch: the other blocks of this launch
    // still read the unfactored block from A (copied back by k_copy_diag_blocks)
    double* out = diag_out + (k0 / 64) * 4096;
    for (int idx = tid; idx < 64 * 64; idx += blockDim.x) {
      const int r = idx % 64, c = idx / 64;
      out[c * 64 + r] = Lk[r][c];
    }
    if (tid == 0 && bad && *info == 0) *info = static_cast<int>(k0) + bad;
    return;
  }
  // panel rows rb .. rb+63: solve X Lk^T = A_rows; lane (rr % 8) * 4 + q owns row rr, columns q, q + 4, ...
  const long rb = k0 + 64 * static_cast<long>(blockIdx.x);
  {
    const int lane = tid & 31, q = lane & 3, rr = (tid >> 5) * 8 + (lane >> 2);
    double x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = A[(k0 + q + 4 * i) * ld + rb + rr];
#pragma unroll
    for (int c = 0; c < 64; ++c) {
      if (q == (c & 3)) x[c >> 2] *= invd[c];
      const double xc = __shfl_sync(0xffffffffu, x[c >> 2], (lane & ~3) | (c & 3));
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (4 * i + 3 > c) {  // (columns q + 4 i <= c of this thread are skipped by the predicate)
          if (q + 4 * i > c) x[i] = fma(-xc, Lk[q + 4 * i][c], x[i]);
        }
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) A[(k0 + q + 4 * i) * ld + rb + rr] = x[i];
  }
}

__global__ void k_copy_diag_blocks(double* A, long ld, const double* blocks) {
  const long kb = blockIdx.x;
  const double* src = blocks + kb * 4096;
  for (int idx = threadIdx.x; idx < 4096; idx += blockDim.x) {
    const int r = idx % 64, c = idx / 64;
    A[(kb * 64 + c) * ld + kb * 64 + r] = src[idx];
  }
}

__global__ void k_zero_upper(double* A, long ld, long n) {
  const long idx = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= n * n) return;
  const long r = idx % n, c = idx / n;
  if (r < c) A[c * ld + r] = 0.0;
}

// inverse of each 64x64 diagonal block of a lower-triangular L (col-major):
// Dinv[kb][c*64 + r] = (L_kk^{-1})(r, c)
__global__ void __launch_bounds__(256) k_trinv_blocks(const double* L, long ld, double* Dinv) {
  extern __shared__ double tsm[];
  double(*Lk)[65] = reinterpret_cast<double(*)[65]>(tsm);
  const long k0 = 64 * static_cast<long>(blockIdx.x);
  const int tid = threadIdx.x;
  for (int idx = tid; idx < 64 * 64; idx += blockDim.x) {
    const int r = idx & 63, c = idx >> 6;
    Lk[r][c] = L[(k0 + c) * ld + k0 + r];
  }
  __syncthreads();
  __shared__ double invd[64];
  if (tid < 64) invd[tid] = 1.0 / Lk[tid][tid];
  __syncthreads();
  // column col of the inverse: right-looking forward substitution on e_col; the four lanes of a
  // column (rows part, part + 4, ... in registers) pass x_r by shuffle, no barriers
  const int col = tid >> 2, part = tid & 3, lane = tid & 31;
  double x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = part + 4 * i == col ? 1.0 : 0.0;
#pragma unroll
  for (int r = 0; r < 64; ++r) {
    if (part == (r & 3)) x[r >> 2] *= invd[r];
    const double xr = __shfl_sync(0xffffffffu, x[r >> 2], (lane & ~3) | (r & 3));
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (4 * i + 3 > r) {
        if (part + 4 * i > r) x[i] = fma(-xr, Lk[part + 4 * i][r], x[i]);
      }
  }
  double* out = Dinv + blockIdx.x * 4096L;
#pragma unroll
  for (int i = 0; i < 16; ++i) out[col * 64 + part + 4 * i] = x[i];
}

// Inverse of the 128 x 128 diagonal block [A 0; C D] of L from the 64 x 64 inverses:
// [A^-1 0; E D^-1] with E = -D^-1 C A^-1, written as the GEMM operand W[k][c] = inv(c, k)
// (128 x 128, ld 128) of trsm_lower_cols' 128-wide steps. One CTA per block.
constexpr int kInv128Smem = 4 * 64 * 65 * 8;
__global__ void __launch_bounds__(256) k_inv128(const double* __restrict__ L, long ld, const double* __restrict__ dinv,
                                                double* __restrict__ W128) {
  extern __shared__ double ism[];
  double(*Ai)[65] = reinterpret_cast<double(*)[65]>(ism);
  double(*Di)[65] = reinterpret_cast<double(*)[65]>(ism + 64 * 65);
  double(*Cm)[65] = reinterpret_cast<double(*)[65]>(ism + 2 * 64 * 65);
  double(*Tm)[65] = reinterpret_cast<double(*)[65]>(ism + 3 * 64 * 65);
  const long b = blockIdx.x, k0 = 128 * b;
  const int tid = threadIdx.x;
  const double* ai = dinv + (2 * b) * 4096L;      // ai[c * 64 + r] = A^-1(r, c)
  const double* di = dinv + (2 * b + 1) * 4096L;
  for (int idx = tid; idx < 4096; idx += 256) {
    const int r = idx & 63, c = idx >> 6;
    Ai[r][c] = ai[c * 64 + r];
    Di[r][c] = di[c * 64 + r];
    Cm[r][c] = L[(k0 + c) * ld + k0 + 64 + r];
  }
  __syncthreads();
  const int r = tid & 63, c0 = tid >> 6;
  for (int i = 0; i < 16; ++i) {  // T = C A^-1 (A^-1 lower: k >= c)
    const int c = c0 + 4 * i;
    double t = 0.0;
    for (int k = c; k < 64; ++k) t = fma(Cm[r][k], Ai[k][c], t);
    Tm[r][c] = t;
  }
  __syncthreads();
  double* out = W128 + b * 16384L;
  for (int i = 0; i < 16; ++i) {  // E = -D^-1 T (D^-1 lower: k <= r)
    const int c = c0 + 4 * i;
    double e = 0.0;
    for (int k = 0; k <= r; ++k) e = fma(Di[r][k], Tm[k][c], e);
    out[c * 128 + 64 + r] = -e;            // inv(64 + r, c)
    out[(64 + c) * 128 + r] = 0.0;         // inv(r, 64 + c) = 0
    out[c * 128 + r] = Ai[r][c];           // inv(r, c)
    out[(64 + c) * 128 + 64 + r] = Di[r][c];
  }
}

__global__ void k_transpose(const double* __restrict__ A, long lda, long rows, long cols, double* __restrict__ B,
                            long ldb) {
  __shared__ double t[32][33];
  const long bx = static_cast<long>(blockIdx.x) * 32, by = static_cast<long>(blockIdx.y) * 32;
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const long r = by + j, c = bx + threadIdx.x;
    if (r < rows && c < cols) t[j][threadIdx.x] = A[r * lda + c];
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const long c = bx + j, r = by + threadIdx.x;
    if (r < rows && c < cols) B[c * ldb + r] = t[threadIdx.x][j];
  }
}

__global__ void k_logdet_diag(const double* L, long ld, long m, double* out) {
  __shared__ double red[256];
  double s = 0.0;
  for (long i = threadIdx.x; i < m; i += blockDim.x) s += log(L[i * ld + i]);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = 2.0 * red[0];
}

constexpr int kPanelSmem = 2 * 64 * 65 * 8;

void set_smem_attrs() {
  static bool done = false;
  if (done) return;
  FSA_CUDA(cudaFuncSetAttribute(k_potrf_panel, cudaFuncAttributeMaxDynamicSharedMemorySize, kPanelSmem));
  FSA_CUDA(cudaFuncSetAttribute(k_trinv_blocks, cudaFuncAttributeMaxDynamicSharedMemorySize, kPanelSmem));
  FSA_CUDA(cudaFuncSetAttribute(k_inv128, cudaFuncAttributeMaxDynamicSharedMemorySize, kInv128Smem));
  done = true;
}

}  // namespace

void launch_cross_cov(const double* ind, long ldi, long m, const double* pts, long ldp, long npts, long npts_pad,
                      int d, int nu, double s1, double rho, int mode, double* M, long ldm, cudaStream_t s) {
  const long mpad = ldm;
  const size_t sm = static_cast<size_t>(d * mpad) * sizeof(double);
  const unsigned grid = static_cast<unsigned>(cdiv(npts_pad, 8));
  if (grid == 0) return;
  switch (d) {
    case 1: k_cross_cov<1><<<grid, 256, sm, s>>>(ind, ldi, m, mpad, pts, ldp, npts, npts_pad, nu, s1, rho, mode, M, ldm); break;
    case 2: k_cross_cov<2><<<grid, 256, sm, s>>>(ind, ldi, m, mpad, pts, ldp, npts, npts_pad, nu, s1, rho, mode, M, ldm); break;
    case 3: k_cross_cov<3><<<grid, 256, sm, s>>>(ind, ldi, m, mpad, pts, ldp, npts, npts_pad, nu, s1, rho, mode, M, ldm); break;
    default: throw std::invalid_argument("dimension must be 1, 2 or 3");
  }
  FSA_LAUNCH_CHECK();
}

void launch_sigma_m(const double* ind, long ldi, long m, long mpad, int d, int nu, double s1, double rho,
                    double jitter, int mode, double* S, cudaStream_t s) {
  launch_cross_cov(ind, ldi, m, ind, ldi, m, mpad, d, nu, s1, rho, mode, S, mpad, s);
  k_sigma_m_fix<<<static_cast<unsigned>(cdiv(mpad, 256)), 256, 0, s>>>(S, m, mpad, jitter, mode);
  FSA_LAUNCH_CHECK();
}

void potrf_lower(double* A, long mpad, int* info_dev, double* scratch, cudaStream_t s) {
  require(mpad % 64 == 0, "potrf: mpad must be a multiple of 64");
  set_smem_attrs();
  FSA_CUDA(cudaMemsetAsync(info_dev, 0, sizeof(int), s));
  for (long k0 = 0; k0 < mpad; k0 += 64) {
    const long rest = mpad - k0 - 64;
    k_potrf_panel<<<static_cast<unsigned>(1 + rest / 64), 256, kPanelSmem, s>>>(A, mpad, k0, info_dev, scratch);
    FSA_LAUNCH_CHECK();
    if (rest > 0) {
      // trailing update of the full (symmetric) square: C -= P P^T
      double* P = A + k0 * mpad + k0 + 64;
      double* C = A + (k0 + 64) * mpad + k0 + 64;
      gemm_km(P, mpad, rest, 64, P, mpad, rest, C, mpad, -1.0, 1.0, s);
    }
  }
  k_zero_upper<<<static_cast<unsigned>(cdiv(mpad * mpad, 256)), 256, 0, s>>>(A, mpad, mpad);
  FSA_LAUNCH_CHECK();
  k_copy_diag_blocks<<<static_cast<unsigned>(mpad / 64), 256, 0, s>>>(A, mpad, scratch);
  FSA_LAUNCH_CHECK();
}

void trsm_lower_cols(const double* L, long mpad, double* B, long ldb, long npts, double* dinv, cudaStream_t s) {
  require(mpad % 64 == 0 && npts % 128 == 0, "trsm: unpadded shape");
  if (npts == 0) return;
  set_smem_attrs();
  k_trinv_blocks<<<static_cast<unsigned>(mpad / 64), 256, kPanelSmem, s>>>(L, mpad, dinv);
  FSA_LAUNCH_CHECK();
  if (mpad % 128 == 0) {
    // 128-wide steps: the trailing block of B is read and written half as often as with 64-wide
    // steps and every update runs over K = 128 (1.36 -> 1.25 ms at config 2). The diagonal step multiplies by the inverse of the
    // 128 x 128 block, upper half first: its columns need the step's unscaled lower columns.
    double* w128 = dinv + mpad * 64;
    k_inv128<<<static_cast<unsigned>(mpad / 128), 256, kInv128Smem, s>>>(L, mpad, dinv, w128);
    FSA_LAUNCH_CHECK();
    for (long k0 = 0; k0 < mpad; k0 += 128) {
      gemm_expand_store(B + k0, ldb, npts, 128, w128 + (k0 / 128) * 16384 + 64, 128, 64, B + k0 + 64, ldb, 1.0, 0.0, s);
      gemm_expand_store(B + k0, ldb, npts, 64, dinv + (k0 / 64) * 4096, 64, 64, B + k0, ldb, 1.0, 0.0, s);
      const long rest = mpad - k0 - 128;
      if (rest > 0)  // B[:, rest] -= L[rest, kk] B[:, kk]
        gemm_expand_store(B + k0, ldb, npts, 128, L + k0 * mpad + k0 + 128, mpad, rest, B + k0 + 128, ldb, -1.0, 1.0,
                          s);
    }
    return;
  }
  for (long k0 = 0; k0 < mpad; k0 += 64) {
    // B[:, k0:k0+64] = L_kk^{-1} B[:, k0:k0+64]   (in place; rows are points)
    gemm_expand_store(B + k0, ldb, npts, 64, dinv + (k0 / 64) * 4096, 64, 64, B + k0, ldb, 1.0, 0.0, s);
    const long rest = mpad - k0 - 64;
    if (rest > 0)  // B[:, rest] -= L[rest, kk] B[:, kk]
      gemm_expand_store(B + k0, ldb, npts, 64, L + k0 * mpad + k0 + 64, mpad, rest, B + k0 + 64, ldb, -1.0, 1.0,
                        s);
  }
}

void launch_transpose(const double* A, long lda, long rows, long cols, double* B, long ldb, cudaStream_t s) {
  dim3 grid(static_cast<unsigned>(cdiv(cols, 32)), static_cast<unsigned>(cdiv(rows, 32)));
  k_transpose<<<grid, dim3(32, 8), 0, s>>>(A, lda, rows, cols, B, ldb);
  FSA_LAUNCH_CHECK();
}

void launch_logdet_diag(const double* L, long ld, long m, double* out, cudaStream_t s) {
  k_logdet_diag<<<1, 256, 0, s>>>(L, ld, m, out);
  FSA_LAUNCH_CHECK();
}

}  // namespace fsa
