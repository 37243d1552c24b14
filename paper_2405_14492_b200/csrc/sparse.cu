// Sparse kernels of the FSA operator:
//  * SDDMM assembly of the tapered residual block straight into CSR
//    (reference fsa.cpp:38-56): value = (C(d) - U_r . U_c) T(d), diagonal
//    max(sigma1_2 - |U_r|^2, 0) + sigma2 with the clamp counted;
//  * its rho derivative on the same pattern (fsa.cpp:101-124, U-form);
//  * the cross block to prediction points (prediction.cpp:16-24);
//  * CSR x dense SpMM on row-major RHS blocks.
// One warp per CSR row; the row's m-vector lives in registers (m/32 per lane).
#include "kernels.cuh"
#include "sparse.cuh"

namespace fsa {

namespace {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int MQ>
__device__ __forceinline__ void load_vec(const double* __restrict__ p, int lane, double* v) {
#pragma unroll
  for (int q = 0; q < MQ; ++q) v[q] = p[lane + 32 * q];
}
template <int MQ>
__device__ __forceinline__ double dot_vec(const double* v, const double* __restrict__ p, int lane) {
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < MQ; ++q) s = fma(v[q], p[lane + 32 * q], s);
  return warp_sum(s);
}

// Sigma_s values on the pattern (rows and cols are the same internal point set)
template <int MQ>
__global__ void k_sddmm_sigma_s(const double* __restrict__ U, long ldu, const long* __restrict__ rowptr,
                                const int* __restrict__ col, const double* __restrict__ dist,
                                const double* __restrict__ lowrank_diag, long n, SddmmParams P,
                                double* __restrict__ val, int* __restrict__ n_clamped) {
  const long r = (static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= n) return;
  double ur[MQ];
  load_vec<MQ>(U + r * ldu, lane, ur);
  const long pe = rowptr[r + 1];
  for (long p = rowptr[r]; p < pe; ++p) {
    const long c = col[p];
    if (c == r) {
      if (lane == 0) {
        double resid = P.sigma1_2 - lowrank_diag[r];
        if (resid < 0.0) {
          resid = 0.0;
          atomicAdd(n_clamped, 1);
        }
        val[p] = resid + P.sigma2;
      }
      continue;
    }
    const double dt = dot_vec<MQ>(ur, U + c * ldu, lane);
    if (lane == 0) {
      const double d = dist[p];
      val[p] = (matern_d(d, P.nu, P.sigma1_2, P.rho) - dt) * taper_d(d, P.family, P.gamma);
    }
  }
}

// d Sigma_s / d rho (U-form of fsa.cpp:107-122): dl = U1_r.U_c + U_r.T_c with
// U1 = L^{-1} dSigma_mn/drho, T = U1 - K2 U, K2 = L^{-1} dSigma_m/drho L^{-T}
template <int MQ>
__global__ void k_sddmm_drho(const double* __restrict__ U, const double* __restrict__ U1,
                             const double* __restrict__ T, long ldu, const long* __restrict__ rowptr,
                             const int* __restrict__ col, const double* __restrict__ dist,
                             const double* __restrict__ lowrank_diag, long n, SddmmParams P,
                             double* __restrict__ val) {
  const long r = (static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= n) return;
  double ur[MQ], u1r[MQ];
  load_vec<MQ>(U + r * ldu, lane, ur);
  load_vec<MQ>(U1 + r * ldu, lane, u1r);
  const long pe = rowptr[r + 1];
  for (long p = rowptr[r]; p < pe; ++p) {
    const long c = col[p];
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < MQ; ++q) {
      s = fma(u1r[q], U[c * ldu + lane + 32 * q], s);
      s = fma(ur[q], T[c * ldu + lane + 32 * q], s);
    }
    const double dl = warp_sum(s);
    if (lane == 0) {
      if (c == r) {
        const bool clamped = P.sigma1_2 - lowrank_diag[r] < 0.0;
        val[p] = clamped ? 0.0 : -dl;
      } else {
        const double d = dist[p];
        val[p] = (matern_drho_d(d, P.nu, P.sigma1_2, P.rho) - dl) * taper_d(d, P.family, P.gamma);
      }
    }
  }
}

// cross block: rows of Rm (training or prediction points), columns of Cm; the
// dot is always U_train . Up_pred so that both orientations agree bitwise.
template <int MQ>
__global__ void k_sddmm_cross(const double* __restrict__ Rm, long ldr, const double* __restrict__ Cm, long ldc,
                              const long* __restrict__ rowptr, const int* __restrict__ col,
                              const double* __restrict__ dist, long nrows, SddmmParams P,
                              double* __restrict__ val) {
  const long r = (static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= nrows) return;
  double vr[MQ];
  load_vec<MQ>(Rm + r * ldr, lane, vr);
  const long pe = rowptr[r + 1];
  for (long p = rowptr[r]; p < pe; ++p) {
    const long c = col[p];
    const double dt = dot_vec<MQ>(vr, Cm + c * ldc, lane);
    if (lane == 0) {
      const double d = dist[p];
      val[p] = (matern_d(d, P.nu, P.sigma1_2, P.rho) - dt) * taper_d(d, P.family, P.gamma);
    }
  }
}

__global__ void k_colnorm2(const double* __restrict__ U, long ldu, long mpad, long n, long n_pad,
                           double* __restrict__ out) {
  const long i = (static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= n_pad) return;
  double s = 0.0;
  if (i < n)
    for (long r = lane; r < mpad; r += 32) {
      const double v = U[i * ldu + r];
      s = fma(v, v, s);
    }
  s = warp_sum(s);
  if (lane == 0) out[i] = s;
}

__global__ void k_extract_diag(const double* __restrict__ val, const long* __restrict__ diagpos, long n, long n_pad,
                               double* __restrict__ D, double* __restrict__ Dinv, double* __restrict__ sqrtD) {
  const long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n_pad) return;
  const double d = i < n ? val[diagpos[i]] : 1.0;
  D[i] = d;
  if (Dinv) Dinv[i] = 1.0 / d;
  if (sqrtD) sqrtD[i] = sqrt(d);
}

// Y[r, c] = alpha * sum_p val[p] X[col[p], c] + beta * Y[r, c]   (warp per row, 2 cols per lane)
__global__ void k_spmm(const long* __restrict__ rowptr, const int* __restrict__ col, const double* __restrict__ val,
                       long nrows, const double* __restrict__ X, long ldx, double* __restrict__ Y, long ldy,
                       long ncols, double alpha, double beta) {
  const long r = (static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= nrows) return;
  const long pb = rowptr[r], pe = rowptr[r + 1];
  for (long c0 = 0; c0 < ncols; c0 += 64) {
    const long c = c0 + 2 * lane;
    if (c >= ncols) break;
    double a0 = 0.0, a1 = 0.0;
    for (long p = pb; p < pe; ++p) {
      const double v = val[p];
      const double2 x = *reinterpret_cast<const double2*>(X + static_cast<long>(col[p]) * ldx + c);
      a0 = fma(v, x.x, a0);
      a1 = fma(v, x.y, a1);
    }
    double2* y = reinterpret_cast<double2*>(Y + r * ldy + c);
    double2 o;
    if (beta == 0.0) {
      o = make_double2(alpha * a0, alpha * a1);
    } else {
      o = *y;
      o.x = alpha * a0 + beta * o.x;
      o.y = alpha * a1 + beta * o.y;
    }
    *y = o;
  }
}

#define FSA_DISPATCH_MQ(KERNEL, mpad, grid, s, ...)                                      \
  do {                                                                                  \
    switch (static_cast<int>((mpad) / 32)) {                                            \
      case 4: KERNEL<4><<<grid, 256, 0, s>>>(__VA_ARGS__); break;                       \
      case 8: KERNEL<8><<<grid, 256, 0, s>>>(__VA_ARGS__); break;                       \
      case 12: KERNEL<12><<<grid, 256, 0, s>>>(__VA_ARGS__); break;                     \
      case 16: KERNEL<16><<<grid, 256, 0, s>>>(__VA_ARGS__); break;                     \
      case 20: KERNEL<20><<<grid, 256, 0, s>>>(__VA_ARGS__); break;                     \
      case 24: KERNEL<24><<<grid, 256, 0, s>>>(__VA_ARGS__); break;                     \
      case 28: KERNEL<28><<<grid, 256, 0, s>>>(__VA_ARGS__); break;                     \
      case 32: KERNEL<32><<<grid, 256, 0, s>>>(__VA_ARGS__); break;                     \
      default: throw std::invalid_argument("more than 1024 inducing points are not supported"); \
    }                                                                                   \
    FSA_LAUNCH_CHECK();                                                                 \
  } while (0)

}  // namespace

void sddmm_sigma_s(const double* U, long ldu, const Csr& pat, const double* lowrank_diag, const SddmmParams& P,
                   double* val, int* n_clamped_dev, cudaStream_t s) {
  FSA_CUDA(cudaMemsetAsync(n_clamped_dev, 0, sizeof(int), s));
  const unsigned grid = static_cast<unsigned>(cdiv(pat.rows * 32, 256));
  if (grid == 0) return;
  FSA_DISPATCH_MQ(k_sddmm_sigma_s, ldu, grid, s, U, ldu, pat.rowptr.get(), pat.col.get(), pat.dist.get(),
                  lowrank_diag, pat.rows, P, val, n_clamped_dev);
}

void sddmm_drho(const double* U, const double* U1, const double* T, long ldu, const Csr& pat,
                const double* lowrank_diag, const SddmmParams& P, double* val, cudaStream_t s) {
  const unsigned grid = static_cast<unsigned>(cdiv(pat.rows * 32, 256));
  if (grid == 0) return;
  FSA_DISPATCH_MQ(k_sddmm_drho, ldu, grid, s, U, U1, T, ldu, pat.rowptr.get(), pat.col.get(), pat.dist.get(),
                  lowrank_diag, pat.rows, P, val);
}

void sddmm_cross(const double* Rm, long ldr, const double* Cm, long ldc, const Csr& pat, const SddmmParams& P,
                 double* val, cudaStream_t s) {
  const unsigned grid = static_cast<unsigned>(cdiv(pat.rows * 32, 256));
  if (grid == 0) return;
  FSA_DISPATCH_MQ(k_sddmm_cross, ldr, grid, s, Rm, ldr, Cm, ldc, pat.rowptr.get(), pat.col.get(),
                  pat.dist.get(), pat.rows, P, val);
}

void colnorm2(const double* U, long ldu, long mpad, long n, long n_pad, double* out, cudaStream_t s) {
  k_colnorm2<<<static_cast<unsigned>(cdiv(n_pad * 32, 256)), 256, 0, s>>>(U, ldu, mpad, n, n_pad, out);
  FSA_LAUNCH_CHECK();
}

void extract_diag(const double* val, const long* diagpos, long n, long n_pad, double* D, double* Dinv,
                  double* sqrtD, cudaStream_t s) {
  k_extract_diag<<<static_cast<unsigned>(cdiv(n_pad, 256)), 256, 0, s>>>(val, diagpos, n, n_pad, D, Dinv, sqrtD);
  FSA_LAUNCH_CHECK();
}

void launch_spmm(const long* rowptr, const int* col, const double* val, long nrows, const double* X, long ldx,
                 double* Y, long ldy, long ncols, double alpha, double beta, cudaStream_t s) {
  if (nrows == 0) return;
  k_spmm<<<static_cast<unsigned>(cdiv(nrows * 32, 256)), 256, 0, s>>>(rowptr, col, val, nrows, X, ldx, Y, ldy,
                                                                     ncols, alpha, beta);
  FSA_LAUNCH_CHECK();
}

}  // namespace fsa
