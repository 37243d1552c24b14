// Device kernels of the FSA iterative core (declarations of the host launchers).
#pragma once

#include "common.cuh"

namespace fsa {

// ---- covariance functions (reference kernels.cpp:7-52) ---------------------------
enum { NU12 = 0, NU32 = 1, NU52 = 2 };

__host__ __device__ __forceinline__ double matern_d(double d, int nu, double s1, double rho) {
  const double s = d / rho;
  if (nu == NU12) return s1 * exp(-s);
  if (nu == NU32) {
    const double x = 1.7320508075688772 * s;
    return s1 * (1.0 + x) * exp(-x);
  }
  const double x = 2.23606797749979 * s;
  return s1 * (1.0 + x + x * x / 3.0) * exp(-x);
}
__host__ __device__ __forceinline__ double matern_drho_d(double d, int nu, double s1, double rho) {
  const double s = d / rho;
  if (nu == NU12) return s1 * exp(-s) * d / (rho * rho);
  if (nu == NU32) {
    const double x = 1.7320508075688772 * s;
    return s1 * 3.0 * d * d / (rho * rho * rho) * exp(-x);
  }
  const double x = 2.23606797749979 * s;
  return s1 * (5.0 * d * d / (3.0 * rho * rho * rho)) * (1.0 + x) * exp(-x);
}
__host__ __device__ __forceinline__ double taper_d(double d, int family, double gamma) {
  const double r = d / gamma;
  if (r >= 1.0) return 0.0;
  const double omr = 1.0 - r;
  const double omr2 = omr * omr;
  if (family == 1) return omr2 * omr2 * (1.0 + 4.0 * r);
  const double omr6 = omr2 * omr2 * omr2;
  return omr6 * (1.0 + 6.0 * r + 35.0 * r * r / 3.0);
}

// Euclidean distance as the reference's contracted Eigen redux: s = d0^2; s = fma(dk, dk, s)
template <int D>
__host__ __device__ __forceinline__ double pdist_soa(const double* a, long lda, long i, const double* b, long ldb,
                                                     long j) {
  const double d0 = a[i] - b[j];
  double s = d0 * d0;
  for (int k = 1; k < D; ++k) {
    const double dk = a[i + k * lda] - b[j + k * ldb];
    s = fma(dk, dk, s);
  }
  return sqrt(s);
}

// ---- launchers ----------------------------------------------------------------------
// coords are SoA [d][ld] (internal point order). Output M column-per-point:
// M[i*ldm + r] = f(|ind_r - pt_i|) for r < m, i < npts; zero padding to (mpad, npts_pad).
// mode: 0 matern, 1 d/drho matern
void launch_cross_cov(const double* ind, long ldi, long m, const double* pts, long ldp, long npts, long npts_pad,
                      int d, int nu, double s1, double rho, int mode, double* M, long ldm, cudaStream_t s);
// Sigma_m (mpad x mpad, symmetric): matern + jitter on the diagonal, identity on the padding.
void launch_sigma_m(const double* ind, long ldi, long m, long mpad, int d, int nu, double s1, double rho,
                    double jitter, int mode, double* S, cudaStream_t s);

// Cholesky (lower, column-major, in place, upper triangle zeroed) of an mpad x mpad
// SPD matrix; *info_dev receives 0 or the first failing column + 1. scratch: mpad*64 doubles.
void potrf_lower(double* A, long mpad, int* info_dev, double* scratch, cudaStream_t s);
// B <- L^{-1} B for B stored one column per "point" (B[i*ldb + r], r < mpad), in place.
// Requires potrf output L (col-major) and scratch of mpad*192 doubles (64 x 64 and 128 x 128
// inverses of the diagonal blocks).
void trsm_lower_cols(const double* L, long mpad, double* B, long ldb, long npts, double* dinv_scratch,
                     cudaStream_t s);
// out = transpose of an mpad x mpad matrix (col-major <-> row-major)
void launch_transpose(const double* A, long lda, long rows, long cols, double* B, long ldb, cudaStream_t s);
// log-determinant partial: out = 2 * sum_i log(L_ii), i < m (single block)
void launch_logdet_diag(const double* L, long ld, long m, double* out, cudaStream_t s);

// ---- taper pattern -------------------------------------------------------------------
struct PatternDev;  // pattern.cu

// ---- sparse -----------------------------------------------------------------------------
// Y (row-major n x ld) = alpha * S X + beta * Y for the first `ncols` columns (ncols <= ld)
void launch_spmm(const long* rowptr, const int* col, const double* val, long nrows, const double* X, long ldx,
                 double* Y, long ldy, long ncols, double alpha, double beta, cudaStream_t s);
// Y (ncols_out rows) = S^T X : transpose SpMM via atomics-free two-pass using the transposed CSR
// (callers pass the transposed pattern).

// ---- blas-1 on n x t row-major blocks --------------------------------------------
// partial[b][j] = sum_{rows in block b} A[i][j] * B[i][j]; then out[j] = sum_b partial[b][j]
size_t coldot_scratch(long n, long t);
void launch_coldot(const double* A, const double* B, long n, long ld, long t, double* out, double* scratch,
                   cudaStream_t s);
void launch_coldot_weighted(const double* A, const double* B, const double* w, long n, long ld, long t,
                            double* out, double* scratch, cudaStream_t s);

}  // namespace fsa
