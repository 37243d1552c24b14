// Column-batched vector kernels and PCG control; see blas1.cu.
#pragma once

#include "common.cuh"

namespace fsa {

enum { kErrNone = 0, kErrOperatorNotPD = 1, kErrPrecondNotPD = 2 };

// Per-column PCG state, device resident (one entry per RHS column).
struct CgState {
  double* rz;
  double* alpha_prev;
  double* beta_prev;
  double* alpha;
  double* beta;
  double* scale;
  int* active;
  int* converged;
  int* iterations;
  double* tdiag;  // [k][max_iter]
  double* toff;   // [k][max_iter]
  double* rnorm;  // [k][max_iter]: ||r||_2 after each iteration (diagnostics: tie margins vs the oracle)
  int* err;
  int* host_flags;  // mapped pinned memory: [num_active, err]
  // graph-captured sweeps (fused single-rank path): the sweep index lives on the device; the
  // control kernels read it, and the last one (k_colsum_ctl<2>) writes the flags into slot
  // 2 (it % 2) of host_flags and advances it. nullptr: `it` comes from the host launch.
  int* it_dev = nullptr;
};

size_t coldot_scratch(long n, long t);
void launch_coldot(const double* A, const double* B, long n, long ld, long t, double* out, double* scratch,
                   cudaStream_t s);
void launch_coldot_weighted(const double* A, const double* B, const double* w, long n, long ld, long t,
                            double* out, double* scratch, cudaStream_t s);

// host layout (column-major n x k, original order, already on the device) ->
// columns [col0, col0 + k) of a row-major n_pad x tp internal-order block (padding rows zeroed)
void pack_cols(const double* in_dev, long n, long k, const int* perm_dev, long n_pad, long tp, long col0,
               double* out, cudaStream_t s);
// same with an input column stride ld_in (n rows of a longer array: a rank's rows)
void pack_cols_ld(const double* in_dev, long ld_in, long n, long k, const int* perm_dev, long n_pad, long tp,
                  long col0, double* out, cudaStream_t s);
// dst[i][j] = src[i][j] for i < n, j < k (row-major blocks of different widths)
void copy_cols(const double* src, long lds, double* dst, long ldd, long n, long k, cudaStream_t s);
void sum_log(const double* x, long n, double* out_dev, cudaStream_t s);
// y[i] = (x[i] + a) * b for i < n, 0 on padding
void affine_vec(double* y, const double* x, double a, double b, long n, long n_pad, cudaStream_t s);
void pinv_diag(double* out, const double* D, const double* q, long n, long n_pad, cudaStream_t s);
void add_identity(double* A, long ld, long m, cudaStream_t s);
// inverse of pack_cols for columns [col0, col0 + k)
void unpack_cols(const double* in, long n, long k, const int* perm_dev, long tp, long col0, double* out_dev,
                 cudaStream_t s);

void cg_start(const double* rr, long k, double tol, const CgState& st, cudaStream_t s);
void cg_start_rz(const double* rz, long k, const CgState& st, cudaStream_t s);
void cg_alpha(const double* hv, long k, int it, int max_iter, const CgState& st, cudaStream_t s);
void cg_check(const double* rr, long k, double tol, int it, int max_iter, const CgState& st, cudaStream_t s);
void cg_beta(const double* rzn, long k, const CgState& st, cudaStream_t s);
void cg_count(long k, const CgState& st, cudaStream_t s);
void update_xr(double* X, double* R, const double* H, const double* V, const double* alpha, long n, long tp, long k,
               cudaStream_t s);
// fused: X += alpha H, R -= alpha V (columns with alpha != 0) and rr[c] = |R_c|^2 (c < k)
void update_xr_dot(double* X, double* R, const double* H, const double* V, const double* alpha, long n, long tp,
                   long k, double* rr, double* scratch, cudaStream_t s);
// same for t_pad <= 64, also leaving the per-chunk column maxima of |dinv R| in ymax
// (atomicMax into [chunk][64], zeroed by the caller) for the Ozaki projection of R
void update_xr_dot_max(double* X, double* R, const double* H, const double* V, const double* alpha, long n, long tp,
                       long k, double* rr, double* scratch, const double* dinv, unsigned long long* ymax,
                       long chunk_rows, cudaStream_t s, bool colsum = true);
long xr_dot_max_blocks(long n);  // partial rows (ld k) left in scratch when colsum = false
// column sums of partials (as colsum_partials) fused with the per-column PCG control of the
// single-rank sweep: mode 0 alpha (cg_alpha), 1 residual test (cg_check), 2 beta + active count
// (cg_beta, cg_count; `ticket` is a zeroed device counter, left zero)
void colsum_ctl(int mode, const double* partial, long nb, long ldp, long t, double* out, long k, int it,
                int max_iter, double tol, const CgState& st, unsigned int* ticket, cudaStream_t s,
                unsigned long long* zero_buf = nullptr, long zero_len = 0,  // zero_buf[0, zero_len) := 0
                const double* partial_b = nullptr, long nb_b = 0, long ldp_b = 0,  // mode 3: the r.z sums
                double* out_b = nullptr);  // zero_buf[0, zero_len) := 0
// Jacobi PCG without a Z block: X += alpha H, R -= alpha V, rr = |R|^2, rz = R' diag(dinv) R;
// scratch holds 2 * coldot_scratch(n, k) doubles
void update_xr_dot_jacobi(double* X, double* R, const double* H, const double* V, const double* alpha,
                          const double* dinv, long n, long tp, long k, double* rr, double* rz, double* scratch,
                          cudaStream_t s);
// H = diag(dinv) R + beta H on the active columns (init: H = active ? diag(dinv) R : 0)
void update_h_jacobi(double* H, const double* R, const double* dinv, const int* active, const double* beta, long n,
                     long tp, long k, bool init, cudaStream_t s);
// m-space recurrence of U H for the active columns: UH = W + beta UH (init: UH = active ? W : 0)
void update_uh(double* UH, const double* W, const int* active, const double* beta, long mpad, long tp, long k,
               bool init, cudaStream_t s);
void update_h(double* H, const double* Z, const int* active, const double* beta, long n, long tp, long k,
              cudaStream_t s);
void init_h(double* H, const double* Z, const int* active, long n, long tp, long k, cudaStream_t s);
// scalar sums of the exact FITC traces: out[7] (see blas1.cu)
void trace_sums(const double* p, const double* d1, const double* dD, const double* f, const double* D, long n,
                const double* Qi, const double* K2, long m, double* out, cudaStream_t s);
// out[i] = sum_{r < len} A[i*ld + r] B[i*ld + r] for i < n (0 for n <= i < n_pad); warp per row
void row_dots(const double* A, const double* B, long ld, long len, long n, long n_pad, double* out, cudaStream_t s);
// H = Z + beta H and Vlr = Lw + beta Vlr on the active columns (tp even)
void update_h2(double* H, const double* Z, double* Vlr, const double* Lw, const int* active, const double* beta,
               long n, long tp, long k, cudaStream_t s);
// out[a * q + c] = sum_{i < n} A[i * lda + a] B[i * ldb + c] (a, c < q; deterministic)
size_t cross_gram_scratch(long q);
void cross_gram(const double* A, long lda, const double* B, long ldb, long n, long q, double* out, double* scratch,
                cudaStream_t s);
// GLS residual column: out[i * ldo] = X[i * ldx] - sum_a X[i * ldx + 1 + a] coef[a]
void gls_residual(const double* X, long ldx, long p, const double* coef_dev, long n, long n_pad, double* out, long ldo,
                  cudaStream_t s);
void scale_rows(double* Y, const double* X, const double* w, long n, long tp, cudaStream_t s);
void axpby(double* Y, const double* X, double a, double b, long len, cudaStream_t s);

}  // namespace fsa
