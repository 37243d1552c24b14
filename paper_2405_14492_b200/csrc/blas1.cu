// Column-batched vector kernels for the lockstep multi-RHS PCG
// (reference krylov.cpp:42-93): per-column dot products with a fixed-order
// two-level reduction (bitwise reproducible), masked axpys, the per-column
// scalar recurrences with Lanczos-tridiagonal capture, and the host<->device
// layout conversions (column-major original order <-> row-major internal order).
#include "blas1.cuh"

namespace fsa {

namespace {

constexpr int kDotBlocks = 2 * kNumSMs;
constexpr int kDotThreads = 256;

// partial[b][c] for columns c in [0, t); rows split into kDotBlocks contiguous chunks
template <bool W>
__global__ void __launch_bounds__(kDotThreads) k_coldot_partial(const double* __restrict__ A,
                                                               const double* __restrict__ B,
                                                               const double* __restrict__ w, long n, long ld, long t,
                                                               double* __restrict__ partial) {
  __shared__ double red[kDotThreads];
  const long chunk = (n + gridDim.x - 1) / gridDim.x;
  const long r0 = static_cast<long>(blockIdx.x) * chunk;
  const long r1 = r0 + chunk < n ? r0 + chunk : n;
  const int tid = threadIdx.x;
  const int cl = tid % 64, rl = tid / 64;  // 64 columns x 4 row lanes
  for (long c0 = 0; c0 < t; c0 += 64) {
    const long c = c0 + cl;
    double s = 0.0;
    if (c < t)
      for (long r = r0 + rl; r < r1; r += 4) {
        const double v = A[r * ld + c] * B[r * ld + c];
        s += W ? v * w[r] : v;
      }
    red[tid] = s;
    __syncthreads();
    if (rl == 0 && c < t)
      partial[static_cast<long>(blockIdx.x) * t + c] = (red[cl] + red[cl + 64]) + (red[cl + 128] + red[cl + 192]);
    __syncthreads();
  }
}

__global__ void k_coldot_final(const double* __restrict__ partial, int nb, long t, double* __restrict__ out) {
  const long c = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c >= t) return;
  double s = 0.0;
  for (int b = 0; b < nb; ++b) s += partial[static_cast<long>(b) * t + c];
  out[c] = s;
}

__global__ void k_pack(const double* __restrict__ in, long n, long k, const int* __restrict__ perm, long n_pad,
                       long tp, long col0, double* __restrict__ out) {
  const long idx = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= n_pad * k) return;
  const long i = idx / k, j = idx % k;
  out[i * tp + col0 + j] = i < n ? in[static_cast<long>(perm[i]) + j * n] : 0.0;
}

__global__ void k_copy_cols(const double* __restrict__ src, long lds, double* __restrict__ dst, long ldd, long n,
                            long k) {
  const long idx = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= n * k) return;
  const long i = idx / k, j = idx % k;
  dst[i * ldd + j] = src[i * lds + j];
}

__global__ void k_sum_log(const double* __restrict__ x, long n, double* out) {
  __shared__ double red[256];
  double s = 0.0;
  for (long i = threadIdx.x; i < n; i += blockDim.x) s += log(x[i]);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

__global__ void k_affine(double* __restrict__ y, const double* __restrict__ x, double a, double b, long n,
                         long n_pad) {
  const long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n_pad) return;
  y[i] = i < n ? (x[i] + a) * b : 0.0;
}

// pinv_i = 1/D_i - q_i / D_i^2 (diag(P^{-1}), preconditioners.cpp:88-92)
__global__ void k_pinv_diag(double* __restrict__ out, const double* __restrict__ D, const double* __restrict__ q,
                            long n, long n_pad) {
  const long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n_pad) return;
  out[i] = i < n ? 1.0 / D[i] - q[i] / (D[i] * D[i]) : 0.0;
}

__global__ void k_add_identity(double* A, long ld, long m) {
  const long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < m) A[i * ld + i] += 1.0;
}

__global__ void k_unpack(const double* __restrict__ in, long n, long k, const int* __restrict__ perm, long tp,
                         long col0, double* __restrict__ out) {
  const long idx = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= n * k) return;
  const long i = idx / k, j = idx % k;
  out[static_cast<long>(perm[i]) + j * n] = in[i * tp + col0 + j];
}

// ---- PCG control (one thread per column) ----------------------------------------------
__global__ void k_cg_start(const double* __restrict__ rr, long k, double tol, CgState st) {
  const long j = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= k) return;
  st.iterations[j] = 0;
  st.alpha_prev[j] = 1.0;
  st.beta_prev[j] = 0.0;
  st.rz[j] = 0.0;
  const bool conv = sqrt(rr[j]) < tol;  // krylov.cpp:44
  st.converged[j] = conv ? 1 : 0;
  st.active[j] = conv ? 0 : 1;
  st.scale[j] = conv ? 0.0 : 1.0;
}

__global__ void k_cg_start_rz(const double* __restrict__ rz, long k, CgState st) {
  const long j = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= k) return;
  if (!st.active[j]) return;
  st.rz[j] = rz[j];
  if (!(rz[j] > 0.0)) atomicCAS(st.err, 0, kErrPrecondNotPD);  // krylov.cpp:51
}

// alpha = rz / h'v, tridiagonal push (krylov.cpp:66-75)
__global__ void k_cg_alpha(const double* __restrict__ hv, long k, int it, int max_iter, CgState st) {
  const long j = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= k) return;
  if (!st.active[j]) {
    st.alpha[j] = 0.0;
    return;
  }
  if (!(hv[j] > 0.0)) {
    atomicCAS(st.err, 0, kErrOperatorNotPD);
    st.alpha[j] = 0.0;
    return;
  }
  const double a = st.rz[j] / hv[j];
  st.alpha[j] = a;
  st.tdiag[j * max_iter + it] = 1.0 / a + st.beta_prev[j] / st.alpha_prev[j];
  if (it > 0) st.toff[j * max_iter + it - 1] = sqrt(st.beta_prev[j]) / st.alpha_prev[j];
  st.iterations[j] = it + 1;
}

// residual test on the unpreconditioned residual (krylov.cpp:77-82)
__global__ void k_cg_check(const double* __restrict__ rr, long k, double tol, CgState st) {
  const long j = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= k) return;
  if (!st.active[j]) return;
  if (sqrt(rr[j]) < tol) {
    st.converged[j] = 1;
    st.active[j] = 0;
  }
}

// beta = rz_new / rz (krylov.cpp:83-90)
__global__ void k_cg_beta(const double* __restrict__ rzn, long k, CgState st) {
  const long j = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= k) return;
  if (!st.active[j]) {
    st.beta[j] = 0.0;
    return;
  }
  if (!(rzn[j] > 0.0)) {
    atomicCAS(st.err, 0, kErrPrecondNotPD);
    st.beta[j] = 0.0;
    return;
  }
  const double b = rzn[j] / st.rz[j];
  st.beta[j] = b;
  st.beta_prev[j] = b;
  st.alpha_prev[j] = st.alpha[j];
  st.rz[j] = rzn[j];
}

__global__ void k_cg_count(long k, CgState st) {
  __shared__ int cnt;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  for (long j = threadIdx.x; j < k; j += blockDim.x)
    if (st.active[j]) atomicAdd(&cnt, 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    st.host_flags[0] = cnt;
    st.host_flags[1] = *st.err;
  }
}

// X += alpha H ; R -= alpha V   (active columns only; alpha = 0 otherwise)
__global__ void k_update_xr(double* __restrict__ X, double* __restrict__ R, const double* __restrict__ H,
                            const double* __restrict__ V, const double* __restrict__ alpha, long n, long tp, long k) {
  const long idx = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= n * tp) return;
  const long j = idx % tp;
  if (j >= k) return;
  const double a = alpha[j];
  if (a == 0.0) return;
  X[idx] += a * H[idx];
  R[idx] -= a * V[idx];
}

// H = Z + beta H for active columns
__global__ void k_update_h(double* __restrict__ H, const double* __restrict__ Z, const int* __restrict__ active,
                           const double* __restrict__ beta, long n, long tp, long k) {
  const long idx = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= n * tp) return;
  const long j = idx % tp;
  if (j >= k || !active[j]) return;
  H[idx] = Z[idx] + beta[j] * H[idx];
}

// H = Z on active columns, 0 elsewhere
__global__ void k_init_h(double* __restrict__ H, const double* __restrict__ Z, const int* __restrict__ active,
                         long n, long tp, long k) {
  const long idx = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= n * tp) return;
  const long j = idx % tp;
  H[idx] = (j < k && active[j]) ? Z[idx] : 0.0;
}

__global__ void k_scale_rows(double* __restrict__ Y, const double* __restrict__ X, const double* __restrict__ w,
                             long n, long tp) {
  const long idx = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= n * tp) return;
  Y[idx] = X[idx] * w[idx / tp];
}

__global__ void k_axpby(double* __restrict__ Y, const double* __restrict__ X, double a, double b, long len) {
  const long idx = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= len) return;
  Y[idx] = a * X[idx] + b * Y[idx];
}

inline unsigned nblk(long total, int th = 256) { return static_cast<unsigned>(cdiv(total, th)); }

}  // namespace

size_t coldot_scratch(long n, long t) {
  (void)n;
  return static_cast<size_t>(kDotBlocks) * static_cast<size_t>(t);
}

void launch_coldot(const double* A, const double* B, long n, long ld, long t, double* out, double* scratch,
                   cudaStream_t s) {
  k_coldot_partial<false><<<kDotBlocks, kDotThreads, 0, s>>>(A, B, nullptr, n, ld, t, scratch);
  FSA_LAUNCH_CHECK();
  k_coldot_final<<<nblk(t, 128), 128, 0, s>>>(scratch, kDotBlocks, t, out);
  FSA_LAUNCH_CHECK();
}

void launch_coldot_weighted(const double* A, const double* B, const double* w, long n, long ld, long t,
                            double* out, double* scratch, cudaStream_t s) {
  k_coldot_partial<true><<<kDotBlocks, kDotThreads, 0, s>>>(A, B, w, n, ld, t, scratch);
  FSA_LAUNCH_CHECK();
  k_coldot_final<<<nblk(t, 128), 128, 0, s>>>(scratch, kDotBlocks, t, out);
  FSA_LAUNCH_CHECK();
}

void pack_cols(const double* in_dev, long n, long k, const int* perm_dev, long n_pad, long tp, long col0,
               double* out, cudaStream_t s) {
  if (k == 0) return;
  k_pack<<<nblk(n_pad * k), 256, 0, s>>>(in_dev, n, k, perm_dev, n_pad, tp, col0, out);
  FSA_LAUNCH_CHECK();
}
void copy_cols(const double* src, long lds, double* dst, long ldd, long n, long k, cudaStream_t s) {
  if (n * k == 0) return;
  k_copy_cols<<<nblk(n * k), 256, 0, s>>>(src, lds, dst, ldd, n, k);
  FSA_LAUNCH_CHECK();
}
void sum_log(const double* x, long n, double* out_dev, cudaStream_t s) {
  k_sum_log<<<1, 256, 0, s>>>(x, n, out_dev);
  FSA_LAUNCH_CHECK();
}
void affine_vec(double* y, const double* x, double a, double b, long n, long n_pad, cudaStream_t s) {
  k_affine<<<nblk(n_pad), 256, 0, s>>>(y, x, a, b, n, n_pad);
  FSA_LAUNCH_CHECK();
}
void pinv_diag(double* out, const double* D, const double* q, long n, long n_pad, cudaStream_t s) {
  k_pinv_diag<<<nblk(n_pad), 256, 0, s>>>(out, D, q, n, n_pad);
  FSA_LAUNCH_CHECK();
}
void add_identity(double* A, long ld, long m, cudaStream_t s) {
  k_add_identity<<<nblk(m), 256, 0, s>>>(A, ld, m);
  FSA_LAUNCH_CHECK();
}
void unpack_cols(const double* in, long n, long k, const int* perm_dev, long tp, long col0, double* out_dev,
                 cudaStream_t s) {
  if (n * k == 0) return;
  k_unpack<<<nblk(n * k), 256, 0, s>>>(in, n, k, perm_dev, tp, col0, out_dev);
  FSA_LAUNCH_CHECK();
}

void cg_start(const double* rr, long k, double tol, const CgState& st, cudaStream_t s) {
  k_cg_start<<<nblk(k, 128), 128, 0, s>>>(rr, k, tol, st);
  FSA_LAUNCH_CHECK();
}
void cg_start_rz(const double* rz, long k, const CgState& st, cudaStream_t s) {
  k_cg_start_rz<<<nblk(k, 128), 128, 0, s>>>(rz, k, st);
  FSA_LAUNCH_CHECK();
}
void cg_alpha(const double* hv, long k, int it, int max_iter, const CgState& st, cudaStream_t s) {
  k_cg_alpha<<<nblk(k, 128), 128, 0, s>>>(hv, k, it, max_iter, st);
  FSA_LAUNCH_CHECK();
}
void cg_check(const double* rr, long k, double tol, const CgState& st, cudaStream_t s) {
  k_cg_check<<<nblk(k, 128), 128, 0, s>>>(rr, k, tol, st);
  FSA_LAUNCH_CHECK();
}
void cg_beta(const double* rzn, long k, const CgState& st, cudaStream_t s) {
  k_cg_beta<<<nblk(k, 128), 128, 0, s>>>(rzn, k, st);
  FSA_LAUNCH_CHECK();
}
void cg_count(long k, const CgState& st, cudaStream_t s) {
  k_cg_count<<<1, 256, 0, s>>>(k, st);
  FSA_LAUNCH_CHECK();
}
void update_xr(double* X, double* R, const double* H, const double* V, const double* alpha, long n, long tp, long k,
               cudaStream_t s) {
  k_update_xr<<<nblk(n * tp), 256, 0, s>>>(X, R, H, V, alpha, n, tp, k);
  FSA_LAUNCH_CHECK();
}
void update_h(double* H, const double* Z, const int* active, const double* beta, long n, long tp, long k,
              cudaStream_t s) {
  k_update_h<<<nblk(n * tp), 256, 0, s>>>(H, Z, active, beta, n, tp, k);
  FSA_LAUNCH_CHECK();
}
void init_h(double* H, const double* Z, const int* active, long n, long tp, long k, cudaStream_t s) {
  k_init_h<<<nblk(n * tp), 256, 0, s>>>(H, Z, active, n, tp, k);
  FSA_LAUNCH_CHECK();
}
void scale_rows(double* Y, const double* X, const double* w, long n, long tp, cudaStream_t s) {
  k_scale_rows<<<nblk(n * tp), 256, 0, s>>>(Y, X, w, n, tp);
  FSA_LAUNCH_CHECK();
}
void axpby(double* Y, const double* X, double a, double b, long len, cudaStream_t s) {
  if (len == 0) return;
  k_axpby<<<nblk(len), 256, 0, s>>>(Y, X, a, b, len);
  FSA_LAUNCH_CHECK();
}

}  // namespace fsa
