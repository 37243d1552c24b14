// Column-batched vector kernels for the lockstep multi-RHS PCG
// (reference krylov.cpp:42-93): per-column dot products with a fixed-order
// two-level reduction (bitwise reproducible), masked axpys, the per-column
// scalar recurrences with Lanczos-tridiagonal capture, and the host<->device
// layout conversions (column-major original order <-> row-major internal order).
#include "blas1.cuh"
#include "bulk.cuh"

#include <algorithm>
#include "dgemm.cuh"

namespace fsa {

namespace {

__global__ void k_pack(const double* __restrict__ in, long ld_in, long n, long k, const int* __restrict__ perm,
                       long n_pad, long tp, long col0, double* __restrict__ out) {
  const long idx = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= n_pad * k) return;
  const long i = idx / k, j = idx % k;
  FSA_DCHECK(i >= n || (perm[i] >= 0 && perm[i] < ld_in), "pack: permutation index out of range");
  out[i * tp + col0 + j] = i < n ? in[static_cast<long>(perm[i]) + j * ld_in] : 0.0;
}

__global__ void k_copy_cols(const double* __restrict__ src, long lds, double* __restrict__ dst, long ldd, long n,
                            long k) {
  const long idx = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= n * k) return;
  const long i = idx / k, j = idx % k;
  dst[i * ldd + j] = src[i * lds + j];
}

// sum_i log x_i in two fixed-order passes (block partials over fixed row ranges, then their sum):
// deterministic, and the logs spread over every SM instead of one block (was 231 us at n = 1e5)
constexpr int kSumLogBlocks = 2 * kNumSMs;
__global__ void k_sum_log(const double* __restrict__ x, long n, double* __restrict__ part) {
  __shared__ double red[256];
  double s = 0.0;
  for (long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += static_cast<long>(gridDim.x) * blockDim.x)
    s += log(x[i]);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}
__global__ void k_sum_parts(const double* __restrict__ part, int nb, double* out) {
  __shared__ double red[256];
  double v = 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) v += part[i];
  red[threadIdx.x] = v;
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
  FSA_DCHECK(perm[i] >= 0 && perm[i] < n, "unpack: permutation index out of range");
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
__global__ void k_cg_check(const double* __restrict__ rr, long k, double tol, int it, int max_iter, CgState st) {
  const long j = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= k) return;
  if (!st.active[j]) return;
  const double rn = sqrt(rr[j]);
  st.rnorm[j * max_iter + it] = rn;
  if (rn < tol) {
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

// H = Z + beta H and Vlr = Lw + beta Vlr for active columns (two columns per thread)
__global__ void k_update_h2(double* __restrict__ H, const double* __restrict__ Z, double* __restrict__ Vlr,
                            const double* __restrict__ Lw, const int* __restrict__ active,
                            const double* __restrict__ beta, long n, long tp, long k) {
  const long idx = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;  // pair index
  if (idx >= n * tp / 2) return;
  const long j = (2 * idx) % tp;
  const bool a0 = j < k && active[j], a1 = j + 1 < k && active[j + 1];
  if (!a0 && !a1) return;
  const double b0 = a0 ? beta[j] : 0.0, b1 = a1 ? beta[j + 1] : 0.0;
  double2 h = reinterpret_cast<double2*>(H)[idx];
  double2 v = reinterpret_cast<double2*>(Vlr)[idx];
  const double2 z = reinterpret_cast<const double2*>(Z)[idx];
  const double2 l = reinterpret_cast<const double2*>(Lw)[idx];
  if (a0) {
    h.x = z.x + b0 * h.x;
    v.x = l.x + b0 * v.x;
  }
  if (a1) {
    h.y = z.y + b1 * h.y;
    v.y = l.y + b1 * v.y;
  }
  reinterpret_cast<double2*>(H)[idx] = h;
  reinterpret_cast<double2*>(Vlr)[idx] = v;
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

// Warp-per-row column dots (fixed grid -> fixed reduction order). Columns
// [c0, c0 + 64*NCH) of row-major blocks; optional row weight w.
// Mode 0: plain dot A.B.  Mode 1: X += alpha H, R -= alpha V (active columns), dot R.R.
template <int NCH, int MODE>
__global__ void __launch_bounds__(256) k_rowdot_cols(const double* __restrict__ A, const double* __restrict__ B,
                                                    const double* __restrict__ w, long n, long ld, long t, long c0,
                                                    double* __restrict__ X, double* __restrict__ R,
                                                    const double* __restrict__ alpha, double* __restrict__ partial,
                                                    long ldp) {
  __shared__ double red[8][64 * NCH];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double d0[NCH], d1[NCH], al0[NCH], al1[NCH];
#pragma unroll
  for (int q = 0; q < NCH; ++q) {
    d0[q] = d1[q] = 0.0;
    if (MODE == 1) {
      const long c = c0 + q * 64 + 2 * lane;
      al0[q] = c < t ? alpha[c] : 0.0;
      al1[q] = c + 1 < t ? alpha[c + 1] : 0.0;
    }
  }
  for (long r = static_cast<long>(blockIdx.x) * 8 + warp; r < n; r += 8L * gridDim.x) {
    const double wr = w != nullptr ? w[r] : 1.0;
#pragma unroll
    for (int q = 0; q < NCH; ++q) {
      const long c = c0 + q * 64 + 2 * lane;
      if (c >= t) break;
      if (MODE == 0) {
        const double2 a = *reinterpret_cast<const double2*>(A + r * ld + c);
        const double2 b = *reinterpret_cast<const double2*>(B + r * ld + c);
        d0[q] = fma(a.x * b.x, wr, d0[q]);
        d1[q] = fma(a.y * b.y, wr, d1[q]);
      } else {
        // A = H, B = V
        double2 x = *reinterpret_cast<const double2*>(X + r * ld + c);
        double2 rr = *reinterpret_cast<const double2*>(R + r * ld + c);
        if (al0[q] != 0.0 || al1[q] != 0.0) {
          const double2 h = *reinterpret_cast<const double2*>(A + r * ld + c);
          const double2 v = *reinterpret_cast<const double2*>(B + r * ld + c);
          x.x += al0[q] * h.x;
          x.y += al1[q] * h.y;
          rr.x -= al0[q] * v.x;
          rr.y -= al1[q] * v.y;
          *reinterpret_cast<double2*>(X + r * ld + c) = x;
          *reinterpret_cast<double2*>(R + r * ld + c) = rr;
        }
        d0[q] = fma(rr.x, rr.x, d0[q]);
        d1[q] = fma(rr.y, rr.y, d1[q]);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < NCH; ++q) {
    red[warp][q * 64 + 2 * lane] = d0[q];
    red[warp][q * 64 + 2 * lane + 1] = d1[q];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < 64 * NCH; c += blockDim.x) {
    if (c0 + c >= t) break;
    double sacc = 0.0;
#pragma unroll
    for (int ww = 0; ww < 8; ++ww) sacc += red[ww][c];
    partial[static_cast<long>(blockIdx.x) * ldp + c0 + c] = sacc;
  }
}

[[maybe_unused]] __global__ void k_colsum(const double* __restrict__ partial, long nb, long ldp,
                                         double* __restrict__ out) {
  const long c = blockIdx.x;
  const int lane = threadIdx.x;
  double sacc = 0.0;
  for (long b = lane; b < nb; b += 32) sacc += partial[b * ldp + c];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
  if (lane == 0) out[c] = sacc;
}

long rowdot_blocks(long n) {
  const long b = cdiv(n, 8);
  return b < 4 * kNumSMs ? (b < 1 ? 1 : b) : 4 * kNumSMs;
}

template <int MODE>
void rowdot_launch(const double* A, const double* B, const double* w, long n, long ld, long t, double* X, double* R,
                   const double* alpha, double* out, double* partial, cudaStream_t s) {
  if (t == 0) return;
  const long nb = rowdot_blocks(n);
  const unsigned g = static_cast<unsigned>(nb);
  for (long c0 = 0; c0 < t; c0 += 256) {
    const long rem = t - c0;
    if (rem <= 64)
      k_rowdot_cols<1, MODE><<<g, 256, 0, s>>>(A, B, w, n, ld, t, c0, X, R, alpha, partial, t);
    else if (rem <= 128)
      k_rowdot_cols<2, MODE><<<g, 256, 0, s>>>(A, B, w, n, ld, t, c0, X, R, alpha, partial, t);
    else
      k_rowdot_cols<4, MODE><<<g, 256, 0, s>>>(A, B, w, n, ld, t, c0, X, R, alpha, partial, t);
    FSA_LAUNCH_CHECK();
  }
  colsum_partials(partial, nb, t, t, out, s);
}

__global__ void k_update_uh(double* __restrict__ UH, const double* __restrict__ W, const int* __restrict__ active,
                            const double* __restrict__ beta, long len, long tp, long k, int init) {
  const long idx = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= len) return;
  const long j = idx % tp;
  if (init) {
    UH[idx] = (j < k && active[j]) ? W[idx] : 0.0;
  } else if (j < k && active[j]) {
    UH[idx] = W[idx] + beta[j] * UH[idx];
  }
}

}  // namespace

size_t coldot_scratch(long n, long t) { return static_cast<size_t>(rowdot_blocks(n)) * static_cast<size_t>(t); }

void launch_coldot(const double* A, const double* B, long n, long ld, long t, double* out, double* scratch,
                   cudaStream_t s) {
  rowdot_launch<0>(A, B, nullptr, n, ld, t, nullptr, nullptr, nullptr, out, scratch, s);
}

void launch_coldot_weighted(const double* A, const double* B, const double* w, long n, long ld, long t,
                            double* out, double* scratch, cudaStream_t s) {
  rowdot_launch<0>(A, B, w, n, ld, t, nullptr, nullptr, nullptr, out, scratch, s);
}

void update_xr_dot(double* X, double* R, const double* H, const double* V, const double* alpha, long n, long tp,
                   long k, double* rr, double* scratch, cudaStream_t s) {
  rowdot_launch<1>(H, V, nullptr, n, tp, k, X, R, alpha, rr, scratch, s);
}

// Jacobi-preconditioned PCG without a Z block: X += alpha H, R -= alpha V, rr = |R|^2 and
// rz = R' D^{-1} R per column in one pass (64-column slabs, fixed-order partials)
__global__ void __launch_bounds__(256) k_xr_dot_jacobi(double* __restrict__ X, double* __restrict__ R,
                                                       const double* __restrict__ H, const double* __restrict__ V,
                                                       const double* __restrict__ alpha,
                                                       const double* __restrict__ dinv, long n, long ld, long t,
                                                       double* __restrict__ prr, double* __restrict__ prz) {
  __shared__ double red[2][8][64];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long c0 = 64L * blockIdx.y;
  const long c = c0 + 2 * lane;
  const bool on = c < t;
  const double al0 = c < t ? alpha[c] : 0.0, al1 = c + 1 < t ? alpha[c + 1] : 0.0;
  double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;
  if (on) {
    for (long r = static_cast<long>(blockIdx.x) * 8 + warp; r < n; r += 8L * gridDim.x) {
      double2 rr = *reinterpret_cast<const double2*>(R + r * ld + c);
      if (al0 != 0.0 || al1 != 0.0) {
        double2 x = *reinterpret_cast<const double2*>(X + r * ld + c);
        const double2 h = *reinterpret_cast<const double2*>(H + r * ld + c);
        const double2 v = *reinterpret_cast<const double2*>(V + r * ld + c);
        x.x += al0 * h.x;
        x.y += al1 * h.y;
        rr.x -= al0 * v.x;
        rr.y -= al1 * v.y;
        *reinterpret_cast<double2*>(X + r * ld + c) = x;
        *reinterpret_cast<double2*>(R + r * ld + c) = rr;
      }
      const double w = dinv[r];
      d0 = fma(rr.x, rr.x, d0);
      d1 = fma(rr.y, rr.y, d1);
      e0 = fma(rr.x * w, rr.x, e0);
      e1 = fma(rr.y * w, rr.y, e1);
    }
  }
  red[0][warp][2 * lane] = d0;
  red[0][warp][2 * lane + 1] = d1;
  red[1][warp][2 * lane] = e0;
  red[1][warp][2 * lane + 1] = e1;
  __syncthreads();
  if (threadIdx.x < 128) {
    const int q = threadIdx.x >> 6, cc = threadIdx.x & 63;
    if (c0 + cc < t) {
      double sacc = 0.0;
#pragma unroll
      for (int w = 0; w < 8; ++w) sacc += red[q][w][cc];
      (q == 0 ? prr : prz)[static_cast<long>(blockIdx.x) * t + c0 + cc] = sacc;
    }
  }
}
void update_xr_dot_jacobi(double* X, double* R, const double* H, const double* V, const double* alpha,
                          const double* dinv, long n, long tp, long k, double* rr, double* rz, double* scratch,
                          cudaStream_t s) {
  const long nb = rowdot_blocks(n);
  const dim3 grid(static_cast<unsigned>(nb), static_cast<unsigned>(cdiv(k, 64)));
  k_xr_dot_jacobi<<<grid, 256, 0, s>>>(X, R, H, V, alpha, dinv, n, tp, k, scratch, scratch + nb * k);
  FSA_LAUNCH_CHECK();
  colsum_partials(scratch, nb, k, k, rr, s);
  colsum_partials(scratch + nb * k, nb, k, k, rz, s);
}
// H = D^{-1} R + beta H on the active columns (init: H = active ? D^{-1} R : 0)
__global__ void k_update_h_jacobi(double* __restrict__ H, const double* __restrict__ R,
                                  const double* __restrict__ dinv, const int* __restrict__ active,
                                  const double* __restrict__ beta, long n, long tp, long k, int init) {
  const long idx = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= n * tp) return;
  const long i = idx / tp, j = idx - i * tp;
  if (j >= k) return;
  if (!active[j]) {
    if (init) H[idx] = 0.0;
    return;
  }
  const double z = R[idx] * dinv[i];
  H[idx] = init ? z : z + beta[j] * H[idx];
}
void update_h_jacobi(double* H, const double* R, const double* dinv, const int* active, const double* beta, long n,
                     long tp, long k, bool init, cudaStream_t s) {
  k_update_h_jacobi<<<nblk(n * tp), 256, 0, s>>>(H, R, dinv, active, beta, n, tp, k, init ? 1 : 0);
  FSA_LAUNCH_CHECK();
}

// update_xr_dot for t <= 64 with contiguous row ranges per block, plus the column maxima
// of |dinv[i] R[i][c]| per chunk of chunk_rows rows (atomicMax on the bit patterns of the
// non-negative doubles: order independent), the exponents of the Ozaki projection
__global__ void __launch_bounds__(256, 3) k_xr_dot_max(double* __restrict__ X, double* __restrict__ R,
                                                    const double* __restrict__ H, const double* __restrict__ V,
                                                    const double* __restrict__ alpha, long n, long ld, long t,
                                                    double* __restrict__ partial, const double* __restrict__ dinv,
                                                    unsigned long long* __restrict__ ymax, long chunk_rows) {
  __shared__ double red[8][64];
  pdl_wait();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const long c = 2 * lane;
  const bool on = c < t;
  const double al0 = c < t ? alpha[c] : 0.0, al1 = c + 1 < t ? alpha[c + 1] : 0.0;
  const long per = (n + gridDim.x - 1) / gridDim.x;
  const long ra = static_cast<long>(blockIdx.x) * per, rb = min(n, ra + per);
  double d0 = 0.0, d1 = 0.0, m0 = 0.0, m1 = 0.0;
  long cur = -1;
  const uint64_t pol_last = l2_evict_last();
  auto flush = [&]() {
    if (cur >= 0 && on) {
      if (m0 > 0.0) atomicMax(ymax + cur * 64 + c, static_cast<unsigned long long>(__double_as_longlong(m0)));
      if (m1 > 0.0) atomicMax(ymax + cur * 64 + c + 1, static_cast<unsigned long long>(__double_as_longlong(m1)));
    }
    m0 = m1 = 0.0;
  };
  long next = 0;  // first row of the chunk after `cur`
  constexpr int kU = 2;  // rows per batch (loads of the batch are issued together)
  for (long rbase = ra + warp; rbase < rb; rbase += 8 * kU) {
    double2 x[kU], rr[kU], h[kU], v[kU];
    double di[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const long r = rbase + 8 * u;
      if (r < rb && on) {
        x[u] = *reinterpret_cast<const double2*>(X + r * ld + c);
        rr[u] = *reinterpret_cast<const double2*>(R + r * ld + c);
        h[u] = *reinterpret_cast<const double2*>(H + r * ld + c);
        v[u] = *reinterpret_cast<const double2*>(V + r * ld + c);
        di[u] = dinv[r];
      }
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const long r = rbase + 8 * u;
      if (r >= rb) break;
      if (r >= next) {  // entering a new chunk (rows only grow)
        flush();
        cur = r / chunk_rows;
        next = (cur + 1) * chunk_rows;
      }
      if (!on) continue;
      if (al0 != 0.0 || al1 != 0.0) {
        x[u].x += al0 * h[u].x;
        x[u].y += al1 * h[u].y;
        rr[u].x -= al0 * v[u].x;
        rr[u].y -= al1 * v[u].y;
        *reinterpret_cast<double2*>(X + r * ld + c) = x[u];
        st_l2(reinterpret_cast<double2*>(R + r * ld + c), rr[u], pol_last);  // read next by the slicing pass
      }
      d0 = fma(rr[u].x, rr[u].x, d0);
      d1 = fma(rr[u].y, rr[u].y, d1);
      m0 = fmax(m0, fabs(rr[u].x * di[u]));
      m1 = fmax(m1, fabs(rr[u].y * di[u]));
    }
  }
  flush();
  red[warp][2 * lane] = d0;
  red[warp][2 * lane + 1] = d1;
  __syncthreads();
  if (threadIdx.x < t && threadIdx.x < 64) {
    double sacc = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) sacc += red[w][threadIdx.x];
    partial[static_cast<long>(blockIdx.x) * t + threadIdx.x] = sacc;
  }
}
long xr_dot_max_blocks(long n) { return std::min(rowdot_blocks(n), 3L * kNumSMs); }  // one wave at 3 blocks/SM
void update_xr_dot_max(double* X, double* R, const double* H, const double* V, const double* alpha, long n, long tp,
                       long k, double* rr, double* scratch, const double* dinv, unsigned long long* ymax,
                       long chunk_rows, cudaStream_t s, bool colsum) {
  require(tp <= 64, "update_xr_dot_max: at most 64 columns");
  const long nb = xr_dot_max_blocks(n);
  launch_pdl(k_xr_dot_max, dim3(static_cast<unsigned>(nb)), dim3(256), 0, s, X, R, H, V, alpha, n, tp, k, scratch, dinv,
             ymax, chunk_rows);
  FSA_LAUNCH_CHECK();
  if (colsum) colsum_partials(scratch, nb, k, k, rr, s);
}

void update_uh(double* UH, const double* W, const int* active, const double* beta, long mpad, long tp, long k,
               bool init, cudaStream_t s) {
  k_update_uh<<<nblk(mpad * tp), 256, 0, s>>>(UH, W, active, beta, mpad * tp, tp, k, init ? 1 : 0);
  FSA_LAUNCH_CHECK();
}

void pack_cols(const double* in_dev, long n, long k, const int* perm_dev, long n_pad, long tp, long col0,
               double* out, cudaStream_t s) {
  if (k == 0) return;
  k_pack<<<nblk(n_pad * k), 256, 0, s>>>(in_dev, n, n, k, perm_dev, n_pad, tp, col0, out);
  FSA_LAUNCH_CHECK();
}
void pack_cols_ld(const double* in_dev, long ld_in, long n, long k, const int* perm_dev, long n_pad, long tp,
                  long col0, double* out, cudaStream_t s) {
  if (k == 0) return;
  k_pack<<<nblk(n_pad * k), 256, 0, s>>>(in_dev, ld_in, n, k, perm_dev, n_pad, tp, col0, out);
  FSA_LAUNCH_CHECK();
}
void copy_cols(const double* src, long lds, double* dst, long ldd, long n, long k, cudaStream_t s) {
  if (n * k == 0) return;
  k_copy_cols<<<nblk(n * k), 256, 0, s>>>(src, lds, dst, ldd, n, k);
  FSA_LAUNCH_CHECK();
}
void sum_log(const double* x, long n, double* out_dev, cudaStream_t s) {
  DBuf<double> part(kSumLogBlocks);
  k_sum_log<<<kSumLogBlocks, 256, 0, s>>>(x, n, part.get());
  FSA_LAUNCH_CHECK();
  k_sum_parts<<<1, 256, 0, s>>>(part.get(), kSumLogBlocks, out_dev);
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
void cg_check(const double* rr, long k, double tol, int it, int max_iter, const CgState& st, cudaStream_t s) {
  k_cg_check<<<nblk(k, 128), 128, 0, s>>>(rr, k, tol, it, max_iter, st);
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
// out[0..3] = sum_i p_i, p.d1, p.dD, f_i / D_i over i < n; out[4..6] = tr Qi, tr K2,
// <K2, Qi> over the m x m blocks. One 1024-thread block, fixed order.
__global__ void __launch_bounds__(1024) k_trace_sums(const double* __restrict__ p, const double* __restrict__ d1,
                                                     const double* __restrict__ dD, const double* __restrict__ f,
                                                     const double* __restrict__ D, long n,
                                                     const double* __restrict__ Qi, const double* __restrict__ K2,
                                                     long m, double* __restrict__ out) {
  __shared__ double red[7][32];
  double a[7] = {0, 0, 0, 0, 0, 0, 0};
  for (long i = threadIdx.x; i < n; i += blockDim.x) {
    a[0] += p[i];
    a[1] += p[i] * d1[i];
    a[2] += p[i] * dD[i];
    a[3] += f[i] / D[i];
  }
  for (long i = threadIdx.x; i < m; i += blockDim.x) {
    a[4] += Qi[i * m + i];
    a[5] += K2[i * m + i];
  }
  for (long i = threadIdx.x; i < m * m; i += blockDim.x) a[6] += K2[i] * Qi[i];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < 7; ++q) {
    double v = a[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[q][warp] = v;
  }
  __syncthreads();
  if (threadIdx.x < 7) {
    double v = 0.0;
    for (int w = 0; w < 32; ++w) v += red[threadIdx.x][w];
    out[threadIdx.x] = v;
  }
}
void trace_sums(const double* p, const double* d1, const double* dD, const double* f, const double* D, long n,
                const double* Qi, const double* K2, long m, double* out, cudaStream_t s) {
  k_trace_sums<<<1, 1024, 0, s>>>(p, d1, dD, f, D, n, Qi, K2, m, out);
  FSA_LAUNCH_CHECK();
}

__global__ void k_row_dots(const double* __restrict__ A, const double* __restrict__ B, long ld, long len, long n,
                           long n_pad, double* __restrict__ out) {
  const long i = (static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= n_pad) return;
  double sacc = 0.0;
  if (i < n)
    for (long r = lane; r < len; r += 32) sacc = fma(A[i * ld + r], B[i * ld + r], sacc);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
  if (lane == 0) out[i] = sacc;
}
void row_dots(const double* A, const double* B, long ld, long len, long n, long n_pad, double* out, cudaStream_t s) {
  k_row_dots<<<nblk(n_pad * 32), 256, 0, s>>>(A, B, ld, len, n, n_pad, out);
  FSA_LAUNCH_CHECK();
}

// cross Gram of two narrow column groups: partial[b][a*q + c] over block b's rows, then a
// fixed-order sum over the blocks (deterministic, independent of timing)
constexpr int kGramBlocks = kNumSMs;
__global__ void __launch_bounds__(256) k_cross_gram(const double* __restrict__ A, long lda,
                                                    const double* __restrict__ B, long ldb, long n, int q,
                                                    double* __restrict__ partial) {
  __shared__ double red[8];
  const long per = (n + gridDim.x - 1) / gridDim.x;
  const long i0 = blockIdx.x * per, i1 = min(n, i0 + per);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int pr = 0; pr < q * q; ++pr) {
    const int a = pr / q, c = pr % q;
    double v = 0.0;
    for (long i = i0 + threadIdx.x; i < i1; i += blockDim.x) v = fma(A[i * lda + a], B[i * ldb + c], v);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < 8; ++w) t += red[w];
      partial[static_cast<long>(blockIdx.x) * q * q + pr] = t;
    }
    __syncthreads();
  }
}
__global__ void k_cross_gram_sum(const double* __restrict__ partial, int nb, int qq, double* __restrict__ out) {
  const int pr = blockIdx.x * blockDim.x + threadIdx.x;
  if (pr >= qq) return;
  double t = 0.0;
  for (int b = 0; b < nb; ++b) t += partial[static_cast<long>(b) * qq + pr];
  out[pr] = t;
}
size_t cross_gram_scratch(long q) { return static_cast<size_t>(kGramBlocks) * static_cast<size_t>(q * q); }
void cross_gram(const double* A, long lda, const double* B, long ldb, long n, long q, double* out, double* scratch,
                cudaStream_t s) {
  if (q == 0) return;
  k_cross_gram<<<kGramBlocks, 256, 0, s>>>(A, lda, B, ldb, n, static_cast<int>(q), scratch);
  FSA_LAUNCH_CHECK();
  k_cross_gram_sum<<<nblk(q * q, 128), 128, 0, s>>>(scratch, kGramBlocks, static_cast<int>(q * q), out);
  FSA_LAUNCH_CHECK();
}

// out[i * ldo] = X[i * ldx] - sum_a X[i * ldx + 1 + a] coef[a] for i < n (0 on padding rows < n_pad)
__global__ void k_gls_residual(const double* __restrict__ X, long ldx, long p, const double* __restrict__ coef,
                               long n, long n_pad, double* __restrict__ out, long ldo) {
  const long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n_pad) return;
  double v = 0.0;
  if (i < n) {
    v = X[i * ldx];
    for (long a = 0; a < p; ++a) v -= X[i * ldx + 1 + a] * coef[a];
  }
  out[i * ldo] = v;
}
void gls_residual(const double* X, long ldx, long p, const double* coef_dev, long n, long n_pad, double* out, long ldo,
                  cudaStream_t s) {
  k_gls_residual<<<nblk(n_pad), 256, 0, s>>>(X, ldx, p, coef_dev, n, n_pad, out, ldo);
  FSA_LAUNCH_CHECK();
}

void update_h2(double* H, const double* Z, double* Vlr, const double* Lw, const int* active, const double* beta,
               long n, long tp, long k, cudaStream_t s) {
  k_update_h2<<<nblk(n * tp / 2), 256, 0, s>>>(H, Z, Vlr, Lw, active, beta, n, tp, k);
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


// ---- column sums fused with the per-column PCG control (single rank) ---------------------
// out[c] = sum_b partial[b][c] exactly as k_colsum_partials (same strided assignment and tree),
// then thread 0 of column c < k runs that column's control step: MODE 0 alpha (k_cg_alpha),
// MODE 1 the residual test (k_cg_check), MODE 2 beta (k_cg_beta) followed, in the last block to
// finish, by the active count for the host (k_cg_count; `ticket` is reset for the next call).
// MODE 3 = MODE 1 on `partial` followed by MODE 2 on `partial_b` (the residual test deferred to
// the end of the sweep: one launch fewer; nothing between them reads the convergence flags)
__device__ __forceinline__ double block_colsum(const double* __restrict__ partial, long nb, long ldp, long c,
                                               double (&red)[8]) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double sacc = strided_colsum(partial, nb, ldp, c);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
  if (lane == 0) red[warp] = sacc;
  __syncthreads();
  double t = 0.0;
  if (tid == 0)
    for (int w = 0; w < 8; ++w) t += red[w];
  __syncthreads();  // (red reused)
  return t;
}
// both sums of MODE 3 in one pass: the loads of the two partial columns are issued together
// (each sum in k_colsum_partials' order), then one shuffle tree and one barrier for both
__device__ __forceinline__ void block_colsum2(const double* __restrict__ pa, long na, long lda,
                                              const double* __restrict__ pb, long nb, long ldb, long c,
                                              double (&red)[2][8], double& ta, double& tb) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double sa = 0.0, sb = 0.0;
  if (na <= 2 * 256 && nb <= 4 * 256) {  // (the sweep's sizes: everything in flight at once)
    double va[2], vb[4];
#pragma unroll
    for (int i = 0; i < 2; ++i) va[i] = tid + 256 * i < na ? pa[(tid + 256 * i) * lda + c] : 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i) vb[i] = tid + 256 * i < nb ? pb[(tid + 256 * i) * ldb + c] : 0.0;
    // the order of strided_colsum: s0 / s1 over pairs of 256-strides, then s0 + s1
    sa = va[0] + va[1];
    sb = (vb[0] + vb[2]) + (vb[1] + vb[3]);
  } else {
    sa = strided_colsum(pa, na, lda, c);
    sb = strided_colsum(pb, nb, ldb, c);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sa += __shfl_xor_sync(0xffffffffu, sa, o);
    sb += __shfl_xor_sync(0xffffffffu, sb, o);
  }
  if (lane == 0) {
    red[0][warp] = sa;
    red[1][warp] = sb;
  }
  __syncthreads();
  ta = tb = 0.0;
  if (tid == 0)
    for (int w = 0; w < 8; ++w) {
      ta += red[0][w];
      tb += red[1][w];
    }
}
template <int MODE>
__global__ void __launch_bounds__(256) k_colsum_ctl(const double* __restrict__ partial, long nb, long ldp,
                                                    double* __restrict__ out, long k, int it, int max_iter,
                                                    double tol, CgState st, unsigned int* ticket,
                                                    unsigned long long* __restrict__ zero_buf, long zero_len,
                                                    const double* __restrict__ partial_b, long nb_b, long ldp_b,
                                                    double* __restrict__ out_b) {
  __shared__ double red[2][8];
  __shared__ bool last;
  pdl_wait();
  const long c = blockIdx.x;
  const long j = c;
  const int tid = threadIdx.x;
  // thread 0's control state, loaded while the partials are summed (independent loads in flight)
  int itv = it, act = 0;
  double rzj = 0.0, bpj = 0.0, apj = 1.0, aj = 0.0;
  if (tid == 0) {
    if (st.it_dev != nullptr) itv = *st.it_dev;
    if (j < k) {
      act = st.active[j];
      rzj = st.rz[j];
      if (MODE == 0) {
        bpj = st.beta_prev[j];
        apj = st.alpha_prev[j];
      }
      if (MODE >= 2) aj = st.alpha[j];
    }
  }
  // clear the next kernel's column-maxima accumulators on the way
  for (long i = c * blockDim.x + tid; i < zero_len; i += static_cast<long>(gridDim.x) * blockDim.x) zero_buf[i] = 0ull;
  double t0, tb = 0.0;
  if (MODE == 3) {
    block_colsum2(partial, nb, ldp, partial_b, nb_b, ldp_b, c, red, t0, tb);
  } else {
    double dummy;
    block_colsum2(partial, nb, ldp, partial, 0, ldp, c, red, t0, dummy);
  }
  if (tid == 0) {
    double t = t0;
    out[c] = t;
    it = itv;
    if (MODE == 3 && j < k && act) {  // residual test first (krylov.cpp:77-82)
      const double rn = sqrt(t);
      st.rnorm[j * max_iter + it] = rn;
      if (rn < tol) {
        st.converged[j] = 1;
        st.active[j] = 0;
        act = 0;
      }
    }
    if (MODE == 3) {
      t = tb;
      out_b[c] = t;
    }
    if (j < k) {
      if (MODE == 0) {  // alpha = rz / h'v, tridiagonal push (krylov.cpp:66-75)
        if (!act) {
          st.alpha[j] = 0.0;
        } else if (!(t > 0.0)) {
          atomicCAS(st.err, 0, kErrOperatorNotPD);
          st.alpha[j] = 0.0;
        } else {
          const double a = rzj / t;
          st.alpha[j] = a;
          st.tdiag[j * max_iter + it] = 1.0 / a + bpj / apj;
          if (it > 0) st.toff[j * max_iter + it - 1] = sqrt(bpj) / apj;
          st.iterations[j] = it + 1;
        }
      } else if (MODE == 1) {  // residual test (krylov.cpp:77-82)
        if (act) {
          const double rn = sqrt(t);
          st.rnorm[j * max_iter + it] = rn;
          if (rn < tol) {
            st.converged[j] = 1;
            st.active[j] = 0;
          }
        }
      } else {  // MODE 2 / 3: beta = rz_new / rz (krylov.cpp:83-90)
        if (!act) {
          st.beta[j] = 0.0;
        } else if (!(t > 0.0)) {
          atomicCAS(st.err, 0, kErrPrecondNotPD);
          st.beta[j] = 0.0;
        } else {
          const double bb = t / rzj;
          st.beta[j] = bb;
          st.beta_prev[j] = bb;
          st.alpha_prev[j] = aj;
          st.rz[j] = t;
        }
      }
    }
    if (MODE >= 2) {
      __threadfence();
      last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
  }
  if (MODE >= 2) {
    __syncthreads();
    if (last) {  // block-uniform: the whole last block counts the active columns
      __threadfence();
      int cnt = 0;
      for (long base = 0; base < k; base += blockDim.x) {
        const long jj = base + tid;
        cnt += __syncthreads_count(jj < k && reinterpret_cast<volatile int*>(st.active)[jj] != 0);
      }
      if (tid == 0) {
        int* hf = st.host_flags;
        if (st.it_dev != nullptr) {  // graph-captured sweep: slot by the device sweep index, then advance it
          hf += 2 * (itv & 1);
          *st.it_dev = itv + 1;
        }
        hf[0] = cnt;
        hf[1] = *reinterpret_cast<volatile int*>(st.err);
        *ticket = 0u;
      }
    }
  }
}
void colsum_ctl(int mode, const double* partial, long nb, long ldp, long t, double* out, long k, int it,
                int max_iter, double tol, const CgState& st, unsigned int* ticket, cudaStream_t s,
                unsigned long long* zero_buf, long zero_len, const double* partial_b, long nb_b, long ldp_b,
                double* out_b) {
  require(t >= k && t > 0, "colsum_ctl: fewer sums than columns");
  require(mode != 3 || (partial_b != nullptr && out_b != nullptr), "colsum_ctl: mode 3 needs the second sums");
  const unsigned g = static_cast<unsigned>(t);
  auto go = [&](auto kern) {
    launch_pdl(kern, dim3(g), dim3(256), 0, s, partial, nb, ldp, out, k, it, max_iter, tol, st, ticket, zero_buf,
               zero_len, partial_b, nb_b, ldp_b, out_b);
  };
  switch (mode) {
    case 0: go(k_colsum_ctl<0>); break;
    case 1: go(k_colsum_ctl<1>); break;
    case 2: go(k_colsum_ctl<2>); break;
    default: go(k_colsum_ctl<3>); break;
  }
  FSA_LAUNCH_CHECK();
}

}  // namespace fsa
