// Sparse kernels of the FSA operator:
//  * SDDMM assembly of the tapered residual block straight into CSR
//    (reference fsa.cpp:38-56): value = (C(d) - U_r . U_c) T(d), diagonal
//    max(sigma1_2 - |U_r|^2, 0) + sigma2 with the clamp counted;
//  * its rho derivative on the same pattern (fsa.cpp:101-124, U-form);
//  * the cross block to prediction points (prediction.cpp:16-24);
//  * CSR x dense SpMM on row-major RHS blocks.
// One warp per CSR row; the row's m-vector lives in registers (m/32 per lane).
#include "dgemm.cuh"
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
// The pattern and the values are symmetric (the warp dot is bitwise symmetric in
// its operands), so each unordered pair is evaluated once: the entry (r, c), c > r,
// also writes its transposed position mirror[p].
template <int MQ>
__global__ void k_sddmm_sigma_s(const double* __restrict__ U, long ldu, const long* __restrict__ rowptr,
                                const int* __restrict__ col, const long* __restrict__ mirror,
                                const double* __restrict__ dist, const double* __restrict__ lowrank_diag, long n,
                                SddmmParams P, double* __restrict__ val, int* __restrict__ n_clamped) {
  const long r = (static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= n) return;
  double ur[MQ];
  load_vec<MQ>(U + r * ldu, lane, ur);
  const long pe = rowptr[r + 1];
  long p = rowptr[r];
  while (p < pe && col[p] < r) ++p;  // columns ascend: skip the lower triangle
  for (; p < pe; ++p) {
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
      const double v = (matern_d(d, P.nu, P.sigma1_2, P.rho) - dt) * taper_d(d, P.family, P.gamma);
      val[p] = v;
      if (mirror[p] >= 0) val[mirror[p]] = v;  // halo columns: the mirror lives on another rank
    }
  }
}

// d Sigma_s / d rho (U-form of fsa.cpp:107-122): dl = U1_r.U_c + U_r.T_c with
// U1 = L^{-1} dSigma_mn/drho, T = U1 - K2 U, K2 = L^{-1} dSigma_m/drho L^{-T}
// (dl is symmetric in (r, c) because K2 is: evaluated once per unordered pair)
template <int MQ>
__global__ void k_sddmm_drho(const double* __restrict__ U, const double* __restrict__ U1,
                             const double* __restrict__ T, long ldu, const long* __restrict__ rowptr,
                             const int* __restrict__ col, const long* __restrict__ mirror,
                             const double* __restrict__ dist, const double* __restrict__ lowrank_diag, long n,
                             SddmmParams P, double* __restrict__ val) {
  const long r = (static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= n) return;
  double ur[MQ], u1r[MQ];
  load_vec<MQ>(U + r * ldu, lane, ur);
  load_vec<MQ>(U1 + r * ldu, lane, u1r);
  const long pe = rowptr[r + 1];
  long p = rowptr[r];
  while (p < pe && col[p] < r) ++p;
  for (; p < pe; ++p) {
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
        const double v = (matern_drho_d(d, P.nu, P.sigma1_2, P.rho) - dl) * taper_d(d, P.family, P.gamma);
        val[p] = v;
        if (mirror[p] >= 0) val[mirror[p]] = v;  // halo columns: the mirror lives on another rank
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

// Fused SpMM + per-column dot: Y = alpha S X + beta Y and dot[c] = sum_r X[r][c] Y[r][c]
// (the PCG's h.v, krylov.cpp:66). Fixed grid: warp w of block b owns rows
// b*8+w, +8*gridDim.x, ...; each lane owns columns 2*lane(+1) of every 64-column chunk,
// so the per-column partials reduce in a fixed order (bitwise reproducible).
constexpr bool kGatherL2 = false;  // RHS gathers through L2 only (the L1 data path bounds them otherwise)
template <int NCH>
__global__ void __launch_bounds__(256) k_spmm_dot(const long* __restrict__ rowptr, const int* __restrict__ col,
                                                 const double* __restrict__ val, long nrows,
                                                 const double* __restrict__ X, long ldx, double* Y,
                                                 long ldy, long ncols, double alpha, double beta,
                                                 double* __restrict__ partial, const double* Y0) {
  __shared__ double red[8][64 * NCH];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double d0[NCH], d1[NCH];
#pragma unroll
  for (int q = 0; q < NCH; ++q) d0[q] = d1[q] = 0.0;
  for (long r = static_cast<long>(blockIdx.x) * 8 + warp; r < nrows; r += 8L * gridDim.x) {
    const long pb = rowptr[r], pe = rowptr[r + 1];
#pragma unroll
    for (int q = 0; q < NCH; ++q) {
      if (q * 64 >= ncols) break;  // warp-uniform
      const long c = q * 64 + 2 * lane;
      const bool on = c < ncols;
      if (!on) continue;
      double a0 = 0.0, a1 = 0.0;
      for (long p = pb; p < pe; ++p) {
        const double v = val[p];
        const double2 x = kGatherL2 ? __ldcg(reinterpret_cast<const double2*>(X + static_cast<long>(col[p]) * ldx + c))
                                    : *reinterpret_cast<const double2*>(X + static_cast<long>(col[p]) * ldx + c);
        a0 = fma(v, x.x, a0);
        a1 = fma(v, x.y, a1);
      }
      double2* y = reinterpret_cast<double2*>(Y + r * ldy + c);
      double2 o;
      if (beta == 0.0) {
        o = make_double2(alpha * a0, alpha * a1);
      } else {
        o = *reinterpret_cast<const double2*>(Y0 + r * ldy + c);
        o.x = alpha * a0 + beta * o.x;
        o.y = alpha * a1 + beta * o.y;
      }
      *y = o;
      const double2 h = *reinterpret_cast<const double2*>(X + r * ldx + c);
      d0[q] = fma(h.x, o.x, d0[q]);
      d1[q] = fma(h.y, o.y, d1[q]);
    }
  }
#pragma unroll
  for (int q = 0; q < NCH; ++q) {
    red[warp][q * 64 + 2 * lane] = d0[q];
    red[warp][q * 64 + 2 * lane + 1] = d1[q];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < 64 * NCH && c < ncols; c += blockDim.x) {
    double sacc = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) sacc += red[w][c];
    partial[static_cast<long>(blockIdx.x) * ncols + c] = sacc;
  }
}

// Grouped SpMM + dot (Csr row groups, build_groups). Each union column of a group of
// kGroup consecutive rows is gathered ONCE and multiplied into the kGroup row accumulators
// by the group's value block (zero where a row lacks the column): the L1/L2 gather traffic,
// which bounds the SpMM, drops by the group's nonzeros / union size (~4x at 80 nnz/row in
// Hilbert order). kSplit warps share a group (interleaved union entries) so that the
// dependent gather chains stay short; their partial sums are combined in shared memory in
// a fixed order. Lanes own column pairs (double2); 64-column chunks.
constexpr int kSplit = 4;
constexpr int kGroupsPerBlock = 8 / kSplit;
template <int NCH>
__global__ void __launch_bounds__(256, 3) k_spmm_group(const long* __restrict__ gptr, const int* __restrict__ gcol,
                                                   const double* __restrict__ gval, long nrows, long ngrp,
                                                   const double* __restrict__ X, long ldx, double* Y, long ldy,
                                                   long ncols, double alpha, double beta,
                                                   double* __restrict__ partial, const double* Y0) {
  __shared__ double2 acc_s[8][kGroup][32];  // [warp][row][lane]; reused for the column dots
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gl = warp / kSplit, part = warp % kSplit;
  const long g = static_cast<long>(blockIdx.x) * kGroupsPerBlock + gl;
  const bool live = g < ngrp;
  const long u0 = live ? gptr[g] : 0, u1 = live ? gptr[g + 1] : 0;
  const long r0 = g * kGroup;
  double dsum[NCH][2];
#pragma unroll
  for (int q = 0; q < NCH; ++q) dsum[q][0] = dsum[q][1] = 0.0;
#pragma unroll
  for (int q = 0; q < NCH; ++q) {
    if (q * 64 >= ncols) break;  // block-uniform
    const long c = q * 64 + 2 * lane;
    const bool on = c < ncols;
    double a0[kGroup], a1[kGroup];
#pragma unroll
    for (int r = 0; r < kGroup; ++r) a0[r] = a1[r] = 0.0;
    // this warp's union entries u0 + part + kSplit k: column indices fetched 32 at a time
    // (one per lane) and broadcast by shuffle, so the gathers of a batch are independent
    for (long ub = u0 + part; ub < u1; ub += 32L * kSplit) {
      const long ul = ub + static_cast<long>(lane) * kSplit;
      const int jl = ul < u1 ? gcol[ul] : 0;
      const int cnt = static_cast<int>(min(32L, (u1 - ub + kSplit - 1) / kSplit));
#pragma unroll 4
      for (int k = 0; k < cnt; ++k) {
        const long j = __shfl_sync(0xffffffffu, jl, k);
        const long u = ub + static_cast<long>(k) * kSplit;
        const double4* vp = reinterpret_cast<const double4*>(gval + u * kGroup);
        double2 x = make_double2(0.0, 0.0);
        if (on) x = *reinterpret_cast<const double2*>(X + j * ldx + c);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const double4 va = vp[h];
          a0[4 * h + 0] = fma(va.x, x.x, a0[4 * h + 0]);
          a1[4 * h + 0] = fma(va.x, x.y, a1[4 * h + 0]);
          a0[4 * h + 1] = fma(va.y, x.x, a0[4 * h + 1]);
          a1[4 * h + 1] = fma(va.y, x.y, a1[4 * h + 1]);
          a0[4 * h + 2] = fma(va.z, x.x, a0[4 * h + 2]);
          a1[4 * h + 2] = fma(va.z, x.y, a1[4 * h + 2]);
          a0[4 * h + 3] = fma(va.w, x.x, a0[4 * h + 3]);
          a1[4 * h + 3] = fma(va.w, x.y, a1[4 * h + 3]);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < kGroup; ++r) acc_s[warp][r][lane] = make_double2(a0[r], a1[r]);
    __syncthreads();
    // warp `part` of the group finishes rows part, part + kSplit, ... (fixed-order sum of the splits)
    if (live && on) {
#pragma unroll
      for (int r = part; r < kGroup; r += kSplit) {
        const long row = r0 + r;
        if (row >= nrows) break;
        double s0 = 0.0, s1 = 0.0;
#pragma unroll
        for (int w = 0; w < kSplit; ++w) {
          const double2 t = acc_s[gl * kSplit + w][r][lane];
          s0 += t.x;
          s1 += t.y;
        }
        double2 o;
        if (beta == 0.0) {
          o = make_double2(alpha * s0, alpha * s1);
        } else {
          o = *reinterpret_cast<const double2*>(Y0 + row * ldy + c);
          o.x = alpha * s0 + beta * o.x;
          o.y = alpha * s1 + beta * o.y;
        }
        *reinterpret_cast<double2*>(Y + row * ldy + c) = o;
        const double2 h = *reinterpret_cast<const double2*>(X + row * ldx + c);
        dsum[q][0] = fma(h.x, o.x, dsum[q][0]);
        dsum[q][1] = fma(h.y, o.y, dsum[q][1]);
      }
    }
    __syncthreads();
  }
  // column dots: fixed order over the block's warps (rows of every warp are disjoint)
  double(*dred)[64 * NCH] = reinterpret_cast<double(*)[64 * NCH]>(&acc_s[0][0][0]);
#pragma unroll
  for (int q = 0; q < NCH; ++q) {
    dred[warp][q * 64 + 2 * lane] = dsum[q][0];
    dred[warp][q * 64 + 2 * lane + 1] = dsum[q][1];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < 64 * NCH && c < ncols; c += blockDim.x) {
    double sacc = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) sacc += dred[w][c];
    partial[static_cast<long>(blockIdx.x) * ncols + c] = sacc;
  }
}
// gval[slot * kGroup + row % kGroup] = val[p] (gval zeroed first)
__global__ void k_group_scatter(const long* __restrict__ rowptr, const int* __restrict__ gslot, long nrows,
                                const double* __restrict__ val, double* __restrict__ gval) {
  const long r = (static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= nrows) return;
  const int rg = static_cast<int>(r % kGroup);
  for (long p = rowptr[r] + lane; p < rowptr[r + 1]; p += 32) gval[static_cast<long>(gslot[p]) * kGroup + rg] = val[p];
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
  FSA_DISPATCH_MQ(k_sddmm_sigma_s, ldu, grid, s, U, ldu, pat.rowptr.get(), pat.col.get(), pat.mirror.get(),
                  pat.dist.get(), lowrank_diag, pat.rows, P, val, n_clamped_dev);
}

void sddmm_drho(const double* U, const double* U1, const double* T, long ldu, const Csr& pat,
                const double* lowrank_diag, const SddmmParams& P, double* val, cudaStream_t s) {
  const unsigned grid = static_cast<unsigned>(cdiv(pat.rows * 32, 256));
  if (grid == 0) return;
  FSA_DISPATCH_MQ(k_sddmm_drho, ldu, grid, s, U, U1, T, ldu, pat.rowptr.get(), pat.col.get(), pat.mirror.get(),
                  pat.dist.get(), lowrank_diag, pat.rows, P, val);
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

void group_values(const Csr& pat, const double* val, double* gval, cudaStream_t s) {
  if (pat.gnnz == 0) return;
  FSA_CUDA(cudaMemsetAsync(gval, 0, sizeof(double) * pat.gnnz * kGroup, s));
  k_group_scatter<<<static_cast<unsigned>(cdiv(pat.rows * 32, 256)), 256, 0, s>>>(pat.rowptr.get(), pat.gslot.get(),
                                                                                 pat.rows, val, gval);
  FSA_LAUNCH_CHECK();
}

long spmm_group_blocks(long ngrp) { return ngrp < 1 ? 1 : cdiv(ngrp, kGroupsPerBlock); }

void spmm_group_dot(const Csr& pat, const double* gval, const double* X, long ldx, double* Y, long ldy, long ncols,
                    double alpha, double beta, double* dot, double* partial, cudaStream_t s, const double* Y0) {
  if (pat.rows == 0) return;
  const long nb = spmm_group_blocks(pat.ngrp);
  const unsigned g = static_cast<unsigned>(nb);
  const double* y0 = Y0 != nullptr ? Y0 : Y;
  for (long c0 = 0; c0 < ncols; c0 += 256) {
    const long w = ncols - c0 < 256 ? ncols - c0 : 256;
    const int nch = static_cast<int>(cdiv(w, 64));
    double* part = partial + c0 * nb;
    switch (nch) {
      case 1: k_spmm_group<1><<<g, 256, 0, s>>>(pat.gptr.get(), pat.gcol.get(), gval, pat.rows, pat.ngrp, X + c0, ldx, Y + c0, ldy, w, alpha, beta, part, y0 + c0); break;
      case 2: k_spmm_group<2><<<g, 256, 0, s>>>(pat.gptr.get(), pat.gcol.get(), gval, pat.rows, pat.ngrp, X + c0, ldx, Y + c0, ldy, w, alpha, beta, part, y0 + c0); break;
      default: k_spmm_group<4><<<g, 256, 0, s>>>(pat.gptr.get(), pat.gcol.get(), gval, pat.rows, pat.ngrp, X + c0, ldx, Y + c0, ldy, w, alpha, beta, part, y0 + c0); break;
    }
    FSA_LAUNCH_CHECK();
    colsum_partials(part, nb, w, w, dot + c0, s);
  }
}

long spmm_dot_blocks(long nrows) {  // one row per warp (the L1-friendly geometry of k_spmm)
  const long b = cdiv(nrows, 8);
  return b < 1 ? 1 : b;
}

void spmm_dot(const long* rowptr, const int* col, const double* val, long nrows, const double* X, long ldx, double* Y,
              long ldy, long ncols, double alpha, double beta, double* dot, double* partial, cudaStream_t s,
              const double* Y0) {
  if (nrows == 0) return;
  const long nb = spmm_dot_blocks(nrows);
  const unsigned g = static_cast<unsigned>(nb);
  const double* y0 = Y0 != nullptr ? Y0 : Y;
  for (long c0 = 0; c0 < ncols; c0 += 256) {  // 256-column slabs (prediction solves use ~m columns)
    const long w = ncols - c0 < 256 ? ncols - c0 : 256;
    const int nch = static_cast<int>(cdiv(w, 64));
    double* part = partial + c0 * nb;
    switch (nch) {
      case 1: k_spmm_dot<1><<<g, 256, 0, s>>>(rowptr, col, val, nrows, X + c0, ldx, Y + c0, ldy, w, alpha, beta, part, y0 + c0); break;
      case 2: k_spmm_dot<2><<<g, 256, 0, s>>>(rowptr, col, val, nrows, X + c0, ldx, Y + c0, ldy, w, alpha, beta, part, y0 + c0); break;
      default: k_spmm_dot<4><<<g, 256, 0, s>>>(rowptr, col, val, nrows, X + c0, ldx, Y + c0, ldy, w, alpha, beta, part, y0 + c0); break;
    }
    FSA_LAUNCH_CHECK();
    colsum_partials(part, nb, w, w, dot + c0, s);
  }
}

void launch_spmm(const long* rowptr, const int* col, const double* val, long nrows, const double* X, long ldx,
                 double* Y, long ldy, long ncols, double alpha, double beta, cudaStream_t s) {
  if (nrows == 0) return;
  k_spmm<<<static_cast<unsigned>(cdiv(nrows * 32, 256)), 256, 0, s>>>(rowptr, col, val, nrows, X, ldx, Y, ldy,
                                                                     ncols, alpha, beta);
  FSA_LAUNCH_CHECK();
}

}  // namespace fsa
