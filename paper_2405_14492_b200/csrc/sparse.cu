// Sparse kernels of the FSA operator:
//  * SDDMM assembly of the tapered residual block straight into CSR
//    (reference fsa.cpp:38-56): value = (C(d) - U_r . U_c) T(d), diagonal
//    max(sigma1_2 - |U_r|^2, 0) + sigma2 with the clamp counted;
//  * its rho derivative on the same pattern (fsa.cpp:101-124, U-form);
//  * the cross block to prediction points (prediction.cpp:16-24);
//  * CSR x dense SpMM on row-major RHS blocks.
// One warp per CSR row; the row's m-vector lives in registers (m/32 per lane).
#include "bulk.cuh"
#include "dgemm.cuh"
#include "kernels.cuh"
#include "sparse.cuh"

#include <algorithm>
#include <cstdlib>
#include <cstring>

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

// Block SpMM + dot on the FP64 tensor cores (Csr row groups, build_groups). A group of
// kGroup = 32 consecutive rows (Hilbert order) and the union of their columns form a
// 32 x u value block, cut into 8 x 4 DMMA A tiles (row tile rt, k-step kb); only the tiles
// holding an entry are stored (Csr::kmask / koff, ~2/3 of them), in A-fragment order. The
// union is consumed in pieces of kPiece rows: the piece's RHS rows (gathered) and stored
// tiles (contiguous) are copied into shared memory with cp.async, double-buffered. Against the
// CSR kernel every RHS row is fetched once per group instead of once per nonzero and the
// arithmetic runs on the tensor pipe. (Measured and removed in round 2: pieces of 8 rows, 3- and
// 4-deep rings -- fewer resident CTAs --, bulk-copy (TMA) gathers of the 448-byte rows, an L2
// prefetch of each group's value tiles.)
constexpr int kPiece = 16;  // union rows per pipeline stage (4 DMMA k-steps)
struct TileSpmmArgs {
  const long* gptr;
  const int* gcol;
  const int2* pmeta;   // Csr::pmeta: per k-step {stored tiles before it, masks of it and the next seven}
  const double* tval;  // stored tiles, 32 doubles each
  long nrows;
  const double* X;
  long ldx;
  double* Y;
  long ldy;
  long ncols;
  const double* Y0;
  double* partial;
  long ldp;
  // fused H update (spmm_block_dot_h): X holds Z, Y0 holds Lw and, unless `first`,
  // H = Z + beta H and V = (Lw + S Z) + beta V on the own rows (beta[j], j < kb; 0 beyond)
  double* Hio = nullptr;
  const double* beta = nullptr;
  long kb = 0;
  int first = 0;
  long xrows = 0;    // rows of X that may be gathered (own + halo); checked builds only
  long ntiles = 0;   // stored value tiles; checked builds only
  int gcap = 0;  // k_spmm_v3: union slots reserved in shared memory (gmax rounded up to whole pieces)
  int epf = 0;   // k_spmm_v3: L2 prefetch of the group's epilogue rows this many pieces before the end (0 off)
};
// the h.v epilogue of the block SpMM: Y = Y0 + S X on this lane's fragments, with the PCG
// direction update when H is given (REC: H = Z + beta H, V = (Lw + S Z) + beta V, krylov.cpp:92;
// else H = Z), and the h.v column partials of the group's 32 rows (fixed order: lane butterfly,
// then the four row tiles in order). The column tile is full (NT * 8 columns, ldx == ldy) and the
// pointers do not alias, so the loads of later column tiles can move above earlier stores.
template <int NT, bool REC, bool UPD, bool HASY0>
__device__ __forceinline__ void spmm_epilogue_cols(const TileSpmmArgs& q, const double (&c)[NT][2], long off, bool rok,
                                                   const double* sbeta, double (&red)[4][NT * 8]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, cl = 2 * (lane & 3);
  const double* __restrict__ zr = q.X + off;
  const double* __restrict__ lr = q.Y0 + off;
  double* __restrict__ vr = q.Y + off;
  double* __restrict__ hr = q.Hio + off;
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    double d0 = 0.0, d1 = 0.0;
    if (rok) {
      double2 o = make_double2(c[j][0], c[j][1]);
      if (HASY0) {
        const double2 y0 = __ldg(reinterpret_cast<const double2*>(lr + 8 * j));
        o.x += y0.x;
        o.y += y0.y;
      }
      double2 h = __ldg(reinterpret_cast<const double2*>(zr + 8 * j));
      if (REC) {
        const double2 b = *reinterpret_cast<const double2*>(sbeta + 8 * j + cl);
        const double2 ho = *reinterpret_cast<const double2*>(hr + 8 * j);
        const double2 vo = *reinterpret_cast<const double2*>(vr + 8 * j);
        h.x = h.x + b.x * ho.x;
        h.y = h.y + b.y * ho.y;
        o.x += b.x * vo.x;
        o.y += b.y * vo.y;
      }
      if (UPD) *reinterpret_cast<double2*>(hr + 8 * j) = h;
      *reinterpret_cast<double2*>(vr + 8 * j) = o;
      d0 = h.x * o.x;
      d1 = h.y * o.y;
    }
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      d0 += __shfl_xor_sync(0xffffffffu, d0, o);
      d1 += __shfl_xor_sync(0xffffffffu, d1, o);
    }
    if (lane < 4) {
      red[warp][j * 8 + cl] = d0;
      red[warp][j * 8 + cl + 1] = d1;
    }
  }
}
template <int NT>
__device__ __forceinline__ void spmm_epilogue(const TileSpmmArgs& q, const double (&c)[NT][2], long g, long c0,
                                              double (&red)[4][NT * 8], const double* sbeta) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long row = g * kGroup + warp * 8 + (lane >> 2);
  const bool rok = row < q.nrows;
  const long off = row * q.ldx + c0 + 2 * (lane & 3);  // (ldx == ldy)
  if (q.Hio != nullptr) {
    if (q.first) spmm_epilogue_cols<NT, false, true, true>(q, c, off, rok, sbeta, red);
    else spmm_epilogue_cols<NT, true, true, true>(q, c, off, rok, sbeta, red);
  } else if (q.Y0 != nullptr) {
    spmm_epilogue_cols<NT, false, false, true>(q, c, off, rok, sbeta, red);
  } else {
    spmm_epilogue_cols<NT, false, false, false>(q, c, off, rok, sbeta, red);
  }
  __syncthreads();
  if (tid < NT * 8) q.partial[c0 + g * q.ldp + tid] = ((red[0][tid] + red[1][tid]) + red[2][tid]) + red[3][tid];
}

// k_spmm_v3: the lean main loop. Everything a piece needs besides its data is precomputed once per
// CTA into shared memory: the gathered rows' element offsets (padded to whole pieces with a valid
// row), each warp's k-step word per piece (bit ks: this row tile has a stored tile in k-step ks; bits
// 4 + 5 ks: its index among the piece's stored tiles) and the piece's {first tile, tile count}.
// Warp w gathers piece rows 4w .. 4w + 3 (one 16-byte vector load of their offsets), so a piece
// costs a warp ~4 copy instructions per row instead of ~25 of 64-bit address arithmetic, and a
// k-step is one bit test plus the fragment loads and DMMAs.
template <int NT, int MINB>
__global__ void __launch_bounds__(128, MINB) k_spmm_v3(TileSpmmArgs q) {
  constexpr int P = kPiece, NS = 2, WN = 4, NTH = 32 * WN, RW = P / WN;
  static_assert(kGroup == 32 && P == 16, "four row tiles per group, four k-steps per piece");
  constexpr int LDH = NT * 8 + 4;  // == 4 or 12 (mod 16): conflict-free B fragments
  constexpr int CH = NT * 4;       // 16-byte chunks per gathered row
  constexpr int HS = P * LDH, AS = P * kGroup;
  extern __shared__ __align__(16) double sm[];  // [NS][HS], [NS][AS], offsets, warp words, piece info
  __shared__ double red[WN][NT * 8];
  __shared__ __align__(16) double sbeta[NT * 8];
  const long g = blockIdx.x;
  const long c0 = 64L * blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long u0 = q.gptr[g];
  const int up = static_cast<int>(q.gptr[g + 1] - u0);
  const int npc = (up + P - 1) / P;
  const long kb0 = u0 / 4;
  uint32_t* soff = reinterpret_cast<uint32_t*>(sm + NS * (HS + AS));
  int* sw = reinterpret_cast<int*>(soff + q.gcap);
  int2* spi = reinterpret_cast<int2*>(sw + 4 * (q.gcap / P));
  // (static metadata: staged before the dependency wait)
  for (int i = tid; i < npc * P; i += NTH) {
    const int col = q.gcol[u0 + (i < up ? i : 0)];
    FSA_DCHECK(col >= 0 && col < q.xrows, "spmm: gathered RHS row out of range");
    soff[i] = static_cast<uint32_t>(col) * static_cast<uint32_t>(q.ldx);
  }
  for (int i = tid; i < npc * WN; i += NTH) {
    const int pc = i >> 2, w = i & 3;
    const int2 pm = q.pmeta[kb0 + pc * (P / 4)];
    const int nks = min(P, up - pc * P) / 4;
    int t = 0, word = 0;
#pragma unroll
    for (int ks = 0; ks < P / 4; ++ks) {
      if (ks < nks) {
        const int m = (pm.y >> (4 * ks)) & 15;
        if ((m >> w) & 1) word |= (1 << ks) | ((t + __popc(m & ((1 << w) - 1))) << (4 + 5 * ks));
        t += __popc(m);
      }
    }
    sw[i] = word;
    if (w == 0) {
      FSA_DCHECK(pm.x >= 0 && pm.x + t <= q.ntiles, "spmm: value tile range out of bounds");
      spi[pc] = make_int2(pm.x, t);
    }
  }
  __syncthreads();
  const double* Xl = q.X + c0 + 2 * lane;  // this lane's 16-byte chunk of every gathered row
  auto issue = [&](int pc) {
    if (pc < npc) {
      const int slot = pc % NS;
      const uint4 v = *reinterpret_cast<const uint4*>(soff + pc * P + RW * warp);
      const uint32_t o[RW] = {v.x, v.y, v.z, v.w};
      double* hd = sm + slot * HS + RW * warp * LDH + 2 * lane;
#pragma unroll
      for (int k = 0; k < (CH + 31) / 32; ++k) {
        if (lane + 32 * k < CH) {
#pragma unroll
          for (int i = 0; i < RW; ++i) cp_async16(hd + 64 * k + i * LDH, Xl + 64 * k + o[i]);
        }
      }
      const int2 pi = spi[pc];
      const double* src = q.tval + 32L * pi.x + 2 * tid;
      double* ad = sm + NS * HS + slot * AS + 2 * tid;
      if (tid < pi.y * 16) cp_async16(ad, src);
      if (tid + NTH < pi.y * 16) cp_async16(ad + 2 * NTH, src + 2 * NTH);
    }
    cp_async_commit();  // (empty groups keep the wait count uniform)
  };
  double c[NT][2];
#pragma unroll
  for (int j = 0; j < NT; ++j) c[j][0] = c[j][1] = 0.0;
  pdl_wait();
  if (tid < NT * 8 && q.Hio != nullptr && !q.first) sbeta[tid] = c0 + tid < q.kb ? q.beta[c0 + tid] : 0.0;
#pragma unroll
  for (int s = 0; s < NS - 1; ++s) issue(s);
  for (int pc = 0; pc < npc; ++pc) {
    cp_async_wait<NS - 2>();
    __syncthreads();  // piece pc visible to all; every warp is done with piece pc - 1, whose slot is refilled next
    issue(pc + NS - 1);
    if (pc == npc - q.epf && tid == 0) {  // the epilogue rows into L2 shortly before they are read
      const uint32_t rb = static_cast<uint32_t>(kGroup * q.ldy * 8);
      if (q.Y0 != nullptr) prefetch_l2(q.Y0 + g * kGroup * q.ldy, rb);
      prefetch_l2(q.X + g * kGroup * q.ldx, static_cast<uint32_t>(kGroup * q.ldx * 8));
      if (q.Hio != nullptr && !q.first) {
        prefetch_l2(q.Hio + g * kGroup * q.ldy, rb);
        prefetch_l2(q.Y + g * kGroup * q.ldy, rb);
      }
    }
    const int slot = pc % NS;
    const int word = sw[pc * WN + warp];
    const double* hs = sm + slot * HS + (lane & 3) * LDH + (lane >> 2);
    const double* as = sm + NS * HS + slot * AS + lane;
#pragma unroll
    for (int ks = 0; ks < P / 4; ++ks) {
      if (word & (1 << ks)) {
        const double a = as[((word >> (4 + 5 * ks)) & 31) * 32];
        const double* hb = hs + ks * 4 * LDH;
        double b[NT];
#pragma unroll
        for (int j = 0; j < NT; ++j) b[j] = hb[j * 8];
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma8x8x4(c[j][0], c[j][1], a, b[j]);
      }
    }
  }
  spmm_epilogue<NT>(q, c, g, c0, red, sbeta);
}
// ---- block SDDMM: dense Gram blocks of the row groups on DMMA ----------------------------------
// G = A_R^T B_C for a group's 32 rows R and a 64-column tile C of its union, over K (the
// inducing dimension): MODE 0 A = B = U (Sigma_s); MODE 1 [U1; U]_R^T [U; T]_C (d Sigma_s /
// d rho, K = 2 m). K pieces of 32 are staged by cp.async (double-buffered) and the block
// product runs as DMMA m8n8k4 tiles; the result is stored in the value-block layout of the
// block SpMM (gslot order), from which k_sddmm_finish picks the pattern's entries.
// Evaluating full blocks costs ~6x the pattern's dot products but turns the L1-bound
// per-nonzero gathers of m-vectors into tensor-core work on staged tiles.
constexpr int kGK = 32;                // K per staged piece
constexpr int kGLd = kGK + 4;          // smem row stride (== 4 mod 16: conflict-free fragments)
template <int SUB, int H>
__device__ __forceinline__ void gram_ksteps(double (&c)[8][2], const double* As, const double* Bs, int rt, int lane) {
#pragma unroll
  for (int ks = 0; ks < kGK / 4; ++ks) {
    const double a = As[(rt * 8 + (lane >> 2)) * kGLd + ks * 4 + (lane & 3)];
#pragma unroll
    for (int q = H; q < 8; q += SUB) {
      const double b = Bs[(q * 8 + (lane >> 2)) * kGLd + ks * 4 + (lane & 3)];
      dmma8x8x4(c[q][0], c[q][1], a, b);
    }
  }
}
template <int MODE>
__global__ void __launch_bounds__(256, 4) k_block_gram(const long* __restrict__ gptr, const int* __restrict__ gcol,
                                                      const int* __restrict__ gneed,
                                                      const int* __restrict__ gneedcnt, long nrows,
                                                      const double* __restrict__ A0,
                                                      const double* __restrict__ B0, const double* __restrict__ A1,
                                                      const double* __restrict__ B1, long ldu, long mp,
                                                      double* __restrict__ G) {
  extern __shared__ __align__(16) double gsm[];
  double(*As)[kGroup * kGLd] = reinterpret_cast<double(*)[kGroup * kGLd]>(gsm);
  double(*Bs)[64 * kGLd] = reinterpret_cast<double(*)[64 * kGLd]>(gsm + 2 * kGroup * kGLd);
  const long g = blockIdx.x;
  const int jt = blockIdx.y;
  // the tile's columns: union slots gneed[u0 + j0 ...] (columns >= the group's first row; entries
  // left of the diagonal are mirrored by k_sddmm_finish and never read from G)
  __shared__ int uslot[64], ucol[64];
  const long u0 = gptr[g];
  const int up = gneedcnt[g];
  const int j0 = jt * 64;
  if (j0 >= up) return;
  const int nc = min(64, up - j0);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < 64) {
    const int u = tid < nc ? gneed[u0 + j0 + tid] : -1;
    uslot[tid] = u;
    ucol[tid] = u >= 0 ? gcol[u0 + u] : 0;
  }
  const int rt = warp & 3, half = warp >> 2;
  const long r0 = g * kGroup;
  const long K = MODE == 0 ? mp : 2 * mp;
  const int npc = static_cast<int>(K / kGK);
  // columns beyond the tile's union and rows beyond nrows stay zero in smem
  for (int i = tid; i < 2 * 64 * kGLd; i += 256) (&Bs[0][0])[i] = 0.0;
  for (int i = tid; i < 2 * kGroup * kGLd; i += 256) (&As[0][0])[i] = 0.0;
  __syncthreads();
  auto issue = [&](int pc) {
    const long k0 = static_cast<long>(pc) * kGK;
    const bool second = MODE == 1 && k0 >= mp;
    const double* A = second ? A1 : A0;
    const double* B = second ? B1 : B0;
    const long kk = second ? k0 - mp : k0;
    double* as = As[pc & 1];
    double* bs = Bs[pc & 1];
    for (int idx = tid; idx < kGroup * (kGK / 2); idx += 256) {
      const int r = idx / (kGK / 2), ch = idx % (kGK / 2);
      if (r0 + r < nrows) cp_async16(as + r * kGLd + ch * 2, A + (r0 + r) * ldu + kk + ch * 2);
    }
    for (int idx = tid; idx < nc * (kGK / 2); idx += 256) {
      const int j = idx / (kGK / 2), ch = idx % (kGK / 2);
      FSA_DCHECK(ucol[j] >= 0, "block gram: negative union column");
      cp_async16(bs + j * kGLd + ch * 2, B + static_cast<long>(ucol[j]) * ldu + kk + ch * 2);
    }
    cp_async_commit();
  };
  double c[8][2];
#pragma unroll
  for (int q = 0; q < 8; ++q) c[q][0] = c[q][1] = 0.0;
  issue(0);
  for (int pc = 0; pc < npc; ++pc) {
    if (pc + 1 < npc) {
      issue(pc + 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    if (half == 0) gram_ksteps<2, 0>(c, As[pc & 1], Bs[pc & 1], rt, lane);
    else gram_ksteps<2, 1>(c, As[pc & 1], Bs[pc & 1], rt, lane);
    __syncthreads();
  }
  const int rr = rt * 8 + (lane >> 2);
  double* gb = G + static_cast<long>(kGroup) * u0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    if ((q & 1) != half) continue;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int u = uslot[q * 8 + 2 * (lane & 3) + e];
      if (u >= 0) gb[((u >> 2) * (kGroup / 8) + (rr >> 3)) * 32 + (rr & 7) * 4 + (u & 3)] = c[q][e];
    }
  }
}
// pattern entries from the Gram blocks: Sigma_s (MODE 0) or d Sigma_s / d rho (MODE 1);
// each unordered pair is evaluated once (from the row with c > r) and mirrored, so the
// result is exactly symmetric; MODE 0 also fills the SpMM value blocks gval
// stored-tile index of dense value-block slot d (Csr::kmask / koff)
__device__ __forceinline__ long tile_slot(int d, const int* __restrict__ kmask, const int* __restrict__ koff) {
  const int kb = d >> 7, rt = (d >> 5) & 3;
  return 32L * (koff[kb] + __popc(kmask[kb] & ((1 << rt) - 1))) + (d & 31);
}
template <int MODE>
__global__ void k_sddmm_finish(const long* __restrict__ rowptr, const int* __restrict__ col,
                               const long* __restrict__ mirror, const int* __restrict__ gslot,
                               const double* __restrict__ dist, const double* __restrict__ lowrank_diag,
                               const double* __restrict__ G, long n, SddmmParams P, double* __restrict__ val,
                               double* __restrict__ gval, const int* __restrict__ kmask,
                               const int* __restrict__ koff, int* __restrict__ n_clamped) {
  const long r = (static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= n) return;
  for (long p = rowptr[r] + lane; p < rowptr[r + 1]; p += 32) {
    const long c = col[p];
    if (c < r) continue;  // written from the mirror entry
    double v;
    if (c == r) {
      const double resid = P.sigma1_2 - lowrank_diag[r];
      if (MODE == 0) {
        if (resid < 0.0) atomicAdd(n_clamped, 1);
        v = (resid < 0.0 ? 0.0 : resid) + P.sigma2;
      } else {
        v = resid < 0.0 ? 0.0 : -G[gslot[p]];
      }
    } else {
      const double d = dist[p];
      const double k = MODE == 0 ? matern_d(d, P.nu, P.sigma1_2, P.rho) : matern_drho_d(d, P.nu, P.sigma1_2, P.rho);
      v = (k - G[gslot[p]]) * taper_d(d, P.family, P.gamma);
    }
    val[p] = v;
    if (MODE == 0 && gval != nullptr) gval[tile_slot(gslot[p], kmask, koff)] = v;
    const long q = mirror[p];
    if (c != r && q >= 0) {
      val[q] = v;
      if (MODE == 0 && gval != nullptr) gval[tile_slot(gslot[q], kmask, koff)] = v;
    }
  }
}

// stored tiles from the CSR values (gval zeroed first)
__global__ void k_group_scatter(const int* __restrict__ gslot, const int* __restrict__ kmask,
                                const int* __restrict__ koff, long nnz, const double* __restrict__ val,
                                double* __restrict__ gval) {
  const long p = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p < nnz) gval[tile_slot(gslot[p], kmask, koff)] = val[p];
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

void sddmm_block(int mode, const double* U, const double* U1, const double* T, long ldu, long mp, const Csr& pat,
                 const double* lowrank_diag, const SddmmParams& P, double* val, double* gval, int* n_clamped_dev,
                 double* gtmp, cudaStream_t s) {
  require(pat.gnnz > 0 && mp % kGK == 0, "sddmm_block: row groups missing");
  const dim3 grid(static_cast<unsigned>(pat.ngrp), static_cast<unsigned>(cdiv(pat.gneedmax, 64)));
  const int smem = static_cast<int>(2 * (kGroup + 64) * kGLd * sizeof(double));
  static bool attr = false;
  if (!attr) {
    FSA_CUDA(cudaFuncSetAttribute(k_block_gram<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    FSA_CUDA(cudaFuncSetAttribute(k_block_gram<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  if (mode == 0)
    k_block_gram<0><<<grid, 256, smem, s>>>(pat.gptr.get(), pat.gcol.get(), pat.gneed.get(), pat.gneedcnt.get(), pat.rows, U, U, U, U, ldu, mp, gtmp);
  else
    k_block_gram<1><<<grid, 256, smem, s>>>(pat.gptr.get(), pat.gcol.get(), pat.gneed.get(), pat.gneedcnt.get(), pat.rows, U1, U, U, T, ldu, mp, gtmp);
  FSA_LAUNCH_CHECK();
  if (mode == 0 && gval != nullptr) FSA_CUDA(cudaMemsetAsync(gval, 0, sizeof(double) * 32 * pat.ntiles, s));
  if (mode == 0 && n_clamped_dev != nullptr) FSA_CUDA(cudaMemsetAsync(n_clamped_dev, 0, sizeof(int), s));
  const unsigned g2 = static_cast<unsigned>(cdiv(pat.rows * 32, 256));
  if (mode == 0)
    k_sddmm_finish<0><<<g2, 256, 0, s>>>(pat.rowptr.get(), pat.col.get(), pat.mirror.get(), pat.gslot.get(),
                                        pat.dist.get(), lowrank_diag, gtmp, pat.rows, P, val, gval, pat.kmask.get(),
                                        pat.koff.get(), n_clamped_dev);
  else
    k_sddmm_finish<1><<<g2, 256, 0, s>>>(pat.rowptr.get(), pat.col.get(), pat.mirror.get(), pat.gslot.get(),
                                        pat.dist.get(), lowrank_diag, gtmp, pat.rows, P, val, nullptr, nullptr, nullptr,
                                        nullptr);
  FSA_LAUNCH_CHECK();
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
  FSA_CUDA(cudaMemsetAsync(gval, 0, sizeof(double) * 32 * pat.ntiles, s));
  k_group_scatter<<<static_cast<unsigned>(cdiv(pat.nnz, 256)), 256, 0, s>>>(pat.gslot.get(), pat.kmask.get(),
                                                                            pat.koff.get(), pat.nnz, val, gval);
  FSA_LAUNCH_CHECK();
}

long spmm_group_blocks(long ngrp) { return ngrp < 1 ? 1 : ngrp; }

bool spmm_block_supported(long ncols) { return ncols % 8 == 0; }

// Y = S X (+ Y0) over ncols (multiple of 8) columns in 64-column tiles; dot[c] = sum_r X[r][c] Y[r][c]
void spmm_block_dot(const Csr& pat, const double* gval, const double* X, long ldx, double* Y, long ldy, long ncols,
                    double* dot, double* partial, const double* Y0, cudaStream_t s) {
  spmm_block_dot_h(pat, gval, X, ldx, Y, ldy, ncols, dot, partial, Y0, nullptr, nullptr, 0, false, s);
}
void spmm_block_dot_h(const Csr& pat, const double* gval, const double* X, long ldx, double* Y, long ldy, long ncols,
                      double* dot, double* partial, const double* Y0, double* H, const double* beta, long kb,
                      bool first, cudaStream_t s, bool colsum) {
  require(spmm_block_supported(ncols) && ldx >= ncols && ldy == ldx && ldx % 2 == 0, "spmm_block_dot: unsupported block");
  if (pat.rows == 0) return;
  static const int epf = [] {  // FSA_SPMM_EPF=k: L2 prefetch of the epilogue rows k pieces before the end (0 off)
    const char* e = std::getenv("FSA_SPMM_EPF");
    return e != nullptr ? std::atoi(e) : 4;
  }();
  auto launch = [&](int nt, long c_first, long tiles) {
    const long ldh = nt * 8 + 4;  // k_spmm_v3's LDH
    const int gcap = static_cast<int>(round_up(pat.gmax, kPiece));
    const int smem = static_cast<int>(2 * (kPiece * ldh + kPiece * kGroup) * 8) + gcap * 4 + (gcap / kPiece) * (16 + 8);
    require((pat.cols > 0 ? pat.cols : pat.rows) * ldx < (1L << 32), "spmm: RHS block too large for 32-bit offsets");
    TileSpmmArgs a{pat.gptr.get(), pat.gcol.get(), reinterpret_cast<const int2*>(pat.pmeta.get()), gval, pat.rows,
                   X + c_first, ldx, Y + c_first, ldy, ncols - c_first, Y0 != nullptr ? Y0 + c_first : nullptr,
                   partial + c_first, ncols, H != nullptr ? H + c_first : nullptr,
                   beta != nullptr ? beta + c_first : nullptr, kb - c_first, first ? 1 : 0,
                   pat.cols > 0 ? pat.cols : pat.rows, pat.ntiles, gcap, epf};
    const dim3 grid(static_cast<unsigned>(pat.ngrp), static_cast<unsigned>(tiles));
    auto go = [&](auto kern) {
      // one fixed opt-in ceiling (not this launch's size: the launch size depends on the pattern's
      // largest union, and thread-group ranks sharing a device would race on a per-launch value)
      constexpr int kSmemCeiling = 160 * 1024;
      require(smem <= kSmemCeiling, "spmm: union too large for shared memory");
      FSA_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemCeiling));
      launch_pdl(kern, grid, dim3(128), static_cast<size_t>(smem), s, a);
    };
    switch (nt) {
      case 1: go(k_spmm_v3<1, 8>); break;
      case 2: go(k_spmm_v3<2, 8>); break;
      case 3: go(k_spmm_v3<3, 8>); break;
      case 4: go(k_spmm_v3<4, 8>); break;
      case 5: go(k_spmm_v3<5, 8>); break;
      case 6: go(k_spmm_v3<6, 7>); break;
      case 7: go(k_spmm_v3<7, 7>); break;  // (7 resident CTAs: 8 -> 4 % slower, 6 -> 6 %)
      case 8: go(k_spmm_v3<8, 7>); break;
      default: go(k_spmm_v3<9, 7>); break;  // 72 columns (t = 65) in one pass
    }
    FSA_LAUNCH_CHECK();
  };
  if (ncols == 72) {  // one 9-n-tile pass instead of 64 + 8 columns (the RHS rows are gathered once)
    launch(9, 0, 1);
  } else {
    const long full = ncols / 64, rem = ncols % 64;
    if (full > 0) launch(8, 0, full);
    if (rem > 0) launch(static_cast<int>(rem / 8), full * 64, 1);
  }
  if (colsum) colsum_partials(partial, pat.ngrp, ncols, ncols, dot, s);
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
