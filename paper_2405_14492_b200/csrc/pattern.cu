// Device taper-neighbour search; see pattern.cuh.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>

#include "kernels.cuh"
#include "pattern.cuh"

namespace fsa {

namespace {

constexpr unsigned kHilbertBits = 21;
constexpr long kMaxCells = (1L << kHilbertBits) - 2;

__host__ __device__ inline unsigned long long hilbert_xy2d(unsigned long long x, unsigned long long y) {
  const unsigned long long n = 1ULL << kHilbertBits;
  unsigned long long d = 0;
  for (unsigned long long s = n / 2; s > 0; s /= 2) {
    const unsigned long long rx = (x & s) > 0 ? 1 : 0;
    const unsigned long long ry = (y & s) > 0 ? 1 : 0;
    d += s * s * ((3 * rx) ^ ry);
    if (ry == 0) {
      if (rx == 1) {
        x = n - 1 - x;
        y = n - 1 - y;
      }
      const unsigned long long t = x;
      x = y;
      y = t;
    }
  }
  return d;
}
__host__ __device__ inline unsigned long long spread3(unsigned long long v) {
  unsigned long long r = 0;
  for (int b = 0; b < 21; ++b) r |= ((v >> b) & 1ULL) << (3 * b);
  return r;
}
template <int D>
__host__ __device__ inline unsigned long long cell_key(const long* c) {
  if (D == 1) return static_cast<unsigned long long>(c[0]);
  if (D == 2) return hilbert_xy2d(static_cast<unsigned long long>(c[0]), static_cast<unsigned long long>(c[1]));
  return spread3(c[0]) | (spread3(c[1]) << 1) | (spread3(c[2]) << 2);
}

struct GridArgs {
  double o0, o1, o2, h;
};
template <int D>
__device__ inline void cell_of(const double* x, long ld, long i, const GridArgs& g, long* c) {
  const double o[3] = {g.o0, g.o1, g.o2};
#pragma unroll
  for (int k = 0; k < D; ++k) {
    long v = static_cast<long>(floor((x[i + k * ld] - o[k]) / g.h));
    v = v < 0 ? 0 : (v > kMaxCells ? kMaxCells : v);
    c[k] = v;
  }
}

// Points are sorted by (cell key, position inside the cell): the cell key keeps every cell
// contiguous for the neighbour search, and the second level (a 2^8 x 2^8 Hilbert curve inside
// the cell for d = 2, the 16-bit offset for d = 1) makes any run of consecutive points
// spatially compact, which is what the 32-row groups of the block SpMM need (smaller column
// unions, fewer stored value tiles). d = 3 keys have no spare bits and keep the cell order.
template <int D>
constexpr int kSubBits = D == 3 ? 0 : 16;
__host__ __device__ inline unsigned hilbert8(unsigned x, unsigned y) {
  unsigned d = 0;
  for (unsigned s = 128; s > 0; s >>= 1) {
    const unsigned rx = (x & s) ? 1 : 0, ry = (y & s) ? 1 : 0;
    d += s * s * ((3 * rx) ^ ry);
    if (ry == 0) {
      if (rx == 1) {
        x = 255 - x;
        y = 255 - y;
      }
      const unsigned t = x;
      x = y;
      y = t;
    }
  }
  return d;
}
template <int D>
__global__ void k_point_keys(const double* __restrict__ xs, long n, GridArgs g, unsigned long long* keys,
                             int* idx) {
  const long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  long c[3] = {0, 0, 0};
  cell_of<D>(xs, n, i, g, c);
  unsigned long long key = cell_key<D>(c);
  if (kSubBits<D> > 0) {
    const double o[2] = {g.o0, g.o1};
    unsigned f[2] = {0, 0};
    const double res = D == 1 ? 65536.0 : 256.0;
#pragma unroll
    for (int k = 0; k < (D < 2 ? D : 2); ++k) {
      const double t = ((xs[i + k * n] - o[k]) / g.h - static_cast<double>(c[k])) * res;
      f[k] = t <= 0.0 ? 0u : (t >= res - 1.0 ? static_cast<unsigned>(res - 1.0) : static_cast<unsigned>(t));
    }
    key = (key << kSubBits<D>) | (D == 1 ? f[0] : hilbert8(f[0], f[1]));
  }
  keys[i] = key;
  idx[i] = static_cast<int>(i);
}
__global__ void k_cell_keys(unsigned long long* keys, long n, int shift) {
  const long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) keys[i] >>= shift;
}

__global__ void k_gather_coords(const double* __restrict__ xs, long n, int d, const int* __restrict__ perm,
                                long n_pad, double* __restrict__ out, int* __restrict__ iperm) {
  const long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n_pad) return;
  if (i < n) {
    const long o = perm[i];
    for (int k = 0; k < d; ++k) out[i + k * n_pad] = xs[o + k * n];
    iperm[o] = static_cast<int>(i);
  } else {
    for (int k = 0; k < d; ++k) out[i + k * n_pad] = 0.0;
  }
}

__device__ inline long lower_bound_key(const unsigned long long* keys, long n, unsigned long long k) {
  long lo = 0, hi = n;
  while (lo < hi) {
    const long mid = (lo + hi) >> 1;
    if (keys[mid] < k) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Visit every column point j within gamma of row point i, in ascending internal
// column order (neighbour cells sorted by key; points within a cell are contiguous).
template <int D, class F>
__device__ inline void visit_neighbours(const double* __restrict__ rx, long rld, long i,
                                        const double* __restrict__ cx, long cld,
                                        const unsigned long long* __restrict__ ckeys, long cn, const GridArgs& g,
                                        double gamma, F&& f) {
  long base[3] = {0, 0, 0};
  cell_of<D>(rx, rld, i, g, base);
  constexpr int NC = D == 1 ? 3 : (D == 2 ? 9 : 27);
  unsigned long long ks[NC];
  int nk = 0;
  for (int q = 0; q < NC; ++q) {
    long c[3] = {0, 0, 0};
    int t = q;
    bool ok = true;
#pragma unroll
    for (int k = 0; k < D; ++k) {
      c[k] = base[k] + (t % 3) - 1;
      t /= 3;
      if (c[k] < 0 || c[k] > kMaxCells) ok = false;
    }
    if (!ok) continue;
    const unsigned long long key = cell_key<D>(c);
    bool dup = false;
    for (int a = 0; a < nk; ++a) dup |= ks[a] == key;
    if (!dup) ks[nk++] = key;
  }
  // insertion sort of the (<= 27) keys
  for (int a = 1; a < nk; ++a) {
    const unsigned long long v = ks[a];
    int b = a - 1;
    while (b >= 0 && ks[b] > v) {
      ks[b + 1] = ks[b];
      --b;
    }
    ks[b + 1] = v;
  }
  for (int a = 0; a < nk; ++a) {
    long p = lower_bound_key(ckeys, cn, ks[a]);
    for (; p < cn && ckeys[p] == ks[a]; ++p) {
      const double dd = pdist_soa<D>(rx, rld, i, cx, cld, p);
      if (dd < gamma) f(p, dd);
    }
  }
}

template <int D>
__global__ void k_count(const double* rx, long rld, long rn, const double* cx, long cld,
                        const unsigned long long* ckeys, long cn, GridArgs g, double gamma, long* counts) {
  const long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= rn) return;
  long cnt = 0;
  visit_neighbours<D>(rx, rld, i, cx, cld, ckeys, cn, g, gamma, [&](long, double) { ++cnt; });
  counts[i] = cnt;
}

// Union of the column indices of kGroup consecutive rows: bitonic sort of the
// group's entries in shared memory, unique, then each entry's union-local index.
constexpr int kUnionSort = 4096;  // max entries per 32-row group handled by the sort
constexpr int kUnionCap = 1024;   // max union size per 32-row group
// (G, sort capacity, union capacity) are runtime: dynamic smem holds 2 x kSortCap ints
// RADIX: the group's (<= 4096) column indices are sorted by a block radix sort over key_bits
// bits (3 to 6 passes instead of the 78 passes of the bitonic network); larger capacities
// (the 128-row groups of the opt-in INT8 SpMM) keep the bitonic sort.
// TILE_ORDER (32-row groups of the block SpMM): the union is then re-ordered so that columns
// referenced by the same subset of the group's four 8-row tiles are adjacent — key = the rank of
// the column's row-tile mask in kMaskRank (a chain 0001, 0011, 0111, 1111, 1110, 1100, 1000 in
// which every tile's columns form one run), ties by column. A 4-column k-step then rarely mixes
// columns of different tiles, so fewer of the 8 x 4 DMMA A tiles are stored and those stored are
// denser (sparse.cu k_spmm_rt does one DMMA per stored tile and n-tile).
__constant__ int kMaskRank[16] = {15, 0, 8, 1, 9, 10, 7, 2, 6, 11, 14, 12, 5, 13, 4, 3};
template <bool RADIX>
__global__ void __launch_bounds__(512) k_group_union(const long* __restrict__ rowptr, const int* __restrict__ col,
                                                     long nrows, int G, int kSortCap, int kCap,
                                                     int* __restrict__ ucols, int* __restrict__ ucount,
                                                     int* __restrict__ lidx, int key_bits, int tile_order) {
  extern __shared__ int ush[];
  int* keys = ush;
  int* flag = ush + kSortCap;
  const long b = blockIdx.x;
  const long r0 = b * G;
  const long r1 = r0 + G < nrows ? r0 + G : nrows;
  const long p0 = rowptr[r0], p1 = rowptr[r1];
  const long cnt = p1 - p0;
  const int tid = threadIdx.x;
  if (cnt > kSortCap) {
    if (tid == 0) ucount[b] = -1;
    return;
  }
  int size = 1;
  while (size < cnt) size <<= 1;
  if constexpr (RADIX) {
    typedef cub::BlockRadixSort<int, 512, 8> BRS;
    __shared__ typename BRS::TempStorage rs;
    int v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int i = tid * 8 + j;
      v[j] = i < cnt ? col[p0 + i] : 0x7fffffff;
    }
    BRS(rs).Sort(v, 0, key_bits < 31 ? key_bits + 1 : 32);  // + 1 bit: the 0x7fffffff padding sorts last
#pragma unroll
    for (int j = 0; j < 8; ++j) keys[tid * 8 + j] = v[j];
    __syncthreads();
    size = 4096;
  } else {
  for (int i = tid; i < size; i += blockDim.x) keys[i] = i < cnt ? col[p0 + i] : 0x7fffffff;
  __syncthreads();
  for (int k = 2; k <= size; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = tid; i < size; i += blockDim.x) {
        const int l = i ^ j;
        if (l > i) {
          const bool up = (i & k) == 0;
          const int a = keys[i], c = keys[l];
          if ((a > c) == up) {
            keys[i] = c;
            keys[l] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  }
  for (int i = tid; i < size; i += blockDim.x) flag[i] = (i < cnt && (i == 0 || keys[i] != keys[i - 1])) ? 1 : 0;
  __syncthreads();
  if (tid < 32) {  // inclusive scan of the flags (one warp)
    int carry = 0;
    for (int base = 0; base < size; base += 32) {
      int v = flag[base + tid];
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, v, o);
        if (tid >= o) v += u;
      }
      flag[base + tid] = v + carry;
      carry += __shfl_sync(0xffffffffu, v, 31);
    }
  }
  __syncthreads();
  const int U = cnt > 0 ? flag[cnt - 1] : 0;
  if (U > kCap) {
    if (tid == 0) ucount[b] = -1;
    return;
  }
  int* out = ucols + b * kCap;
  for (int i = tid; i < cnt; i += blockDim.x)
    if (i == 0 || keys[i] != keys[i - 1]) out[flag[i] - 1] = keys[i];
  __syncthreads();
  for (long p = p0 + tid; p < p1; p += blockDim.x) {
    const int c = col[p];
    int lo = 0, hi = U;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (out[mid] < c) lo = mid + 1; else hi = mid;
    }
    lidx[p] = lo;
  }
  if (tile_order && U > 0) {
    __syncthreads();  // lidx (global, written by this block) and `out` complete
    int* umask = flag;       // [U] row-tile masks
    int* okey = keys;        // [U] order keys
    int* oldc = keys + 2048; // [U] union columns in ascending order (U <= kCap <= 1024)
    for (int i = tid; i < U; i += blockDim.x) {
      umask[i] = 0;
      oldc[i] = out[i];
    }
    __syncthreads();
    const int warp = tid >> 5, lane = tid & 31;
    for (long r = r0 + warp; r < r1; r += blockDim.x / 32)
      for (long p = rowptr[r] + lane; p < rowptr[r + 1]; p += 32) atomicOr(&umask[lidx[p]], 1 << ((r - r0) >> 3));
    __syncthreads();
    for (int i = tid; i < U; i += blockDim.x) okey[i] = (kMaskRank[umask[i] & 15] << 12) | i;
    __syncthreads();
    int* pos1 = keys + 3072;  // [U] position of old slot i in the mask order
    for (int i = tid; i < U; i += blockDim.x) {  // rank of key i (keys are distinct)
      const int ki = okey[i];
      int pos = 0;
      for (int j = 0; j < U; ++j) pos += okey[j] < ki ? 1 : 0;
      pos1[i] = pos;
    }
    __syncthreads();
    // tile_order 2: the k-steps (4 consecutive slots; their composition, hence the stored tiles,
    // unchanged) are dealt round-robin into the 16-row pieces of the block SpMM, so each piece
    // mixes k-steps from the whole mask chain and the four row tiles' warps get similar work
    // between two barriers (in mask order a piece often belongs to one row tile). A partial last
    // k-step (U % 4 != 0, padded after it) keeps its place.
    int* fin = flag + 2048;  // [U] final position of old slot i
    const int K4 = U >> 2, npc = (K4 + 3) >> 2;
    int* newk = flag + 1024;  // [K4]
    if (tile_order == 2) {
      for (int k = tid; k < K4; k += blockDim.x) {
        const int kk = ((k % npc) << 12) | (k / npc);
        int pos = 0;
        for (int j = 0; j < K4; ++j) pos += (((j % npc) << 12) | (j / npc)) < kk ? 1 : 0;
        newk[k] = pos;
      }
      __syncthreads();
    }
    for (int i = tid; i < U; i += blockDim.x) {
      const int p = pos1[i], k = p >> 2;
      fin[i] = tile_order == 2 && k < K4 ? (newk[k] << 2) | (p & 3) : p;
    }
    __syncthreads();
    for (int i = tid; i < U; i += blockDim.x) out[fin[i]] = oldc[i];
    for (long p = p0 + tid; p < p1; p += blockDim.x) lidx[p] = fin[lidx[p]];
  }
  if (tid == 0) ucount[b] = U;
}
__global__ void k_group_compact(const int* __restrict__ ucols, int kCap, const int* __restrict__ ucount,
                                const long* __restrict__ gptr, long ngrp, int* __restrict__ gcol) {
  const long b = blockIdx.x;
  if (b >= ngrp) return;
  const long o = gptr[b], up = gptr[b + 1] - o;
  const int u = ucount[b];
  for (long i = threadIdx.x; i < up; i += blockDim.x) gcol[o + i] = ucols[b * kCap + (i < u ? i : 0)];
}
// union slots whose column is >= the group's first row, in slot order (one warp per group)
__global__ void k_group_need(const long* __restrict__ gptr, const int* __restrict__ gcol, long ngrp,
                             int* __restrict__ gneed, int* __restrict__ gneedcnt, int* __restrict__ cntmax) {
  const long g = blockIdx.x;
  if (g >= ngrp) return;
  const int lane = threadIdx.x;
  const long o = gptr[g];
  const int up = static_cast<int>(gptr[g + 1] - o);
  const int r0 = static_cast<int>(g * kGroup);
  int cnt = 0;
  for (int u0 = 0; u0 < up; u0 += 32) {
    const int u = u0 + lane;
    const bool keep = u < up && gcol[o + u] >= r0;
    const unsigned b = __ballot_sync(0xffffffffu, keep);
    if (keep) gneed[o + cnt + __popc(b & ((1u << lane) - 1u))] = u;
    cnt += __popc(b);
  }
  if (lane == 0) {
    gneedcnt[g] = cnt;
    atomicMax(cntmax, cnt);
  }
}
// value index of entry p (row r, union slot u of group g): A-fragment order of the
// 8 x 4 DMMA tiles: [k-step u/4][warp (r%32)/8][lane ((r%8)*4 + u%4)]
__global__ void k_group_slots(const long* __restrict__ rowptr, long nrows, const long* __restrict__ gptr,
                              int* __restrict__ lidx_to_slot) {
  const long r = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  const long o = gptr[r / kGroup];
  const int rr = static_cast<int>(r % kGroup);
  for (long p = rowptr[r]; p < rowptr[r + 1]; ++p) {
    const int u = lidx_to_slot[p];
    lidx_to_slot[p] = static_cast<int>(kGroup * o + ((u >> 2) * (kGroup / 8) + (rr >> 3)) * 32 + (rr & 7) * 4 + (u & 3));
  }
}
// kmask[kb] |= 1 << rt for every entry (dense slot = kb * 128 + rt * 32 + lane)
__global__ void k_tile_mask(const int* __restrict__ gslot, long nnz, int* __restrict__ kmask) {
  const long p = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= nnz) return;
  const int d = gslot[p];
  atomicOr(kmask + (d >> 7), 1 << ((d >> 5) & 3));
}
__global__ void k_tile_count(const int* __restrict__ kmask, long nkb, int* __restrict__ cnt) {
  const long k = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k <= nkb) cnt[k] = k < nkb ? __popc(kmask[k]) : 0;
}
__global__ void k_piece_meta(const int* __restrict__ kmask, const int* __restrict__ koff, long nkb,
                             int2* __restrict__ pmeta) {
  const long k = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= nkb) return;
  int m = 0;
  for (int i = 0; i < 8 && k + i < nkb; ++i) m |= kmask[k + i] << (4 * i);
  pmeta[k] = make_int2(koff[k], m);
}
__global__ void k_group_ok(const int* __restrict__ ucount, long ngrp, int pad, int* __restrict__ bad,
                           long* __restrict__ sizes) {
  const long b = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (b >= ngrp) return;
  const int u = ucount[b];
  if (u < 0) atomicExch(bad, 1);
  sizes[b] = u < 0 ? 0 : (u + pad - 1) / pad * pad;
}
// unions of G consecutive rows, padded to `pad`; false if a group exceeds the capacities
bool build_unions(const Csr& pat, int G, int pad, int sort_cap, int cap, long& ngrp, long& gnnz, int& gmax,
                  DBuf<long>& gptr, DBuf<int>& gcol, DBuf<int>& lidx, cudaStream_t s, int tile_order = 0) {
  gnnz = 0;
  ngrp = cdiv(pat.rows, G);
  if (ngrp == 0 || pat.nnz == 0) return false;
  DBuf<int> ucols(static_cast<size_t>(ngrp) * cap), ucount(ngrp), bad(1);
  DBuf<long> sizes(ngrp + 1);
  lidx.alloc(pat.nnz);
  const int smem = 2 * sort_cap * static_cast<int>(sizeof(int));
  int key_bits = 1;  // column indices (extended indexing) are < 2^key_bits
  {
    long maxc = pat.cols > 0 ? pat.cols : pat.rows;
    while ((1L << key_bits) < maxc + 1 && key_bits < 31) ++key_bits;
  }
  if (sort_cap == 4096) {
    FSA_CUDA(cudaFuncSetAttribute(k_group_union<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    k_group_union<true><<<static_cast<unsigned>(ngrp), 512, smem, s>>>(
        pat.rowptr.get(), pat.col.get(), pat.rows, G, sort_cap, cap, ucols.get(), ucount.get(), lidx.get(), key_bits,
        tile_order);
  } else {
    FSA_CUDA(cudaFuncSetAttribute(k_group_union<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    k_group_union<false><<<static_cast<unsigned>(ngrp), 512, smem, s>>>(
        pat.rowptr.get(), pat.col.get(), pat.rows, G, sort_cap, cap, ucols.get(), ucount.get(), lidx.get(), key_bits,
        tile_order);
  }
  FSA_LAUNCH_CHECK();
  bad.zero(s);
  FSA_CUDA(cudaMemsetAsync(sizes.get() + ngrp, 0, sizeof(long), s));
  k_group_ok<<<static_cast<unsigned>(cdiv(ngrp, 256)), 256, 0, s>>>(ucount.get(), ngrp, pad, bad.get(), sizes.get());
  FSA_LAUNCH_CHECK();
  int hbad = 0;
  FSA_CUDA(cudaMemcpyAsync(&hbad, bad.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
  FSA_CUDA(cudaStreamSynchronize(s));
  if (hbad) {
    lidx.release();
    return false;
  }
  gptr.alloc(ngrp + 1);
  size_t tmp_bytes = 0;
  FSA_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, sizes.get(), gptr.get(), ngrp + 1, s));
  DBuf<unsigned char> tmp(tmp_bytes);
  FSA_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), tmp_bytes, sizes.get(), gptr.get(), ngrp + 1, s));
  FSA_CUDA(cudaMemcpyAsync(&gnnz, gptr.get() + ngrp, sizeof(long), cudaMemcpyDeviceToHost, s));
  FSA_CUDA(cudaStreamSynchronize(s));
  gcol.alloc(gnnz > 0 ? gnnz : 1);
  k_group_compact<<<static_cast<unsigned>(ngrp), 128, 0, s>>>(ucols.get(), cap, ucount.get(), gptr.get(), ngrp,
                                                              gcol.get());
  FSA_LAUNCH_CHECK();
  std::vector<long> gp(static_cast<size_t>(ngrp + 1));
  FSA_CUDA(cudaMemcpyAsync(gp.data(), gptr.get(), sizeof(long) * (ngrp + 1), cudaMemcpyDeviceToHost, s));
  FSA_CUDA(cudaStreamSynchronize(s));
  long mx = 0;
  for (long g = 0; g < ngrp; ++g) mx = std::max(mx, gp[static_cast<size_t>(g + 1)] - gp[static_cast<size_t>(g)]);
  gmax = static_cast<int>(mx);
  if (std::getenv("FSA_DEBUG"))
    std::fprintf(stderr, "[fsa] row groups of %d: %ld groups, union %ld (%.1f per group, max %d), nnz %ld (%.2f x)\n",
                 G, ngrp, gnnz, static_cast<double>(gnnz) / ngrp, gmax, pat.nnz,
                 static_cast<double>(pat.nnz) / std::max<long>(gnnz, 1));
  return true;
}

// mirror[p] = position of (c, r) for p = (r, c): binary search of r in row c (warp per row)
__global__ void k_mirror(const long* __restrict__ rowptr, const int* __restrict__ col, long n,
                         long* __restrict__ mirror) {
  const long r = (static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= n) return;
  for (long p = rowptr[r] + lane; p < rowptr[r + 1]; p += 32) {
    const long c = col[p];
    long lo = rowptr[c], hi = rowptr[c + 1];
    while (lo < hi) {
      const long mid = (lo + hi) >> 1;
      if (col[mid] < r) lo = mid + 1; else hi = mid;
    }
    mirror[p] = lo;
  }
}

template <int D>
__global__ void k_fill(const double* rx, long rld, long rn, const double* cx, long cld,
                       const unsigned long long* ckeys, long cn, GridArgs g, double gamma, const long* rowptr,
                       int* col, double* dist, long* diagpos, int square) {
  const long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= rn) return;
  long p = rowptr[i];
  long dp = -1;
  visit_neighbours<D>(rx, rld, i, cx, cld, ckeys, cn, g, gamma, [&](long j, double dd) {
    col[p] = static_cast<int>(j);
    if (square && j == i) {
      dp = p;
      dd = 0.0;
    }
    dist[p] = dd;
    ++p;
  });
  if (square) diagpos[i] = dp;
}

}  // namespace

CellGrid make_grid(const double* coords, long n, int d, double gamma, const double* coords2, long n2) {
  require(d >= 1 && d <= 3, "dimension must be 1, 2 or 3");
  require(gamma > 0.0, "taper range must be positive");
  CellGrid g;
  g.d = d;
  double ext = 0.0;
  for (int k = 0; k < d; ++k) {
    double lo = coords[k * n], hi = coords[k * n];
    for (long i = 1; i < n; ++i) {
      lo = std::min(lo, coords[i + k * n]);
      hi = std::max(hi, coords[i + k * n]);
    }
    for (long i = 0; coords2 && i < n2; ++i) {
      lo = std::min(lo, coords2[i + k * n2]);
      hi = std::max(hi, coords2[i + k * n2]);
    }
    g.origin[k] = lo;
    ext = std::max(ext, hi - lo);
  }
  // cells of edge >= gamma keep the 3^d neighbourhood exhaustive
  g.h = std::max(gamma, ext / static_cast<double>(kMaxCells - 2));
  return g;
}

void sort_points(const double* coords_host, long n, int d, const CellGrid& g, long n_pad, SortedPoints& out,
                 cudaStream_t s) {
  require(n > 0, "empty location set");
  out.n = n;
  out.n_pad = n_pad;
  out.d = d;
  out.grid = g;
  DBuf<double> raw(static_cast<size_t>(n * d));
  FSA_CUDA(cudaMemcpyAsync(raw.get(), coords_host, sizeof(double) * n * d, cudaMemcpyHostToDevice, s));
  DBuf<unsigned long long> keys_in(n);
  DBuf<int> idx_in(n);
  out.keys.alloc(n);
  out.perm_d.alloc(n);
  out.iperm_d.alloc(n);
  out.coords.alloc(static_cast<size_t>(d * n_pad));
  GridArgs ga{g.origin[0], g.origin[1], g.origin[2], g.h};
  const unsigned nb = static_cast<unsigned>(cdiv(n, 256));
  switch (d) {
    case 1: k_point_keys<1><<<nb, 256, 0, s>>>(raw.get(), n, ga, keys_in.get(), idx_in.get()); break;
    case 2: k_point_keys<2><<<nb, 256, 0, s>>>(raw.get(), n, ga, keys_in.get(), idx_in.get()); break;
    default: k_point_keys<3><<<nb, 256, 0, s>>>(raw.get(), n, ga, keys_in.get(), idx_in.get()); break;
  }
  FSA_LAUNCH_CHECK();
  size_t tmp_bytes = 0;
  FSA_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys_in.get(), out.keys.get(), idx_in.get(),
                                           out.perm_d.get(), static_cast<int>(n), 0, 64, s));
  DBuf<unsigned char> tmp(tmp_bytes);
  FSA_CUDA(cub::DeviceRadixSort::SortPairs(tmp.get(), tmp_bytes, keys_in.get(), out.keys.get(), idx_in.get(),
                                           out.perm_d.get(), static_cast<int>(n), 0, 64, s));
  const int sub = d == 1 ? kSubBits<1> : (d == 2 ? kSubBits<2> : kSubBits<3>);
  if (sub > 0) {  // back to the cell keys of the neighbour search
    k_cell_keys<<<nb, 256, 0, s>>>(out.keys.get(), n, sub);
    FSA_LAUNCH_CHECK();
  }
  k_gather_coords<<<static_cast<unsigned>(cdiv(n_pad, 256)), 256, 0, s>>>(raw.get(), n, d, out.perm_d.get(), n_pad,
                                                                         out.coords.get(), out.iperm_d.get());
  FSA_LAUNCH_CHECK();
  out.perm.resize(n);
  out.iperm.resize(n);
  FSA_CUDA(cudaMemcpyAsync(out.perm.data(), out.perm_d.get(), sizeof(int) * n, cudaMemcpyDeviceToHost, s));
  FSA_CUDA(cudaMemcpyAsync(out.iperm.data(), out.iperm_d.get(), sizeof(int) * n, cudaMemcpyDeviceToHost, s));
  FSA_CUDA(cudaStreamSynchronize(s));
}

void build_groups(Csr& pat, cudaStream_t s) {
  // FSA_UNION_ORDER=plain (ascending columns) | mask (row-tile-mask order) | default: mask order with
  // the k-steps interleaved across pieces
  static const int order = [] {
    const char* e = std::getenv("FSA_UNION_ORDER");
    if (e != nullptr && std::strcmp(e, "plain") == 0) return 0;
    if (e != nullptr && std::strcmp(e, "mask") == 0) return 1;
    return 2;
  }();
  if (!build_unions(pat, kGroup, 4, kUnionSort, kUnionCap, pat.ngrp, pat.gnnz, pat.gmax, pat.gptr, pat.gcol, pat.gslot,
                    s, order)) {
    pat.gnnz = 0;
    return;
  }
  k_group_slots<<<static_cast<unsigned>(cdiv(pat.rows, 256)), 256, 0, s>>>(pat.rowptr.get(), pat.rows, pat.gptr.get(),
                                                                          pat.gslot.get());
  FSA_LAUNCH_CHECK();
  DBuf<int> needmax(1);
  {  // columns the Gram blocks have to evaluate (the rest comes from mirror entries)
    pat.gneed.alloc(pat.gnnz);
    pat.gneedcnt.alloc(pat.ngrp);
    needmax.zero(s);
    k_group_need<<<static_cast<unsigned>(pat.ngrp), 32, 0, s>>>(pat.gptr.get(), pat.gcol.get(), pat.ngrp,
                                                               pat.gneed.get(), pat.gneedcnt.get(), needmax.get());
    FSA_LAUNCH_CHECK();  // (its maximum is read back with the tile count below)
  }
  {  // compact tiles of the value blocks
    pat.nkb = pat.gnnz / 4;
    pat.kmask.alloc(pat.nkb);
    pat.kmask.zero(s);
    pat.koff.alloc(pat.nkb + 1);
    k_tile_mask<<<static_cast<unsigned>(cdiv(pat.nnz, 256)), 256, 0, s>>>(pat.gslot.get(), pat.nnz, pat.kmask.get());
    FSA_LAUNCH_CHECK();
    DBuf<int> cnt(pat.nkb + 1);
    k_tile_count<<<static_cast<unsigned>(cdiv(pat.nkb + 1, 256)), 256, 0, s>>>(pat.kmask.get(), pat.nkb, cnt.get());
    FSA_LAUNCH_CHECK();
    size_t tb = 0;
    FSA_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.get(), pat.koff.get(), static_cast<int>(pat.nkb + 1), s));
    DBuf<unsigned char> tmp(tb);
    FSA_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), tb, cnt.get(), pat.koff.get(), static_cast<int>(pat.nkb + 1), s));
    int nt = 0;
    FSA_CUDA(cudaMemcpyAsync(&nt, pat.koff.get() + pat.nkb, sizeof(int), cudaMemcpyDeviceToHost, s));
    FSA_CUDA(cudaMemcpyAsync(&pat.gneedmax, needmax.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
    FSA_CUDA(cudaStreamSynchronize(s));
    pat.ntiles = nt;
    pat.pmeta.alloc(2 * std::max<long>(pat.nkb, 1));
    k_piece_meta<<<static_cast<unsigned>(cdiv(pat.nkb, 256)), 256, 0, s>>>(
        pat.kmask.get(), pat.koff.get(), pat.nkb, reinterpret_cast<int2*>(pat.pmeta.get()));
    FSA_LAUNCH_CHECK();
    if (std::getenv("FSA_DEBUG"))
      std::fprintf(stderr, "[fsa] value tiles: %ld of %ld (%.3f), %.2f entries per tile\n", pat.ntiles, pat.nkb * 4,
                   static_cast<double>(pat.ntiles) / std::max<long>(1, pat.nkb * 4),
                   static_cast<double>(pat.nnz) / std::max<long>(1, pat.ntiles));
  }
  FSA_CUDA(cudaStreamSynchronize(s));
}

void build_pattern(const SortedPoints& rows, const SortedPoints& cols, double gamma, bool force_diag, Csr& out,
                   cudaStream_t s) {
  require(rows.d == cols.d, "location sets must share the dimension");
  const int d = rows.d;
  const CellGrid& g = cols.grid;
  GridArgs ga{g.origin[0], g.origin[1], g.origin[2], g.h};
  out.rows = rows.n;
  out.cols = cols.n;
  DBuf<long> counts(rows.n + 1);
  const unsigned nb = static_cast<unsigned>(cdiv(rows.n, 128));
#define FSA_PAT_ARGS rows.coords.get(), rows.n_pad, rows.n, cols.coords.get(), cols.n_pad, cols.keys.get(), cols.n, ga, gamma
  switch (d) {
    case 1: k_count<1><<<nb, 128, 0, s>>>(FSA_PAT_ARGS, counts.get()); break;
    case 2: k_count<2><<<nb, 128, 0, s>>>(FSA_PAT_ARGS, counts.get()); break;
    default: k_count<3><<<nb, 128, 0, s>>>(FSA_PAT_ARGS, counts.get()); break;
  }
  FSA_LAUNCH_CHECK();
  FSA_CUDA(cudaMemsetAsync(counts.get() + rows.n, 0, sizeof(long), s));
  out.rowptr.alloc(rows.n + 1);
  size_t tmp_bytes = 0;
  FSA_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, counts.get(), out.rowptr.get(),
                                         static_cast<int>(rows.n + 1), s));
  DBuf<unsigned char> tmp(tmp_bytes);
  FSA_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), tmp_bytes, counts.get(), out.rowptr.get(),
                                         static_cast<int>(rows.n + 1), s));
  long nnz = 0;
  FSA_CUDA(cudaMemcpyAsync(&nnz, out.rowptr.get() + rows.n, sizeof(long), cudaMemcpyDeviceToHost, s));
  FSA_CUDA(cudaStreamSynchronize(s));
  out.nnz = nnz;
  out.col.alloc(nnz > 0 ? nnz : 1);
  out.dist.alloc(nnz > 0 ? nnz : 1);
  if (force_diag) out.diagpos.alloc(rows.n);
  long* dp = force_diag ? out.diagpos.get() : nullptr;
  const int sq = force_diag ? 1 : 0;
  switch (d) {
    case 1: k_fill<1><<<nb, 128, 0, s>>>(FSA_PAT_ARGS, out.rowptr.get(), out.col.get(), out.dist.get(), dp, sq); break;
    case 2: k_fill<2><<<nb, 128, 0, s>>>(FSA_PAT_ARGS, out.rowptr.get(), out.col.get(), out.dist.get(), dp, sq); break;
    default: k_fill<3><<<nb, 128, 0, s>>>(FSA_PAT_ARGS, out.rowptr.get(), out.col.get(), out.dist.get(), dp, sq); break;
  }
#undef FSA_PAT_ARGS
  FSA_LAUNCH_CHECK();
  if (force_diag && nnz > 0) {  // transposed positions: the pattern is symmetric
    out.mirror.alloc(nnz);
    k_mirror<<<static_cast<unsigned>(cdiv(rows.n * 32, 256)), 256, 0, s>>>(out.rowptr.get(), out.col.get(), rows.n,
                                                                           out.mirror.get());
    FSA_LAUNCH_CHECK();
  }
}

}  // namespace fsa
