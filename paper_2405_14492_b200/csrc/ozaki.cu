// INT8 tensor-core (tcgen05) emulation of the fp64 skinny GEMMs; see ozaki.cuh.
#include <algorithm>
#include <cstdlib>

#include "bulk.cuh"
#include "dgemm.cuh"
#include "ozaki.cuh"

namespace fsa {
namespace {

constexpr int kStages = 4;  // (a fifth 42 KB stage measured no faster)
constexpr int kKb = 32;                            // K bytes per stage = one kind::i8 MMA
constexpr int kATile = kOzSlices * 128 * kKb;      // 28 KB: 7 planes x 128 rows x 32 K
constexpr int kBTile = kOzSlices * kOzCols * kKb;  // 14 KB: 7 planes x 64 cols x 32 K
constexpr int kSmem = kStages * (kATile + kBTile);
constexpr long kMaxChunk = 16384;  // int32 exactness: <= 7 pairs x K x 128^2 < 2^31

// ---- PTX wrappers ---------------------------------------------------------------------------
// (no L2 prefetch ahead of the bulk copies: measured slower, it competes with the copies)

// UMMA shared-memory descriptor, K-major, no swizzle: core matrices of 8 rows x 16 B,
// lbo = byte stride between the two 16-B K halves, sbo = byte stride between 8-row groups
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // descriptor version (sm_100)
  return d;                             // base offset 0, layout SWIZZLE_NONE
}
// instruction descriptor: s8 x s8 -> s32, both K-major
__device__ __forceinline__ uint32_t idesc_i8(int M, int N) {
  return (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
// 16 columns [col0, col0 + 16) of this lane's row: 2^4 sum_{d=2..9} 2^{-8d} C_d with the eight int32
// accumulators combined exactly in three int64 groups (|g| < 2^53: exact conversions)
__device__ __forceinline__ double recombine8(uint32_t c2, uint32_t c3, uint32_t c4, uint32_t c5, uint32_t c6,
                                             uint32_t c7, uint32_t c8, uint32_t c9) {
  const long long g1 = (static_cast<long long>(static_cast<int>(c2)) << 16) +
                       (static_cast<long long>(static_cast<int>(c3)) << 8) + static_cast<int>(c4);
  const long long g2 = (static_cast<long long>(static_cast<int>(c5)) << 16) +
                       (static_cast<long long>(static_cast<int>(c6)) << 8) + static_cast<int>(c7);
  const long long g3 = (static_cast<long long>(static_cast<int>(c8)) << 8) + static_cast<int>(c9);
  return fma(static_cast<double>(g1), 0x1p-28, fma(static_cast<double>(g2), 0x1p-52, static_cast<double>(g3) * 0x1p-68));
}
template <int NW = kOzWeights>  // NW = 8: weights 2..9; NW = 7: weights 2..8 (weight 9 not accumulated)
__device__ __forceinline__ void drain16(uint32_t trow, int col0, double (&out)[16], int wstride = kOzCols) {
  uint32_t v[NW][16];
#pragma unroll
  for (int dd = 0; dd < NW; ++dd) tmem_ld16_nowait(trow + static_cast<uint32_t>(dd * wstride + col0), v[dd]);
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int c = 0; c < 16; ++c)
    out[c] = recombine8(v[0][c], v[1][c], v[2][c], v[3][c], v[4][c], v[5][c], v[6][c], NW == 8 ? v[NW - 1][c] : 0u);
}

__device__ __forceinline__ void tmem_ld8_nowait(uint32_t taddr, uint32_t (&v)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
               : "r"(taddr));
}
// drain16 for 8 columns (half the registers)
template <int NW = kOzWeights>
__device__ __forceinline__ void drain8(uint32_t trow, int col0, double (&out)[8], int wstride = kOzCols) {
  uint32_t v[NW][8];
#pragma unroll
  for (int dd = 0; dd < NW; ++dd) tmem_ld8_nowait(trow + static_cast<uint32_t>(dd * wstride + col0), v[dd]);
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int c = 0; c < 8; ++c)
    out[c] = recombine8(v[0][c], v[1][c], v[2][c], v[3][c], v[4][c], v[5][c], v[6][c], NW == 8 ? v[NW - 1][c] : 0u);
}

// exponent e with |x| < 2^e for all x of a group whose max magnitude is mx (0 -> 0)
__device__ __forceinline__ int group_exp(double mx) {
  int e = 0;
  if (mx > 0.0) frexp(mx, &e);
  return e;
}
// exact 2^k (normal range; ldexp outside it)
__device__ __forceinline__ double pow2(int k) {
  return (k > -1023 && k < 1024) ? __hiloint2double((k + 1023) << 20, 0) : ldexp(1.0, k);
}
// 16 values -> 7 balanced base-256 digit planes of 16 signed bytes each (ozaki.cuh): X = trunc(x
// 2^{54-e}) is exact for the group maximum (|x| < 2^e, 53-bit mantissa) and |X| < 2^54. The balanced
// digits d_a in [-128, 127] with X = sum_a d_a 256^a are all read off at once: X + sum_a 128 256^a
// has the ordinary base-256 digits d_a + 128 (the add carries exactly as peeling the signed low byte
// and (X + 128) >> 8 does), and byte ^ 0x80 is d_a as a signed byte. Plane a - 1 holds digit a (weight
// 2^{-8a}), i.e. byte 7 - a of the biased word; the bytes of four values are transposed into plane
// words with byte permutes.
__device__ __forceinline__ void digits16(const double (&v)[16], int e, int4 (&out)[kOzSlices]) {
  static_assert(kOzSlices == 7, "digit planes: 7 bytes of the biased 64-bit word");
  const double sc = pow2(54 - e);
  uint32_t w[kOzSlices][4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint32_t lo[4], hi[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const unsigned long long bias = 0x0080808080808080ULL;
      const unsigned long long Y = (static_cast<unsigned long long>(__double2ll_rz(v[4 * j + q] * sc)) + bias) ^ bias;
      lo[q] = static_cast<uint32_t>(Y);
      hi[q] = static_cast<uint32_t>(Y >> 32);
    }
    // 4 x 4 byte transposes: bytes 0..3 (lo) are digits 7..4, bytes 4..6 (hi) digits 3..1
    const uint32_t t0 = __byte_perm(lo[0], lo[1], 0x5140), t1 = __byte_perm(lo[2], lo[3], 0x5140);
    const uint32_t t2 = __byte_perm(lo[0], lo[1], 0x7362), t3 = __byte_perm(lo[2], lo[3], 0x7362);
    w[6][j] = __byte_perm(t0, t1, 0x5410);
    w[5][j] = __byte_perm(t0, t1, 0x7632);
    w[4][j] = __byte_perm(t2, t3, 0x5410);
    w[3][j] = __byte_perm(t2, t3, 0x7632);
    const uint32_t h0 = __byte_perm(hi[0], hi[1], 0x5140), h1 = __byte_perm(hi[2], hi[3], 0x5140);
    const uint32_t h2 = __byte_perm(hi[0], hi[1], 0x7362), h3 = __byte_perm(hi[2], hi[3], 0x7362);
    w[2][j] = __byte_perm(h0, h1, 0x5410);
    w[1][j] = __byte_perm(h0, h1, 0x7632);
    w[0][j] = __byte_perm(h2, h3, 0x5410);
  }
#pragma unroll
  for (int a = 0; a < kOzSlices; ++a)
    out[a] = make_int4(static_cast<int>(w[a][0]), static_cast<int>(w[a][1]), static_cast<int>(w[a][2]),
                       static_cast<int>(w[a][3]));
}

// One K step of plane-pair MMAs into the weight accumulators (weights a + b <= MAXW of the 7 x 7
// digit planes). MAXW = 9: 34 products in 12 instructions of N <= 4 NC; MAXW = 8 (the projection):
// 28 products in 10 instructions. `first` (the first K step of an accumulation) overwrites
// instead of accumulating: weights 2..8 are first written by a = 1; with MAXW = 9, weight 9 by
// (a = 2, b = 7), which shares its instruction with weights 7 and 8 and is split off.
template <int MAXW = kOzMaxW>
__device__ __forceinline__ void ozaki_kstep(uint32_t tmem, uint32_t a0, uint32_t b0, int NC, bool first) {
#pragma unroll
  for (int a = 1; a <= kOzSlices; ++a) {
    const int bmax = min(kOzSlices, MAXW - a);
    const uint64_t ad = umma_desc(a0 + (a - 1) * 4096, 2048, 128);
#pragma unroll
    for (int bs = 1; bs <= bmax; bs += 4) {
      const int nb = min(4, bmax - bs + 1);
      const uint32_t td = tmem + static_cast<uint32_t>((a + bs - 2) * NC);
      const uint64_t bd = umma_desc(b0 + (bs - 1) * 16 * NC, kOzSlices * 16 * NC, 128);
      if (a == 1) {
        mma_i8(td, ad, bd, idesc_i8(128, nb * NC), first ? 0u : 1u);
      } else if (MAXW == 9 && a == 2 && bs + nb - 1 == MAXW - a && first) {  // weights 7, 8 (accumulate) | 9 (new)
        mma_i8(td, ad, bd, idesc_i8(128, (nb - 1) * NC), 1u);
        mma_i8(td + static_cast<uint32_t>((nb - 1) * NC), ad,
               umma_desc(b0 + (bs + nb - 2) * 16 * NC, kOzSlices * 16 * NC, 128), idesc_i8(128, NC), 0u);
      } else {
        mma_i8(td, ad, bd, idesc_i8(128, nb * NC), 1u);
      }
    }
  }
}

// ---- the GEMM ---------------------------------------------------------------------------------
// CTA (blockIdx.x = 128-row tile of A, blockIdx.y = K chunk). A planes: [tile][kb][plane][kc][rg][8][16],
// B planes: [kb][kc][plane * 8 + col / 8][col % 8][16]. All MMAs of a stage are issued by one thread
// into 8 TMEM accumulators (weights d = 2..9), 4-stage bulk-copy pipeline, epilogue per mode:
//   0: project partials   part[chunk][row][c] = acc * 2^(er[chunk][row] + f[chunk][c])
//   1: expand keep        Lw, Z = Dinv (R - Lw), per-tile column partials of R.Z
//   2: expand plain       Y = acc * 2^(ec[row] + h[c])
struct OzEpi {
  int mode;
  long m_pad;   // mode 0: rows of the partial blocks
  long tp;      // real columns to write (modes 1, 2)
  long ld;      // row stride of R / Z / Lw (modes 1, 2)
  const int* erow;  // exponents of A rows: mode 0 [nchunks][m_pad], else [n_pad]
  const int* ecol;  // exponents of B columns: mode 0 [nchunks][64], else [64]
  double* part;     // mode 0 partials / mode 1 rz partials [tiles][tp]
  double* Z;
  double* Lw;       // modes 1, 2 (Y)
  const double* R;
  const double* Dinv;
  const double* A2 = nullptr;  // mode 4: second row operand
};
// expansion epilogue modes (k_oz_expand): 1 Woodbury keep, 2 plain Y = acc,
// 3 Y = R - acc (R, Y with row stride ld), 4 row dots of acc with R and A2 (row stride ld):
//   Z[i] = sum_c acc[i][c] R[i][c], Lw[i] = sum_c acc[i][c] A2[i][c]

// Two column tiles of one wider RHS block in one launch (t_pad in (64, 128], config 4's 72): the
// two CTAs of a (row tile, K chunk) -- or, in the persistent expansion, of a pair -- are adjacent
// in the launch order, run concurrently and stream the SAME A (U digit-plane) tiles, so the second
// read of each A tile comes from L2: the U planes cross HBM once per pass, where a 64-column INT8
// pass plus an 8-column fp64 DMMA remainder read 8 + 8 bytes of U per entry.
// The block is split evenly (72 = 36 + 36) and both tiles use the same B width nc (a multiple of
// 16, <= 48 here): equal MMA work, so the two CTAs of a pair run in step and the second read of
// every A tile hits L2 (a 64 + 8 split ran the short tile ahead and paid the A stream twice).
struct OzPair {
  const int8_t* B[2];
  OzEpi epi[2];
  int nc = kOzCols;  // B tile width of both column tiles (PAIRED)
};
template <bool PAIRED, int MAXW = kOzProjMaxW>
__global__ void __launch_bounds__(128, 1)
    k_oz_gemm(const int8_t* __restrict__ A, OzPair pr, int nkb_all, int kb_per_chunk) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages], done;
  __shared__ uint32_t tmem_base_s;
  const int ct = PAIRED ? blockIdx.x : 0;
  const int tile = PAIRED ? blockIdx.y : blockIdx.x, chunk = PAIRED ? blockIdx.z : blockIdx.y;
  const int8_t* __restrict__ B = pr.B[ct];
  const OzEpi& epi = pr.epi[ct];
  // B tile width NC: 64, or the pair's nc (layout of k_oz_planes_*: plane stride 16 NC bytes,
  // K-half stride 128 NC bytes; one accumulator weight per NC TMEM columns)
  const int NC = PAIRED ? pr.nc : kOzCols;
  const uint32_t btile = static_cast<uint32_t>(kOzSlices * kKb * NC);
  const int kb0 = chunk * kb_per_chunk;
  const int nk = min(nkb_all - kb0, kb_per_chunk);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint8_t* sA = smem;
  uint8_t* sB = smem + kStages * kATile;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(&done, 1);
    mbar_init_fence();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_s;
  pdl_wait();  // (TMEM allocation and barrier setup overlap the predecessor)

  // warp-specialised issue: lane 0 of warp 1 streams the stages (waiting only for a stage to be
  // released), lane 0 of warp 0 issues the MMAs (waiting only for a stage to land) -- the loads no
  // longer queue behind the MMA thread's waits
  if (tid == 32) {
    const int8_t* Ablk = A + (static_cast<long>(tile) * nkb_all + kb0) * kATile;
    const int8_t* Bblk = B + static_cast<long>(kb0) * btile;
    const uint64_t pol_a = l2_evict_first();  // the U digit planes pass through L2 once (bulk.cuh)
    for (int j = 0; j < nk; ++j) {
      const int st = j % kStages;
      if (j >= kStages) mbar_wait(&empty[st], ((j / kStages) - 1) & 1);
      mbar_expect_tx(&full[st], kATile + btile);
      bulk_g2s_hint(sA + st * kATile, Ablk + static_cast<long>(j) * kATile, kATile, &full[st], pol_a);
      bulk_g2s(sB + st * kBTile, Bblk + static_cast<long>(j) * btile, btile, &full[st]);
    }
  }
  if (tid == 0) {
    for (int j = 0; j < nk; ++j) {
      const int st = j % kStages;
      mbar_wait(&full[st], (j / kStages) & 1);
      tc_fence_after();
      const uint32_t a0 = smem_u32(sA + st * kATile), b0 = smem_u32(sB + st * kBTile);
      ozaki_kstep<MAXW>(tmem, a0, b0, NC, j == 0);
      mma_commit(&empty[st]);
    }
    mma_commit(&done);
  }
  __syncwarp();
  mbar_wait(&done, 0);
  tc_fence_after();

  // ---- epilogue: warp w owns TMEM lanes [32 w, 32 w + 32) = rows of the tile ----
  const int row = warp * 32 + lane;
  const uint32_t trow = tmem + (static_cast<uint32_t>(warp * 32) << 16);
  // modes 1, 2: [128][kLd] tiles of Lw and R.Z in the (now idle) pipeline buffers
  constexpr int kLd = kOzCols + 1;
  double* lws = reinterpret_cast<double*>(smem);
  double* rzs = lws + 128 * kLd;
  for (int hh = 0; hh < 2; ++hh) {
    if (hh * 32 >= NC) break;  // (NC = 16 or 48: the last half is partial)
    double acc[32];
    {
      double y0[16], y1[16];
      drain16<MAXW - 1>(trow, hh * 32, y0, NC);
      if (hh * 32 + 16 < NC) {
        drain16<MAXW - 1>(trow, hh * 32 + 16, y1, NC);
      } else {
#pragma unroll
        for (int c = 0; c < 16; ++c) y1[c] = 0.0;
      }
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        acc[c] = y0[c];
        acc[16 + c] = y1[c];
      }
    }
    if (epi.mode == 0) {
      const long r = static_cast<long>(tile) * 128 + row;
      const int er = epi.erow[static_cast<long>(chunk) * epi.m_pad + r];
      double* out = epi.part + (static_cast<long>(chunk) * epi.m_pad + r) * kOzCols + hh * 32;
      const int* fc = epi.ecol + static_cast<long>(chunk) * kOzCols + hh * 32;
#pragma unroll
      for (int c = 0; c < 32; c += 2)
        if (hh * 32 + c < NC)
          *reinterpret_cast<double2*>(out + c) = make_double2(acc[c] * pow2(er + fc[c]), acc[c + 1] * pow2(er + fc[c + 1]));
    } else {  // modes 1, 2: Lw (and Z) through shared memory, coalesced row copies
      const long i = static_cast<long>(tile) * 128 + row;
      const double sci = pow2(epi.erow[i]);
      const int* hc = epi.ecol + hh * 32;
#pragma unroll
      for (int c = 0; c < 32; ++c) lws[row * kLd + hh * 32 + c] = acc[c] * sci * pow2(hc[c]);
    }
  }
  if (epi.mode != 0) {
    const long r0 = static_cast<long>(tile) * 128;
    const long tp = epi.tp;
    __syncthreads();
    if (epi.mode == 2) {
      for (long idx = tid; idx < 128 * tp; idx += 128) {
        const long rr = idx / tp, c = idx - rr * tp;
        epi.Lw[(r0 + rr) * epi.ld + c] = lws[rr * kLd + c];
      }
    } else {
      // R tile in, Z = Dinv (R - Lw) and Lw out, row-major tiles are contiguous in HBM
      for (long idx = tid; idx < 128 * tp; idx += 128) {
        const long rr = idx / tp, c = idx - rr * tp;
        const double x = epi.R[(r0 + rr) * epi.ld + c];
        const double lw = lws[rr * kLd + c];
        const double z = (x - lw) * epi.Dinv[r0 + rr];
        epi.Lw[(r0 + rr) * epi.ld + c] = lw;
        epi.Z[(r0 + rr) * epi.ld + c] = z;
        rzs[rr * kLd + c] = x * z;
      }
      __syncthreads();
      if (tid < tp) {  // fixed-order column sums of R.Z over the tile's rows
        double sacc = 0.0;
        for (int rr = 0; rr < 128; ++rr) sacc += rzs[rr * kLd + tid];
        epi.part[static_cast<long>(tile) * tp + tid] = sacc;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// Persistent, warp-specialized expansion Y = U^T W (+ Woodbury epilogue): one CTA per SM loops
// over 128-point tiles; warp 0 streams A/B stages (bulk copies), warp 1 issues the MMAs, warps
// 2-5 drain TMEM (one lane quadrant each) and write the outputs. The producer runs ahead across
// tile boundaries and the next tile's MMAs start as soon as TMEM is drained, so loads and the
// output writes of tile t overlap the MMAs of tile t + 1.
constexpr int kXStages = 3;
constexpr int kXLd = kOzCols + 1;  // odd stride: conflict-free row-per-lane access
constexpr int kXSmem = kXStages * (kATile + kBTile) + 128 * kXLd * 8;
constexpr int kXEpi = 512;  // epilogue threads: four warps per TMEM lane quadrant, 16 columns each
// the sweep's Woodbury pass (mode 1, <= 56 columns): a 57-double staging stride leaves room for a
// fourth pipeline stage (4 x 42 KB + 57 KB)
constexpr int kXStages4 = 4, kXLd56 = 57;
constexpr int kXSmem4 = kXStages4 * (kATile + kBTile) + 128 * kXLd56 * 8;
// MULTI (the wide passes, modes 3 and 4): ncolt 64-column tiles of W per point tile, innermost, so the
// tile's U digit planes cross HBM once and are re-streamed from L2 for the other column tiles (148
// CTAs x 458 KB of planes stay resident); column tile j uses the W planes B + j * bstride, exponents
// ecol + 64 j, columns 64 j ... of R / Y / A2 and, in mode 4, the partial rows Z / Lw + j * zstride.
template <bool PAIRED, int STAGES = kXStages, int LDY = kXLd, int MAXW = kOzMaxW, bool MULTI = false>
__global__ void __launch_bounds__(64 + kXEpi, 1)
    k_oz_expand(const int8_t* __restrict__ A, OzPair pr, int tiles, int mkb, int ncolt_arg, long bstride,
                long zstride) {
  constexpr int kStages = STAGES;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[kStages], empty[kStages], tfull, tempty;
  __shared__ uint32_t tmem_base_s;
  // PAIRED: CTAs 2j and 2j + 1 process the same point tiles j, j + G/2, ... for column tiles 0 / 1
  const int ct = PAIRED ? (blockIdx.x & 1) : 0;
  const int t_first = PAIRED ? (blockIdx.x >> 1) : blockIdx.x;
  const int t_step = PAIRED ? (gridDim.x >> 1) : gridDim.x;
  const int8_t* __restrict__ B = pr.B[ct];
  const OzEpi& epi = pr.epi[ct];
  const int NC = PAIRED ? pr.nc : kOzCols;  // B tile width (see k_oz_gemm)
  const uint32_t btile = static_cast<uint32_t>(kOzSlices * kKb * NC);
  const int ncolt = MULTI ? ncolt_arg : 1;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint8_t* sA = smem;
  uint8_t* sB = smem + kStages * kATile;
  double* tileY = reinterpret_cast<double*>(smem + kStages * (kATile + kBTile));  // [128][LDY]
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 32) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(&tfull, 1);
    mbar_init(&tempty, kXEpi / 32);
    mbar_init_fence();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base_s;
  pdl_wait();

  if (warp == 0) {
    if (lane == 0) {  // producer
      long g = 0;
      for (int t = t_first; t < tiles; t += t_step) {
        const int8_t* At = A + static_cast<long>(t) * mkb * kATile;
        for (int j = 0; j < ncolt; ++j) {
          const int8_t* Bj = B + j * bstride;
          for (int kb = 0; kb < mkb; ++kb, ++g) {
            const int st = static_cast<int>(g % kStages);
            if (g >= kStages) mbar_wait(&empty[st], static_cast<uint32_t>((g / kStages - 1) & 1));
            mbar_expect_tx(&full[st], kATile + btile);
            bulk_g2s(sA + st * kATile, At + static_cast<long>(kb) * kATile, kATile, &full[st]);
            bulk_g2s(sB + st * kBTile, Bj + static_cast<long>(kb) * btile, btile, &full[st]);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      long g = 0;
      int lt = 0;
      for (int t = t_first; t < tiles; t += t_step) {
        for (int j = 0; j < ncolt; ++j, ++lt) {
          if (lt > 0) {
            mbar_wait(&tempty, static_cast<uint32_t>((lt - 1) & 1));
            tc_fence_after();
          }
          for (int kb = 0; kb < mkb; ++kb, ++g) {
            const int st = static_cast<int>(g % kStages);
            mbar_wait(&full[st], static_cast<uint32_t>((g / kStages) & 1));
            tc_fence_after();
            const uint32_t a0 = smem_u32(sA + st * kATile), b0 = smem_u32(sB + st * kBTile);
            ozaki_kstep<MAXW>(tmem, a0, b0, NC, kb == 0);
            mma_commit(&empty[st]);
          }
          mma_commit(&tfull);
        }
      }
    }
    __syncwarp();
  } else {  // epilogue warps 2..17: TMEM lane quadrant q = warp % 4, column group (warp - 2) / 4
    const int q = warp & 3, gq = (warp - 2) >> 2;
    const int row = q * 32 + lane;
    const uint32_t trow = tmem + (static_cast<uint32_t>(q * 32) << 16);
    const long tp = epi.tp;
    const int et = tid - 64;  // 0 .. kXEpi - 1
    int lt = 0;
    for (int t = t_first; t < tiles; t += t_step)
    for (int j = 0; j < ncolt; ++j, ++lt) {
      const long r0 = static_cast<long>(t) * 128;
      // this column tile's operands (MULTI: see above)
      const int* e_ecol = epi.ecol + (MULTI ? j * kOzCols : 0);
      const double* e_R = epi.R + (MULTI ? j * kOzCols : 0);
      const double* e_A2 = epi.A2 + (MULTI ? j * kOzCols : 0);
      double* e_Lw = epi.Lw + (MULTI ? (epi.mode == 4 ? j * zstride : static_cast<long>(j) * kOzCols) : 0);
      double* e_Z = epi.Z + (MULTI && epi.mode == 4 ? j * zstride : 0);
      if (epi.mode == 1 || epi.mode == 3 || epi.mode == 4) {
        // pull the tile's R entries (128 rows x tp columns, row stride ld) into L2 while the MMAs
        // run, so the write-out below reads them at L2 latency
        const char* rb = reinterpret_cast<const char*>(e_R + r0 * epi.ld);
        const int lpr = static_cast<int>((tp * 8 + 127) / 128);  // 128-byte lines per row
        for (int li = et; li < 128 * lpr; li += kXEpi)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(rb + (li / lpr) * epi.ld * 8 + (li % lpr) * 128));
      }
      mbar_wait(&tfull, static_cast<uint32_t>(lt & 1));
      tc_fence_after();
      const int ei = epi.erow[r0 + row];
#pragma unroll 1
      for (int h8 = 0; h8 < 2; ++h8) {  // stage this warp's 16 columns in shared memory
        const int c0 = gq * 16 + h8 * 8;
        if (c0 >= tp || c0 >= NC) break;
        double y[8];
        drain8<MAXW - 1>(trow, c0, y, NC);
#pragma unroll
        for (int c = 0; c < 8; ++c) tileY[row * LDY + c0 + c] = y[c] * pow2(ei + e_ecol[c0 + c]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tempty)) : "memory");
      // TMEM is free for the next tile already; coalesced copies of the staged rows
      asm volatile("bar.sync 1, %0;" ::"n"(kXEpi) : "memory");
      if (epi.mode == 4) {  // one thread per row: dots of the staged row with R and A2 rows
        if (et < 128) {
          const long i = r0 + et;
          double s1 = 0.0, s2 = 0.0;
          for (int c = 0; c < tp; ++c) {
            const double yv = tileY[et * LDY + c];
            s1 = fma(yv, __ldg(e_R + i * epi.ld + c), s1);
            s2 = fma(yv, __ldg(e_A2 + i * epi.ld + c), s2);
          }
          e_Z[i] = s1;
          e_Lw[i] = s2;
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kXEpi) : "memory");  // tileY reused by the next tile
        continue;
      }
      // thread (column c, row phase h): rows h, h + 4, ..., coalesced across c; loads are
      // batched ahead of the stores (R and Dinv are read-only here)
      constexpr int kPh = kXEpi / 64;  // row phases
      const int c = et & 63, h = et >> 6;
      if (c < tp) {
        double sacc = 0.0;
        const long base = r0 * epi.ld + c;
#pragma unroll 1
        for (int rb = h; rb < 128; rb += 8 * kPh) {
          double x[8], di[8], lw[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int rr = rb + kPh * u;
            lw[u] = tileY[rr * LDY + c];
            if (epi.mode == 1) {
              x[u] = __ldg(e_R + base + static_cast<long>(rr) * epi.ld);
              di[u] = __ldg(epi.Dinv + r0 + rr);
            } else if (epi.mode == 3) {
              x[u] = __ldg(e_R + base + static_cast<long>(rr) * epi.ld);
            }
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const long off = base + static_cast<long>(rb + kPh * u) * epi.ld;
            e_Lw[off] = epi.mode == 3 ? x[u] - lw[u] : lw[u];
            if (epi.mode == 1) {
              const double z = (x[u] - lw[u]) * di[u];
              e_Z[off] = z;
              sacc = fma(x[u], z, sacc);
            }
          }
        }
        if (epi.mode == 1) tileY[h * LDY + c] = sacc;  // (row h, column c) was read only by this thread
      }
      if (epi.mode == 1) {
        asm volatile("bar.sync 1, %0;" ::"n"(kXEpi) : "memory");
        if (h == 0 && c < tp) {  // fixed order over the row phases
          double sum = tileY[c];
          for (int ph = 1; ph < kPh; ++ph) sum += tileY[ph * LDY + c];
          epi.part[static_cast<long>(t) * tp + c] = sum;
        }
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kXEpi) : "memory");  // tileY reused by the next tile
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// ---- digit planes ---------------------------------------------------------------------------------
// project A: exponent per (chunk, inducing row) over the chunk's points
__global__ void __launch_bounds__(1024) k_oz_exp_rows(const double* __restrict__ U, long mp, long n_pad,
                                                      int kb_per_chunk, int* __restrict__ er) {
  // 8 point phases x 128 rows, eight independent loads in flight per thread (max is order-free)
  __shared__ double red[1024];
  const int chunk = blockIdx.x, tile = blockIdx.y;
  const int r = threadIdx.x & 127, ph = threadIdx.x >> 7;
  const long i0 = static_cast<long>(chunk) * kb_per_chunk * kKb;
  const long i1 = min(n_pad, i0 + static_cast<long>(kb_per_chunk) * kKb);
  const double* __restrict__ p = U + tile * 128 + r;
  double mx[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) mx[u] = 0.0;
  long i = i0 + ph;
  for (; i + 56 < i1; i += 64) {
#pragma unroll
    for (int u = 0; u < 8; ++u) mx[u] = fmax(mx[u], fabs(p[(i + 8 * u) * mp]));
  }
  for (; i < i1; i += 8) mx[0] = fmax(mx[0], fabs(p[i * mp]));
#pragma unroll
  for (int u = 1; u < 8; ++u) mx[0] = fmax(mx[0], mx[u]);
  red[threadIdx.x] = mx[0];
  __syncthreads();
  if (ph == 0) {
    double m = mx[0];
#pragma unroll
    for (int q = 1; q < 8; ++q) m = fmax(m, red[q * 128 + r]);
    er[static_cast<long>(chunk) * mp + tile * 128 + r] = group_exp(m);
  }
}
__global__ void __launch_bounds__(256) k_oz_planes_rows(const double* __restrict__ U, long mp, int nkb,
                                                        int kb_per_chunk, const int* __restrict__ er,
                                                        int8_t* __restrict__ Ar) {
  __shared__ double tileU[kKb][129];
  const int kb = blockIdx.x, tile = blockIdx.y;
  for (int idx = threadIdx.x; idx < kKb * 128; idx += 256) {
    const int p = idx >> 7, r = idx & 127;
    tileU[p][r] = U[(static_cast<long>(kb) * kKb + p) * mp + tile * 128 + r];
  }
  __syncthreads();
  const int r = threadIdx.x & 127, kc = threadIdx.x >> 7;
  const int e = er[static_cast<long>(kb / kb_per_chunk) * mp + tile * 128 + r];
  double v[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) v[q] = tileU[kc * 16 + q][r];
  int4 out[kOzSlices];
  digits16(v, e, out);
  int8_t* base = Ar + (static_cast<long>(tile) * nkb + kb) * kATile + kc * 2048 + (r >> 3) * 128 + (r & 7) * 16;
#pragma unroll
  for (int a = 0; a < kOzSlices; ++a) *reinterpret_cast<int4*>(base + a * 4096) = out[a];
}
// expand A: exponent per point over the inducing rows
__global__ void k_oz_exp_points(const double* __restrict__ U, long mp, long n_pad, int* __restrict__ ec) {
  const long i = (static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= n_pad) return;
  double mx = 0.0;
  for (long r = lane; r < mp; r += 32) mx = fmax(mx, fabs(U[i * mp + r]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) ec[i] = group_exp(mx);
}
__global__ void __launch_bounds__(256) k_oz_planes_points(const double* __restrict__ U, long mp, int mkb,
                                                          const int* __restrict__ ec, int8_t* __restrict__ Ac) {
  const int kb = blockIdx.x, tile = blockIdx.y;
  const int il = threadIdx.x & 127, kc = threadIdx.x >> 7;
  const long i = static_cast<long>(tile) * 128 + il;
  const double* src = U + i * mp + kb * kKb + kc * 16;
  double v[16];
#pragma unroll
  for (int q = 0; q < 16; q += 2) {
    const double2 x = *reinterpret_cast<const double2*>(src + q);
    v[q] = x.x;
    v[q + 1] = x.y;
  }
  int4 out[kOzSlices];
  digits16(v, ec[i], out);
  int8_t* base = Ac + (static_cast<long>(tile) * mkb + kb) * kATile + kc * 2048 + (il >> 3) * 128 + (il & 7) * 16;
#pragma unroll
  for (int a = 0; a < kOzSlices; ++a) *reinterpret_cast<int4*>(base + a * 4096) = out[a];
}

// per-sweep B planes of Y = diag(scale) V (project): column max per chunk, then digits
__global__ void __launch_bounds__(256) k_oz_ymax(const double* __restrict__ V, long ld, long tp,
                                                 const double* __restrict__ scale,
                                                 long n_pad, int kb_per_chunk, int parts,
                                                 unsigned long long* __restrict__ ymax) {
  __shared__ double red[256];
  pdl_wait();
  const int chunk = blockIdx.x, part = blockIdx.y;
  const int c = threadIdx.x & 63, ph = threadIdx.x >> 6;
  const long i0 = static_cast<long>(chunk) * kb_per_chunk * kKb;
  const long i1 = min(n_pad, i0 + static_cast<long>(kb_per_chunk) * kKb);
  const long len = i1 - i0, per = (len + parts - 1) / parts;
  const long a0 = i0 + part * per, a1 = min(i1, a0 + per);
  double mx = 0.0;
  if (c < tp)
    for (long i = a0 + ph; i < a1; i += 4) mx = fmax(mx, fabs(scale ? V[i * ld + c] * scale[i] : V[i * ld + c]));
  red[threadIdx.x] = mx;
  __syncthreads();
  if (ph == 0) {
    mx = fmax(fmax(mx, red[threadIdx.x + 64]), fmax(red[threadIdx.x + 128], red[threadIdx.x + 192]));
    if (mx > 0.0) atomicMax(ymax + static_cast<long>(chunk) * kOzCols + c, static_cast<unsigned long long>(__double_as_longlong(mx)));
  }
}
// B planes in the layout [kb][kc][plane * nc / 8 + col / 8][col % 8][16] of an nc-column tile
// (nc = 64, or 16 for the narrow second tile of a pair)
__global__ void __launch_bounds__(128, 11) k_oz_planes_y(const double* __restrict__ V, long ld, long tp,
                                                     const double* __restrict__ scale, int kb_per_chunk,
                                                     const unsigned long long* __restrict__ ymax,
                                                     int* __restrict__ f, int8_t* __restrict__ Ys, int nc = kOzCols) {
  pdl_wait();
  const int kb = blockIdx.x;
  const int c = threadIdx.x & 63, kc = threadIdx.x >> 6;
  if (c >= nc) return;
  const int chunk = kb / kb_per_chunk;
  const int e = group_exp(__longlong_as_double(static_cast<long long>(ymax[static_cast<long>(chunk) * kOzCols + c])));
  if (kb % kb_per_chunk == 0 && kc == 0) f[static_cast<long>(chunk) * kOzCols + c] = e;
  double v[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const long i = static_cast<long>(kb) * kKb + kc * 16 + q;
    v[q] = c < tp ? (scale ? V[i * ld + c] * scale[i] : V[i * ld + c]) : 0.0;
  }
  int4 out[kOzSlices];
  digits16(v, e, out);
  int8_t* base = Ys + static_cast<long>(kb) * (kOzSlices * kKb * nc) + kc * (kOzSlices * 16 * nc) + c * 16;
  const uint64_t pol_last = l2_evict_last();  // read next by the projection's row-tile CTAs (bulk.cuh)
#pragma unroll
  for (int b = 0; b < kOzSlices; ++b) st_l2(reinterpret_cast<int4*>(base + b * (16 * nc)), out[b], pol_last);
}
// per-sweep B planes of W (expand): column exponents over all rows, then digits
__global__ void __launch_bounds__(1024) k_oz_wexp(const double* __restrict__ W, long ld, long tp, long mp,
                                                  int* __restrict__ h) {
  __shared__ double red[1024];
  pdl_wait();
  const int c = threadIdx.x & 63, ph = threadIdx.x >> 6;  // 16 row phases
  double mx = 0.0;
  if (c < tp)
    for (long r = ph; r < mp; r += 16) mx = fmax(mx, fabs(W[r * ld + c]));
  red[threadIdx.x] = mx;
  __syncthreads();
  if (ph == 0) {
    for (int q = 1; q < 16; ++q) mx = fmax(mx, red[q * 64 + c]);
    h[c] = group_exp(mx);
  }
}
__global__ void __launch_bounds__(128) k_oz_planes_w(const double* __restrict__ W, long ld, long tp,
                                                     int* __restrict__ h, int8_t* __restrict__ Ws,
                                                     const unsigned long long* __restrict__ wmax, int nc = kOzCols) {
  pdl_wait();
  const int kb = blockIdx.x;
  const int c = threadIdx.x & 63, kc = threadIdx.x >> 6;
  if (c >= nc) return;
  int e;
  if (wmax != nullptr) {  // column maxima left by the producer of W (core_apply)
    e = c < tp ? group_exp(__longlong_as_double(static_cast<long long>(wmax[c]))) : 0;
    if (kb == 0 && kc == 0) h[c] = e;
  } else {
    e = h[c];
  }
  double v[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) v[q] = c < tp ? W[(static_cast<long>(kb) * kKb + kc * 16 + q) * ld + c] : 0.0;
  int4 out[kOzSlices];
  digits16(v, e, out);
  int8_t* base = Ws + static_cast<long>(kb) * (kOzSlices * kKb * nc) + kc * (kOzSlices * 16 * nc) + c * 16;
#pragma unroll
  for (int b = 0; b < kOzSlices; ++b) *reinterpret_cast<int4*>(base + b * (16 * nc)) = out[b];
}
// S[r][c] = sum_chunk part[chunk][r][c] in a fixed order: four lanes per entry each add a
// contiguous quarter of the chunks (all its loads in flight), then the quarters in order
__global__ void k_oz_reduce(const double* __restrict__ part, int nchunks, long mp, long ld, long tp,
                            double* __restrict__ S) {
  pdl_wait();
  const long idx = (static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 2;
  const int qp = threadIdx.x & 3;
  const bool ok = idx < mp * tp;
  const long r = ok ? idx / tp : 0, c = ok ? idx % tp : 0;
  const int per = (nchunks + 3) / 4, q0 = qp * per, q1 = min(nchunks, q0 + per);
  double sacc = 0.0;
  if (ok) {
#pragma unroll 16
    for (int q = q0; q < q1; ++q) sacc += part[(static_cast<long>(q) * mp + r) * kOzCols + c];
  }
  const double s1 = __shfl_down_sync(0xffffffffu, sacc, 1), s2 = __shfl_down_sync(0xffffffffu, sacc, 2),
               s3 = __shfl_down_sync(0xffffffffu, sacc, 3);
  if (ok && qp == 0) S[r * ld + c] = ((sacc + s1) + s2) + s3;
}

// projection weights: 2..8 (kOzProjMaxW); FSA_OZ_PROJ_W9=1 keeps weight 9 too (A/B switch)
static bool proj_w9() {
  static const bool w9 = [] {
    const char* e = std::getenv("FSA_OZ_PROJ_W9");
    return e != nullptr && e[0] == '1';
  }();
  return w9;
}
template <bool PAIRED, int MAXW>
void launch_gemm_t(const int8_t* A, const OzPair& pr, dim3 grid, int nkb_all, int kb_per_chunk, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    FSA_CUDA(cudaFuncSetAttribute(k_oz_gemm<PAIRED, MAXW>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    attr = true;
  }
  launch_pdl(k_oz_gemm<PAIRED, MAXW>, grid, dim3(128), kSmem, s, A, pr, nkb_all, kb_per_chunk);
  FSA_LAUNCH_CHECK();
}
void launch_gemm(const int8_t* A, const int8_t* B, int tiles, int chunks, int nkb_all, int kb_per_chunk,
                 const OzEpi& epi, cudaStream_t s) {
  OzPair pr{{B, B}, {epi, epi}};
  if (proj_w9()) launch_gemm_t<false, 9>(A, pr, dim3(tiles, chunks), nkb_all, kb_per_chunk, s);
  else launch_gemm_t<false, kOzProjMaxW>(A, pr, dim3(tiles, chunks), nkb_all, kb_per_chunk, s);
}
void launch_gemm_pair(const int8_t* A, const OzPair& pr, int tiles, int chunks, int nkb_all, int kb_per_chunk,
                      cudaStream_t s) {
  if (proj_w9()) launch_gemm_t<true, 9>(A, pr, dim3(2, tiles, chunks), nkb_all, kb_per_chunk, s);
  else launch_gemm_t<true, kOzProjMaxW>(A, pr, dim3(2, tiles, chunks), nkb_all, kb_per_chunk, s);
}

// q[i] = sum_j qp[j][i], f likewise (fixed order)
__global__ void k_sum_tiles(const double* __restrict__ qp, const double* __restrict__ fp, long tiles, long n,
                            double* __restrict__ q, double* __restrict__ f) {
  const long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double a = 0.0, b = 0.0;
  for (long j = 0; j < tiles; ++j) {
    a += qp[j * n + i];
    b += fp[j * n + i];
  }
  q[i] = a;
  f[i] = b;
}

template <bool PAIRED, int STAGES, int LDY, int MAXW, bool MULTI = false>
void launch_expand_t(const int8_t* A, const OzPair& pr, int grid, int smem, int tiles, int mkb, cudaStream_t s,
                     int ncolt = 1, long bstride = 0, long zstride = 0) {
  static bool attr = false;
  if (!attr) {
    FSA_CUDA(cudaFuncSetAttribute(k_oz_expand<PAIRED, STAGES, LDY, MAXW, MULTI>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  launch_pdl(k_oz_expand<PAIRED, STAGES, LDY, MAXW, MULTI>, dim3(grid), dim3(64 + kXEpi), smem, s, A, pr, tiles, mkb,
             ncolt, bstride, zstride);
  FSA_LAUNCH_CHECK();
}
void launch_expand(const OzakiPlan& p, const OzEpi& epi, cudaStream_t s, const int8_t* Ws = nullptr) {
  const int grid = std::min(p.ptiles, kNumSMs);
  const int8_t* B = Ws != nullptr ? Ws : p.Ws.get();
  const int8_t* A = p.Ac.get();
  OzPair pr{{B, B}, {epi, epi}};
  // (weight 9 kept: dropping it -- 28 products -- measured 7 us faster per pass at config 2 and
  // 13 % at config 4, but breaks the normwise fp64-class bound, 1.11x of it in tests/test_gpu_ozaki.py)
  if (epi.mode == 1 && epi.tp <= kXLd56 - 1)
    launch_expand_t<false, kXStages4, kXLd56, kOzMaxW>(A, pr, grid, kXSmem4, p.ptiles, p.mkb, s);
  else
    launch_expand_t<false, kXStages, kXLd, kOzMaxW>(A, pr, grid, kXSmem, p.ptiles, p.mkb, s);
}
void launch_expand_pair(const OzakiPlan& p, const OzPair& pr, cudaStream_t s) {
  const int grid = 2 * std::min(p.ptiles, kNumSMs / 2);
  launch_expand_t<true, kXStages, kXLd, kOzMaxW>(p.Ac.get(), pr, grid, kXSmem, p.ptiles, p.mkb, s);
}

// digit planes of diag(scale) V (columns [0, tp) of a row-stride-ld block) for the projection
void slice_y(OzakiPlan& p, const double* V, long ld, long tp, const double* scale, unsigned long long* ymax, int* f,
             int8_t* Ys, cudaStream_t s, bool ymax_ready, int nc = kOzCols) {
  if (!ymax_ready) {
    FSA_CUDA(cudaMemsetAsync(ymax, 0, sizeof(unsigned long long) * p.nchunks * kOzCols, s));
    launch_pdl(k_oz_ymax, dim3(p.nchunks, 16), dim3(256), 0, s, V, ld, tp, scale, p.n_pad, p.kb_per_chunk, 16, ymax);
    FSA_LAUNCH_CHECK();
  }
  launch_pdl(k_oz_planes_y, dim3(p.nkb), dim3(128), 0, s, V, ld, tp, scale, p.kb_per_chunk,
             static_cast<const unsigned long long*>(ymax), f, Ys, nc);
  FSA_LAUNCH_CHECK();
}
void project_impl(OzakiPlan& p, const double* V, long ld, long tp, const double* scale, double* S, cudaStream_t s,
                  bool ymax_ready) {
  require(p.ready && tp <= kOzCols && tp <= ld, "ozaki: plan not prepared or too many columns");
  slice_y(p, V, ld, tp, scale, p.ymax.get(), p.f.get(), p.Ys.get(), s, ymax_ready);
  OzEpi epi{0, p.m_pad, tp, ld, p.er.get(), p.f.get(), p.part.get(), nullptr, nullptr, nullptr, nullptr};
  launch_gemm(p.Ar.get(), p.Ys.get(), p.mtiles, p.nchunks, p.nkb, p.kb_per_chunk, epi, s);
  launch_pdl(k_oz_reduce, dim3(static_cast<unsigned>(cdiv(4 * p.m_pad * tp, 256))), dim3(256), 0, s, p.part.get(),
             p.nchunks, p.m_pad, ld, tp, S);
  FSA_LAUNCH_CHECK();
}

void slice_w_to(OzakiPlan& p, const double* W, long ld, long tp, int8_t* Ws, int* h, cudaStream_t s,
                const unsigned long long* wmax = nullptr, int nc = kOzCols) {
  require(p.ready && tp <= kOzCols && tp <= ld, "ozaki: plan not prepared or too many columns");
  if (wmax == nullptr) {
    launch_pdl(k_oz_wexp, dim3(1), dim3(1024), 0, s, W, ld, tp, p.m_pad, h);
    FSA_LAUNCH_CHECK();
  }
  launch_pdl(k_oz_planes_w, dim3(p.mkb), dim3(128), 0, s, W, ld, tp, h, Ws, wmax, nc);
  FSA_LAUNCH_CHECK();
}
void slice_w(OzakiPlan& p, const double* W, long ld, long tp, cudaStream_t s) {
  slice_w_to(p, W, ld, tp, p.Ws.get(), p.h.get(), s);
}

}  // namespace

void ozaki_prepare(OzakiPlan& p, const double* U, long m_pad, long n_pad, cudaStream_t s) {
  require(m_pad % 128 == 0 && n_pad % 128 == 0, "ozaki: padded sizes must be multiples of 128");
  p.m_pad = m_pad;
  p.n_pad = n_pad;
  p.mtiles = static_cast<int>(m_pad / 128);
  p.ptiles = static_cast<int>(n_pad / 128);
  p.nkb = static_cast<int>(n_pad / kKb);
  p.mkb = static_cast<int>(m_pad / kKb);
  // split-K chunks: whole waves of CTAs (one per SM), chunk <= kMaxChunk points
  for (int waves = 1;; ++waves) {
    const int chunks = std::max(1, kNumSMs * waves / p.mtiles);
    const int kbpc = static_cast<int>(cdiv(p.nkb, chunks));
    if (static_cast<long>(kbpc) * kKb <= kMaxChunk) {
      p.kb_per_chunk = kbpc;
      p.nchunks = static_cast<int>(cdiv(p.nkb, kbpc));
      break;
    }
  }
  p.U = U;
  p.Ar.alloc(static_cast<size_t>(m_pad * n_pad * kOzSlices));
  p.Ac.alloc(static_cast<size_t>(m_pad * n_pad * kOzSlices));
  p.er.alloc(static_cast<size_t>(p.nchunks * m_pad));
  p.ec.alloc(static_cast<size_t>(n_pad));
  p.Ys.alloc(static_cast<size_t>(p.nkb) * kBTile);
  p.Ws.alloc(static_cast<size_t>(p.mkb) * kBTile);
  p.ymax.alloc(static_cast<size_t>(p.nchunks * kOzCols));
  p.f.alloc(static_cast<size_t>(p.nchunks * kOzCols));
  p.h.alloc(kOzCols);
  p.part.alloc(static_cast<size_t>(p.nchunks * m_pad * kOzCols));
  k_oz_exp_rows<<<dim3(p.nchunks, p.mtiles), 1024, 0, s>>>(U, m_pad, n_pad, p.kb_per_chunk, p.er.get());
  FSA_LAUNCH_CHECK();
  k_oz_planes_rows<<<dim3(p.nkb, p.mtiles), 256, 0, s>>>(U, m_pad, p.nkb, p.kb_per_chunk, p.er.get(), p.Ar.get());
  FSA_LAUNCH_CHECK();
  k_oz_exp_points<<<static_cast<unsigned>(cdiv(n_pad * 32, 256)), 256, 0, s>>>(U, m_pad, n_pad, p.ec.get());
  FSA_LAUNCH_CHECK();
  k_oz_planes_points<<<dim3(p.mkb, p.ptiles), 256, 0, s>>>(U, m_pad, p.mkb, p.ec.get(), p.Ac.get());
  FSA_LAUNCH_CHECK();
  p.ready = true;
}

void ozaki_project(OzakiPlan& p, const double* R, long ld, long ncols, const double* Dinv, double* S, cudaStream_t s,
                   bool ymax_ready) {
  project_impl(p, R, ld, ncols, Dinv, S, s, ymax_ready);
}
void ozaki_project_plain(OzakiPlan& p, const double* V, long tp, const double* scale, double* S, cudaStream_t s) {
  project_impl(p, V, tp, tp, scale, S, s, false);
}

void ozaki_expand_keep(OzakiPlan& p, const double* W, long ld, long ncols, double* Z, double* Lw, const double* R,
                       const double* Dinv, double* rz, double* partial, cudaStream_t s, bool colsum,
                       const unsigned long long* wmax) {
  slice_w_to(p, W, ld, ncols, p.Ws.get(), p.h.get(), s, wmax);
  OzEpi epi{1, p.m_pad, ncols, ld, p.ec.get(), p.h.get(), partial, Z, Lw, R, Dinv};
  launch_expand(p, epi, s);
  if (colsum) colsum_partials(partial, p.ptiles, ncols, ncols, rz, s);
}
// second column tile's per-sweep buffers (lazily, 65..96 columns)
static void ensure_pair(OzakiPlan& p) {
  if (p.Ys2.n == 0) {
    p.Ys2.alloc(static_cast<size_t>(p.nkb) * kBTile);
    p.Ws2.alloc(static_cast<size_t>(p.mkb) * kBTile);
    p.ymax2.alloc(static_cast<size_t>(p.nchunks * kOzCols));
    p.f2.alloc(static_cast<size_t>(p.nchunks * kOzCols));
    p.h2.alloc(kOzCols);
    p.part2.alloc(static_cast<size_t>(p.nchunks * p.m_pad * kOzCols));
  }
}
// even split of ncols: n0 + n1 columns, both tiles nc = round_up(n0, 16) wide
static void pair_split(long ncols, long& n0, long& n1, int& nc) {
  n0 = (ncols + 1) / 2;
  n1 = ncols - n0;
  nc = static_cast<int>(round_up(n0, 16));
}
void ozaki_project_pair(OzakiPlan& p, const double* R, long ld, long ncols, const double* Dinv, double* S,
                        cudaStream_t s) {
  require(p.ready && ncols > kOzCols && ncols <= kOzPairCols && ncols <= ld, "ozaki pair: 65..96 columns");
  ensure_pair(p);
  long n0, n1;
  int nc;
  pair_split(ncols, n0, n1, nc);
  slice_y(p, R, ld, n0, Dinv, p.ymax.get(), p.f.get(), p.Ys.get(), s, false, nc);
  slice_y(p, R + n0, ld, n1, Dinv, p.ymax2.get(), p.f2.get(), p.Ys2.get(), s, false, nc);
  OzPair pr{{p.Ys.get(), p.Ys2.get()},
            {OzEpi{0, p.m_pad, n0, ld, p.er.get(), p.f.get(), p.part.get(), nullptr, nullptr, nullptr, nullptr},
             OzEpi{0, p.m_pad, n1, ld, p.er.get(), p.f2.get(), p.part2.get(), nullptr, nullptr, nullptr, nullptr}},
            nc};
  launch_gemm_pair(p.Ar.get(), pr, p.mtiles, p.nchunks, p.nkb, p.kb_per_chunk, s);
  launch_pdl(k_oz_reduce, dim3(static_cast<unsigned>(cdiv(4 * p.m_pad * n0, 256))), dim3(256), 0, s, p.part.get(),
             p.nchunks, p.m_pad, ld, n0, S);
  FSA_LAUNCH_CHECK();
  launch_pdl(k_oz_reduce, dim3(static_cast<unsigned>(cdiv(4 * p.m_pad * n1, 256))), dim3(256), 0, s, p.part2.get(),
             p.nchunks, p.m_pad, ld, n1, S + n0);
  FSA_LAUNCH_CHECK();
}
void ozaki_expand_keep_pair(OzakiPlan& p, const double* W, long ld, long ncols, double* Z, double* Lw, const double* R,
                            const double* Dinv, double* rz, double* partial, cudaStream_t s) {
  require(p.ready && ncols > kOzCols && ncols <= kOzPairCols && ncols <= ld, "ozaki pair: 65..96 columns");
  ensure_pair(p);
  long n0, n1;
  int nc;
  pair_split(ncols, n0, n1, nc);
  slice_w_to(p, W, ld, n0, p.Ws.get(), p.h.get(), s, nullptr, nc);
  slice_w_to(p, W + n0, ld, n1, p.Ws2.get(), p.h2.get(), s, nullptr, nc);
  double* part2 = partial + static_cast<long>(p.ptiles) * n0;
  OzPair pr{{p.Ws.get(), p.Ws2.get()},
            {OzEpi{1, p.m_pad, n0, ld, p.ec.get(), p.h.get(), partial, Z, Lw, R, Dinv},
             OzEpi{1, p.m_pad, n1, ld, p.ec.get(), p.h2.get(), part2, Z + n0, Lw + n0, R + n0, Dinv}},
            nc};
  launch_expand_pair(p, pr, s);
  colsum_partials(partial, p.ptiles, n0, n0, rz, s);
  colsum_partials(part2, p.ptiles, n1, n1, rz + n0, s);
}
namespace {
// W planes and exponents of all 64-column tiles of a wide W, then ONE launch that loops the column
// tiles inside each point tile (k_oz_expand<MULTI>): the U digit planes cross HBM once per wide
// pass instead of once per column tile.
void launch_expand_wide(OzakiPlan& p, const double* W, long ldw, OzEpi epi, long zstride, cudaStream_t s,
                        bool side_buffers) {
  const int ncolt = static_cast<int>(ldw / kOzCols);
  const long wsz = static_cast<long>(kOzSlices) * kKb * kOzCols * p.mkb;  // bytes of one tile's W planes
  DBuf<int8_t>& Wb = side_buffers ? p.Ws_wide_side : p.Ws_wide;  // (the side stream has its own)
  DBuf<int>& hb = side_buffers ? p.h_wide_side : p.h_wide;
  if (Wb.n < static_cast<size_t>(ncolt * wsz)) Wb.alloc(static_cast<size_t>(ncolt * wsz));
  if (hb.n < static_cast<size_t>(ncolt * kOzCols)) hb.alloc(static_cast<size_t>(ncolt * kOzCols));
  for (int j = 0; j < ncolt; ++j)
    slice_w_to(p, W + j * kOzCols, ldw, kOzCols, Wb.get() + j * wsz, hb.get() + j * kOzCols, s);
  epi.ecol = hb.get();
  OzPair pr{{Wb.get(), Wb.get()}, {epi, epi}};
  launch_expand_t<false, kXStages, kXLd, kOzMaxW, true>(p.Ac.get(), pr, std::min(p.ptiles, kNumSMs), kXSmem, p.ptiles,
                                                       p.mkb, s, ncolt, wsz, zstride);
}
}  // namespace

void ozaki_expand_sub(OzakiPlan& p, const double* W, long ldw, const double* A, double* Y, long ld, cudaStream_t s,
                      bool side_buffers) {
  require(ldw % kOzCols == 0 && ld % kOzCols == 0, "ozaki: wide passes need 64-column tiles");
  OzEpi epi{3, p.m_pad, kOzCols, ld, p.ec.get(), nullptr, nullptr, nullptr, Y, A, nullptr};
  launch_expand_wide(p, W, ldw, epi, 0, s, side_buffers);
}
void ozaki_expand_rowdots(OzakiPlan& p, const double* W, long ldw, const double* B1, const double* B2, long ld,
                          double* q, double* f, cudaStream_t s, bool side_buffers) {
  require(ldw % kOzCols == 0 && ld % kOzCols == 0, "ozaki: wide passes need 64-column tiles");
  const long tiles = ldw / kOzCols;
  DBuf<double> qp(static_cast<size_t>(tiles * p.n_pad)), fp(static_cast<size_t>(tiles * p.n_pad));
  OzEpi epi{4, p.m_pad, kOzCols, ld, p.ec.get(), nullptr, nullptr, qp.get(), fp.get(), B1, nullptr};
  epi.A2 = B2;
  launch_expand_wide(p, W, ldw, epi, p.n_pad, s, side_buffers);
  k_sum_tiles<<<static_cast<unsigned>(cdiv(p.n_pad, 256)), 256, 0, s>>>(qp.get(), fp.get(), tiles, p.n_pad, q, f);
  FSA_LAUNCH_CHECK();
}
void ozaki_project_wide(OzakiPlan& p, const double* V, long ldv, const double* scale, double* S, long lds,
                        cudaStream_t s) {
  require(ldv % kOzCols == 0 && lds >= ldv, "ozaki: wide passes need 64-column tiles");
  for (long j = 0; j < ldv; j += kOzCols) project_impl(p, V + j, ldv, kOzCols, scale, S + j, s, false);
}
void ozaki_expand_plain(OzakiPlan& p, const double* W, long tp, double* Y, cudaStream_t s) {
  slice_w(p, W, tp, tp, s);
  OzEpi epi{2, p.m_pad, tp, tp, p.ec.get(), p.h.get(), nullptr, nullptr, Y, nullptr, nullptr};
  launch_expand(p, epi, s);
}

}  // namespace fsa
