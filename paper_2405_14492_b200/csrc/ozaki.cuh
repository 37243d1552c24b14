// FP64-accurate skinny GEMMs on the INT8 tensor cores (tcgen05.mma kind::i8).
//
// The two dense passes of a fused FITC-PCG sweep (fsa_core.cu) are
//   project  S  = U diag(D^{-1}) R      (m x t, K = n points)
//   expand   Lw = U^T W                 (n x t, K = m)
// with U fixed for a parameter set. On sm_100a the FP64 tensor path (DMMA) peaks
// near 40 TF/s, so both passes are compute bound; the INT8 tensor cores run
// ~100x faster. Each fp64 operand is split (Ozaki scheme) into kOzSlices = 7 signed
// BALANCED base-256 digit planes sharing one power-of-two exponent per scaling group
// (round 2: base 256 with digits in [-128, 127] instead of base 128 with 8 sign-magnitude
// digits -- 7 bytes per entry of U instead of 8, and 34 plane products instead of 36):
//   |x| < 2^e:  X = trunc(x 2^{54-e}) (an integer, |X| < 2^54; the group maximum keeps its
//   whole 53-bit mantissa),  X = sum_a d_a 2^{8(7-a)},  so  x = 2^{e+2} sum_a d_a 2^{-8a} + r,
//   |r| < 2^{e-54},
// and the product is recovered from the exact int32 products of digit planes, grouped by
// total weight d = a + b, d <= 9 kept (8 TMEM accumulators, C_d = sum_{a+b=d} X_a Y_b):
//   (X Y)_{ij} = 2^{e_i + f_j + 4} sum_{d=2..9} 2^{-8d} C_d[i][j].
// Scaling groups: project -> U per (inducing row, K chunk), D^{-1}R per (column,
// K chunk); expand -> U per point, W per column. Every operand loses at most 2^-54 of
// its group's power-of-two bound (<= 2^-53 of the group's largest magnitude) and the dropped
// weight >= 10 products are below 2^-63, so per output entry
//   |dY_ij| <= 2^-53 (max_k|X_ik| sum_k|Y_kj| + sum_k|X_ik| max_k|Y_kj|)  (+ the final rounding)
// -- an fp64-GEMM-class NORMWISE bound per scaling group. Measured against the
// componentwise sum_k |X_ik||Y_kj| (tests/test_gpu_ozaki.py): see DESIGN.md §4; the expansion
// has a tail at entries where a W entry happens to be tiny exactly where a point's U column is
// concentrated (a per-column exponent cannot resolve it; an fp64 GEMM would).
//
// The U digit planes are built once per parameter set (2 x 7 bytes per entry, less than
// fp64 U); R and W are sliced every sweep. Operand tiles are stored in the
// UMMA canonical K-major no-swizzle layout, so one bulk copy (cp.async.bulk)
// moves a whole stage into shared memory and the MMA descriptors address it
// directly. Accumulators live in TMEM: 8 weights x 64 columns = all 512 columns.
#pragma once

#include <cstdint>

#include "common.cuh"
#include "pattern.cuh"

namespace fsa {

constexpr int kOzSlices = 7;   // digit planes per operand (balanced base 256)
constexpr int kOzMaxW = 9;     // largest kept weight a + b
constexpr int kOzWeights = kOzMaxW - 1;  // TMEM accumulators: weights 2 .. 9
// the projection keeps weights 2 .. 8 (28 plane products per K step instead of 34; see above)
constexpr int kOzProjMaxW = 8;
constexpr int kOzCols = 64;  // RHS columns per accumulator (t_pad <= 64)
constexpr int kOzPairCols = 96;  // widest block of the paired passes (two column tiles of <= 48)

struct OzakiPlan {
  long m_pad = 0, n_pad = 0;
  int mtiles = 0;        // m_pad / 128
  int ptiles = 0;        // n_pad / 128
  int nkb = 0;           // n_pad / 32 (project K blocks)
  int mkb = 0;           // m_pad / 32 (expand K blocks)
  int kb_per_chunk = 0;  // project split-K chunk, in K blocks
  int nchunks = 0;
  const double* U = nullptr;  // the fp64 block the planes were built from
  DBuf<int8_t> Ar, Ac;        // project / expand digit planes of U
  DBuf<int> er, ec;           // their exponents: [nchunks][m_pad], [n_pad]
  DBuf<int8_t> Ys, Ws;        // per-sweep planes of D^{-1} R and W
  DBuf<int8_t> Ws_wide, Ws_wide_side;  // W planes of all column tiles of a wide pass (main / side stream)
  DBuf<int> h_wide, h_wide_side;
  DBuf<unsigned long long> ymax;
  DBuf<int> f, h;             // [nchunks][64], [64]
  DBuf<double> part;          // project partials [nchunks][m_pad][64]
  // second column tile of 65..128-column blocks (ozaki_*_pair), allocated on first use
  DBuf<int8_t> Ys2, Ws2;
  DBuf<unsigned long long> ymax2;
  DBuf<int> f2, h2;
  DBuf<double> part2;
  bool ready = false;
};

inline bool ozaki_supported(long tp) { return tp <= kOzCols; }

// digit planes of U (m_pad x n_pad, column per point, ld m_pad); n_pad % 128 == 0, m_pad % 128 == 0
void ozaki_prepare(OzakiPlan& p, const double* U, long m_pad, long n_pad, cudaStream_t s);
// S (m_pad x ncols, row stride ld) = U diag(Dinv) R over the plan's n_pad rows of R (row stride
// ld, columns [0, ncols), ncols <= 64). With ymax_ready the per-chunk column maxima of
// |Dinv R| are already in p.ymax (update_xr_dot_max)
void ozaki_project(OzakiPlan& p, const double* R, long ld, long ncols, const double* Dinv, double* S, cudaStream_t s,
                   bool ymax_ready = false);
inline long ozaki_chunk_rows(const OzakiPlan& p) { return static_cast<long>(p.kb_per_chunk) * 32; }
// same contract as gemm_expand_woodbury_keep on columns [0, ncols) of row-stride-ld blocks:
// Lw = U^T W, Z = Dinv (R - Lw), rz = column sums of R.Z
void ozaki_expand_keep(OzakiPlan& p, const double* W, long ld, long ncols, double* Z, double* Lw, const double* R,
                       const double* Dinv, double* rz, double* partial, cudaStream_t s,
                       bool colsum = true,  // colsum = false: partials [ptiles][ncols] only
                       const unsigned long long* wmax = nullptr);  // column maxima of |W| (core_apply)
// 65..128 columns (t_pad = 72 at config 4) as two column tiles in ONE launch whose CTA pairs stream
// the same U digit-plane tiles (the second read hits L2): same contracts as ozaki_project /
// ozaki_expand_keep; `partial` holds ptiles * ncols doubles
void ozaki_project_pair(OzakiPlan& p, const double* R, long ld, long ncols, const double* Dinv, double* S,
                        cudaStream_t s);
void ozaki_expand_keep_pair(OzakiPlan& p, const double* W, long ld, long ncols, double* Z, double* Lw, const double* R,
                            const double* Dinv, double* rz, double* partial, cudaStream_t s);
// wide passes (64-column tiles of row-major operands whose widths are multiples of 64):
//   Y = A - U^T W            (W m_pad x ldw, A / Y n_pad x ld)
//   q[i] = (U^T W)_i . B1_i, f[i] = (U^T W)_i . B2_i   (row dots, B1 / B2 n_pad x ld)
//   S = U diag(scale) V      (V n_pad x ldv, S m_pad x lds)
void ozaki_expand_sub(OzakiPlan& p, const double* W, long ldw, const double* A, double* Y, long ld, cudaStream_t s,
                      bool side_buffers = false);  // side_buffers: own W-plane buffers (side-stream passes)
void ozaki_expand_rowdots(OzakiPlan& p, const double* W, long ldw, const double* B1, const double* B2, long ld,
                          double* q, double* f, cudaStream_t s, bool side_buffers = false);
void ozaki_project_wide(OzakiPlan& p, const double* V, long ldv, const double* scale, double* S, long lds,
                        cudaStream_t s);
// plain products for tests: S = U diag(scale) V (scale may be null), Y = U^T W
void ozaki_project_plain(OzakiPlan& p, const double* V, long tp, const double* scale, double* S, cudaStream_t s);
void ozaki_expand_plain(OzakiPlan& p, const double* W, long tp, double* Y, cudaStream_t s);

}  // namespace fsa
