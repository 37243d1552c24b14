// Taper-neighbour search on the device (reference GridIndex / taper_pattern /
// cross_taper_pattern, locations.cpp:19-62,139-184).
//
// Points are binned into cells of edge h >= gamma, the cells are ordered along a
// Hilbert curve (d = 2; row-major for d = 1, Morton for d = 3) and the points are
// radix-sorted by (cell key, original index). That order is the library's
// internal point order: it makes the 3^d-cell neighbourhood of a row a handful of
// contiguous index ranges (L2-friendly SpMM gathers) and is the row-sharding order
// for multiple GPUs. Rows list their columns in ascending internal order.
#pragma once

#include <vector>

#include "common.cuh"

namespace fsa {

struct CellGrid {
  int d = 2;
  double origin[3] = {0, 0, 0};
  double h = 1.0;
};

// A point set in internal (cell-sorted) order.
struct SortedPoints {
  long n = 0, n_pad = 0;
  int d = 2;
  CellGrid grid;
  std::vector<int> perm;        // internal -> original (host)
  std::vector<int> iperm;       // original -> internal (host)
  DBuf<int> perm_d, iperm_d;    // same on device
  DBuf<double> coords;          // SoA [d][n_pad], internal order, zero padding
  DBuf<unsigned long long> keys;  // sorted cell keys, length n
};


struct Csr {
  long rows = 0, cols = 0, nnz = 0;
  DBuf<long> rowptr;   // rows + 1
  DBuf<int> col;       // internal column index
  DBuf<double> dist;   // stored distances (parameter independent)
  DBuf<long> diagpos;  // position of (i,i) (square patterns only)
  DBuf<long> mirror;   // position of (c,r) for the entry (r,c) (square patterns only)
  // Row groups: kGroup consecutive rows (Hilbert order) share one column list, the
  // union of their columns, padded to a multiple of 4 (parameter independent, built
  // once). The group's values form a dense kGroup x union block (zeros where a row lacks
  // the column), stored in DMMA m8n8k4 A-fragment order, so the SpMM is a dense block
  // product on the FP64 tensor cores with every RHS row of the union staged in shared
  // memory once per group (sparse.cu, spmm_block_dot).
  long ngrp = 0, gnnz = 0;     // gnnz = total padded union size (0: groups not built)
  DBuf<long> gptr;             // ngrp + 1 offsets into gcol (multiples of 4)
  DBuf<int> gcol;              // union columns (row-tile-mask order, see k_group_union; padding repeats a valid column)
  DBuf<int> gslot;             // per entry: its index in the value blocks (kGroup * gnnz)
  int gmax = 0;                // largest padded union
  // Gram blocks (sddmm_block) only evaluate the union columns c >= the group's first row: every
  // entry (r, c) with c < r is taken from its mirror (c, r). gneed[gptr[g] + j], j < gneedcnt[g]:
  // the union slots of those columns, in slot order.
  DBuf<int> gneed, gneedcnt;
  int gneedmax = 0;            // largest gneedcnt
  // Compact value tiles: of the dense block only the 8 x 4 DMMA A tiles (row tile rt of the
  // group, k-step kb = union slot / 4) that hold an entry are stored (~2/3 of them at 80
  // entries per row). kmask[kb] bit rt marks them; koff[kb] = stored tiles before k-step kb.
  long nkb = 0, ntiles = 0;    // k-steps (gnnz / 4) and stored tiles
  DBuf<int> kmask, koff;       // nkb, nkb + 1
  DBuf<int> pmeta;             // per k-step (int2): {koff[kb], kmask[kb + i] << 4 i for i < 8}
};
constexpr int kGroup = 32;
// builds the row groups (leaves gnnz = 0 if some group has more than 4096 entries)
void build_groups(Csr& pat, cudaStream_t s);

// grid covering both point sets (cross patterns use one grid for rows and cols)
CellGrid make_grid(const double* coords, long n, int d, double gamma, const double* coords2, long n2);
void sort_points(const double* coords_host, long n, int d, const CellGrid& g, long n_pad, SortedPoints& out,
                 cudaStream_t s);
// rows x cols pattern of pairs with |x_row - x_col| < gamma; force_diag adds (i,i)
// (rows and cols must be the same set then).
void build_pattern(const SortedPoints& rows, const SortedPoints& cols, double gamma, bool force_diag, Csr& out,
                   cudaStream_t s);

}  // namespace fsa
