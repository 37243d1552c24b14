// Row sharding of the taper pattern for multi-GPU operation.
//
// Rank r owns the contiguous block [r0, r1) of the Hilbert-sorted points. Its
// "extended" point set is E = local rows (padded to n_loc_pad) followed by the
// halo: the points outside the block that its rows reference, in ascending
// global order. The local CSR uses E indices, so the SpMM reads one array
// [local | halo] whose halo part is refreshed by a neighbour exchange. Because the
// halo is sorted by global index and every rank's block is contiguous, the rows
// received from one peer form one contiguous segment of the halo, and the peer
// sends exactly its rows in that segment, in the same order.
#pragma once

#include <vector>

#include "common.cuh"
#include "pattern.cuh"

namespace fsa {

struct ShardPlan {
  int rank = 0, world = 1;
  long n = 0;                      // global number of points
  long r0 = 0, r1 = 0;             // owned global internal rows
  long n_loc = 0, n_loc_pad = 0;   // owned rows, padded to 128
  long n_halo = 0, n_ext_pad = 0;  // halo points; n_loc_pad + n_halo padded to 128
  DBuf<double> coords_ext;         // SoA [d][n_ext_pad] (empty when world == 1)
  std::vector<long> halo_global;   // global internal index of each halo point
  // exchange plan (per peer with something to send or receive)
  std::vector<int> peer;
  std::vector<long> send_off, send_cnt;  // rows into send_idx
  std::vector<long> recv_off, recv_cnt;  // rows into the halo region
  DBuf<int> send_idx;                    // local row indices to send, concatenated per peer
};

// Builds the plan and replaces `local` with the rank's rows of `full` in E indexing.
void shard_pattern(const Csr& full, const SortedPoints& pts, int rank, int world, ShardPlan& plan, Csr& local,
                   cudaStream_t s);

// dst[i][j] = src[idx[i]][j] (rows of width tp)
void gather_rows(const double* src, long tp, const int* idx, long count, double* dst, cudaStream_t s);

}  // namespace fsa
