// Row sharding of the pattern; see shard.cuh.
#include <cub/cub.cuh>

#include <algorithm>

#include "shard.cuh"

namespace fsa {

namespace {

inline unsigned nb(long total, int th = 256) { return static_cast<unsigned>(cdiv(total, th)); }

__global__ void k_flag_outside(const long* __restrict__ rowptr, const int* __restrict__ col, long q0, long q1,
                               long lo, long hi, int inside, int* __restrict__ flags, long flag_base) {
  // entries of rows [q0, q1): flag column c when (c in [lo, hi)) == inside
  const long p = rowptr[q0] + static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= rowptr[q1]) return;
  const long c = col[p];
  const bool in = c >= lo && c < hi;
  if (in == (inside != 0)) flags[c - flag_base] = 1;
}

__global__ void k_compact(const int* __restrict__ flags, const int* __restrict__ pos, long n, long base,
                          long* __restrict__ out_long, int* __restrict__ out_int) {
  const long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n || !flags[i]) return;
  if (out_long) out_long[pos[i]] = base + i;
  if (out_int) out_int[pos[i]] = static_cast<int>(base + i);
}

// local rows in E indexing, each row sorted by E index (local part first, halo after)
__global__ void k_local_rows(const long* __restrict__ rowptr, const int* __restrict__ col,
                             const double* __restrict__ dist, long r0, long r1, long n_loc_pad,
                             const int* __restrict__ pos, long n_loc, const long* __restrict__ rowptr_loc,
                             int* __restrict__ col_loc, double* __restrict__ dist_loc, long* __restrict__ diagpos) {
  const long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n_loc) return;
  const long src = rowptr[r0 + i], dst = rowptr_loc[i];
  const long len = rowptr[r0 + i + 1] - src;
  for (long q = 0; q < len; ++q) {
    const long c = col[src + q];
    const int e = (c >= r0 && c < r1) ? static_cast<int>(c - r0) : static_cast<int>(n_loc_pad + pos[c]);
    const double dd = dist[src + q];
    long b = q - 1;  // insertion sort by E index
    while (b >= 0 && col_loc[dst + b] > e) {
      col_loc[dst + b + 1] = col_loc[dst + b];
      dist_loc[dst + b + 1] = dist_loc[dst + b];
      --b;
    }
    col_loc[dst + b + 1] = e;
    dist_loc[dst + b + 1] = dd;
  }
  long dp = -1;
  for (long q = 0; q < len; ++q)
    if (col_loc[dst + q] == i) dp = dst + q;
  diagpos[i] = dp;
}

// transposed position for local columns, -1 for halo columns (their mirror lives on another rank)
__global__ void k_mirror_local(const long* __restrict__ rowptr, const int* __restrict__ col, long n_loc,
                               long* __restrict__ mirror) {
  const long r = (static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= n_loc) return;
  for (long p = rowptr[r] + lane; p < rowptr[r + 1]; p += 32) {
    const long c = col[p];
    if (c >= n_loc) {
      mirror[p] = -1;
      continue;
    }
    long lo = rowptr[c], hi = rowptr[c + 1];
    while (lo < hi) {
      const long mid = (lo + hi) >> 1;
      if (col[mid] < r) lo = mid + 1; else hi = mid;
    }
    mirror[p] = lo;
  }
}

__global__ void k_coords_ext(const double* __restrict__ xs, long ld, long r0, long n_loc, long n_loc_pad,
                             const long* __restrict__ halo, long n_halo, long n_ext_pad, int d,
                             double* __restrict__ out) {
  const long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n_ext_pad) return;
  long src = -1;
  if (i < n_loc) src = r0 + i;
  else if (i >= n_loc_pad && i < n_loc_pad + n_halo) src = halo[i - n_loc_pad];
  for (int k = 0; k < d; ++k) out[i + k * n_ext_pad] = src >= 0 ? xs[src + k * ld] : 0.0;
}

__global__ void k_gather_rows(const double* __restrict__ src, long tp, const int* __restrict__ idx, long count,
                              double* __restrict__ dst) {
  const long e = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (e >= count * tp) return;
  const long i = e / tp, j = e % tp;
  dst[e] = src[static_cast<long>(idx[i]) * tp + j];
}

// exclusive scan of int flags (length n) -> pos, returns the total
long scan_flags(const int* flags, int* pos, long n, cudaStream_t s) {
  size_t bytes = 0;
  FSA_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, flags, pos, static_cast<int>(n), s));
  DBuf<unsigned char> tmp(bytes);
  FSA_CUDA(cub::DeviceScan::ExclusiveSum(tmp.get(), bytes, flags, pos, static_cast<int>(n), s));
  int last_pos = 0, last_flag = 0;
  FSA_CUDA(cudaMemcpyAsync(&last_pos, pos + n - 1, sizeof(int), cudaMemcpyDeviceToHost, s));
  FSA_CUDA(cudaMemcpyAsync(&last_flag, flags + n - 1, sizeof(int), cudaMemcpyDeviceToHost, s));
  FSA_CUDA(cudaStreamSynchronize(s));
  return static_cast<long>(last_pos) + last_flag;
}

}  // namespace

void gather_rows(const double* src, long tp, const int* idx, long count, double* dst, cudaStream_t s) {
  if (count == 0) return;
  k_gather_rows<<<nb(count * tp), 256, 0, s>>>(src, tp, idx, count, dst);
  FSA_LAUNCH_CHECK();
}

void shard_pattern(const Csr& full, const SortedPoints& pts, int rank, int world, ShardPlan& plan, Csr& local,
                   cudaStream_t s) {
  const long n = full.rows;
  plan.rank = rank;
  plan.world = world;
  plan.n = n;
  auto range = [&](int q, long& a, long& b) {
    a = n * q / world;
    b = n * (q + 1) / world;
  };
  range(rank, plan.r0, plan.r1);
  const long r0 = plan.r0, r1 = plan.r1;
  plan.n_loc = r1 - r0;
  plan.n_loc_pad = round_up(plan.n_loc, 128);
  std::vector<long> hrow(static_cast<size_t>(n + 1));
  FSA_CUDA(cudaMemcpyAsync(hrow.data(), full.rowptr.get(), sizeof(long) * (n + 1), cudaMemcpyDeviceToHost, s));
  FSA_CUDA(cudaStreamSynchronize(s));

  // halo: columns of the owned rows outside [r0, r1)
  DBuf<int> flags(n), pos(n);
  flags.zero(s);
  {
    const long cnt = hrow[static_cast<size_t>(r1)] - hrow[static_cast<size_t>(r0)];
    if (cnt > 0)
      k_flag_outside<<<nb(cnt), 256, 0, s>>>(full.rowptr.get(), full.col.get(), r0, r1, r0, r1, 0, flags.get(), 0);
    FSA_LAUNCH_CHECK();
  }
  plan.n_halo = scan_flags(flags.get(), pos.get(), n, s);
  plan.n_ext_pad = round_up(plan.n_loc_pad + plan.n_halo, 128);
  DBuf<long> halo_d(plan.n_halo > 0 ? plan.n_halo : 1);
  k_compact<<<nb(n), 256, 0, s>>>(flags.get(), pos.get(), n, 0, halo_d.get(), nullptr);
  FSA_LAUNCH_CHECK();
  plan.halo_global.resize(static_cast<size_t>(plan.n_halo));
  if (plan.n_halo > 0)
    FSA_CUDA(cudaMemcpyAsync(plan.halo_global.data(), halo_d.get(), sizeof(long) * plan.n_halo,
                             cudaMemcpyDeviceToHost, s));

  // local CSR in E indexing
  local.rows = plan.n_loc;
  local.cols = plan.n_ext_pad;
  std::vector<long> lrow(static_cast<size_t>(plan.n_loc + 1));
  for (long i = 0; i <= plan.n_loc; ++i)
    lrow[static_cast<size_t>(i)] = hrow[static_cast<size_t>(r0 + i)] - hrow[static_cast<size_t>(r0)];
  local.nnz = lrow[static_cast<size_t>(plan.n_loc)];
  local.rowptr.alloc(plan.n_loc + 1);
  local.col.alloc(local.nnz > 0 ? local.nnz : 1);
  local.dist.alloc(local.nnz > 0 ? local.nnz : 1);
  local.diagpos.alloc(plan.n_loc > 0 ? plan.n_loc : 1);
  local.mirror.alloc(local.nnz > 0 ? local.nnz : 1);
  FSA_CUDA(cudaMemcpyAsync(local.rowptr.get(), lrow.data(), sizeof(long) * (plan.n_loc + 1), cudaMemcpyHostToDevice,
                           s));
  k_local_rows<<<nb(plan.n_loc, 128), 128, 0, s>>>(full.rowptr.get(), full.col.get(), full.dist.get(), r0, r1,
                                                   plan.n_loc_pad, pos.get(), plan.n_loc, local.rowptr.get(),
                                                   local.col.get(), local.dist.get(), local.diagpos.get());
  FSA_LAUNCH_CHECK();
  k_mirror_local<<<nb(plan.n_loc * 32), 256, 0, s>>>(local.rowptr.get(), local.col.get(), plan.n_loc,
                                                     local.mirror.get());
  FSA_LAUNCH_CHECK();

  // extended coordinates
  plan.coords_ext.alloc(static_cast<size_t>(pts.d * plan.n_ext_pad));
  k_coords_ext<<<nb(plan.n_ext_pad), 256, 0, s>>>(pts.coords.get(), pts.n_pad, r0, plan.n_loc, plan.n_loc_pad,
                                                  halo_d.get(), plan.n_halo, plan.n_ext_pad, pts.d,
                                                  plan.coords_ext.get());
  FSA_LAUNCH_CHECK();
  FSA_CUDA(cudaStreamSynchronize(s));

  // exchange plan: for every peer q, the owned rows q's rows reference (sent, ascending)
  // and the halo segment of q's range (received, ascending)
  std::vector<int> send_all;
  DBuf<int> sflags(plan.n_loc > 0 ? plan.n_loc : 1), spos(plan.n_loc > 0 ? plan.n_loc : 1);
  for (int q = 0; q < world; ++q) {
    if (q == rank) continue;
    long q0, q1;
    range(q, q0, q1);
    long scnt = 0;
    const long base = static_cast<long>(send_all.size());
    if (plan.n_loc > 0) {
      sflags.zero(s);
      const long cnt = hrow[static_cast<size_t>(q1)] - hrow[static_cast<size_t>(q0)];
      if (cnt > 0)
        k_flag_outside<<<nb(cnt), 256, 0, s>>>(full.rowptr.get(), full.col.get(), q0, q1, r0, r1, 1, sflags.get(),
                                               r0);
      FSA_LAUNCH_CHECK();
      scnt = scan_flags(sflags.get(), spos.get(), plan.n_loc, s);
      if (scnt > 0) {
        DBuf<int> idx(scnt);
        k_compact<<<nb(plan.n_loc), 256, 0, s>>>(sflags.get(), spos.get(), plan.n_loc, 0, nullptr, idx.get());
        FSA_LAUNCH_CHECK();
        send_all.resize(static_cast<size_t>(base + scnt));
        FSA_CUDA(cudaMemcpyAsync(send_all.data() + base, idx.get(), sizeof(int) * scnt, cudaMemcpyDeviceToHost, s));
        FSA_CUDA(cudaStreamSynchronize(s));
      }
    }
    const long ra = std::lower_bound(plan.halo_global.begin(), plan.halo_global.end(), q0) - plan.halo_global.begin();
    const long rb = std::lower_bound(plan.halo_global.begin(), plan.halo_global.end(), q1) - plan.halo_global.begin();
    if (scnt > 0 || rb > ra) {
      plan.peer.push_back(q);
      plan.send_off.push_back(base);
      plan.send_cnt.push_back(scnt);
      plan.recv_off.push_back(ra);
      plan.recv_cnt.push_back(rb - ra);
    }
  }
  plan.send_idx.alloc(send_all.empty() ? 1 : send_all.size());
  if (!send_all.empty())
    FSA_CUDA(cudaMemcpyAsync(plan.send_idx.get(), send_all.data(), sizeof(int) * send_all.size(),
                             cudaMemcpyHostToDevice, s));
  FSA_CUDA(cudaStreamSynchronize(s));
}

}  // namespace fsa
