// Host orchestration of the FSA iterative core on one B200; see fsa_core.cuh.
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <random>

#include "blas1.cuh"
#include "dgemm.cuh"
#include "fsa_core.cuh"
#include "kernels.cuh"
#include "sparse.cuh"

namespace fsa {


// ---- RNG (types.h:104-129; identical libstdc++ distributions) ------------------------------
unsigned long long splitmix64(unsigned long long x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
static std::mt19937_64 probe_rng(unsigned long long seed, unsigned long long i) {
  return std::mt19937_64(splitmix64(splitmix64(seed) ^ splitmix64(i + 0x51ed2701ULL)));
}
void probe_gaussian(unsigned long long seed, unsigned long long i, long n1, double* e1, long n2, double* e2) {
  std::mt19937_64 rng = probe_rng(seed, i);
  {
    std::normal_distribution<double> N01(0.0, 1.0);  // fresh object per vector
    for (long j = 0; j < n1; ++j) e1[j] = N01(rng);
  }
  {
    std::normal_distribution<double> N01(0.0, 1.0);
    for (long j = 0; j < n2; ++j) e2[j] = N01(rng);
  }
}
// probe_gaussian on the device, one CTA per probe: the same MT19937-64 stream (seeding, twist in
// two parallel halves, tempering), generate_canonical<double, 53> (one 64-bit draw per uniform)
// and libstdc++'s polar normal_distribution: draws are consumed in pairs, a pair is accepted when
// 0 < x^2 + y^2 <= 1 and yields y m then x m (m = sqrt(-2 log r2 / r2)); a fresh distribution per
// vector, so e1 takes the first ceil(n1 / 2) accepted pairs and e2 the following ones. The
// products, sums and quotients are issued unfused and correctly rounded like the host's (SSE, no
// FMA); log is CUDA's (<= 1 ulp, the host's glibc < 0.52 ulp), so a draw can differ from the host's
// in its last bit. e1 goes to E1[r * ld1 + i] (r < n1), e2 to E2[i * n2 + r].
namespace {
__device__ __forceinline__ unsigned long long splitmix64_d(unsigned long long x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}
constexpr int kMtN = 312, kMtM = 156;
__global__ void __launch_bounds__(320) k_probe_gaussian(unsigned long long seed, long n1, long ld1, double* E1, long n2,
                                                        double* E2) {
  __shared__ unsigned long long mt[kMtN];
  __shared__ double us[kMtN];
  __shared__ int wsum[10];  // (320 threads)
  const unsigned long long i = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr unsigned long long kUpper = 0xFFFFFFFF80000000ULL, kLower = 0x7FFFFFFFULL, kA = 0xB5026F5AA96619E9ULL;
  if (tid == 0) {
    unsigned long long x = splitmix64_d(splitmix64_d(seed) ^ splitmix64_d(i + 0x51ed2701ULL));
    mt[0] = x;
    for (int k = 1; k < kMtN; ++k) {
      x = 6364136223846793005ULL * (x ^ (x >> 62)) + static_cast<unsigned long long>(k);
      mt[k] = x;
    }
  }
  __syncthreads();
  const long p1 = (n1 + 1) / 2, ptot = p1 + (n2 + 1) / 2;
  long done = 0;
  while (done < ptot) {
    unsigned long long a0 = 0, a1 = 0, b = 0;
    if (tid < kMtM) a0 = mt[tid], a1 = mt[tid + 1], b = mt[tid + kMtM];
    __syncthreads();
    if (tid < kMtM) {
      const unsigned long long y = (a0 & kUpper) | (a1 & kLower);
      mt[tid] = b ^ (y >> 1) ^ ((y & 1ULL) ? kA : 0ULL);
    }
    __syncthreads();
    const int k2 = kMtM + tid;
    if (tid < kMtM) a0 = mt[k2], a1 = k2 + 1 < kMtN ? mt[k2 + 1] : mt[0], b = mt[k2 - kMtM];
    __syncthreads();
    if (tid < kMtM) {
      const unsigned long long y = (a0 & kUpper) | (a1 & kLower);
      mt[k2] = b ^ (y >> 1) ^ ((y & 1ULL) ? kA : 0ULL);
    }
    __syncthreads();
    if (tid < kMtN) {
      unsigned long long z = mt[tid];
      z ^= (z >> 29) & 0x5555555555555555ULL;
      z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
      z ^= (z << 37) & 0xFFF7EEE000000000ULL;
      z ^= z >> 43;
      double u = __dmul_rn(__ull2double_rn(z), 0x1p-64);
      if (u >= 1.0) u = 0x1.fffffffffffffp-1;  // nextafter(1, 0)
      us[tid] = u;
    }
    __syncthreads();
    double xv = 0.0, yv = 0.0, r2 = 0.0;
    int acc = 0;
    if (tid < kMtM) {
      xv = __dsub_rn(__dmul_rn(2.0, us[2 * tid]), 1.0);
      yv = __dsub_rn(__dmul_rn(2.0, us[2 * tid + 1]), 1.0);
      r2 = __dadd_rn(__dmul_rn(xv, xv), __dmul_rn(yv, yv));
      acc = (r2 > 1.0 || r2 == 0.0) ? 0 : 1;
    }
    // exclusive rank of this pair among the accepted ones (pairs in order)
    const unsigned bal = __ballot_sync(0xffffffffu, acc);
    if (lane == 0) wsum[warp] = __popc(bal);
    __syncthreads();
    int before = 0, total = 0;
    for (int w = 0; w < 10; ++w) {
      before += w < warp ? wsum[w] : 0;
      total += wsum[w];
    }
    const long P = done + before + __popc(bal & ((1u << lane) - 1u));
    if (acc && P < ptot) {
      const double mult = __dsqrt_rn(__ddiv_rn(__dmul_rn(-2.0, log(r2)), r2));
      const double v0 = __dmul_rn(yv, mult), v1 = __dmul_rn(xv, mult);
      if (P < p1) {
        const long r = 2 * P;
        E1[r * ld1 + static_cast<long>(i)] = v0;
        if (r + 1 < n1) E1[(r + 1) * ld1 + static_cast<long>(i)] = v1;
      } else {
        const long r = 2 * (P - p1);
        E2[static_cast<long>(i) * n2 + r] = v0;
        if (r + 1 < n2) E2[static_cast<long>(i) * n2 + r + 1] = v1;
      }
    }
    done += total;
    __syncthreads();  // (wsum, us and mt are rewritten by the next round)
  }
}
}  // namespace
void probe_rademacher(unsigned long long seed, unsigned long long i, long n, double* z) {
  std::mt19937_64 rng = probe_rng(seed, i);
  std::bernoulli_distribution coin(0.5);
  for (long j = 0; j < n; ++j) z[j] = coin(rng) ? 1.0 : -1.0;
}

// ---- context ------------------------------------------------------------------------------
Context::Context(int dev) : device(dev) {
  FSA_CUDA(cudaSetDevice(dev));
  {  // the main stream outranks the side stream (the rho-derivative build fills idle SMs only)
    int least = 0, greatest = 0;
    FSA_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    FSA_CUDA(cudaStreamCreateWithPriority(&stream, cudaStreamNonBlocking, greatest));
  }
  alloc_stream() = stream;
  cudaMemPool_t pool = nullptr;
  FSA_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
  unsigned long long keep = ~0ULL;  // keep freed blocks for reuse across evaluations
  FSA_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  {  // prime the device pool once per process: later per-evaluation temporaries are carved
     // from retained memory instead of mapping new pages mid-evaluation
    static bool primed = false;
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    if (!primed) {
      size_t free_b = 0, total_b = 0;
      FSA_CUDA(cudaMemGetInfo(&free_b, &total_b));
      const size_t want = std::min<size_t>(free_b / 4, size_t(16) << 30);
      void* p = nullptr;
      if (want > 0 && cudaMallocAsync(&p, want, stream) == cudaSuccess) {
        cudaFreeAsync(p, stream);
        cudaStreamSynchronize(stream);
      }
      cudaGetLastError();
      primed = true;
    }
  }
  FSA_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&host_flags), 4 * sizeof(int), cudaHostAllocMapped));
  FSA_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&host_flags_dev), host_flags, 0));
  if (const char* g = std::getenv("FSA_GEMM")) gemm_mode = std::strcmp(g, "dmma") == 0 ? 1 : (std::strcmp(g, "ozaki") == 0 ? 2 : 0);
}
cudaStream_t Context::side_stream() {
  if (side == nullptr) {
    int least = 0, greatest = 0;
    FSA_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    FSA_CUDA(cudaStreamCreateWithPriority(&side, cudaStreamNonBlocking, least));
  }
  return side;
}
Context::~Context() {
  if (side) cudaStreamSynchronize(side);
  cudaStreamSynchronize(stream);
  cgw.reset();
  cudaStreamSynchronize(stream);
  if (alloc_stream() == stream) alloc_stream() = nullptr;  // later frees go to the legacy stream
  for (auto& r : pending) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (auto e : pool) cudaEventDestroy(e);
  if (host_flags) cudaFreeHost(host_flags);
  if (side) cudaStreamDestroy(side);
  if (stream) cudaStreamDestroy(stream);
}
cudaEvent_t Context::ev() {
  if (!pool.empty()) {
    cudaEvent_t e = pool.back();
    pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  FSA_CUDA(cudaEventCreate(&e));
  return e;
}
void Context::flush_timers() {
  FSA_CUDA(cudaStreamSynchronize(stream));
  for (auto& r : pending) {
    float ms = 0.f;
    FSA_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
    Acc& a = totals[r.name];
    a.ms += ms;
    a.count += 1;
    a.units += r.units;
    pool.push_back(r.a);
    pool.push_back(r.b);
  }
  pending.clear();
}
void Context::sync() { FSA_CUDA(cudaStreamSynchronize(stream)); }

KTimer::KTimer(Context* ctx, const char* name, double units) : c(ctx) {
  if (c == nullptr || !c->profile) return;
  Context::Rec r{name, c->ev(), c->ev(), units};
  FSA_CUDA(cudaEventRecord(r.a, c->stream));
  c->pending.push_back(r);
  idx = c->pending.size() - 1;
}
KTimer::~KTimer() {
  if (idx == static_cast<size_t>(-1)) return;
  cudaEventRecord(c->pending[idx].b, c->stream);
}

// ---- geometry --------------------------------------------------------------------------------
std::shared_ptr<Geometry> make_geometry(Context* ctx, const double* coords, long n, int d, double gamma) {
  require(n > 0, "empty location set");
  require(gamma > 0.0, "taper range gamma must be positive");
  require(d >= 1 && d <= 3, "dimension must be 1, 2 or 3");
  auto g = std::make_shared<Geometry>();
  g->gamma = gamma;
  g->coords_host.assign(coords, coords + n * d);
  const CellGrid grid = make_grid(coords, n, d, gamma, nullptr, 0);
  sort_points(coords, n, d, grid, round_up(n, 128), g->pts, ctx->stream);
  const int world = ctx->row_sharded() ? ctx->comm->size() : 1, rank = ctx->row_sharded() ? ctx->comm->rank() : 0;
  if (world == 1) {
    build_pattern(g->pts, g->pts, gamma, true, g->pat, ctx->stream);
    g->shard.n = g->shard.n_loc = g->shard.r1 = n;
    g->shard.n_loc_pad = g->shard.n_ext_pad = g->pts.n_pad;
  } else {
    // every rank derives the same global order and pattern, then keeps its row block
    Csr full;
    build_pattern(g->pts, g->pts, gamma, true, full, ctx->stream);
    shard_pattern(full, g->pts, rank, world, g->shard, g->pat, ctx->stream);
  }
  // row groups of the block SpMM (FSA_SPMM=csr keeps the per-row gather kernel)
  static const bool csr_only = std::getenv("FSA_SPMM") && std::strcmp(std::getenv("FSA_SPMM"), "csr") == 0;
  if (!csr_only) build_groups(g->pat, ctx->stream);
  ctx->sync();
  return g;
}

// Matern (mode 0) or its rho derivative (mode 1) between the inducing points and the
// extended point set (owned rows, zero padding, halo points): column-per-point m_pad x n_ext_pad
void Model::cross_cov_ext(int mode, double* out, cudaStream_t s) {
  const ShardPlan& sp = geo->shard;
  if (s == nullptr) s = ctx->stream;
  launch_cross_cov(ind.get(), m, m, geo->coords_ext(), n_ext_pad, n, n_pad, d, P.nu, P.sigma1_2, P.rho, mode, out,
                   m_pad, s);
  if (n_ext_pad > n_pad)
    launch_cross_cov(ind.get(), m, m, geo->coords_ext() + n_pad, n_ext_pad, sp.n_halo, n_ext_pad - n_pad, d, P.nu,
                     P.sigma1_2, P.rho, mode, out + n_pad * m_pad, m_pad, s);
}

void Model::halo_exchange(double* X, long tp) {
  if (world() == 1) return;
  const ShardPlan& sp = geo->shard;
  cudaStream_t s = ctx->stream;
  KTimer t(ctx, "halo_exchange");
  long total = 0;
  for (long c : sp.send_cnt) total += c;
  if (halo_send.n < static_cast<size_t>(total * tp)) halo_send.alloc(static_cast<size_t>(total * tp));
  gather_rows(X, tp, sp.send_idx.get(), total, halo_send.get(), s);
  std::vector<HaloPeer> peers;
  for (size_t q = 0; q < sp.peer.size(); ++q)
    peers.push_back(HaloPeer{sp.peer[q], halo_send.get() + sp.send_off[q] * tp, sp.send_cnt[q] * tp,
                             X + (n_pad + sp.recv_off[q]) * tp, sp.recv_cnt[q] * tp});
  rcomm->exchange(peers, s);
}

// ---- model --------------------------------------------------------------------------------------
static void validate(const Params& p) {  // types.h:80-84, fsa.cpp:9-13
  require(p.sigma2 > 0.0 && std::isfinite(p.sigma2), "sigma2 must be positive and finite");
  require(p.sigma1_2 > 0.0 && std::isfinite(p.sigma1_2), "sigma1_2 must be positive and finite");
  require(p.rho > 0.0 && std::isfinite(p.rho), "rho must be positive and finite");
  require(p.gamma > 0.0, "taper range gamma must be positive");
  require(p.nu >= 0 && p.nu <= 2, "Matern smoothness must be one of 0.5, 1.5, 2.5");
  require(p.family == 1 || p.family == 2, "taper family must be wendland1 or wendland2");
}

double* Model::mt_buf(int which, long tp) {
  DBuf<double>& b = which == 0 ? mt1 : mt2;
  const size_t need = static_cast<size_t>(m_pad * tp);
  if (b.n < need) b.alloc(need);
  return b.get();
}

void Model::ensure_ozaki() {
  if (oz_pending) {
    FSA_CUDA(cudaStreamWaitEvent(ctx->stream, oz_done, 0));
    oz_pending = false;
  }
  if (oz.ready && oz.U == U.get()) return;
  KTimer t(ctx, "ozaki_prepare", 16.0 * m_pad * n_pad);
  ozaki_prepare(oz, U.get(), m_pad, n_pad, ctx->stream);
}

// The digit planes depend on U only: started on the side stream as soon as U exists, they are
// built while the main stream runs the Sigma_s SDDMM and the FITC core (SYRK, the latency-bound
// Cholesky panels); ensure_ozaki joins. The plan's per-call B-side buffers are only allocated here.
void Model::start_ozaki() {
  if (ctx->gemm_mode == 1 || (oz.ready && oz.U == U.get())) return;
  cudaStream_t side = ctx->side_stream();
  cudaEvent_t go = ctx->ev();
  FSA_CUDA(cudaEventRecord(go, ctx->stream));
  FSA_CUDA(cudaStreamWaitEvent(side, go, 0));
  ctx->pool.push_back(go);
  cudaStream_t saved = alloc_stream();
  alloc_stream() = side;
  try {
    ozaki_prepare(oz, U.get(), m_pad, n_pad, side);
  } catch (...) {
    alloc_stream() = saved;
    throw;
  }
  alloc_stream() = saved;
  if (oz_done == nullptr) oz_done = ctx->ev();
  FSA_CUDA(cudaEventRecord(oz_done, side));
  oz_pending = true;
}


void Model::project(const double* M, const double* V, long tp, double* out, const double* scale) {
  const double flops = 2.0 * m * n * (cols_hint > 0 && cols_hint <= tp ? cols_hint : tp);
  if (M == U.get() && use_ozaki(tp)) {  // INT8 tensor cores, fp64-accurate (ozaki.cuh)
    ensure_ozaki();
    KTimer t(ctx, "lowrank_project", flops);
    ozaki_project_plain(oz, V, tp, scale, out, ctx->stream);
  } else {
    const size_t need = gemm_reduce_scratch(m_pad, tp, n_pad);
    if (red_scratch.n < need) red_scratch.alloc(need);
    KTimer t(ctx, "lowrank_project", flops);
    gemm_reduce(M, m_pad, m_pad, n_pad, V, tp, tp, scale, out, tp, 1.0, 0.0, red_scratch.get(), ctx->stream);
  }
  if (world() > 1) {  // m x t partials of the row blocks
    KTimer t(ctx, "allreduce");
    rcomm->allreduce(out, m_pad * tp, ctx->stream);
  }
}

void Model::expand(const double* W, long tp, double* Y) {
  KTimer t(ctx, "lowrank_expand", 2.0 * m * n * (cols_hint > 0 && cols_hint <= tp ? cols_hint : tp));
  if (use_ozaki(tp)) {
    ensure_ozaki();
    ozaki_expand_plain(oz, W, tp, Y, ctx->stream);
  } else {
    gemm_expand_store(U.get(), m_pad, n_pad, m_pad, W, tp, tp, Y, tp, 1.0, 0.0, ctx->stream);
  }
}

std::unique_ptr<Model> Model::assemble(Context* ctx, std::shared_ptr<Geometry> geo, const double* inducing, long m,
                                       const Params& p) {
  NvtxRange nvtx_("fsa::assemble");
  validate(p);
  require(geo != nullptr, "geometry missing");
  require(m > 0, "empty inducing set");
  require(std::fabs(geo->gamma - p.gamma) == 0.0, "geometry built for another taper range");
  auto md = std::make_unique<Model>();
  Model& M = *md;
  cudaStream_t s = ctx->stream;
  M.ctx = ctx;
  M.geo = geo;
  M.P = p;
  require(geo->shard.world == (ctx->row_sharded() ? ctx->comm->size() : 1), "geometry built for another communicator");
  M.rcomm = geo->shard.world > 1 ? ctx->comm.get() : &ctx->self_comm;
  M.n = geo->shard.n_loc;
  M.n_pad = geo->shard.n_loc_pad;
  M.n_ext_pad = geo->shard.n_ext_pad;
  M.d = geo->pts.d;
  M.m = m;
  M.m_pad = round_up(m, 128);
  require(M.m_pad <= 1024, "more than 1024 inducing points are not supported");
  const long mp = M.m_pad, np = M.n_pad, ne = M.n_ext_pad;
  M.ind_host.assign(inducing, inducing + m * M.d);
  M.ind.alloc(m * M.d);
  FSA_CUDA(cudaMemcpyAsync(M.ind.get(), inducing, sizeof(double) * m * M.d, cudaMemcpyHostToDevice, s));
  M.info.alloc(4);
  M.info.zero(s);  // [0] Cholesky status, [1] clamped residual diagonals
  M.dinv_scratch.alloc(mp * 192);  // potrf: mp * 64; trsm: mp * 192
  M.dot_scratch.alloc(coldot_scratch(np, 128));
  DBuf<double> scal(4);

  // Sigma_m + jitter, Cholesky (fsa.cpp:23-30); Sigma_mn (fsa.cpp:32-35, owned and halo points) is
  // evaluated on the side stream meanwhile: the Cholesky panels are a few CTAs wide and leave the
  // GPU idle
  M.Sm.alloc(mp * mp);
  M.L.alloc(mp * mp);
  M.U.alloc(mp * ne);
  M.lowrank.alloc(np);
  static const bool serial_cov = std::getenv("FSA_SERIAL_CROSS_COV") != nullptr;
  cudaEvent_t cov_done = nullptr;
  if (!serial_cov) {
    cudaStream_t side = ctx->side_stream();
    cudaEvent_t ready = ctx->ev();
    FSA_CUDA(cudaEventRecord(ready, s));  // inducing points uploaded, U allocated
    FSA_CUDA(cudaStreamWaitEvent(side, ready, 0));
    ctx->pool.push_back(ready);
    M.cross_cov_ext(0, M.U.get(), side);
    cov_done = ctx->ev();
    FSA_CUDA(cudaEventRecord(cov_done, side));
  }
  {
    KTimer t(ctx, "setup_sigma_m");
    launch_sigma_m(M.ind.get(), m, m, mp, M.d, p.nu, p.sigma1_2, p.rho, p.jitter_rel * p.sigma1_2, 0, M.Sm.get(), s);
    FSA_CUDA(cudaMemcpyAsync(M.L.get(), M.Sm.get(), sizeof(double) * mp * mp, cudaMemcpyDeviceToDevice, s));
    potrf_lower(M.L.get(), mp, M.info.get(), M.dinv_scratch.get(), s);
    launch_logdet_diag(M.L.get(), mp, m, scal.get(), s);
  }
  // U = L^{-1} Sigma_mn
  if (cov_done != nullptr) {
    FSA_CUDA(cudaStreamWaitEvent(s, cov_done, 0));
    ctx->pool.push_back(cov_done);
  } else {
    KTimer t(ctx, "setup_cross_cov");
    M.cross_cov_ext(0, M.U.get());
  }
  {
    KTimer t(ctx, "setup_trsm", 1.0 * mp * mp * ne);
    trsm_lower_cols(M.L.get(), mp, M.U.get(), mp, ne, M.dinv_scratch.get(), s);
  }
  colnorm2(M.U.get(), mp, mp, M.n, np, M.lowrank.get(), s);
  M.start_ozaki();  // INT8 digit planes of U on the side stream, under the SDDMM / FITC build
  // Sigma_s on the taper pattern (fsa.cpp:37-56)
  const Csr& pat = geo->pat;
  M.sval.alloc(pat.nnz > 0 ? pat.nnz : 1);
  SddmmParams sp{p.nu, p.family, p.sigma2, p.sigma1_2, p.rho, p.gamma};
  {
    KTimer t(ctx, "setup_sddmm", 2.0 * mp * pat.nnz);
    if (pat.gnnz > 0 && mp % 32 == 0) {  // dense Gram blocks on DMMA; fills the SpMM value blocks too
      M.gval.alloc(static_cast<size_t>(32 * pat.ntiles));
      DBuf<double> gtmp(static_cast<size_t>(pat.gnnz * kGroup));
      sddmm_block(0, M.U.get(), nullptr, nullptr, mp, mp, pat, M.lowrank.get(), sp, M.sval.get(), M.gval.get(),
                  M.info.get() + 1, gtmp.get(), s);
    } else {
      sddmm_sigma_s(M.U.get(), mp, pat, M.lowrank.get(), sp, M.sval.get(), M.info.get() + 1, s);
    }
  }
  if (pat.gnnz > 0 && !(mp % 32 == 0)) {  // value blocks of the row groups (block SpMM of the PCG sweeps)
    KTimer t(ctx, "setup_group_values", 16.0 * pat.nnz + 8.0 * 32 * pat.ntiles);
    M.gval.alloc(static_cast<size_t>(32 * pat.ntiles));
    group_values(pat, M.sval.get(), M.gval.get(), s);
  }
  M.D.alloc(np);
  M.Dinv.alloc(np);
  M.sqrtD.alloc(np);
  extract_diag(M.sval.get(), pat.diagpos.get(), M.n, np, M.D.get(), M.Dinv.get(), M.sqrtD.get(), s);
  int hinfo[2] = {0, 0};
  double hld = 0.0;
  FSA_CUDA(cudaMemcpyAsync(hinfo, M.info.get(), 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
  FSA_CUDA(cudaMemcpyAsync(&hld, scal.get(), sizeof(double), cudaMemcpyDeviceToHost, s));
  FSA_CUDA(cudaStreamSynchronize(s));
  if (hinfo[0] != 0) throw NumericalError("inducing covariance is not positive definite");
  M.logdet_sigma_m = hld;
  M.n_clamped = hinfo[1];
  return md;
}

// The rho-derivative blocks (fsa.cpp:101-124 in U-form) are needed only by the gradient, so
// make_preconditioner starts them on the context's side stream (start_rho_derivs): they run
// during the PCG sweeps, filling the SMs the sweep kernels leave idle (wave tails, the small
// control kernels). Every consumer calls ensure_rho_derivs, which joins the side stream. The
// side-stream build allocates and frees on the side stream and touches no scratch shared with
// the main stream (own TRSM scratch; the T product on DMMA rather than through the Ozaki plan's
// W-plane buffers, which the sweep's expansions use).
void Model::ensure_rho_derivs() {
  if (have_rho) {
    if (rho_pending) {
      FSA_CUDA(cudaStreamWaitEvent(ctx->stream, rho_done, 0));
      rho_pending = false;
    }
    return;
  }
  KTimer t(ctx, "setup_rho_derivs");
  build_rho_derivs(ctx->stream, dinv_scratch.get(), false);
  have_rho = true;
}

void Model::start_rho_derivs() {
  if (have_rho) return;
  cudaStream_t side = ctx->side_stream();
  cudaEvent_t go = ctx->ev();
  FSA_CUDA(cudaEventRecord(go, ctx->stream));
  FSA_CUDA(cudaStreamWaitEvent(side, go, 0));
  ctx->pool.push_back(go);
  cudaStream_t saved = alloc_stream();
  alloc_stream() = side;  // allocations and frees of the build are ordered on the side stream
  try {
    rho_scratch.alloc(m_pad * 192);
    build_rho_derivs(side, rho_scratch.get(), true);
  } catch (...) {
    alloc_stream() = saved;
    throw;
  }
  alloc_stream() = saved;
  if (rho_done == nullptr) rho_done = ctx->ev();
  FSA_CUDA(cudaEventRecord(rho_done, side));
  have_rho = true;
  rho_pending = true;
}

Model::~Model() {
  // frees below are ordered after the side-stream builds
  if (rho_pending) cudaStreamWaitEvent(ctx->stream, rho_done, 0);
  if (oz_pending) cudaStreamWaitEvent(ctx->stream, oz_done, 0);
  if (rho_done != nullptr) ctx->pool.push_back(rho_done);
  if (oz_done != nullptr) ctx->pool.push_back(oz_done);
}

void Model::build_rho_derivs(cudaStream_t s, double* trsm_scratch, bool side) {
  const long mp = m_pad, np = n_pad;
  // K2 = L^{-1} dSigma_m/drho L^{-T}
  K2.alloc(mp * mp);
  {
    DBuf<double> tmp(mp * mp);
    launch_sigma_m(ind.get(), m, m, mp, d, P.nu, P.sigma1_2, P.rho, 0.0, 1, tmp.get(), s);
    trsm_lower_cols(L.get(), mp, tmp.get(), mp, mp, trsm_scratch, s);  // X = L^{-1} dSm
    launch_transpose(tmp.get(), mp, mp, mp, K2.get(), mp, s);
  }
  trsm_lower_cols(L.get(), mp, K2.get(), mp, mp, trsm_scratch, s);   // L^{-1} X^T
  // U1 = L^{-1} dSigma_mn/drho ; T = U1 - K2 U
  const long ne = n_ext_pad;
  U1.alloc(mp * ne);
  T.alloc(mp * ne);
  cross_cov_ext(1, U1.get(), s);
  {
    KTimer t1(side ? nullptr : ctx, "rho_trsm", 1.0 * mp * mp * ne);
    trsm_lower_cols(L.get(), mp, U1.get(), mp, ne, trsm_scratch, s);
  }
  {
    KTimer t2(side ? nullptr : ctx, "rho_T_gemm", 2.0 * m * m * n);
    if (ctx->gemm_mode != 1 && ne == np && (!side || (oz.ready && oz.U == U.get()))) {
      // INT8 tensor cores, 64-column tiles of K2; on the side stream the digit planes of U were
      // queued on this same stream (start_ozaki) and the W planes use the side buffers
      if (!side) ensure_ozaki();
      ozaki_expand_sub(oz, K2.get(), mp, U1.get(), T.get(), mp, s, side);
    } else {
      FSA_CUDA(cudaMemcpyAsync(T.get(), U1.get(), sizeof(double) * mp * ne, cudaMemcpyDeviceToDevice, s));
      gemm_expand_store(U.get(), mp, ne, mp, K2.get(), mp, mp, T.get(), mp, -1.0, 1.0, s);
    }
  }
  const Csr& pat = geo->pat;
  dsval.alloc(pat.nnz > 0 ? pat.nnz : 1);
  SddmmParams sp{P.nu, P.family, P.sigma2, P.sigma1_2, P.rho, P.gamma};
  {
    KTimer t3(side ? nullptr : ctx, "rho_sddmm", 4.0 * m * pat.nnz / 2);
    if (pat.gnnz > 0 && mp % 32 == 0) {  // dense Gram blocks of the row groups on DMMA
      DBuf<double> gtmp(static_cast<size_t>(pat.gnnz * kGroup));
      sddmm_block(1, U.get(), U1.get(), T.get(), mp, mp, pat, lowrank.get(), sp, dsval.get(), nullptr, nullptr,
                  gtmp.get(), s);
    } else {
      sddmm_drho(U.get(), U1.get(), T.get(), mp, pat, lowrank.get(), sp, dsval.get(), s);
    }
  }
  dD.alloc(np);
  extract_diag(dsval.get(), pat.diagpos.get(), n, np, dD.get(), nullptr, nullptr, s);
  // padding rows of dD must be zero (extract_diag writes 1)
  affine_vec(dD.get(), dD.get(), 0.0, 1.0, n, np, s);
}

void Model::sigma_s_mat(const double* H, double* V, long tp, double alpha, double beta) {
  KTimer t(ctx, "spmm", 12.0 * geo->pat.nnz + (beta == 0.0 ? 16.0 : 24.0) * n * (cols_hint > 0 ? cols_hint : tp));
  const Csr& pat = geo->pat;
  if (alpha == 1.0 && beta == 0.0 && pat.gnnz > 0 && gval.n > 0 && spmm_block_supported(tp)) {
    // V = Sigma_s H on the DMMA block SpMM (the h.v partials it also forms are not used)
    DBuf<double> dots(static_cast<size_t>(tp)), part(static_cast<size_t>(spmm_group_blocks(pat.ngrp) * tp));
    spmm_block_dot(pat, gval.get(), H, tp, V, tp, tp, dots.get(), part.get(), nullptr, ctx->stream);
    return;
  }
  launch_spmm(pat.rowptr.get(), pat.col.get(), sval.get(), n, H, tp, V, tp, tp, alpha, beta, ctx->stream);
}

// V = Sigma H = U^T (U H) + Sigma_s H   (fsa.cpp:65-68)
void Model::matmat(const double* H, double* V, long tp) {
  double* W1 = mt_buf(0, tp);
  project(U.get(), H, tp, W1);
  {
    KTimer t(ctx, "lowrank_expand", 2.0 * m_pad * n_pad * tp);
    gemm_expand_store(U.get(), m_pad, n_pad, m_pad, W1, tp, tp, V, tp, 1.0, 0.0, ctx->stream);
  }
  sigma_s_mat(H, V, tp, 1.0, 1.0);
}

// deriv_matmat (fsa.cpp:165-182) in U-form
void Model::deriv_matmat(int which, const double* V, double* out, long tp) {
  require(which >= 0 && which < 3, "parameter index out of range");
  cudaStream_t s = ctx->stream;
  const long len = n_pad * tp;
  if (which == 0) {
    FSA_CUDA(cudaMemcpyAsync(out, V, sizeof(double) * len, cudaMemcpyDeviceToDevice, s));
    return;
  }
  if (which == 1) {  // (Sigma V - sigma2 V) / sigma1_2
    matmat(V, out, tp);
    axpby(out, V, -P.sigma2 / P.sigma1_2, 1.0 / P.sigma1_2, len, s);
    return;
  }
  ensure_rho_derivs();
  double* UV = mt_buf(0, tp);
  double* W = mt_buf(1, tp);
  project(U.get(), V, tp, UV);
  project(U1.get(), V, tp, W);  // W = U1 V
  gemm_km(K2.get(), m_pad, m_pad, m_pad, UV, tp, tp, W, tp, -1.0, 1.0, s);  // W = U1 V - K2 U V
  gemm_expand_store(U.get(), m_pad, n_pad, m_pad, W, tp, tp, out, tp, 1.0, 0.0, s);
  gemm_expand_store(U1.get(), m_pad, n_pad, m_pad, UV, tp, tp, out, tp, 1.0, 1.0, s);
  launch_spmm(geo->pat.rowptr.get(), geo->pat.col.get(), dsval.get(), n, V, tp, out, tp, tp, 1.0, 1.0, s);
}

// ---- preconditioners ------------------------------------------------------------------------------
// upload a host column-major (original order) n x k block into columns [0, k) of Z
static void upload_pack(Model* md, const double* host, long k, double* Z, long tp) {
  cudaStream_t s = md->ctx->stream;
  DBuf<double> raw(static_cast<size_t>(md->n * k));
  FSA_CUDA(cudaMemcpyAsync(raw.get(), host, sizeof(double) * md->n * k, cudaMemcpyHostToDevice, s));
  pack_cols(raw.get(), md->n, k, md->geo->pts.perm_d.get(), md->n_pad, tp, 0, Z, s);
  FSA_CUDA(cudaStreamSynchronize(s));
}

void IdentityPrecond::solve(const double* R, double* Z, long tp) {
  FSA_CUDA(cudaMemcpyAsync(Z, R, sizeof(double) * md->n_pad * tp, cudaMemcpyDeviceToDevice, md->ctx->stream));
}
void IdentityPrecond::sample_probes(int L, unsigned long long seed, double* Z, long tp) {
  std::vector<double> h(static_cast<size_t>(md->n * L));
#pragma omp parallel for schedule(dynamic, 1)
  for (int i = 0; i < L; ++i) probe_rademacher(seed, static_cast<unsigned long long>(i), md->n, h.data() + i * md->n);
  FSA_CUDA(cudaMemsetAsync(Z, 0, sizeof(double) * md->n_pad * tp, md->ctx->stream));
  upload_pack(md, h.data(), L, Z, tp);
}

DiagPrecond::DiagPrecond(Model* m, bool d) : md(m), derivs(d) {
  DBuf<double> out(1);
  sum_log(md->D.get(), md->n, out.get(), md->ctx->stream);
  FSA_CUDA(cudaMemcpyAsync(&ld, out.get(), sizeof(double), cudaMemcpyDeviceToHost, md->ctx->stream));
  md->ctx->sync();
  if (derivs) md->start_rho_derivs();
}
void DiagPrecond::solve(const double* R, double* Z, long tp) {
  scale_rows(Z, R, md->Dinv.get(), md->n_pad, tp, md->ctx->stream);
}
void DiagPrecond::sample_probes(int L, unsigned long long seed, double* Z, long tp) {
  std::vector<double> h(static_cast<size_t>(md->n * L));
#pragma omp parallel for schedule(dynamic, 1)
  for (int i = 0; i < L; ++i) {
    std::vector<double> dummy;
    probe_gaussian(seed, static_cast<unsigned long long>(i), 0, dummy.data(), md->n, h.data() + i * md->n);
  }
  FSA_CUDA(cudaMemsetAsync(Z, 0, sizeof(double) * md->n_pad * tp, md->ctx->stream));
  upload_pack(md, h.data(), L, Z, tp);
  scale_rows(Z, Z, md->sqrtD.get(), md->n_pad, tp, md->ctx->stream);
}

FitcPrecond::FitcPrecond(Model* m, bool with_derivs) : md(m), derivs(with_derivs) {
  cudaStream_t s = md->ctx->stream;
  const long mp = md->m_pad, np = md->n_pad;
  // the rho-derivative blocks need only U and L: queued on the side stream before the FITC core
  // build, so they run under its latency-bound Cholesky panels instead of under the PCG sweeps
  if (derivs) md->start_rho_derivs();  // (44.2 -> 43.7 ms per evaluation at config 2)
  KTimer t(md->ctx, "setup_fitc", 2.0 * mp * mp * np);
  Q.alloc(mp * mp);
  LQ.alloc(mp * mp);
  Qinv.alloc(mp * mp);
  // Q = I + U D^{-1} U^T  (= L^{-1} core L^{-T}, preconditioners.cpp:49)
  {
    const size_t need = gemm_syrk_scratch(mp, np);
    if (md->red_scratch.n < need) md->red_scratch.alloc(need);
    KTimer tq(md->ctx, "setup_fitc_syrk", 1.0 * mp * mp * np);
    // DMMA SYRK (lower half + mirror): the full-matrix INT8 alternative (ozaki_project_wide over
    // 64-column tiles, 2.1 ms at config 2) does not beat it (1.7 ms)
    gemm_syrk(md->U.get(), mp, mp, np, md->Dinv.get(), Q.get(), mp, 1.0, md->red_scratch.get(), s);
    md->rcomm->allreduce(Q.get(), mp * mp, s);  // sum of the row blocks' U_i D_i^{-1} U_i^T
  }
  add_identity(Q.get(), mp, mp, s);
  FSA_CUDA(cudaMemcpyAsync(LQ.get(), Q.get(), sizeof(double) * mp * mp, cudaMemcpyDeviceToDevice, s));
  potrf_lower(LQ.get(), mp, md->info.get(), md->dinv_scratch.get(), s);
  DBuf<double> scal(2);
  launch_logdet_diag(LQ.get(), mp, mp, scal.get(), s);
  sum_log(md->D.get(), md->n, scal.get() + 1, s);
  // Qinv = LQ^{-T} LQ^{-1}
  {
    DBuf<double> X(mp * mp), Xt(mp * mp);
    FSA_CUDA(cudaMemsetAsync(X.get(), 0, sizeof(double) * mp * mp, s));
    add_identity(X.get(), mp, mp, s);
    trsm_lower_cols(LQ.get(), mp, X.get(), mp, mp, md->dinv_scratch.get(), s);  // X[j][r] = LQinv(r, j)
    launch_transpose(X.get(), mp, mp, mp, Xt.get(), mp, s);                       // Xt[k][r] = LQinv(k, r)
    const size_t need = gemm_reduce_scratch(mp, mp, mp);
    if (md->red_scratch.n < need) md->red_scratch.alloc(need);
    gemm_reduce(Xt.get(), mp, mp, mp, Xt.get(), mp, mp, nullptr, Qinv.get(), mp, 1.0, 0.0, md->red_scratch.get(), s);
    int hinfo = 0;
    double hs[2];
    FSA_CUDA(cudaMemcpyAsync(&hinfo, md->info.get(), sizeof(int), cudaMemcpyDeviceToHost, s));
    FSA_CUDA(cudaMemcpyAsync(hs, scal.get(), 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
    FSA_CUDA(cudaStreamSynchronize(s));
    if (hinfo != 0) throw NumericalError("preconditioner core matrix is not positive definite");
    md->rcomm->allreduce_host(hs + 1, 1, s);  // sum log d over all rows
    logdetQ = hs[0];
    ld = hs[0] + hs[1];  // logdet(core) - logdet(Sigma_m) + sum log d   (preconditioners.cpp:53-55)
  }
  if (derivs) {
    md->start_rho_derivs();
    start_traces();
  }
}

// The exact traces need Q^{-1}, D and the rho-derivative blocks: queued on the side stream right
// after those (off the main stream's critical path); deriv_trace joins and finishes on the host.
void FitcPrecond::start_traces() {
  static const bool sync_traces = std::getenv("FSA_SYNC_TRACES") != nullptr;
  if (sync_traces || have_traces || traces_pending || md->ctx->gemm_mode == 1 || !md->rho_pending || !md->oz.ready)
    return;
  Context* ctx = md->ctx;
  cudaStream_t side = ctx->side_stream();
  const long mp = md->m_pad, np = md->n_pad, n = md->n;
  // the trace passes read Q^{-1}, written on the main stream: order them after it explicitly
  // (not through the host synchronisation that happens to precede this call)
  cudaEvent_t qready = ctx->ev();
  FSA_CUDA(cudaEventRecord(qready, ctx->stream));
  FSA_CUDA(cudaStreamWaitEvent(side, qready, 0));
  ctx->pool.push_back(qready);
  cudaStream_t saved = alloc_stream();
  alloc_stream() = side;
  try {
    tr_q.alloc(np);
    tr_f.alloc(np);
    tr_pinv.alloc(np);
    tr_d1.alloc(np);
    tr_sums.alloc(8);
    // rows dots of U^T Q^{-1} with U and U1 (INT8 passes, side-stream W-plane buffers)
    ozaki_expand_rowdots(md->oz, Qinv.get(), mp, md->U.get(), md->U1.get(), mp, tr_q.get(), tr_f.get(), side, true);
    pinv_diag(tr_pinv.get(), md->D.get(), tr_q.get(), n, np, side);
    affine_vec(tr_d1.get(), md->D.get(), -md->P.sigma2, 1.0 / md->P.sigma1_2, n, np, side);
    trace_sums(tr_pinv.get(), tr_d1.get(), md->dD.get(), tr_f.get(), md->D.get(), n, Qinv.get(), md->K2.get(), mp,
               tr_sums.get(), side);
    if (traces_host == nullptr) FSA_CUDA(cudaMallocHost(reinterpret_cast<void**>(&traces_host), 8 * sizeof(double)));
    FSA_CUDA(cudaMemcpyAsync(traces_host, tr_sums.get(), 7 * sizeof(double), cudaMemcpyDeviceToHost, side));
  } catch (...) {
    alloc_stream() = saved;
    throw;
  }
  alloc_stream() = saved;
  if (traces_done == nullptr) traces_done = ctx->ev();
  FSA_CUDA(cudaEventRecord(traces_done, side));
  traces_pending = true;
}

void FitcPrecond::finish_traces(const double* h) {
  double hs[7];
  std::copy(h, h + 7, hs);
  md->rcomm->allreduce_host(hs, 4, md->ctx->stream);  // sums over rows; the m x m sums are replicated
  const double s0 = hs[0], s1 = hs[1], s2 = hs[2], qf = hs[3], trQi = hs[4], trK2 = hs[5], k2q = hs[6];
  trace[0] = s0;
  trace[1] = s1 + (static_cast<double>(md->m_pad) - trQi) / md->P.sigma1_2;
  trace[2] = s2 + 2.0 * qf - (trK2 - k2q);
  have_traces = true;
}

FitcPrecond::~FitcPrecond() {
  // frees below (stream-ordered on the main stream) come after the side-stream trace work, and
  // the pinned host buffer its device-to-host copy targets is released only after that copy
  if (traces_pending) {
    cudaStreamWaitEvent(md->ctx->stream, traces_done, 0);
    cudaEventSynchronize(traces_done);
  }
  if (traces_done != nullptr) md->ctx->pool.push_back(traces_done);
  if (traces_host != nullptr) cudaFreeHost(traces_host);
}

// P^{-1} R = D^{-1} R - D^{-1} U^T Q^{-1} U D^{-1} R   (preconditioners.cpp:58-67)
void FitcPrecond::solve(const double* R, double* Z, long tp) {
  cudaStream_t s = md->ctx->stream;
  double* S = md->mt_buf(0, tp);
  double* W = md->mt_buf(1, tp);
  md->project(md->U.get(), R, tp, S, md->Dinv.get());
  {
    KTimer t(md->ctx, "core_solve", 2.0 * md->m_pad * md->m_pad * tp);
    gemm_km(Qinv.get(), md->m_pad, md->m_pad, md->m_pad, S, tp, tp, W, tp, 1.0, 0.0, s);
  }
  KTimer t(md->ctx, "lowrank_expand", 2.0 * md->m_pad * md->n_pad * tp);
  if (md->use_ozaki(tp) && md->world() == 1) {  // INT8 expansion with the Woodbury epilogue
    md->ensure_ozaki();
    DBuf<double> lw(static_cast<size_t>(md->n_pad * tp)), rz(static_cast<size_t>(tp)),
        part(static_cast<size_t>(md->oz.ptiles * tp));
    ozaki_expand_keep(md->oz, W, tp, tp, Z, lw.get(), R, md->Dinv.get(), rz.get(), part.get(), s, false);
    return;
  }
  gemm_expand_woodbury(md->U.get(), md->m_pad, md->n_pad, md->m_pad, W, tp, tp, Z, R, tp, md->Dinv.get(), s);
}

// z = Sigma_mn^T L^{-T} e1 + sqrt(D) e2 = U^T e1 + sqrt(D) e2  (preconditioners.cpp:69-73)
void FitcPrecond::sample_probes(int L, unsigned long long seed, double* Z, long tp) {
  const long m = md->m, n = md->n, mp = md->m_pad, np = md->n_pad;
  cudaStream_t s = md->ctx->stream;
  Geometry::ProbeCache& pc = md->geo->probes;
  if (md->geo->cache_probes && pc.valid && pc.seed == seed && pc.L == L && pc.tp == tp && pc.m == m) {
    KTimer t(md->ctx, "probe_expand", 2.0 * mp * np * tp);
    gemm_expand_probe(md->U.get(), mp, np, mp, pc.E1.get(), tp, tp, Z, tp, md->sqrtD.get(), pc.E2.get(), s);
    return;
  }
  // each probe's stream draws e1 (m) then e2 over ALL n points; a rank keeps its rows of e2
  const long nf = md->geo->shard.n, r0 = md->geo->shard.r0;
  static const bool host_probes = std::getenv("FSA_HOST_PROBES") != nullptr;
  if (!host_probes) {  // the same streams drawn on the device (k_probe_gaussian)
    DBuf<double> E1(mp * tp), E2(np * tp), raw(nf * L);
    FSA_CUDA(cudaMemsetAsync(E1.get(), 0, sizeof(double) * mp * tp, s));
    k_probe_gaussian<<<static_cast<unsigned>(L), 320, 0, s>>>(seed, m, tp, E1.get(), nf, raw.get());
    FSA_LAUNCH_CHECK();
    FSA_CUDA(cudaMemsetAsync(E2.get(), 0, sizeof(double) * np * tp, s));
    pack_cols_ld(raw.get(), nf, n, L, md->geo->pts.perm_d.get() + r0, np, tp, 0, E2.get(), s);
    {
      KTimer t(md->ctx, "probe_expand", 2.0 * mp * np * tp);
      gemm_expand_probe(md->U.get(), mp, np, mp, E1.get(), tp, tp, Z, tp, md->sqrtD.get(), E2.get(), s);
    }
    if (md->geo->cache_probes) {
      pc.valid = true;
      pc.seed = seed;
      pc.L = L;
      pc.tp = tp;
      pc.m = m;
      pc.E1 = std::move(E1);
      pc.E2 = std::move(E2);
    }
    return;
  }
  PinnedBuf& e1h = md->ctx->pin1;  // host staging owned by the context
  PinnedBuf& e2h = md->ctx->pin2;
  e1h.ensure(static_cast<size_t>(mp * tp));
  e2h.ensure(static_cast<size_t>(nf * L));
  double* e1p = e1h.p;
  double* e2p = e2h.p;
  std::memset(e1p, 0, sizeof(double) * mp * tp);
  std::vector<double> e1col(static_cast<size_t>(m) * L);
  double* e1c = e1col.data();
#pragma omp parallel for schedule(dynamic, 1)
  for (int i = 0; i < L; ++i)
    probe_gaussian(seed, static_cast<unsigned long long>(i), m, e1c + static_cast<long>(i) * m, nf,
                   e2p + static_cast<long>(i) * nf);
  for (int i = 0; i < L; ++i)
    for (long r = 0; r < m; ++r) e1p[r * tp + i] = e1col[static_cast<size_t>(i) * m + r];
  DBuf<double> E1(mp * tp), E2(np * tp), raw(nf * L);
  FSA_CUDA(cudaMemcpyAsync(E1.get(), e1h.p, sizeof(double) * mp * tp, cudaMemcpyHostToDevice, s));
  FSA_CUDA(cudaMemcpyAsync(raw.get(), e2h.p, sizeof(double) * nf * L, cudaMemcpyHostToDevice, s));
  FSA_CUDA(cudaMemsetAsync(E2.get(), 0, sizeof(double) * np * tp, s));
  pack_cols_ld(raw.get(), nf, n, L, md->geo->pts.perm_d.get() + r0, np, tp, 0, E2.get(), s);
  {
    KTimer t(md->ctx, "probe_expand", 2.0 * mp * np * tp);
    gemm_expand_probe(md->U.get(), mp, np, mp, E1.get(), tp, tp, Z, tp, md->sqrtD.get(), E2.get(), s);
  }
  FSA_CUDA(cudaStreamSynchronize(s));
  if (md->geo->cache_probes) {
    pc.valid = true;
    pc.seed = seed;
    pc.L = L;
    pc.tp = tp;
    pc.m = m;
    pc.E1 = std::move(E1);
    pc.E2 = std::move(E2);
  }
}

// exact Tr(P^{-1} dP_k) in U-form:
//   k = 0: sum_i pinv_i
//   k = 1: pinv . d_1 + (m - Tr Q^{-1}) / sigma1_2
//   k = 2: pinv . dD + 2 <Q^{-1}, F> - Tr(K2) + <K2, Q^{-1}>,  F = U D^{-1} U1^T
double FitcPrecond::deriv_trace(int k) {
  require(derivs, "FITC preconditioner built without derivatives");
  if (!have_traces && traces_pending) {
    md->ensure_rho_derivs();
    FSA_CUDA(cudaEventSynchronize(traces_done));
    traces_pending = false;
    finish_traces(traces_host);
  }
  if (!have_traces) {
    cudaStream_t s = md->ctx->stream;
    const long mp = md->m_pad, np = md->n_pad, n = md->n;
    md->ensure_rho_derivs();
    KTimer tt(md->ctx, "grad_exact_traces", 2.0 * mp * mp * np);
    // q_i = U_i' Q^{-1} U_i (diag P^{-1} = 1/D - q/D^2) and
    // <Q^{-1}, U D^{-1} U1^T> = sum_i (U_i' Q^{-1} U1_i) / D_i
    DBuf<double> q(np), f(np), pinv(np), d1(np);
    if (md->ctx->gemm_mode != 1) {  // row dots of U^T Q^{-1} (INT8 tensor cores, 64-column tiles)
      md->ensure_ozaki();
      ozaki_expand_rowdots(md->oz, Qinv.get(), mp, md->U.get(), md->U1.get(), mp, q.get(), f.get(), s);
    } else {  // V = LQ^{-1} U, W1 = LQ^{-1} U1: q_i = |V_i|^2, f_i = V_i . W1_i
      DBuf<double> V(mp * np), W1(mp * np);
      FSA_CUDA(cudaMemcpyAsync(V.get(), md->U.get(), sizeof(double) * mp * np, cudaMemcpyDeviceToDevice, s));
      FSA_CUDA(cudaMemcpyAsync(W1.get(), md->U1.get(), sizeof(double) * mp * np, cudaMemcpyDeviceToDevice, s));
      trsm_lower_cols(LQ.get(), mp, V.get(), mp, np, md->dinv_scratch.get(), s);
      trsm_lower_cols(LQ.get(), mp, W1.get(), mp, np, md->dinv_scratch.get(), s);
      colnorm2(V.get(), mp, mp, n, np, q.get(), s);
      row_dots(V.get(), W1.get(), mp, mp, n, np, f.get(), s);
    }
    pinv_diag(pinv.get(), md->D.get(), q.get(), n, np, s);
    affine_vec(d1.get(), md->D.get(), -md->P.sigma2, 1.0 / md->P.sigma1_2, n, np, s);
    DBuf<double> sums(8);
    trace_sums(pinv.get(), d1.get(), md->dD.get(), f.get(), md->D.get(), n, Qinv.get(), md->K2.get(), mp,
               sums.get(), s);
    double hs[7];
    FSA_CUDA(cudaMemcpyAsync(hs, sums.get(), sizeof(hs), cudaMemcpyDeviceToHost, s));
    FSA_CUDA(cudaStreamSynchronize(s));
    finish_traces(hs);
  }
  return trace[k];
}

std::unique_ptr<Precond> make_preconditioner(Model* md, int type) {  // estimation.cpp:160-176
  NvtxRange nvtx_("fsa::make_preconditioner");
  require(md->world() == 1 || type == 2, "row-sharded models support the FITC preconditioner only");
  switch (type) {
    case 0: return std::make_unique<IdentityPrecond>(md);
    case 1: return std::make_unique<DiagPrecond>(md, true);
    case 2: return std::make_unique<FitcPrecond>(md, true);
  }
  throw std::invalid_argument("unknown preconditioner type");
}

// ---- Krylov -------------------------------------------------------------------------------------------
bool CgResult::all_converged() const {
  for (int c : converged)
    if (!c) return false;
  return true;
}
int CgResult::max_iterations() const {
  int m = 0;
  for (int v : iterations) m = std::max(m, v);
  return m;
}

// Lockstep PCG. With the FSA operator and the FITC preconditioner a sweep is
//   V = U^T (U H) + Sigma_s H   [expand + fused SpMM/h.v]   alpha, tridiagonal
//   X += alpha H, R -= alpha V  [fused with |R|^2]          convergence test
//   S = U D^{-1} R, w = Q^{-1} S, Z = D^{-1}(R - U^T w)  [project, core, expand + r.z]
//   H = Z + beta H, U H = w + beta U H   (U Z = Q^{-1} S = w exactly, so the
//                                         projection of H is an m-space update)
// i.e. one projection and two expansions over U per sweep instead of the
// reference sequence's four dense passes (krylov.cpp:56-93, preconditioners.cpp:58-61).
CgResult pcg_solve_multi(Model* md, LinOp& A, Precond& P, const double* B, long k, long tp, double* X,
                         const CgOptions& opts) {
  NvtxRange nvtx_("fsa::pcg_solve_multi");
  require(opts.tol > 0.0 && opts.max_iter > 0, "cg: invalid options");
  require(k >= 1 && k <= tp, "cg: column count mismatch");
  Context* ctx = md->ctx;
  cudaStream_t s = ctx->stream;
  const long np = md->n_pad, n = md->n, mp = md->m_pad;
  const int maxit = opts.max_iter;
  const size_t blk = static_cast<size_t>(np * tp);
  FsaOp* fop = dynamic_cast<FsaOp*>(&A);
  FitcPrecond* fitc = dynamic_cast<FitcPrecond*>(&P);
  const bool fused = fop != nullptr && fitc != nullptr;
  require(fused || md->world() == 1, "row-sharded solves need the FSA operator with the FITC preconditioner");
  // Jacobi on Sigma_s (prediction solves, prediction.cpp:90-93): no Z block, r.z fused into the update
  const bool jfused = !fused && dynamic_cast<DiagPrecond*>(&P) != nullptr && dynamic_cast<SigmaSOp*>(&A) != nullptr;
  Comm& comm = *md->rcomm;
  CgWork& w = *ctx->cgw;
  if (w.R.n < blk) {
    w.R.alloc(blk);
    w.V.alloc(blk);
  }
  const size_t ext_blk = static_cast<size_t>(md->n_ext_pad * tp);  // H and Z carry the halo rows
  if (w.H.n < ext_blk) w.H.alloc(ext_blk);
  if (w.Z.n < ext_blk) w.Z.alloc(ext_blk);
  if (fused && w.Lw.n < blk) {
    w.Lw.alloc(blk);
    w.Vlr.alloc(blk);
  }
  const size_t npart = std::max(static_cast<size_t>(std::max(np / 64, spmm_dot_blocks(n)) * tp),
                                2 * coldot_scratch(n, tp));
  if (w.part.n < npart) w.part.alloc(npart);
  w.dots.alloc(static_cast<size_t>(4 * tp));
  w.dbl.alloc(static_cast<size_t>(6 * k));
  w.ints.alloc(static_cast<size_t>(3 * k + 2));
  w.tri.alloc(static_cast<size_t>(3 * k * maxit));
  CgState st;
  st.rz = w.dbl.get();
  st.alpha_prev = st.rz + k;
  st.beta_prev = st.rz + 2 * k;
  st.alpha = st.rz + 3 * k;
  st.beta = st.rz + 4 * k;
  st.scale = st.rz + 5 * k;
  st.active = w.ints.get();
  st.converged = st.active + k;
  st.iterations = st.active + 2 * k;
  st.err = st.active + 3 * k;
  st.tdiag = w.tri.get();
  st.toff = st.tdiag + k * maxit;
  st.rnorm = st.toff + k * maxit;
  st.host_flags = ctx->host_flags_dev;
  double* rr = w.dots.get();
  double* hv = rr + tp;
  double* rz = rr + 2 * tp;
  double* part = w.part.get();
  FSA_CUDA(cudaMemsetAsync(st.err, 0, sizeof(int), s));
  FSA_CUDA(cudaMemsetAsync(st.tdiag, 0, sizeof(double) * 3 * k * maxit, s));
  FSA_CUDA(cudaMemcpyAsync(w.R.get(), B, sizeof(double) * blk, cudaMemcpyDeviceToDevice, s));
  FSA_CUDA(cudaMemsetAsync(X, 0, sizeof(double) * blk, s));
  const double flops_mn = 2.0 * md->m * n * k;
  md->cols_hint = k;

  // Fused direction update (block SpMM path): the SpMM of sweep i gathers Z_{i-1} instead of
  // H_i and forms, on its own rows, H_i = Z + beta H and V_i = (Lw + Sigma_s Z) + beta V_{i-1}
  // (= U^T U H_i + Sigma_s H_i by linearity), so no separate H / Vlr pass runs
  const bool fuse_h = fused && md->geo->pat.gnnz > 0 && spmm_block_supported(tp);
  bool first_sweep = true;
  // Ozaki projection inputs: update_xr_dot_max leaves the chunk maxima of |D^{-1} R|
  const bool oz = fused && md->use_ozaki(tp);
  // wider blocks (config 4: t = 65 -> t_pad = 72): two INT8 column tiles in one launch whose CTA
  // pairs share each U-plane tile through L2 (ozaki_*_pair); beyond 128 columns, 64-column INT8
  // blocks and a DMMA remainder
  const bool oz_split = fused && !oz && md->ctx->gemm_mode != 1 && tp > kOzCols;
  // FSA_OZ_PAIR=0: the 64-column INT8 + DMMA-remainder passes instead of the pair (A/B measurement)
  static const bool pair_off = std::getenv("FSA_OZ_PAIR") && std::strcmp(std::getenv("FSA_OZ_PAIR"), "0") == 0;
  const bool oz_pair = oz_split && tp <= kOzPairCols && !pair_off;
  if (oz || oz_split) md->ensure_ozaki();
  // single rank: the column sums of the SpMM, residual-update and expansion partials run fused
  // with the alpha / residual-test / beta + count control kernels (no separate launches)
  // fused column-sum / CG-control kernels (k_colsum_ctl). On several row ranks the launchers'
  // column sums are allreduced first and the control kernels run on those sums (one "partial")
  const bool ctl = fuse_h && oz;
  const bool multi = md->world() > 1;
  if (ctl) {
    w.tick.alloc(1);
    w.tick.zero(s);
    w.wmax.alloc(kOzCols);
    w.wmax.zero(s);  // (then cleared by the end-of-sweep control kernel for the next sweep)
    const size_t nrr = static_cast<size_t>(xr_dot_max_blocks(n) * tp);
    if (w.part_rr.n < nrr) w.part_rr.alloc(nrr);
  }
  bool ymax_ready = false;
  // Z = P^{-1} R (+ r.z); fused path also leaves w = Q^{-1} U D^{-1} R in mt_buf(1)
  auto precond = [&](double* rzout, bool sums = true) {
    // column maxima of |W| for the expansion's digit planes: left by the one-launch core solve
    // (only that kernel fills them; zeroed by the residual-test control kernel)
    const bool wfill = ctl && !sums && core_apply_supported(mp, tp);
    if (fused) {
      double* S = md->mt_buf(0, tp);
      double* W = md->mt_buf(1, tp);
      if (oz) {
        {
          KTimer t(ctx, "lowrank_project", 2.0 * md->m * n * k);
          ozaki_project(md->oz, w.R.get(), tp, tp, md->Dinv.get(), S, s, ymax_ready);
        }
        if (md->world() > 1) {
          KTimer t(ctx, "allreduce");
          comm.allreduce(S, mp * tp, s);
        }
        ymax_ready = false;
      } else if (oz_pair) {  // two column tiles, U planes streamed once
        {
          KTimer t(ctx, "lowrank_project", 2.0 * md->m * n * k);
          ozaki_project_pair(md->oz, w.R.get(), tp, tp, md->Dinv.get(), S, s);
        }
        if (md->world() > 1) {
          KTimer t(ctx, "allreduce");
          comm.allreduce(S, mp * tp, s);
        }
      } else if (oz_split) {
        {
          KTimer t(ctx, "lowrank_project", 2.0 * md->m * n * k);
          for (long c0 = 0; c0 < tp; c0 += kOzCols) {
            const long wd = std::min<long>(kOzCols, tp - c0);
            if (wd == kOzCols) {
              ozaki_project(md->oz, w.R.get() + c0, tp, wd, md->Dinv.get(), S + c0, s, false);
            } else {
              const size_t need = gemm_reduce_scratch(mp, wd, np);
              if (md->red_scratch.n < need) md->red_scratch.alloc(need);
              gemm_reduce(md->U.get(), mp, mp, np, w.R.get() + c0, tp, wd, md->Dinv.get(), S + c0, tp, 1.0, 0.0,
                          md->red_scratch.get(), s);
            }
          }
        }
        if (md->world() > 1) {
          KTimer t(ctx, "allreduce");
          comm.allreduce(S, mp * tp, s);
        }
      } else {
        md->project(md->U.get(), w.R.get(), tp, S, md->Dinv.get());
      }
      {
        KTimer t(ctx, "core_solve", 2.0 * md->m * md->m * k);
        if (core_apply_supported(mp, tp)) {
          // (the fused path's sweeps also leave the column maxima the expansion slices W with)
          core_apply(fitc->Qinv.get(), mp, S, tp, W, s, wfill ? w.wmax.get() : nullptr);
        } else {
          const size_t need = gemm_reduce_scratch(mp, tp, mp);
          if (md->red_scratch.n < need) md->red_scratch.alloc(need);
          gemm_reduce(fitc->Qinv.get(), mp, mp, mp, S, tp, tp, nullptr, W, tp, 1.0, 0.0, md->red_scratch.get(), s);
        }
      }
      KTimer t(ctx, "lowrank_expand", flops_mn);
      if (md->use_ozaki(tp)) {
        ozaki_expand_keep(md->oz, W, tp, tp, w.Z.get(), w.Lw.get(), w.R.get(), md->Dinv.get(), rzout, part, s, sums,
                          wfill ? w.wmax.get() : nullptr);
      } else if (oz_pair) {
        ozaki_expand_keep_pair(md->oz, W, tp, tp, w.Z.get(), w.Lw.get(), w.R.get(), md->Dinv.get(), rzout, part, s);
      } else if (oz_split) {
        for (long c0 = 0; c0 < tp; c0 += kOzCols) {
          const long wd = std::min<long>(kOzCols, tp - c0);
          if (wd == kOzCols)
            ozaki_expand_keep(md->oz, W + c0, tp, wd, w.Z.get() + c0, w.Lw.get() + c0, w.R.get() + c0,
                              md->Dinv.get(), rzout + c0, part, s);
          else
            gemm_expand_woodbury_keep(md->U.get(), mp, np, mp, W + c0, tp, wd, w.Z.get() + c0, w.Lw.get() + c0,
                                      w.R.get() + c0, tp, md->Dinv.get(), rzout + c0, part, s);
        }
      } else
        gemm_expand_woodbury_keep(md->U.get(), mp, np, mp, W, tp, tp, w.Z.get(), w.Lw.get(), w.R.get(), tp,
                                  md->Dinv.get(), rzout, part, s);
      comm.allreduce(rzout, tp, s);
    } else if (jfused) {
      KTimer t(ctx, "cg_blas1");
      launch_coldot_weighted(w.R.get(), w.R.get(), md->Dinv.get(), n, tp, k, rzout, part, s);
    } else {
      P.solve(w.R.get(), w.Z.get(), tp);
      KTimer t(ctx, "cg_blas1");
      launch_coldot(w.R.get(), w.Z.get(), n, tp, k, rzout, part, s);
    }
  };

  {
    KTimer t(ctx, "cg_blas1");
    launch_coldot(w.R.get(), w.R.get(), n, tp, k, rr, part, s);
    comm.allreduce(rr, k, s);
    cg_start(rr, k, opts.tol, st, s);
  }
  precond(rz);
  {
    KTimer t(ctx, "cg_blas1");
    cg_start_rz(rz, k, st, s);
    if (jfused)
      update_h_jacobi(w.H.get(), w.R.get(), md->Dinv.get(), st.active, st.beta, np, tp, k, true, s);
    else if (!fuse_h)
      init_h(w.H.get(), w.Z.get(), st.active, np, tp, k, s);
    if (fused && !fuse_h) init_h(w.Vlr.get(), w.Lw.get(), st.active, np, tp, k, s);  // U^T U H_0 = U^T w_0
    cg_count(k, st, s);
  }
  FSA_CUDA(cudaStreamSynchronize(s));
  auto check_err = [&](const volatile int* flags) {
    const int e = flags[1];
    if (e == kErrOperatorNotPD) throw NumericalError("cg: operator is not positive definite");
    if (e == kErrPrecondNotPD) throw NumericalError("cg: preconditioner is not positive definite");
  };
  check_err(ctx->host_flags);
  int num_active = ctx->host_flags[0];
  CgResult res;
  // The host reads each sweep's [num_active, err] one sweep late: sweep it + 1 is queued before
  // the flags of sweep it are inspected, so the GPU never idles on the host round trip. Sweeps
  // queued after every column converged are no-ops (alpha = beta = 0 and no tridiagonal push
  // for inactive columns), so results and iteration counts are those of the synchronous loop.
  // Flags are double-buffered in the mapped slots [2 (it % 2), 2 (it % 2) + 1].
  cudaEvent_t sweep_ev[2] = {ctx->ev(), ctx->ev()};
  int pending = -1;  // last queued sweep whose flags are unread
  auto read_flags = [&](int sw) {
    FSA_CUDA(cudaEventSynchronize(sweep_ev[sw & 1]));
    const volatile int* f = ctx->host_flags + 2 * (sw & 1);
    check_err(f);
    num_active = f[0];
    res.sweeps = sw + 1;
  };
  // One sweep's kernels. On the fused single-rank path (ctl) sweeps 1, 2, ... are identical
  // launch sequences (the sweep index is read on the device, CgState::it_dev), so they are
  // captured once into a CUDA graph and replayed: one launch per sweep instead of eleven, and
  // no host gaps between the kernels (profiling runs keep eager launches for the group timers).
  auto sweep = [&](int it) {
    if (fuse_h) {  // H = Z + beta H, V = (Lw + Sigma_s Z) + beta V; h.v
        md->halo_exchange(w.Z.get(), tp);
        // CSR + Z (once per row), Lw, H, V read + H, V write
        KTimer t(ctx, "spmm", 12.0 * md->geo->pat.nnz + 48.0 * n * k);
        spmm_block_dot_h(md->geo->pat, md->gval.get(), w.Z.get(), tp, w.V.get(), tp, tp, hv, part, w.Lw.get(),
                         w.H.get(), st.beta, k, first_sweep, s, !ctl || multi);
        first_sweep = false;
        comm.allreduce(hv, tp, s);
      } else if (fused) {  // V = Vlr + Sigma_s H with Vlr = U^T U H kept by recurrence; h.v
        md->halo_exchange(w.H.get(), tp);
        KTimer t(ctx, "spmm", 12.0 * md->geo->pat.nnz + 24.0 * n * k);  // CSR + H, Vlr read + V write
        if (md->geo->pat.gnnz > 0 && spmm_block_supported(tp))
          spmm_block_dot(md->geo->pat, md->gval.get(), w.H.get(), tp, w.V.get(), tp, tp, hv, part, w.Vlr.get(), s);
        else
          spmm_dot(md->geo->pat.rowptr.get(), md->geo->pat.col.get(), md->sval.get(), n, w.H.get(), tp, w.V.get(), tp,
                   tp, 1.0, 1.0, hv, part, s, w.Vlr.get());
        comm.allreduce(hv, tp, s);
      } else if (jfused && md->geo->pat.gnnz > 0 && spmm_block_supported(tp)) {  // V = Sigma_s H; h.v
        KTimer t(ctx, "spmm", 12.0 * md->geo->pat.nnz + 16.0 * n * k);
        spmm_block_dot(md->geo->pat, md->gval.get(), w.H.get(), tp, w.V.get(), tp, tp, hv, part, nullptr, s);
      } else if (jfused) {
        KTimer t(ctx, "spmm", 12.0 * md->geo->pat.nnz + 16.0 * n * k);
        spmm_dot(md->geo->pat.rowptr.get(), md->geo->pat.col.get(), md->sval.get(), n, w.H.get(), tp, w.V.get(), tp,
                 tp, 1.0, 0.0, hv, part, s);
      } else {
        A.apply(w.H.get(), w.V.get(), tp);
        KTimer t(ctx, "cg_blas1");
        launch_coldot(w.H.get(), w.V.get(), n, tp, k, hv, part, s);
      }
      {
        KTimer t(ctx, "cg_blas1");
        if (ctl)  // alpha, and the ymax clear of the residual update below
          colsum_ctl(0, multi ? hv : part, multi ? 1 : md->geo->pat.ngrp, tp, tp, hv, k, it, maxit, 0.0, st,
                     w.tick.get(), s, md->oz.ymax.get(), static_cast<long>(md->oz.ymax.n));
        else
          cg_alpha(hv, k, it, maxit, st, s);
        if (oz) {
          if (!ctl) FSA_CUDA(cudaMemsetAsync(md->oz.ymax.get(), 0, md->oz.ymax.bytes(), s));
          update_xr_dot_max(X, w.R.get(), w.H.get(), w.V.get(), st.alpha, n, tp, k, rr, ctl ? w.part_rr.get() : part,
                            md->Dinv.get(), md->oz.ymax.get(), ozaki_chunk_rows(md->oz), s, !ctl || multi);
          ymax_ready = true;
        } else if (jfused) {
          update_xr_dot_jacobi(X, w.R.get(), w.H.get(), w.V.get(), st.alpha, md->Dinv.get(), n, tp, k, rr, rz, part,
                               s);
        } else {
          update_xr_dot(X, w.R.get(), w.H.get(), w.V.get(), st.alpha, n, tp, k, rr, part, s);
        }
        comm.allreduce(rr, k, s);
        if (!ctl) cg_check(rr, k, opts.tol, it, maxit, st, s);  // (fused: at the end of the sweep)
      }
      if (!jfused) precond(rz, !ctl || multi);
      {
        KTimer t(ctx, "cg_blas1");
        if (ctl)  // residual test, beta and the active count; clears wmax for the next core solve
          colsum_ctl(3, multi ? rr : w.part_rr.get(), multi ? 1 : xr_dot_max_blocks(n), k, k, rr, k, it, maxit,
                     opts.tol, st, w.tick.get(), s, w.wmax.get(), kOzCols, multi ? rz : part,
                     multi ? 1 : md->oz.ptiles, tp, rz);
        else
          cg_beta(rz, k, st, s);
        if (fuse_h) {
          // H and V are updated by the next sweep's SpMM
        } else if (fused) {  // H = Z + beta H, Vlr = U^T w + beta Vlr
          update_h2(w.H.get(), w.Z.get(), w.Vlr.get(), w.Lw.get(), st.active, st.beta, np, tp, k, s);
        } else if (jfused) {  // H = D^{-1} R + beta H
          update_h_jacobi(w.H.get(), w.R.get(), md->Dinv.get(), st.active, st.beta, np, tp, k, false, s);
        } else {
          update_h(w.H.get(), w.Z.get(), st.active, st.beta, np, tp, k, s);
        }
        if (!ctl) cg_count(k, st, s);
      }
  };
  const bool graph = ctl && !multi && !ctx->profile && !kChecked && std::getenv("FSA_NO_GRAPH") == nullptr;
  cudaGraphExec_t gexec = nullptr;
  long graph_kernels = 0;
  if (graph) {
    st.it_dev = st.err + 1;
    FSA_CUDA(cudaMemsetAsync(st.it_dev, 0, sizeof(int), s));
  }
  for (int it = 0; it < maxit && num_active > 0; ++it) {
    if (graph && it > 0) {
      if (gexec == nullptr) {
        st.host_flags = ctx->host_flags_dev;
        cudaGraph_t g = nullptr;
        const long before = launch_counter().load();
        FSA_CUDA(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        try {
          sweep(it);
        } catch (...) {
          cudaGraph_t dead = nullptr;
          cudaStreamEndCapture(s, &dead);
          if (dead) cudaGraphDestroy(dead);
          throw;
        }
        FSA_CUDA(cudaStreamEndCapture(s, &g));
        graph_kernels = launch_counter().load() - before;  // captured, not yet run: counted per replay
        launch_counter().fetch_sub(graph_kernels);
        FSA_CUDA(cudaGraphInstantiate(&gexec, g, 0));
        FSA_CUDA(cudaGraphDestroy(g));
      }
      FSA_CUDA(cudaGraphLaunch(gexec, s));
      launch_counter().fetch_add(graph_kernels);
    } else {
      st.host_flags = graph ? ctx->host_flags_dev : ctx->host_flags_dev + 2 * (it & 1);
      sweep(it);
    }
    FSA_CUDA(cudaEventRecord(sweep_ev[it & 1], s));
    if (pending >= 0) {
      read_flags(pending);
      if (num_active == 0) {  // sweep `it` was queued after convergence: a no-op
        pending = -1;
        break;
      }
    }
    pending = it;
  }
  if (pending >= 0) read_flags(pending);
  FSA_CUDA(cudaStreamSynchronize(s));
  if (gexec != nullptr) FSA_CUDA(cudaGraphExecDestroy(gexec));
  ctx->pool.push_back(sweep_ev[0]);
  ctx->pool.push_back(sweep_ev[1]);
  md->cols_hint = 0;
  if (num_active > 0 && opts.error_on_max_iter) throw NumericalError("cg: no convergence within max_iter");
  res.iterations.resize(static_cast<size_t>(k));
  res.converged.resize(static_cast<size_t>(k));
  // only the first `sweeps` entries of each column's tridiagonal can be set: strided copy
  // into pinned staging (2 k sweeps doubles instead of 2 k max_iter)
  const long used = res.sweeps > 0 ? res.sweeps : 1;
  ctx->pin1.ensure(static_cast<size_t>(3 * k * used + 2 * k));
  double* td = ctx->pin1.p;
  int* hint = reinterpret_cast<int*>(td + 3 * k * used);
  FSA_CUDA(cudaMemcpyAsync(hint, st.iterations, sizeof(int) * k, cudaMemcpyDeviceToHost, s));
  FSA_CUDA(cudaMemcpyAsync(hint + k, st.converged, sizeof(int) * k, cudaMemcpyDeviceToHost, s));
  FSA_CUDA(cudaMemcpy2DAsync(td, sizeof(double) * used, st.tdiag, sizeof(double) * maxit, sizeof(double) * used,
                             3 * k, cudaMemcpyDeviceToHost, s));
  FSA_CUDA(cudaStreamSynchronize(s));
  res.iterations.assign(hint, hint + k);
  res.converged.assign(hint + k, hint + 2 * k);
  res.tdiag.resize(static_cast<size_t>(k));
  res.toff.resize(static_cast<size_t>(k));
  res.rnorm.resize(static_cast<size_t>(k));
  for (long j = 0; j < k; ++j) {
    const int it = res.iterations[static_cast<size_t>(j)];
    res.tdiag[static_cast<size_t>(j)].assign(td + j * used, td + j * used + it);
    if (it > 1) res.toff[static_cast<size_t>(j)].assign(td + (k + j) * used, td + (k + j) * used + it - 1);
    res.rnorm[static_cast<size_t>(j)].assign(td + (2 * k + j) * used, td + (2 * k + j) * used + it);
  }
  ctx->last_cg_iterations = res.iterations;
  ctx->last_cg_rnorm = res.rnorm;
  return res;
}

// e1' log(T) e1 (krylov.cpp:120-142): implicit-QL eigensolve of the symmetric
// tridiagonal, tracking only the first row of the eigenvector matrix.
double tridiag_log_quadrature(const std::vector<double>& diag, const std::vector<double>& off) {
  const long n = static_cast<long>(diag.size());
  if (n == 0) return 0.0;
  std::vector<double> d(diag), e(static_cast<size_t>(n), 0.0), z(static_cast<size_t>(n), 0.0);
  for (long i = 0; i + 1 < n; ++i) e[static_cast<size_t>(i)] = off[static_cast<size_t>(i)];
  z[0] = 1.0;
  for (long l = 0; l < n; ++l) {
    int iter = 0;
    long mm;
    do {
      for (mm = l; mm < n - 1; ++mm) {
        const double dd = std::fabs(d[static_cast<size_t>(mm)]) + std::fabs(d[static_cast<size_t>(mm + 1)]);
        if (std::fabs(e[static_cast<size_t>(mm)]) <= std::numeric_limits<double>::epsilon() * dd) break;
      }
      if (mm != l) {
        if (iter++ == 60) throw NumericalError("tridiagonal eigendecomposition failed");
        double g = (d[static_cast<size_t>(l + 1)] - d[static_cast<size_t>(l)]) / (2.0 * e[static_cast<size_t>(l)]);
        double r = std::hypot(g, 1.0);
        g = d[static_cast<size_t>(mm)] - d[static_cast<size_t>(l)] + e[static_cast<size_t>(l)] / (g + std::copysign(r, g));
        double sn = 1.0, c = 1.0, p = 0.0;
        bool early = false;
        for (long i = mm - 1; i >= l; --i) {
          double f = sn * e[static_cast<size_t>(i)];
          const double b = c * e[static_cast<size_t>(i)];
          r = std::hypot(f, g);
          e[static_cast<size_t>(i + 1)] = r;
          if (r == 0.0) {
            d[static_cast<size_t>(i + 1)] -= p;
            e[static_cast<size_t>(mm)] = 0.0;
            early = true;
            break;
          }
          sn = f / r;
          c = g / r;
          g = d[static_cast<size_t>(i + 1)] - p;
          r = (d[static_cast<size_t>(i)] - g) * sn + 2.0 * c * b;
          p = sn * r;
          d[static_cast<size_t>(i + 1)] = g + p;
          g = c * r - b;
          f = z[static_cast<size_t>(i + 1)];
          z[static_cast<size_t>(i + 1)] = sn * z[static_cast<size_t>(i)] + c * f;
          z[static_cast<size_t>(i)] = c * z[static_cast<size_t>(i)] - sn * f;
        }
        if (early) continue;
        d[static_cast<size_t>(l)] -= p;
        e[static_cast<size_t>(l)] = g;
        e[static_cast<size_t>(mm)] = 0.0;
      }
    } while (mm != l);
  }
  double q = 0.0;
  for (long i = 0; i < n; ++i) {
    const double lam = d[static_cast<size_t>(i)];
    if (!(lam > 0.0)) throw NumericalError("tridiagonal has a nonpositive Ritz value");
    q += z[static_cast<size_t>(i)] * z[static_cast<size_t>(i)] * std::log(lam);
  }
  return q;
}

static std::vector<double> small_spd_solve(std::vector<double> G, long p, std::vector<double> b) {
  // Cholesky of the p x p symmetrised GLS matrix (estimation.cpp:207 uses LDLT)
  for (long j = 0; j < p; ++j) {
    double sdiag = G[static_cast<size_t>(j + j * p)];
    for (long k = 0; k < j; ++k) sdiag -= G[static_cast<size_t>(j + k * p)] * G[static_cast<size_t>(j + k * p)];
    if (!(sdiag > 0.0)) throw NumericalError("nll: GLS normal matrix is not positive definite");
    const double ljj = std::sqrt(sdiag);
    G[static_cast<size_t>(j + j * p)] = ljj;
    for (long i = j + 1; i < p; ++i) {
      double t = G[static_cast<size_t>(i + j * p)];
      for (long k = 0; k < j; ++k) t -= G[static_cast<size_t>(i + k * p)] * G[static_cast<size_t>(j + k * p)];
      G[static_cast<size_t>(i + j * p)] = t / ljj;
    }
  }
  for (long i = 0; i < p; ++i) {
    double t = b[static_cast<size_t>(i)];
    for (long k = 0; k < i; ++k) t -= G[static_cast<size_t>(i + k * p)] * b[static_cast<size_t>(k)];
    b[static_cast<size_t>(i)] = t / G[static_cast<size_t>(i + i * p)];
  }
  for (long i = p - 1; i >= 0; --i) {
    double t = b[static_cast<size_t>(i)];
    for (long k = i + 1; k < p; ++k) t -= G[static_cast<size_t>(k + i * p)] * b[static_cast<size_t>(k)];
    b[static_cast<size_t>(i)] = t / G[static_cast<size_t>(i + i * p)];
  }
  return b;
}

NllResult iterative_nll_grad(Model* md, Precond& P, const double* y, const double* Xc, long p, int L,
                             unsigned long long seed, const CgOptions& cg, int cv_mode, bool want_grad) {
  NvtxRange nvtx_("fsa::iterative_nll_grad");
  require(L > 0, "nll: need at least one probe");
  const bool resident = y == nullptr;
  if (resident) {  // response kept in HBM by fsa_geometry_set_response
    require(md->geo->resp_p >= 0, "nll: no resident response on the geometry");
    p = md->geo->resp_p;
    y = md->geo->resp_host.data();
    Xc = p > 0 ? md->geo->resp_host.data() + md->n : nullptr;
  }
  Context* ctx = md->ctx;
  cudaStream_t s = ctx->stream;
  // Row sharding: this rank holds rows [r0, r0 + n) of the N sorted points; every
  // global scalar (dots, Gram, traces) is a sum of rank partials.
  Comm& comm = *md->rcomm;
  const long N = md->geo->pts.n, r0 = md->world() > 1 ? md->geo->shard.r0 : 0;
  const long n = md->n, np = md->n_pad, mp = md->m_pad;
  const long k = L + 1 + p;
  const long tp = pad_cols(k);
  cudaEvent_t e0 = ctx->ev(), e1 = ctx->ev(), e2 = ctx->ev(), e3 = ctx->ev();
  FSA_CUDA(cudaEventRecord(e0, s));
  DBuf<double> B(static_cast<size_t>(np * tp)), Xs(static_cast<size_t>(np * tp));
  P.sample_probes(L, seed, B.get(), tp);  // columns [0, L)
  const int* perm_loc = md->geo->pts.perm_d.get() + r0;
  if (resident) {
    pack_cols_ld(md->geo->resp_dev.get(), N, n, 1 + p, perm_loc, np, tp, L, B.get(), s);
  } else {
    std::vector<double> yx(static_cast<size_t>(N * (1 + p)));
    std::copy(y, y + N, yx.begin());
    if (p > 0) std::copy(Xc, Xc + N * p, yx.begin() + N);
    DBuf<double> raw(static_cast<size_t>(N * (1 + p)));
    FSA_CUDA(cudaMemcpyAsync(raw.get(), yx.data(), sizeof(double) * N * (1 + p), cudaMemcpyHostToDevice, s));
    pack_cols_ld(raw.get(), N, n, 1 + p, perm_loc, np, tp, L, B.get(), s);
    FSA_CUDA(cudaStreamSynchronize(s));
  }
  FsaOp op(md);
  FSA_CUDA(cudaEventRecord(e1, s));
  CgResult sol = pcg_solve_multi(md, op, P, B.get(), k, tp, Xs.get(), cg);
  FSA_CUDA(cudaEventRecord(e2, s));
  if (!sol.all_converged()) throw NumericalError("nll: cg did not converge");
  NllResult out;
  out.cg_iterations = sol.max_iterations();
  out.sweeps = sol.sweeps;
  for (int it : sol.iterations) out.rhs_iterations += it;
  std::vector<double> quad(static_cast<size_t>(L));
#pragma omp parallel for schedule(dynamic, 1)
  for (int i = 0; i < L; ++i)
    quad[static_cast<size_t>(i)] =
        tridiag_log_quadrature(sol.tdiag[static_cast<size_t>(i)], sol.toff[static_cast<size_t>(i)]);
  double acc = 0.0;
  for (int i = 0; i < L; ++i) acc += quad[static_cast<size_t>(i)];
  out.logdet = static_cast<double>(N) / static_cast<double>(L) * acc + P.logdet();  // estimation.cpp:198-200

  // u and the GLS coefficients (estimation.cpp:202-212) from the cross Gram
  // C[a][c] = [y|X]_a . Sigma^{-1}[y|X]_c of the packed columns (q = 1 + p)
  const long q = 1 + p;
  std::vector<double> C(static_cast<size_t>(q * q));
  {
    DBuf<double> Cd(static_cast<size_t>(q * q)), scr(cross_gram_scratch(q));
    cross_gram(B.get() + L, tp, Xs.get() + L, tp, n, q, Cd.get(), scr.get(), s);
    comm.allreduce(Cd.get(), q * q, s);
    FSA_CUDA(cudaMemcpyAsync(C.data(), Cd.get(), sizeof(double) * q * q, cudaMemcpyDeviceToHost, s));
    FSA_CUDA(cudaStreamSynchronize(s));
  }
  auto Cx = [&](long a, long c) { return C[static_cast<size_t>(a * q + c)]; };
  double quad_form = Cx(0, 0);  // resid' Sigma^{-1} resid = y'u0 - 2 b'(X'u0) + b'Gb (G symmetric part)
  if (p > 0) {
    std::vector<double> Gs(static_cast<size_t>(p * p)), rhs(static_cast<size_t>(p));
    for (long a = 0; a < p; ++a)
      for (long b = 0; b < p; ++b) Gs[static_cast<size_t>(a + b * p)] = 0.5 * (Cx(1 + a, 1 + b) + Cx(1 + b, 1 + a));
    for (long a = 0; a < p; ++a) rhs[static_cast<size_t>(a)] = Cx(0, 1 + a);  // y . Sigma^{-1} X_a
    out.beta = small_spd_solve(Gs, p, rhs);
    for (long a = 0; a < p; ++a) {
      const double ba = out.beta[static_cast<size_t>(a)];
      quad_form -= ba * (Cx(1 + a, 0) + Cx(0, 1 + a));
      for (long b = 0; b < p; ++b) quad_form += ba * Cx(1 + a, 1 + b) * out.beta[static_cast<size_t>(b)];
    }
  }
  constexpr double log2pi = 1.8378770664093454836;
  out.nll = 0.5 * (out.logdet + quad_form + static_cast<double>(N) * log2pi);

  if (want_grad) {
    // STE gradient traces (krylov.cpp:163-206, estimation.cpp:217-225), U-form:
    // columns [0, L) hold the probes, column L holds u so that u' dSigma_k u comes
    // out of the same batched quadratic forms.
    const long t2 = pad_cols(L + 1);
    const long ne = md->n_ext_pad;  // Yb carries the halo rows for the Sigma_s products
    DBuf<double> Zb(np * t2), Wb(np * t2), Yb(ne * t2), SY(np * t2);
    FSA_CUDA(cudaMemsetAsync(Zb.get(), 0, sizeof(double) * np * t2, s));
    FSA_CUDA(cudaMemsetAsync(Wb.get(), 0, sizeof(double) * np * t2, s));
    copy_cols(B.get(), tp, Zb.get(), t2, np, L, s);
    copy_cols(Xs.get(), tp, Wb.get(), t2, np, L, s);
    {
      // u = Sigma^{-1} (y - X beta) = Xs[:, L] - SX beta, written into column L
      DBuf<double> coef(static_cast<size_t>(std::max<long>(p, 1)));
      if (p > 0)
        FSA_CUDA(cudaMemcpyAsync(coef.get(), out.beta.data(), sizeof(double) * p, cudaMemcpyHostToDevice, s));
      gls_residual(Xs.get() + L, tp, p, coef.get(), n, np, Zb.get() + L, t2, s);
      copy_cols(Zb.get() + L, t2, Wb.get() + L, t2, np, 1, s);
      P.solve(Zb.get(), Yb.get(), t2);
      copy_cols(Zb.get() + L, t2, Yb.get() + L, t2, np, 1, s);
      FSA_CUDA(cudaStreamSynchronize(s));
    }
    md->halo_exchange(Yb.get(), t2);
    const bool rho_needed = true;
    if (rho_needed) md->ensure_rho_derivs();
    DBuf<double> UY(mp * t2), UW(mp * t2), U1Y(mp * t2), U1W(mp * t2), K2UY(mp * t2), d1(np);
    md->project(md->U.get(), Yb.get(), t2, UY.get());
    md->project(md->U.get(), Wb.get(), t2, UW.get());
    md->project(md->U1.get(), Yb.get(), t2, U1Y.get());
    md->project(md->U1.get(), Wb.get(), t2, U1W.get());
    gemm_km(md->K2.get(), mp, mp, mp, UY.get(), t2, t2, K2UY.get(), t2, 1.0, 0.0, s);
    affine_vec(d1.get(), md->D.get(), -md->P.sigma2, 1.0 / md->P.sigma1_2, n, np, s);
    const long nd = 12;
    DBuf<double> dots(static_cast<size_t>(nd * t2));
    FSA_CUDA(cudaMemsetAsync(dots.get(), 0, sizeof(double) * nd * t2, s));
    double* sc = md->dot_scratch.get();
    auto dd = [&](int slot) { return dots.get() + slot * t2; };
    // n-space dots (rank partials, summed below) ...
    launch_coldot(Wb.get(), Yb.get(), n, t2, t2, dd(0), sc, s);           // w.y
    launch_coldot(Yb.get(), Yb.get(), n, t2, t2, dd(1), sc, s);           // y.y
    md->sigma_s_mat(Yb.get(), SY.get(), t2);
    launch_coldot(Wb.get(), SY.get(), n, t2, t2, dd(2), sc, s);           // w.Ss y
    launch_coldot_weighted(Yb.get(), Yb.get(), d1.get(), n, t2, t2, dd(4), sc, s);  // y.d1 y
    launch_spmm(md->geo->pat.rowptr.get(), md->geo->pat.col.get(), md->dsval.get(), n, Yb.get(), t2, SY.get(), t2,
                t2, 1.0, 0.0, s);
    launch_coldot(Wb.get(), SY.get(), n, t2, t2, dd(6), sc, s);           // w.dSs y
    launch_coldot_weighted(Yb.get(), Yb.get(), md->dD.get(), n, t2, t2, dd(10), sc, s);  // y.dD y
    comm.allreduce(dots.get(), nd * t2, s);
    // ... m-space dots of the (already summed) projections
    launch_coldot(UW.get(), UY.get(), mp, t2, t2, dd(3), sc, s);          // Uw.Uy
    launch_coldot(UY.get(), UY.get(), mp, t2, t2, dd(5), sc, s);          // |Uy|^2
    launch_coldot(U1W.get(), UY.get(), mp, t2, t2, dd(7), sc, s);         // U1w.Uy
    launch_coldot(UW.get(), U1Y.get(), mp, t2, t2, dd(8), sc, s);         // Uw.U1y
    launch_coldot(UW.get(), K2UY.get(), mp, t2, t2, dd(9), sc, s);        // Uw.K2Uy
    launch_coldot(U1Y.get(), UY.get(), mp, t2, t2, dd(11), sc, s);        // U1y.Uy  (dd(9)-style K2 term below)
    std::vector<double> h(static_cast<size_t>(nd * t2));
    DBuf<double> uk(t2);
    launch_coldot(UY.get(), K2UY.get(), mp, t2, t2, uk.get(), sc, s);    // Uy.K2Uy
    std::vector<double> hk(static_cast<size_t>(t2));
    FSA_CUDA(cudaMemcpyAsync(h.data(), dots.get(), sizeof(double) * nd * t2, cudaMemcpyDeviceToHost, s));
    FSA_CUDA(cudaMemcpyAsync(hk.data(), uk.get(), sizeof(double) * t2, cudaMemcpyDeviceToHost, s));
    FSA_CUDA(cudaStreamSynchronize(s));
    auto H = [&](int slot, long i) { return h[static_cast<size_t>(slot * t2 + i)]; };
    const double s2 = md->P.sigma2, s12 = md->P.sigma1_2;
    for (int kk = 0; kk < 3; ++kk) {
      std::vector<double> a(static_cast<size_t>(L + 1)), b(static_cast<size_t>(L));
      for (long i = 0; i <= L; ++i) {
        double av;
        if (kk == 0) av = H(0, i);
        else if (kk == 1) av = ((H(2, i) - s2 * H(0, i)) + H(3, i)) / s12;
        else av = ((H(6, i) + H(7, i)) + H(8, i)) - H(9, i);
        a[static_cast<size_t>(i)] = av;
        if (i < L) {
          double bv;
          if (kk == 0) bv = H(1, i);
          else if (kk == 1) bv = H(4, i) + H(5, i) / s12;
          else bv = (H(10, i) + 2.0 * H(11, i)) - hk[static_cast<size_t>(i)];
          b[static_cast<size_t>(i)] = bv;
        }
      }
      const double quad = a[static_cast<size_t>(L)];  // u' dSigma_k u
      const double dl = static_cast<double>(L);
      double abar = 0.0;
      for (long i = 0; i < L; ++i) abar += a[static_cast<size_t>(i)];
      abar /= dl;
      double value = abar;
      const bool cv_on = cv_mode != 0 && P.has_derivs();
      if (cv_on) {
        double exact_b = 0.0;
        if (P.kind() == 2) exact_b = static_cast<FitcPrecond&>(P).deriv_trace(kk);
        else exact_b = -1.0;  // set below for the diagonal preconditioner
        if (P.kind() == 1) {
          // Tr(D^{-1} dD_k) with dD_0 = 1, dD_1 = d1, dD_2 = dD
          std::vector<double> hD(static_cast<size_t>(np)), hv(static_cast<size_t>(np));
          FSA_CUDA(cudaMemcpy(hD.data(), md->D.get(), sizeof(double) * np, cudaMemcpyDeviceToHost));
          const double* src = kk == 1 ? d1.get() : md->dD.get();
          if (kk > 0) FSA_CUDA(cudaMemcpy(hv.data(), src, sizeof(double) * np, cudaMemcpyDeviceToHost));
          exact_b = 0.0;
          for (long i = 0; i < n; ++i) exact_b += (kk == 0 ? 1.0 : hv[static_cast<size_t>(i)]) / hD[static_cast<size_t>(i)];
          // diagonal preconditioner: b_i = y_i' dD_k y_i (no low-rank part)
          for (long i = 0; i < L; ++i) b[static_cast<size_t>(i)] = kk == 0 ? H(1, i) : (kk == 1 ? H(4, i) : H(10, i));
        }
        double bbar = 0.0;
        for (long i = 0; i < L; ++i) bbar += b[static_cast<size_t>(i)];
        bbar /= dl;
        double c = 1.0;
        if (cv_mode == 2) {
          double sbb = 0.0, sab = 0.0, mx = 0.0;
          for (long i = 0; i < L; ++i) {
            sbb += (b[static_cast<size_t>(i)] - bbar) * (b[static_cast<size_t>(i)] - bbar);
            sab += (a[static_cast<size_t>(i)] - abar) * (b[static_cast<size_t>(i)] - bbar);
            mx = std::max(mx, std::fabs(b[static_cast<size_t>(i)]));
          }
          const double scale = std::max(mx, 1.0);
          c = sbb > dl * 1e-28 * scale * scale ? sab / sbb : 0.0;  // krylov.cpp:192-197
        }
        value = abar - c * (bbar - exact_b);
      }
      out.grad[kk] = 0.5 * (value - quad);
    }
  }
  FSA_CUDA(cudaEventRecord(e3, s));
  FSA_CUDA(cudaEventSynchronize(e3));
  float ms1 = 0.f, ms2 = 0.f;
  FSA_CUDA(cudaEventElapsedTime(&ms1, e1, e2));
  FSA_CUDA(cudaEventElapsedTime(&ms2, e0, e3));
  out.pcg_ms = ms1;
  out.total_ms = ms2;
  ctx->pool.push_back(e0);
  ctx->pool.push_back(e1);
  ctx->pool.push_back(e2);
  ctx->pool.push_back(e3);
  return out;
}

FisherResult fisher_ste(Model* md, Precond& P, int L, unsigned long long seed, bool rademacher, const CgOptions& cg) {
  NvtxRange nvtx_("fsa::fisher_ste");
  require(L > 0, "need at least one probe");  // fsa.cpp:285
  Context* ctx = md->ctx;
  cudaStream_t s = ctx->stream;
  Comm& comm = *md->rcomm;
  const long N = md->geo->pts.n, r0 = md->world() > 1 ? md->geo->shard.r0 : 0;
  const long n = md->n, np = md->n_pad, ne = md->n_ext_pad;
  const long t1 = pad_cols(L), t3 = pad_cols(3L * L);
  // probes z_i = gaussian_vector / rademacher_vector of probe_rng(seed, i) over all N points
  // (fsa.cpp:288-289); a rank keeps its rows. Z lives in an extended block (owned rows +
  // halo) so that the Sigma_s products see the neighbours.
  DBuf<double> Z(static_cast<size_t>(ne * t1));
  {
    std::vector<double> h(static_cast<size_t>(N * L));
#pragma omp parallel for schedule(dynamic, 1)
    for (int i = 0; i < L; ++i) {
      double* zi = h.data() + static_cast<size_t>(i) * N;
      if (rademacher) probe_rademacher(seed, static_cast<unsigned long long>(i), N, zi);
      else probe_gaussian(seed, static_cast<unsigned long long>(i), 0, nullptr, N, zi);
    }
    DBuf<double> raw(static_cast<size_t>(N * L));
    FSA_CUDA(cudaMemcpyAsync(raw.get(), h.data(), sizeof(double) * N * L, cudaMemcpyHostToDevice, s));
    FSA_CUDA(cudaMemsetAsync(Z.get(), 0, sizeof(double) * ne * t1, s));
    pack_cols_ld(raw.get(), N, n, L, md->geo->pts.perm_d.get() + r0, np, t1, 0, Z.get(), s);
    FSA_CUDA(cudaStreamSynchronize(s));
  }
  md->halo_exchange(Z.get(), t1);
  FisherResult out;
  FsaOp op(md);
  // W = Sigma^{-1} Z (fsa.cpp:290)
  DBuf<double> W(static_cast<size_t>(ne * t1));
  FSA_CUDA(cudaMemsetAsync(W.get(), 0, sizeof(double) * ne * t1, s));
  {
    CgResult r = pcg_solve_multi(md, op, P, Z.get(), L, t1, W.get(), cg);
    if (!r.all_converged()) throw NumericalError("fisher: cg did not converge");
    out.cg_iterations = r.max_iterations();
    out.sweeps += r.sweeps;
  }
  md->halo_exchange(W.get(), t1);
  // B = [dSigma_0 Z | dSigma_1 Z | dSigma_2 Z] and A_k = dSigma_k W (fsa.cpp:292-295)
  DBuf<double> B(static_cast<size_t>(np * t3)), A(static_cast<size_t>(3 * np * t1)), tmp(static_cast<size_t>(np * t1));
  FSA_CUDA(cudaMemsetAsync(B.get(), 0, sizeof(double) * np * t3, s));
  for (int k = 0; k < 3; ++k) {
    md->deriv_matmat(k, Z.get(), tmp.get(), t1);
    copy_cols(tmp.get(), t1, B.get() + k * L, t3, np, L, s);
    md->deriv_matmat(k, W.get(), A.get() + k * np * t1, t1);
  }
  // T = Sigma^{-1} B, one batched solve over the 3 L columns
  DBuf<double> T(static_cast<size_t>(ne * t3));
  FSA_CUDA(cudaMemsetAsync(T.get(), 0, sizeof(double) * ne * t3, s));
  {
    CgResult r = pcg_solve_multi(md, op, P, B.get(), 3L * L, t3, T.get(), cg);
    if (!r.all_converged()) throw NumericalError("fisher: cg did not converge");
    out.cg_iterations = std::max(out.cg_iterations, r.max_iterations());
    out.sweeps += r.sweeps;
  }
  // F_kl = sum_i a_k,i . t_l,i: column dots of A_k against the l-th slice of T
  DBuf<double> dots(static_cast<size_t>(9 * t1));
  FSA_CUDA(cudaMemsetAsync(dots.get(), 0, sizeof(double) * 9 * t1, s));
  for (int l = 0; l < 3; ++l) {
    copy_cols(T.get() + l * L, t3, tmp.get(), t1, np, L, s);
    for (int k = 0; k < 3; ++k)
      launch_coldot(A.get() + k * np * t1, tmp.get(), n, t1, t1, dots.get() + (k + 3 * l) * t1, md->dot_scratch.get(),
                    s);
  }
  comm.allreduce(dots.get(), 9 * t1, s);
  std::vector<double> h(static_cast<size_t>(9 * t1));
  FSA_CUDA(cudaMemcpyAsync(h.data(), dots.get(), sizeof(double) * 9 * t1, cudaMemcpyDeviceToHost, s));
  FSA_CUDA(cudaStreamSynchronize(s));
  double F[9];
  for (int c = 0; c < 9; ++c) {
    double acc = 0.0;
    for (long i = 0; i < L; ++i) acc += h[static_cast<size_t>(c * t1 + i)];  // probe order, as F += a^T t
    F[c] = acc / (2.0 * L);
  }
  for (int k = 0; k < 3; ++k)
    for (int l = 0; l < 3; ++l) out.F[k + 3 * l] = 0.5 * (F[k + 3 * l] + F[l + 3 * k]);  // fsa.cpp:299-300
  return out;
}

}  // namespace fsa
