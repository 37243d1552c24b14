// extern "C" boundary (include/fsa_b200.h) over the device FSA core.
#include "../../include/fsa_b200.h"

#include <algorithm>
#include <cmath>
#include <atomic>
#include <cstring>
#include <memory>
#include <numeric>
#include <string>
#include <vector>

#include "blas1.cuh"
#include "fit.h"
#include "fsa_core.cuh"
#include "inputs.h"
#include "kmeans.cuh"
#include "predict.cuh"
#include "sparse.cuh"

using namespace fsa;

// Handles are reference counted: a geometry or model keeps its context alive and a
// preconditioner or prediction set keeps its model alive, so the caller may destroy them in any
// order (a garbage collector tearing down a Python session does).
struct fsa_ctx {
  std::unique_ptr<Context> c;
  std::atomic<int> refs{1};
};
struct fsa_geometry {
  fsa_ctx* ctx;
  std::shared_ptr<Geometry> g;
};
struct fsa_model {
  fsa_ctx* ctx;
  std::unique_ptr<Model> m;
  std::atomic<int> refs{1};
};
struct fsa_precond {
  fsa_model* md;
  std::unique_ptr<Precond> p;
};
struct fsa_pred {
  fsa_model* md;
  std::unique_ptr<PredictionSet> p;
};

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return FSA_OK;
  } catch (const NumericalError& e) {
    g_err = e.what();
    return FSA_ENUMERIC;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return FSA_EINVAL;
  } catch (const CudaError& e) {
    g_err = e.what();
    return FSA_ECUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return FSA_ECUDA;
  }
}

void need(const void* p, const char* what) {
  if (!p) throw std::invalid_argument(std::string(what) + " is null");
}

// Stream-ordered temporaries (DBuf) are allocated and freed on the calling thread's
// alloc_stream(): bind it (and the device) to the handle's context on every entry, so that a
// context driven from any host thread keeps its temporaries ordered on its own stream.
struct Bind {
  explicit Bind(Context* c) {
    if (c == nullptr) return;
    alloc_stream() = c->stream;
    cudaSetDevice(c->device);
  }
};

// entry points whose host buffers hold every point (caller order) exist on one rank only;
// a row-sharded context runs the fit path (iterative_nll_grad) alone
void single_rank(const Context* c, const char* what) {
  if (c->row_sharded())
    throw std::invalid_argument(std::string(what) + " is not available on a row-sharded context");
}

Params to_params(const fsa_params* p) {
  need(p, "params");
  Params q;
  q.nu = p->nu_code;
  q.family = p->taper_family;
  q.gamma = p->gamma;
  q.sigma2 = p->sigma2;
  q.sigma1_2 = p->sigma1_2;
  q.rho = p->rho;
  q.jitter_rel = p->jitter_rel;
  return q;
}

CgOptions to_cg(const fsa_cg_options* c) {
  CgOptions o;
  if (c) {
    o.tol = c->tol;
    o.max_iter = c->max_iter;
    o.error_on_max_iter = c->error_on_max_iter != 0;
  }
  return o;
}

// host column-major (original order) n x k -> device internal block (n_pad x tp)
DBuf<double> to_device_block(Model* md, const double* host, long k, long tp) {
  cudaStream_t s = md->ctx->stream;
  DBuf<double> raw(static_cast<size_t>(md->n * k)), blk(static_cast<size_t>(md->n_pad * tp));
  FSA_CUDA(cudaMemcpyAsync(raw.get(), host, sizeof(double) * md->n * k, cudaMemcpyHostToDevice, s));
  FSA_CUDA(cudaMemsetAsync(blk.get(), 0, sizeof(double) * md->n_pad * tp, s));
  pack_cols(raw.get(), md->n, k, md->geo->pts.perm_d.get(), md->n_pad, tp, 0, blk.get(), s);
  FSA_CUDA(cudaStreamSynchronize(s));
  return blk;
}
void to_host_block(Model* md, const double* blk, long k, long tp, double* host) {
  cudaStream_t s = md->ctx->stream;
  DBuf<double> raw(static_cast<size_t>(md->n * k));
  unpack_cols(blk, md->n, k, md->geo->pts.perm_d.get(), tp, 0, raw.get(), s);
  FSA_CUDA(cudaMemcpyAsync(host, raw.get(), sizeof(double) * md->n * k, cudaMemcpyDeviceToHost, s));
  FSA_CUDA(cudaStreamSynchronize(s));
}

// internal CSR (rows/cols in sorted order) -> caller order, columns ascending
void export_csr(const Csr& pat, const double* vals_dev, const SortedPoints& rows, const SortedPoints& cols,
                cudaStream_t s, int64_t* rowptr, int32_t* col, double* val) {
  const long nr = pat.rows, nnz = pat.nnz;
  std::vector<long> rp(static_cast<size_t>(nr + 1));
  std::vector<int> ci(static_cast<size_t>(nnz));
  std::vector<double> v(static_cast<size_t>(nnz));
  FSA_CUDA(cudaMemcpyAsync(rp.data(), pat.rowptr.get(), sizeof(long) * (nr + 1), cudaMemcpyDeviceToHost, s));
  if (nnz > 0) {
    FSA_CUDA(cudaMemcpyAsync(ci.data(), pat.col.get(), sizeof(int) * nnz, cudaMemcpyDeviceToHost, s));
    FSA_CUDA(cudaMemcpyAsync(v.data(), vals_dev, sizeof(double) * nnz, cudaMemcpyDeviceToHost, s));
  }
  FSA_CUDA(cudaStreamSynchronize(s));
  rowptr[0] = 0;
  for (long ro = 0; ro < nr; ++ro) {
    const long i = rows.iperm[static_cast<size_t>(ro)];
    rowptr[ro + 1] = rowptr[ro] + (rp[static_cast<size_t>(i + 1)] - rp[static_cast<size_t>(i)]);
  }
  std::vector<std::pair<int, double>> tmp;
  for (long ro = 0; ro < nr; ++ro) {
    const long i = rows.iperm[static_cast<size_t>(ro)];
    tmp.clear();
    for (long p = rp[static_cast<size_t>(i)]; p < rp[static_cast<size_t>(i + 1)]; ++p)
      tmp.emplace_back(cols.perm[static_cast<size_t>(ci[static_cast<size_t>(p)])], v[static_cast<size_t>(p)]);
    std::sort(tmp.begin(), tmp.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    long q = rowptr[ro];
    for (const auto& e : tmp) {
      if (col) col[q] = e.first;
      if (val) val[q] = e.second;
      ++q;
    }
  }
}
}  // namespace

extern "C" {

const char* fsa_last_error(void) { return g_err.c_str(); }
int fsa_version(void) { return 1; }

int fsa_ctx_create(int device, fsa_ctx** out) {
  return guard([&] {
    need(out, "out");
    auto c = std::make_unique<fsa_ctx>();
    c->c = std::make_unique<Context>(device);
    *out = c.release();
  });
}
namespace {
fsa_ctx* ctx_acquire(fsa_ctx* ctx) {
  ctx->refs.fetch_add(1);
  return ctx;
}
void ctx_release(fsa_ctx* ctx) {
  if (ctx->refs.fetch_sub(1) != 1) return;
  Bind bind_(ctx->c.get());
  delete ctx;
}
fsa_model* model_acquire(fsa_model* md) {
  md->refs.fetch_add(1);
  return md;
}
void model_release(fsa_model* md) {
  if (md->refs.fetch_sub(1) != 1) return;
  fsa_ctx* ctx = md->ctx;
  {
    Bind bind_(md->m->ctx);
    cudaStreamSynchronize(md->m->ctx->stream);
    delete md;
  }
  ctx_release(ctx);
}
}  // namespace
void fsa_ctx_destroy(fsa_ctx* ctx) {
  if (ctx == nullptr) return;
  ctx_release(ctx);
}
int fsa_nccl_unique_id(void* id_out) {
  return guard([&] {
    need(id_out, "id_out");
    nccl_unique_id(id_out);
  });
}
int fsa_ctx_create_nccl(int device, int rank, int world, const void* unique_id, fsa_ctx** out) {
  return guard([&] {
    need(out, "out");
    need(unique_id, "unique_id");
    require(world >= 1 && rank >= 0 && rank < world, "rank out of range");
    auto c = std::make_unique<fsa_ctx>();
    c->c = std::make_unique<Context>(device);
    c->c->comm = std::make_unique<NcclComm>(rank, world, unique_id);
    *out = c.release();
  });
}
int fsa_ctx_group_create(int device, int world, fsa_ctx** out) {
  return guard([&] {
    need(out, "out");
    require(world >= 1, "group size must be positive");
    std::vector<std::unique_ptr<fsa_ctx>> made;
    auto comms = make_thread_group(world);
    for (int r = 0; r < world; ++r) {
      auto c = std::make_unique<fsa_ctx>();
      c->c = std::make_unique<Context>(device);
      c->c->comm = std::move(comms[static_cast<size_t>(r)]);
      made.push_back(std::move(c));
    }
    for (int r = 0; r < world; ++r) out[r] = made[static_cast<size_t>(r)].release();
  });
}
int fsa_ctx_set_replicated(fsa_ctx* ctx, int on) {
  return guard([&] {
    need(ctx, "ctx");
    ctx->c->shard_rows = on == 0;
  });
}
int fsa_ctx_rank(fsa_ctx* ctx, int* rank, int* world) {
  return guard([&] {
    need(ctx, "ctx");
    Bind bind_(ctx->c.get());
    if (rank) *rank = ctx->c->comm->rank();
    if (world) *world = ctx->c->comm->size();
  });
}
int fsa_ctx_set_gemm_mode(fsa_ctx* ctx, int mode) {
  return guard([&] {
    need(ctx, "ctx");
    Bind bind_(ctx->c.get());
    require(mode >= 0 && mode <= 2, "gemm mode must be 0 (auto), 1 (dmma) or 2 (ozaki)");
    ctx->c->gemm_mode = mode;
  });
}
int fsa_ctx_last_cg(fsa_ctx* ctx, int64_t* k, int64_t cap_k, int64_t cap_len, int* iterations, double* rnorm) {
  return guard([&] {
    need(ctx, "ctx");
    const Context& c = *ctx->c;
    const int64_t kk = static_cast<int64_t>(c.last_cg_iterations.size());
    if (k) *k = kk;
    for (int64_t j = 0; j < std::min(kk, cap_k); ++j) {
      if (iterations) iterations[j] = c.last_cg_iterations[static_cast<size_t>(j)];
      if (!rnorm) continue;
      const auto& h = c.last_cg_rnorm[static_cast<size_t>(j)];
      for (int64_t i = 0; i < cap_len; ++i)
        rnorm[j * cap_len + i] = i < static_cast<int64_t>(h.size()) ? h[static_cast<size_t>(i)] : 0.0;
    }
  });
}
int fsa_ctx_synchronize(fsa_ctx* ctx) {
  return guard([&] {
    need(ctx, "ctx");
    Bind bind_(ctx->c.get());
    ctx->c->sync();
  });
}
int fsa_ctx_stream(fsa_ctx* ctx, void** stream) {
  return guard([&] {
    need(ctx, "ctx");
    Bind bind_(ctx->c.get());
    *stream = ctx->c->stream;
  });
}
int fsa_ctx_set_profiling(fsa_ctx* ctx, int on) {
  return guard([&] {
    need(ctx, "ctx");
    Bind bind_(ctx->c.get());
    ctx->c->flush_timers();
    ctx->c->profile = on != 0;
  });
}
int fsa_ctx_reset_timers(fsa_ctx* ctx) {
  return guard([&] {
    need(ctx, "ctx");
    Bind bind_(ctx->c.get());
    ctx->c->flush_timers();
    ctx->c->totals.clear();
  });
}
int fsa_ctx_timer_names(fsa_ctx* ctx, char* buf, size_t len) {
  return guard([&] {
    need(ctx, "ctx");
    Bind bind_(ctx->c.get());
    ctx->c->flush_timers();
    std::string s;
    for (const auto& kv : ctx->c->totals) s += kv.first + "\n";
    if (buf && len > 0) {
      std::strncpy(buf, s.c_str(), len - 1);
      buf[len - 1] = 0;
    }
  });
}
int fsa_ctx_timer(fsa_ctx* ctx, const char* name, double* ms, int64_t* count, double* units) {
  return guard([&] {
    need(ctx, "ctx");
    Bind bind_(ctx->c.get());
    need(name, "name");
    ctx->c->flush_timers();
    auto it = ctx->c->totals.find(name);
    const Context::Acc a = it == ctx->c->totals.end() ? Context::Acc{} : it->second;
    if (ms) *ms = a.ms;
    if (count) *count = a.count;
    if (units) *units = a.units;
  });
}

int fsa_uniform_locations(int64_t n, int d, uint64_t seed, double* out) {
  return guard([&] { uniform_locations(n, d, seed, out); });
}
int fsa_select_random(const double* coords, int64_t n, int d, int64_t m, uint64_t seed, double* out) {
  return guard([&] { select_random(coords, n, d, m, seed, out); });
}
int fsa_select_kmeanspp(const double* coords, int64_t n, int d, int64_t m, uint64_t seed, int max_iter,
                        double rel_tol, double* out) {
  return guard([&] { select_kmeanspp(coords, n, d, m, seed, max_iter, rel_tol, out); });
}
int fsa_select_kmeanspp_device(fsa_ctx* ctx, const double* coords, int64_t n, int d, int64_t m, uint64_t seed,
                               int max_iter, double rel_tol, double* out) {
  return guard([&] {
    need(ctx, "context");
    need(coords, "coords");
    need(out, "out");
    Bind bind_(ctx->c.get());
    select_kmeanspp_device(ctx->c->stream, coords, n, d, m, seed, max_iter, rel_tol, out);
  });
}
double fsa_gamma_for_avg_row_nnz(int64_t n, double target) {
  double g = 0.0;
  if (guard([&] { g = gamma_for_avg_row_nnz(n, target); }) != FSA_OK) return -1.0;
  return g;
}
int fsa_simulate_rff(const double* coords, int64_t n, int d, int nu_code, double sigma1_2, double rho, double nugget,
                     int features, uint64_t seed, double* y) {
  return guard([&] { simulate_rff(coords, n, d, nu_code, sigma1_2, rho, nugget, features, seed, y); });
}
int fsa_blob_locations(int64_t n, int d, int blobs, double sd, uint64_t seed, double* out) {
  return guard([&] { blob_locations(n, d, blobs, sd, seed, out); });
}
int fsa_probe_gaussian(uint64_t seed, uint64_t index, int64_t n1, double* e1, int64_t n2, double* e2) {
  return guard([&] { probe_gaussian(seed, index, n1, e1, n2, e2); });
}
int fsa_probe_rademacher(uint64_t seed, uint64_t index, int64_t n, double* z) {
  return guard([&] { probe_rademacher(seed, index, n, z); });
}

int fsa_geometry_create(fsa_ctx* ctx, const double* coords, int64_t n, int d, double gamma, fsa_geometry** out) {
  return guard([&] {
    need(ctx, "ctx");
    Bind bind_(ctx->c.get());
    need(coords, "coords");
    auto g = std::make_unique<fsa_geometry>();
    g->g = make_geometry(ctx->c.get(), coords, n, d, gamma);
    g->ctx = ctx_acquire(ctx);
    *out = g.release();
  });
}
void fsa_geometry_destroy(fsa_geometry* g) {
  if (g == nullptr) return;
  fsa_ctx* ctx = g->ctx;
  {
    Bind bind_(ctx->c.get());
    cudaStreamSynchronize(ctx->c->stream);
    delete g;
  }
  ctx_release(ctx);
}
int fsa_geometry_info(fsa_geometry* g, int64_t* n, int64_t* nnz) {
  return guard([&] {
    need(g, "geometry");
    Bind bind_(g->ctx->c.get());
    if (n) *n = g->g->pts.n;
    if (nnz) *nnz = g->g->pat.nnz;
  });
}
int fsa_geometry_shard_info(fsa_geometry* g, int64_t* r0, int64_t* r1, int64_t* n_halo) {
  return guard([&] {
    need(g, "geometry");
    Bind bind_(g->ctx->c.get());
    const ShardPlan& sp = g->g->shard;
    const bool one = sp.world <= 1;
    if (r0) *r0 = one ? 0 : sp.r0;
    if (r1) *r1 = one ? g->g->pts.n : sp.r1;
    if (n_halo) *n_halo = one ? 0 : sp.n_halo;
  });
}
int fsa_geometry_pattern(fsa_geometry* g, int64_t* rowptr, int32_t* col, double* dist) {
  return guard([&] {
    need(g, "geometry");
    Bind bind_(g->ctx->c.get());
    single_rank(g->ctx->c.get(), "taper_pattern export");
    export_csr(g->g->pat, g->g->pat.dist.get(), g->g->pts, g->g->pts, g->ctx->c->stream, rowptr, col, dist);
  });
}
int fsa_geometry_permutation(fsa_geometry* g, int32_t* perm) {
  return guard([&] {
    need(g, "geometry");
    Bind bind_(g->ctx->c.get());
    std::copy(g->g->pts.perm.begin(), g->g->pts.perm.end(), perm);
  });
}

int fsa_geometry_set_response(fsa_geometry* g, const double* y, const double* X, int64_t pcols) {
  return guard([&] {
    need(g, "geometry");
    Bind bind_(g->ctx->c.get());
    need(y, "y");
    require(pcols >= 0 && (pcols == 0 || X != nullptr), "nll: shape mismatch");
    Geometry& G = *g->g;
    const long n = G.pts.n;
    G.resp_host.assign(y, y + n);
    if (pcols > 0) G.resp_host.insert(G.resp_host.end(), X, X + n * pcols);
    G.resp_dev.alloc(static_cast<size_t>(n * (1 + pcols)));
    FSA_CUDA(cudaMemcpyAsync(G.resp_dev.get(), G.resp_host.data(), sizeof(double) * n * (1 + pcols),
                             cudaMemcpyHostToDevice, g->ctx->c->stream));
    FSA_CUDA(cudaStreamSynchronize(g->ctx->c->stream));
    G.resp_p = pcols;
  });
}
int fsa_geometry_cache_probes(fsa_geometry* g, int on) {
  return guard([&] {
    need(g, "geometry");
    Bind bind_(g->ctx->c.get());
    g->g->cache_probes = on != 0;
    if (!on) {
      g->g->probes.valid = false;
      g->g->probes.E1.release();
      g->g->probes.E2.release();
    }
  });
}
int64_t fsa_launch_count(void) { return launch_counter().load(); }

int fsa_model_assemble(fsa_ctx* ctx, const double* coords, int64_t n, int d, const double* inducing, int64_t m,
                       const fsa_params* params, fsa_model** out) {
  return guard([&] {
    need(ctx, "ctx");
    Bind bind_(ctx->c.get());
    need(coords, "coords");
    need(inducing, "inducing");
    const Params p = to_params(params);
    require(p.gamma > 0.0, "taper range gamma must be positive");
    auto geo = make_geometry(ctx->c.get(), coords, n, d, p.gamma);
    auto md = std::make_unique<fsa_model>();
    md->m = Model::assemble(ctx->c.get(), geo, inducing, m, p);
    md->ctx = ctx_acquire(ctx);
    *out = md.release();
  });
}
int fsa_model_assemble_geo(fsa_geometry* g, const double* inducing, int64_t m, const fsa_params* params,
                           fsa_model** out) {
  return guard([&] {
    need(g, "geometry");
    Bind bind_(g->ctx->c.get());
    need(inducing, "inducing");
    auto md = std::make_unique<fsa_model>();
    md->m = Model::assemble(g->ctx->c.get(), g->g, inducing, m, to_params(params));
    md->ctx = ctx_acquire(g->ctx);
    *out = md.release();
  });
}
void fsa_model_destroy(fsa_model* md) {
  if (md == nullptr) return;
  model_release(md);
}
int fsa_model_info(fsa_model* md, int64_t* n, int64_t* m, int64_t* nnz, int64_t* n_clamped, double* ldsm) {
  return guard([&] {
    need(md, "model");
    Bind bind_(md->m->ctx);
    Model& M = *md->m;
    if (n) *n = M.geo->pts.n;  // all points (a sharded rank owns a row block of them)
    if (m) *m = M.m;
    if (nnz) *nnz = M.geo->pat.nnz;
    if (n_clamped) *n_clamped = M.n_clamped;
    if (ldsm) *ldsm = M.logdet_sigma_m;
  });
}
int fsa_model_sigma_s(fsa_model* md, int which, int64_t* rowptr, int32_t* col, double* val) {
  return guard([&] {
    need(md, "model");
    Bind bind_(md->m->ctx);
    Model& M = *md->m;
    single_rank(M.ctx, "Sigma_s export");
    require(which == 0 || which == 1, "which must be 0 (sigma_s) or 1 (d sigma_s / d rho)");
    if (which == 1) M.ensure_rho_derivs();
    export_csr(M.geo->pat, which == 0 ? M.sval.get() : M.dsval.get(), M.geo->pts, M.geo->pts, M.ctx->stream,
               rowptr, col, val);
  });
}
int fsa_model_matmat(fsa_model* md, const double* V, int64_t k, double* out) {
  return guard([&] {
    need(md, "model");
    Bind bind_(md->m->ctx);
    Model* M = md->m.get();
    single_rank(M->ctx, "matmat");
    require(k >= 1, "matrix row mismatch");
    const long tp = pad_cols(k);
    DBuf<double> in = to_device_block(M, V, k, tp);
    DBuf<double> o(static_cast<size_t>(M->n_pad * tp));
    M->matmat(in.get(), o.get(), tp);
    to_host_block(M, o.get(), k, tp, out);
  });
}
int fsa_model_deriv_matmat(fsa_model* md, int which, const double* V, int64_t k, double* out) {
  return guard([&] {
    need(md, "model");
    Bind bind_(md->m->ctx);
    Model* M = md->m.get();
    single_rank(M->ctx, "matmat");
    require(k >= 1, "matrix row mismatch");
    const long tp = pad_cols(k);
    DBuf<double> in = to_device_block(M, V, k, tp);
    DBuf<double> o(static_cast<size_t>(M->n_pad * tp));
    M->deriv_matmat(which, in.get(), o.get(), tp);
    to_host_block(M, o.get(), k, tp, out);
  });
}
int fsa_model_lowrank_project(fsa_model* md, const double* V, int64_t k, double* out) {
  return guard([&] {
    need(md, "model");
    Bind bind_(md->m->ctx);
    need(V, "V");
    need(out, "out");
    Model* M = md->m.get();
    single_rank(M->ctx, "lowrank_project");
    require(k >= 1, "matrix row mismatch");
    const long tp = pad_cols(k), mp = M->m_pad;
    DBuf<double> in = to_device_block(M, V, k, tp);
    DBuf<double> o(static_cast<size_t>(mp * tp));
    M->project(M->U.get(), in.get(), tp, o.get());
    std::vector<double> h(static_cast<size_t>(mp * tp));
    FSA_CUDA(cudaMemcpyAsync(h.data(), o.get(), sizeof(double) * mp * tp, cudaMemcpyDeviceToHost, M->ctx->stream));
    FSA_CUDA(cudaStreamSynchronize(M->ctx->stream));
    for (long c = 0; c < k; ++c)
      for (long r = 0; r < M->m; ++r) out[r + c * M->m] = h[static_cast<size_t>(r * tp + c)];
  });
}
int fsa_model_lowrank_expand(fsa_model* md, const double* W, int64_t k, double* out) {
  return guard([&] {
    need(md, "model");
    Bind bind_(md->m->ctx);
    need(W, "W");
    need(out, "out");
    Model* M = md->m.get();
    single_rank(M->ctx, "lowrank_expand");
    require(k >= 1, "matrix row mismatch");
    const long tp = pad_cols(k), mp = M->m_pad;
    std::vector<double> h(static_cast<size_t>(mp * tp), 0.0);
    for (long c = 0; c < k; ++c)
      for (long r = 0; r < M->m; ++r) h[static_cast<size_t>(r * tp + c)] = W[r + c * M->m];
    cudaStream_t s = M->ctx->stream;
    DBuf<double> Wd(static_cast<size_t>(mp * tp)), Y(static_cast<size_t>(M->n_pad * tp));
    FSA_CUDA(cudaMemcpyAsync(Wd.get(), h.data(), sizeof(double) * mp * tp, cudaMemcpyHostToDevice, s));
    M->expand(Wd.get(), tp, Y.get());
    to_host_block(M, Y.get(), k, tp, out);
  });
}
int fsa_debug_kernel_bench(fsa_model* md, int which, int64_t k, int reps, int flags, double* ms_out) {
  return guard([&] {
    need(md, "model");
    Bind bind_(md->m->ctx);
    need(ms_out, "ms_out");
    Model* M = md->m.get();
    single_rank(M->ctx, "debug_kernel_bench");
    require(k >= 1 && reps >= 1, "invalid sizes");
    cudaStream_t s = M->ctx->stream;
    const long tp = pad_cols(k), np = M->n_pad, mp = M->m_pad;
    const size_t blk = static_cast<size_t>(M->n_ext_pad * tp);
    DBuf<double> Z(blk), Lw(blk), H(blk), V(blk), R(blk), part(static_cast<size_t>((np / 32 + 1) * tp * 4)),
        dots(static_cast<size_t>(4 * tp)), beta(static_cast<size_t>(tp)), W(static_cast<size_t>(mp * tp));
    std::vector<double> h(blk);
    for (size_t i = 0; i < blk; ++i) h[i] = std::sin(0.37 * static_cast<double>(i)) * 0.5;
    for (DBuf<double>* b : {&Z, &Lw, &H, &V, &R})
      FSA_CUDA(cudaMemcpyAsync(b->get(), h.data(), sizeof(double) * blk, cudaMemcpyHostToDevice, s));
    std::vector<double> hb(static_cast<size_t>(tp), 0.3), hw(static_cast<size_t>(mp * tp));
    for (size_t i = 0; i < hw.size(); ++i) hw[i] = std::cos(0.11 * static_cast<double>(i));
    FSA_CUDA(cudaMemcpyAsync(beta.get(), hb.data(), sizeof(double) * tp, cudaMemcpyHostToDevice, s));
    FSA_CUDA(cudaMemcpyAsync(W.get(), hw.data(), sizeof(double) * mp * tp, cudaMemcpyHostToDevice, s));
    if (which != 0) M->ensure_ozaki();
    auto run = [&] {
      switch (which) {
        case 0:
          spmm_block_dot_h(M->geo->pat, M->gval.get(), Z.get(), tp, V.get(), tp, tp, dots.get(), part.get(),
                           Lw.get(), H.get(), beta.get(), k, false, s, false);
          break;
        case 1:
          ozaki_project(M->oz, R.get(), tp, tp, M->Dinv.get(), W.get(), s, false);
          break;
        default:
          ozaki_expand_keep(M->oz, W.get(), tp, tp, Z.get(), Lw.get(), R.get(), M->Dinv.get(), dots.get(),
                            part.get(), s, false, nullptr);
          break;
      }
    };
    require(flags == 0, "debug_kernel_bench: flags must be 0");
    run();
    cudaEvent_t a = M->ctx->ev(), b = M->ctx->ev();
    FSA_CUDA(cudaEventRecord(a, s));
    for (int i = 0; i < reps; ++i) run();
    FSA_CUDA(cudaEventRecord(b, s));
    FSA_CUDA(cudaEventSynchronize(b));
    float ms = 0.f;
    FSA_CUDA(cudaEventElapsedTime(&ms, a, b));
    *ms_out = static_cast<double>(ms) / reps;
    M->ctx->pool.push_back(a);
    M->ctx->pool.push_back(b);
  });
}
int fsa_model_diagonals(fsa_model* md, double* sdiag, double* lowrank) {
  return guard([&] {
    need(md, "model");
    Bind bind_(md->m->ctx);
    Model* M = md->m.get();
    single_rank(M->ctx, "diagonals");
    cudaStream_t s = M->ctx->stream;
    DBuf<double> raw(static_cast<size_t>(M->n));
    if (sdiag) {
      unpack_cols(M->D.get(), M->n, 1, M->geo->pts.perm_d.get(), 1, 0, raw.get(), s);
      FSA_CUDA(cudaMemcpyAsync(sdiag, raw.get(), sizeof(double) * M->n, cudaMemcpyDeviceToHost, s));
      FSA_CUDA(cudaStreamSynchronize(s));
    }
    if (lowrank) {
      unpack_cols(M->lowrank.get(), M->n, 1, M->geo->pts.perm_d.get(), 1, 0, raw.get(), s);
      FSA_CUDA(cudaMemcpyAsync(lowrank, raw.get(), sizeof(double) * M->n, cudaMemcpyDeviceToHost, s));
      FSA_CUDA(cudaStreamSynchronize(s));
    }
  });
}

int fsa_make_preconditioner(fsa_model* md, int type, fsa_precond** out) {
  return guard([&] {
    need(md, "model");
    Bind bind_(md->m->ctx);
    auto p = std::make_unique<fsa_precond>();
    p->p = make_preconditioner(md->m.get(), type);
    p->md = model_acquire(md);
    *out = p.release();
  });
}
int fsa_make_jacobi(fsa_model* md, fsa_precond** out) {
  return guard([&] {
    need(md, "model");
    Bind bind_(md->m->ctx);
    auto p = std::make_unique<fsa_precond>();
    single_rank(md->m->ctx, "the Jacobi preconditioner");
    p->p = std::make_unique<DiagPrecond>(md->m.get(), false);
    p->md = model_acquire(md);
    *out = p.release();
  });
}
void fsa_precond_destroy(fsa_precond* p) {
  if (p == nullptr) return;
  fsa_model* md = p->md;
  {
    Bind bind_(md->m->ctx);
    cudaStreamSynchronize(md->m->ctx->stream);
    delete p;
  }
  model_release(md);
}
int fsa_precond_logdet(fsa_precond* p, double* out) {
  return guard([&] {
    need(p, "preconditioner");
    Bind bind_(p->md->m->ctx);
    *out = p->p->logdet();
  });
}
int fsa_precond_solve_mat(fsa_precond* p, const double* R, int64_t k, double* out) {
  return guard([&] {
    need(p, "preconditioner");
    Bind bind_(p->md->m->ctx);
    Model* M = p->md->m.get();
    single_rank(M->ctx, "solve_mat");
    const long tp = pad_cols(k);
    DBuf<double> in = to_device_block(M, R, k, tp);
    DBuf<double> o(static_cast<size_t>(M->n_pad * tp));
    p->p->solve(in.get(), o.get(), tp);
    to_host_block(M, o.get(), k, tp, out);
  });
}
int fsa_precond_sample_probes(fsa_precond* p, int L, uint64_t seed, double* Z) {
  return guard([&] {
    need(p, "preconditioner");
    Bind bind_(p->md->m->ctx);
    require(L > 0, "need at least one probe");
    Model* M = p->md->m.get();
    single_rank(M->ctx, "sample_probes");
    const long tp = pad_cols(L);
    DBuf<double> o(static_cast<size_t>(M->n_pad * tp));
    p->p->sample_probes(L, seed, o.get(), tp);
    to_host_block(M, o.get(), L, tp, Z);
  });
}
int fsa_precond_deriv_trace(fsa_precond* p, int which, double* out) {
  return guard([&] {
    need(p, "preconditioner");
    Bind bind_(p->md->m->ctx);
    require(which >= 0 && which < 3, "parameter index out of range");
    require(p->p->kind() == 2, "deriv_trace is implemented for the FITC preconditioner");
    *out = static_cast<FitcPrecond*>(p->p.get())->deriv_trace(which);
  });
}

int fsa_pcg_solve_multi(fsa_model* md, fsa_precond* p, int op_kind, const double* B, int64_t k,
                        const fsa_cg_options* cg, double* X, int* iterations, int* converged, double* tdiag,
                        double* toff, int* sweeps) {
  return guard([&] {
    need(md, "model");
    Bind bind_(md->m->ctx);
    need(p, "preconditioner");
    Model* M = md->m.get();
    single_rank(M->ctx, "pcg_solve_multi on host blocks");
    const CgOptions o = to_cg(cg);
    const long tp = pad_cols(k);
    DBuf<double> Bd = to_device_block(M, B, k, tp);
    DBuf<double> Xd(static_cast<size_t>(M->n_pad * tp));
    FsaOp fop(M);
    SigmaSOp sop(M);
    LinOp& op = op_kind == 0 ? static_cast<LinOp&>(fop) : static_cast<LinOp&>(sop);
    CgResult r = pcg_solve_multi(M, op, *p->p, Bd.get(), k, tp, Xd.get(), o);
    to_host_block(M, Xd.get(), k, tp, X);
    for (long j = 0; j < k; ++j) {
      if (iterations) iterations[j] = r.iterations[static_cast<size_t>(j)];
      if (converged) converged[j] = r.converged[static_cast<size_t>(j)];
      if (tdiag) std::copy(r.tdiag[static_cast<size_t>(j)].begin(), r.tdiag[static_cast<size_t>(j)].end(), tdiag + j * o.max_iter);
      if (toff) std::copy(r.toff[static_cast<size_t>(j)].begin(), r.toff[static_cast<size_t>(j)].end(), toff + j * o.max_iter);
    }
    if (sweeps) *sweeps = r.sweeps;
  });
}
int fsa_tridiag_log_quadrature(const double* diag, const double* off, int64_t len, double* out) {
  return guard([&] {
    std::vector<double> d(diag, diag + len), e;
    if (len > 1) e.assign(off, off + len - 1);
    *out = tridiag_log_quadrature(d, e);
  });
}
int fsa_iterative_nll_grad(fsa_model* md, fsa_precond* p, const double* y, const double* X, int64_t pcols, int L,
                           uint64_t seed, const fsa_cg_options* cg, int cv_mode, int want_grad, fsa_nll_result* out,
                           double* beta) {
  return guard([&] {
    need(md, "model");
    Bind bind_(md->m->ctx);
    need(p, "preconditioner");
    need(out, "out");
    require(pcols == 0 || X != nullptr, "nll: shape mismatch");
    require(cv_mode >= 0 && cv_mode <= 2, "unknown control-variate mode");
    NllResult r = iterative_nll_grad(md->m.get(), *p->p, y, X, pcols, L, seed, to_cg(cg), cv_mode, want_grad != 0);
    out->nll = r.nll;
    for (int k = 0; k < 3; ++k) out->grad[k] = r.grad[k];
    out->logdet = r.logdet;
    out->cg_iterations = r.cg_iterations;
    out->sweeps = r.sweeps;
    out->rhs_iterations = r.rhs_iterations;
    out->pcg_ms = r.pcg_ms;
    out->total_ms = r.total_ms;
    for (long a = 0; a < pcols; ++a)
      if (beta) beta[a] = r.beta[static_cast<size_t>(a)];
  });
}

int fsa_fisher_ste(fsa_model* md, fsa_precond* p, int num_probes, uint64_t seed, int rademacher,
                   const fsa_cg_options* cg, double* F_out, int* cg_iterations) {
  return guard([&] {
    need(md, "model");
    Bind bind_(md->m->ctx);
    need(p, "preconditioner");
    need(F_out, "F_out");
    FisherResult r = fisher_ste(md->m.get(), *p->p, num_probes, seed, rademacher != 0, to_cg(cg));
    std::copy(r.F, r.F + 9, F_out);
    if (cg_iterations) *cg_iterations = r.cg_iterations;
  });
}

void fsa_fit_options_default(fsa_fit_options* o) {
  if (o == nullptr) return;
  FitOptions d;
  o->nu_code = d.nu;
  o->taper_family = d.family;
  o->num_inducing = d.num_inducing;
  o->taper_range = d.taper_range;
  o->target_row_nnz = d.target_row_nnz;
  o->precond = d.precond;
  o->num_probes = d.num_probes;
  o->cv_mode = d.cv_mode;
  o->seed = d.seed;
  o->cg_tol = d.cg_tol;
  o->cg_max_iter = d.cg_max_iter;
  o->jitter_rel = d.jitter_rel;
  o->max_evals = d.lbfgs.max_evals;
  o->lbfgs_memory = d.lbfgs.memory;
  o->armijo_c1 = d.lbfgs.armijo_c1;
  o->max_backtracks = d.lbfgs.max_backtracks;
  o->f_rel_tol = d.lbfgs.f_rel_tol;
  o->grad_tol_per_n = d.grad_tol_per_n;
}
int fsa_fit(fsa_ctx* ctx, const double* coords, int64_t n, int d, const double* y, const double* X, int64_t pcols,
            const fsa_fit_options* opts, fsa_fit_result* out, double* beta, double* inducing, double* nll_trace,
            int64_t trace_cap) {
  return guard([&] {
    need(ctx, "ctx");
    Bind bind_(ctx->c.get());
    need(coords, "coords");
    need(y, "y");
    need(opts, "opts");
    need(out, "out");
    single_rank(ctx->c.get(), "fit");
    FitOptions o;
    o.nu = opts->nu_code;
    o.family = opts->taper_family;
    o.num_inducing = opts->num_inducing;
    o.taper_range = opts->taper_range;
    o.target_row_nnz = opts->target_row_nnz;
    o.precond = opts->precond;
    o.num_probes = opts->num_probes;
    o.cv_mode = opts->cv_mode;
    o.seed = opts->seed;
    o.cg_tol = opts->cg_tol;
    o.cg_max_iter = opts->cg_max_iter;
    o.jitter_rel = opts->jitter_rel;
    o.lbfgs.max_evals = opts->max_evals;
    o.lbfgs.memory = opts->lbfgs_memory;
    o.lbfgs.armijo_c1 = opts->armijo_c1;
    o.lbfgs.max_backtracks = opts->max_backtracks;
    o.lbfgs.f_rel_tol = opts->f_rel_tol;
    o.grad_tol_per_n = opts->grad_tol_per_n;
    require(o.nu >= 0 && o.nu <= 2 && (o.family == 1 || o.family == 2), "fit: invalid kernel or taper");
    require(o.precond >= 0 && o.precond <= 2 && o.cv_mode >= 0 && o.cv_mode <= 2, "fit: invalid options");
    FitOutput r = fit_fsa(ctx->c.get(), coords, n, d, y, X, pcols, o);
    out->sigma2 = r.sigma2;
    out->sigma1_2 = r.sigma1_2;
    out->rho = r.rho;
    out->nll = r.nll;
    out->gamma = r.gamma;
    for (int k = 0; k < 3; ++k) out->grad_log[k] = k < static_cast<int>(r.grad_log.size()) ? r.grad_log[k] : 0.0;
    out->evals = r.evals;
    out->converged = r.converged ? 1 : 0;
    out->n_trace = static_cast<int64_t>(r.nll_trace.size());
    if (beta)
      for (int64_t a = 0; a < pcols; ++a) beta[a] = r.beta[static_cast<size_t>(a)];
    if (inducing) std::copy(r.inducing.begin(), r.inducing.end(), inducing);
    if (nll_trace)
      for (int64_t i = 0; i < std::min<int64_t>(trace_cap, out->n_trace); ++i) nll_trace[i] = r.nll_trace[static_cast<size_t>(i)];
  });
}

int fsa_pred_setup(fsa_model* md, const double* pcoords, int64_t np, fsa_pred** out) {
  return guard([&] {
    need(md, "model");
    Bind bind_(md->m->ctx);
    need(pcoords, "pcoords");
    single_rank(md->m->ctx, "prediction");
    auto pr = std::make_unique<fsa_pred>();
    pr->p = make_prediction_set(md->m.get(), pcoords, np);
    pr->md = model_acquire(md);
    *out = pr.release();
  });
}
void fsa_pred_destroy(fsa_pred* pr) {
  if (pr == nullptr) return;
  fsa_model* md = pr->md;
  {
    Bind bind_(md->m->ctx);
    cudaStreamSynchronize(md->m->ctx->stream);
    delete pr;
  }
  model_release(md);
}
int fsa_pred_info(fsa_pred* pr, int64_t* np, int64_t* nnz) {
  return guard([&] {
    need(pr, "prediction set");
    Bind bind_(pr->md->m->ctx);
    if (np) *np = pr->p->np;
    if (nnz) *nnz = pr->p->rows.nnz;
  });
}
int fsa_cross_apply_t(fsa_pred* pr, const double* u, double* out) {
  return guard([&] {
    need(pr, "prediction set");
    Bind bind_(pr->md->m->ctx);
    cross_apply_t(*pr->p, u, out);
  });
}
int fsa_predict_mean_iterative(fsa_pred* pr, const double* resid, fsa_precond* p, const fsa_cg_options* cg,
                               double* mean_out) {
  return guard([&] {
    need(pr, "prediction set");
    Bind bind_(pr->md->m->ctx);
    need(p, "preconditioner");
    predict_mean_iterative(*pr->p, resid, *p->p, to_cg(cg), mean_out);
  });
}
int fsa_predict_var_sim(fsa_pred* pr, int num_probes, uint64_t seed, const fsa_cg_options* cg,
                        const fsa_cg_options* cg_s, int control_variate, double floor_rel, double* var, double* se,
                        fsa_predvar_info* info) {
  return guard([&] {
    need(pr, "prediction set");
    Bind bind_(pr->md->m->ctx);
    PredVarInfo pi = predict_var_sim(*pr->p, num_probes, seed, to_cg(cg), to_cg(cg_s), control_variate != 0,
                                     floor_rel, var, se);
    if (info) {
      info->clamped = pi.clamped;
      info->cg_iterations = pi.cg_iterations;
      info->det_ms = pi.det_ms;
      info->sim_ms = pi.sim_ms;
    }
  });
}
int fsa_pred_det_pieces(fsa_pred* pr, const fsa_cg_options* cg, const fsa_cg_options* cg_s, double* d1, double* d2,
                        double* d3, int* cg_iterations) {
  return guard([&] {
    need(pr, "prediction set");
    Bind bind_(pr->md->m->ctx);
    int it = 0;
    deterministic_pieces_host(*pr->p, to_cg(cg), to_cg(cg_s), d1, d2, d3, &it);
    if (cg_iterations) *cg_iterations = it;
  });
}

}  // extern "C"
