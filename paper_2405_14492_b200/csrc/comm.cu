// Communicators; see comm.cuh.
#include <dlfcn.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <mutex>

#include "comm.cuh"

namespace fsa {

void Comm::allreduce_host(double* host, long count, cudaStream_t s) {
  if (size() == 1 || count == 0) return;
  DBuf<double> d(static_cast<size_t>(count));
  FSA_CUDA(cudaMemcpyAsync(d.get(), host, sizeof(double) * count, cudaMemcpyHostToDevice, s));
  allreduce(d.get(), count, s);
  FSA_CUDA(cudaMemcpyAsync(host, d.get(), sizeof(double) * count, cudaMemcpyDeviceToHost, s));
  FSA_CUDA(cudaStreamSynchronize(s));
}

// ---- in-process thread group -------------------------------------------------------------
constexpr int kMaxThreadRanks = 16;

struct ThreadGroup {
  int world = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long generation = 0;
  const double* bufs[kMaxThreadRanks] = {};
  const double* send[kMaxThreadRanks][kMaxThreadRanks] = {};
  long send_count[kMaxThreadRanks][kMaxThreadRanks] = {};
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long gen = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen; });
    }
  }
};

namespace {
struct PtrSet {
  const double* p[kMaxThreadRanks];
};
// out[i] = sum_j p[j][i] in rank order (identical on every rank)
__global__ void k_sum_ptrs(PtrSet ps, int world, long count, double* __restrict__ out) {
  const long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= count) return;
  double s = 0.0;
  for (int j = 0; j < world; ++j) s += ps.p[j][i];
  out[i] = s;
}
// out[i] = sum_j g[j * count + i] in rank order (the gathered partials of NcclComm::allreduce)
__global__ void k_sum_ranks(const double* __restrict__ g, int world, long count, double* __restrict__ out) {
  const long i = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= count) return;
  double s = 0.0;
  for (int j = 0; j < world; ++j) s += g[static_cast<long>(j) * count + i];
  out[i] = s;
}
}  // namespace

ThreadComm::ThreadComm(std::shared_ptr<ThreadGroup> g, int rank) : g_(std::move(g)), rank_(rank) {}
int ThreadComm::size() const { return g_->world; }

void ThreadComm::allreduce(double* dev, long count, cudaStream_t s) {
  if (g_->world == 1 || count == 0) return;
  FSA_CUDA(cudaStreamSynchronize(s));
  g_->bufs[rank_] = dev;
  g_->barrier();
  PtrSet ps{};
  for (int j = 0; j < g_->world; ++j) ps.p[j] = g_->bufs[j];
  DBuf<double> tmp(static_cast<size_t>(count));
  k_sum_ptrs<<<static_cast<unsigned>(cdiv(count, 256)), 256, 0, s>>>(ps, g_->world, count, tmp.get());
  FSA_LAUNCH_CHECK();
  FSA_CUDA(cudaStreamSynchronize(s));
  g_->barrier();  // every rank has read every buffer
  FSA_CUDA(cudaMemcpyAsync(dev, tmp.get(), sizeof(double) * count, cudaMemcpyDeviceToDevice, s));
  FSA_CUDA(cudaStreamSynchronize(s));
}

void ThreadComm::exchange(const std::vector<HaloPeer>& peers, cudaStream_t s) {
  if (g_->world == 1) return;
  FSA_CUDA(cudaStreamSynchronize(s));
  for (int q = 0; q < g_->world; ++q) {
    g_->send[rank_][q] = nullptr;
    g_->send_count[rank_][q] = 0;
  }
  for (const HaloPeer& p : peers) {
    g_->send[rank_][p.rank] = p.send;
    g_->send_count[rank_][p.rank] = p.send_count;
  }
  g_->barrier();
  for (const HaloPeer& p : peers) {
    if (p.recv_count == 0) continue;
    require(g_->send_count[p.rank][rank_] == p.recv_count, "halo exchange: size mismatch between ranks");
    FSA_CUDA(cudaMemcpyAsync(p.recv, g_->send[p.rank][rank_], sizeof(double) * p.recv_count,
                             cudaMemcpyDeviceToDevice, s));
  }
  FSA_CUDA(cudaStreamSynchronize(s));
  g_->barrier();  // senders may reuse their buffers
}

std::vector<std::unique_ptr<Comm>> make_thread_group(int world) {
  require(world >= 1 && world <= kMaxThreadRanks, "thread group size must be in [1, 16]");
  auto g = std::make_shared<ThreadGroup>();
  g->world = world;
  std::vector<std::unique_ptr<Comm>> out;
  for (int r = 0; r < world; ++r) out.push_back(std::make_unique<ThreadComm>(g, r));
  return out;
}

// ---- NCCL (dlopen) -------------------------------------------------------------------------
namespace {
struct NcclApi {
  bool loaded = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
NcclApi& nccl() {
  static NcclApi api;
  if (api.loaded) return api;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) throw CudaError(std::string("NCCL unavailable: ") + dlerror());
  auto sym = [&](const char* name) {
    void* f = dlsym(h, name);
    if (!f) throw CudaError(std::string("NCCL symbol missing: ") + name);
    return f;
  };
  api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
  api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
  api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
  api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
  api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
  api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
  api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
  api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
  api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
  api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
  api.loaded = true;
  return api;
}
void nccl_check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) throw CudaError(std::string(what) + ": " + nccl().GetErrorString(r));
}
}  // namespace

void nccl_unique_id(void* out) {
  ncclUniqueId id;
  nccl_check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
  static_assert(sizeof(ncclUniqueId) == 128, "unexpected ncclUniqueId size");
  std::memcpy(out, &id, sizeof(id));
}

NcclComm::NcclComm(int rank, int world, const void* unique_id) : rank_(rank), world_(world) {
  require(world >= 1 && rank >= 0 && rank < world, "invalid rank / world size");
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof(id));
  ncclComm_t c = nullptr;
  nccl_check(nccl().CommInitRank(&c, world, id, rank), "ncclCommInitRank");
  comm_ = c;
}
NcclComm::~NcclComm() {
  if (comm_) nccl().CommDestroy(static_cast<ncclComm_t>(comm_));
}
// Fixed-order sum over ranks (SURVEY §8e "determinism needs fixed-order reductions"): the rank
// partials are all-gathered and every rank adds them in rank order, so the result is bitwise
// identical on every rank, run to run, and equal to the in-process ThreadComm's k_sum_ptrs order
// (whatever ring / tree / NVLS algorithm NCCL picks for the transfer). The payloads are an m x t
// projection (<= 0.6 MB at config 4) and t-long dot vectors: at W <= 8 the W-fold gather volume
// costs a few microseconds on NVLink, the same launch count as ncclAllReduce.
void NcclComm::allreduce(double* dev, long count, cudaStream_t s) {
  if (world_ == 1 || count == 0) return;
  const size_t need = static_cast<size_t>(count) * static_cast<size_t>(world_);
  if (gather_.n < need) gather_.alloc(need);
  nccl_check(nccl().AllGather(dev, gather_.get(), static_cast<size_t>(count), ncclDouble,
                              static_cast<ncclComm_t>(comm_), s),
             "ncclAllGather");
  k_sum_ranks<<<static_cast<unsigned>(cdiv(count, 256)), 256, 0, s>>>(gather_.get(), world_, count, dev);
  FSA_LAUNCH_CHECK();
}
void NcclComm::exchange(const std::vector<HaloPeer>& peers, cudaStream_t s) {
  if (world_ == 1) return;
  nccl_check(nccl().GroupStart(), "ncclGroupStart");
  for (const HaloPeer& p : peers) {
    if (p.send_count > 0)
      nccl_check(nccl().Send(p.send, static_cast<size_t>(p.send_count), ncclDouble, p.rank,
                             static_cast<ncclComm_t>(comm_), s),
                 "ncclSend");
    if (p.recv_count > 0)
      nccl_check(nccl().Recv(p.recv, static_cast<size_t>(p.recv_count), ncclDouble, p.rank,
                             static_cast<ncclComm_t>(comm_), s),
                 "ncclRecv");
  }
  nccl_check(nccl().GroupEnd(), "ncclGroupEnd");
}

}  // namespace fsa
