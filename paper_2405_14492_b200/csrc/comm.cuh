// Communicators for the row-sharded FSA core.
//
// Ranks own contiguous row blocks of the Hilbert-sorted points. Per PCG sweep
// they exchange the halo rows of the RHS block (neighbour-to-neighbour) and
// sum m x t projections and per-column dot products. Three implementations:
//   SelfComm   world = 1, every collective is a no-op
//   NcclComm   one process per GPU, NCCL over NVLink/NVSwitch (libnccl is
//              dlopen'ed when the first distributed context is created)
//   ThreadComm P ranks as P host threads of one process; collectives are host
//              barriers plus device copies (no kernel ever waits on another),
//              which lets the sharded path be checked on a single GPU.
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "common.cuh"

namespace fsa {

struct HaloPeer {
  int rank;
  const double* send;  // contiguous send rows (device)
  long send_count;     // doubles
  double* recv;        // contiguous receive rows (device)
  long recv_count;     // doubles
};

class Comm {
 public:
  virtual ~Comm() = default;
  virtual int rank() const = 0;
  virtual int size() const = 0;
  virtual std::string kind() const = 0;
  // in-place sum over ranks of a device array, added in rank order: bitwise identical on every
  // rank and for every implementation (thread group, NCCL)
  virtual void allreduce(double* dev, long count, cudaStream_t s) = 0;
  // point-to-point exchange with each listed peer
  virtual void exchange(const std::vector<HaloPeer>& peers, cudaStream_t s) = 0;
  // sum of a small host array (through the device path)
  void allreduce_host(double* host, long count, cudaStream_t s);
};

class SelfComm final : public Comm {
 public:
  int rank() const override { return 0; }
  int size() const override { return 1; }
  std::string kind() const override { return "self"; }
  void allreduce(double*, long, cudaStream_t) override {}
  void exchange(const std::vector<HaloPeer>&, cudaStream_t) override {}
};

// shared state of an in-process group
struct ThreadGroup;
class ThreadComm final : public Comm {
 public:
  ThreadComm(std::shared_ptr<ThreadGroup> g, int rank);
  int rank() const override { return rank_; }
  int size() const override;
  std::string kind() const override { return "thread"; }
  void allreduce(double* dev, long count, cudaStream_t s) override;
  void exchange(const std::vector<HaloPeer>& peers, cudaStream_t s) override;

 private:
  std::shared_ptr<ThreadGroup> g_;
  int rank_;
};
std::vector<std::unique_ptr<Comm>> make_thread_group(int world);

class NcclComm final : public Comm {
 public:
  NcclComm(int rank, int world, const void* unique_id /* 128 bytes */);
  ~NcclComm() override;
  int rank() const override { return rank_; }
  int size() const override { return world_; }
  std::string kind() const override { return "nccl"; }
  void allreduce(double* dev, long count, cudaStream_t s) override;
  void exchange(const std::vector<HaloPeer>& peers, cudaStream_t s) override;

 private:
  int rank_, world_;
  void* comm_ = nullptr;  // ncclComm_t
  DBuf<double> gather_;   // [world][count] partials of the fixed-order allreduce
};
// fills 128 bytes with a fresh ncclUniqueId (rank 0 calls it and broadcasts)
void nccl_unique_id(void* out);

}  // namespace fsa
