// Shared helpers for the B200 (sm_100a) FSA iterative core.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <stdexcept>
#include <string>

namespace fsa {

// ---- errors: mirror fsagp::NumericalError / std::invalid_argument (types.h:22-29)
struct NumericalError : std::runtime_error {
  explicit NumericalError(const std::string& w) : std::runtime_error(w) {}
};
struct CudaError : std::runtime_error {
  explicit CudaError(const std::string& w) : std::runtime_error(w) {}
};
inline void require(bool c, const char* msg) {
  if (!c) throw std::invalid_argument(msg);
}

#define FSA_CUDA(x)                                                                          \
  do {                                                                                       \
    cudaError_t e_ = (x);                                                                    \
    if (e_ != cudaSuccess)                                                                   \
      throw ::fsa::CudaError(std::string("CUDA error ") + cudaGetErrorString(e_) + " at " + \
                             __FILE__ + ":" + std::to_string(__LINE__));                     \
  } while (0)

// number of kernels this library has launched (every launch site ends with FSA_LAUNCH_CHECK)
inline std::atomic<long>& launch_counter() {
  static std::atomic<long> c{0};
  return c;
}

#ifdef FSA_CHECKED
#define FSA_LAUNCH_CHECK()                        \
  do {                                            \
    ::fsa::launch_counter().fetch_add(1);         \
    FSA_CUDA(cudaGetLastError());                 \
    FSA_CUDA(cudaDeviceSynchronize());            \
  } while (0)
#else
#define FSA_LAUNCH_CHECK()                        \
  do {                                            \
    ::fsa::launch_counter().fetch_add(1);         \
    FSA_CUDA(cudaGetLastError());                 \
  } while (0)
#endif

// NVTX phase range (assemble / FITC setup / PCG / SLQ / traces / prediction): visible in nsys /
// ncu --nvtx; no-ops without a tool attached (NVTX v3 is header-only)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

// ---- checked build (make checked -> build/checked/libfsa_b200.so, FSA_LIB selects it) ----------
// Bounds checks on the gather / scatter indices of the sweep kernels, and a stream synchronisation
// after every launch so a fault is reported at the kernel that caused it (graph capture is then
// off). The pool's compute-sanitizer is closed; this is the substitute.
#ifdef FSA_CHECKED
#define FSA_DCHECK(cond, what)                                                                     \
  do {                                                                                            \
    if (!(cond)) {                                                                                \
      printf("FSA_DCHECK failed: %s (%s:%d) block %d thread %d\n", what, __FILE__, __LINE__,      \
             static_cast<int>(blockIdx.x), static_cast<int>(threadIdx.x));                        \
      __trap();                                                                                   \
    }                                                                                             \
  } while (0)
constexpr bool kChecked = true;
#else
#define FSA_DCHECK(cond, what) \
  do {                         \
  } while (0)
constexpr bool kChecked = false;
#endif

// ---- programmatic dependent launch (PDL) -------------------------------------------------
// The PCG sweep kernels are launched with programmatic stream serialisation: a kernel's CTAs
// may be scheduled while its predecessor drains, and each such kernel executes pdl_wait()
// (griddepcontrol.wait) before it touches anything the predecessor writes (setup such as TMEM
// allocation and mbarrier initialisation goes first). Without the attribute the wait is a no-op.
// FSA_PDL=0 disables it (A/B measurement).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("FSA_PDL");
    return !(e != nullptr && e[0] == '0');
  }();
  return on;
}
template <typename... Params, typename... Args>
inline void launch_pdl(void (*kern)(Params...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, static_cast<Params>(args)...);
  if (e != cudaSuccess) throw CudaError(std::string("kernel launch: ") + cudaGetErrorString(e));
}

inline long round_up(long x, long a) { return (x + a - 1) / a * a; }
inline long cdiv(long x, long a) { return (x + a - 1) / a; }

// column padding of an n x t right-hand-side block (row-major, ld = tpad)
inline long pad_cols(long t) { return t <= 72 ? round_up(t < 1 ? 1 : t, 8) : round_up(t, 64); }

constexpr int kNumSMs = 148;

// ---- device buffers ------------------------------------------------------------
// Stream-ordered allocation from the device's default memory pool (release
// threshold raised by Context), so per-evaluation temporaries neither hit
// cudaMalloc nor serialise the stream on cudaFree.
inline cudaStream_t& alloc_stream() {
  static thread_local cudaStream_t s = nullptr;
  return s;
}

template <class T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;
  DBuf() = default;
  explicit DBuf(size_t count) { alloc(count); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~DBuf() { release(); }
  void alloc(size_t count) {
    if (count == n && p) return;
    release();
    n = count;
    if (count) FSA_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), alloc_stream()));
  }
  void release() {
    if (p) cudaFreeAsync(p, alloc_stream());
    p = nullptr;
    n = 0;
  }
  void zero(cudaStream_t s) {
    if (n) FSA_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s));
  }
  T* get() const { return p; }
  size_t bytes() const { return n * sizeof(T); }
};

}  // namespace fsa
