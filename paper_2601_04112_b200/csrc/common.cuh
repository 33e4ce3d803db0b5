// common.cuh — error plumbing, device buffers and cooperative "teams" shared
// by every kernel of the B200 AMG-DD library.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../../include/lsamgdd_b200.h"

namespace lsb {

// Status-carrying exception; the C ABI maps it to lsamgdd_status and the
// reference exception class of the same name (errors.hpp:11-69).
struct Error : std::runtime_error {
  int status;
  Error(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};

[[noreturn]] inline void raise(int status, const std::string& msg) { throw Error(status, msg); }

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
  if (e != cudaSuccess) {
    const int st = (e == cudaErrorMemoryAllocation) ? LSAMGDD_ERR_OOM : LSAMGDD_ERR_CUDA;
    raise(st, std::string("CUDA error in ") + what + " (" + file + ":" + std::to_string(line) +
                  "): " + cudaGetErrorString(e));
  }
}
// Kernels launched by this thread (the bench's gpu_launches claim).
inline int64_t& launch_counter() {
  static thread_local int64_t n = 0;
  return n;
}
#define LSB_CUDA(call) ::lsb::cuda_check((call), #call, __FILE__, __LINE__)
#define LSB_LAUNCH()                                                             \
  do {                                                                           \
    ++::lsb::launch_counter();                                                   \
    ::lsb::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__); \
  } while (0)

// The library's own memory pool of the current device: every DBuf comes from it. Freed blocks stay
// mapped between calls (release threshold = max, like a caching allocator), so repeated setups do
// not pay for remapping tens of GB each time and the host application's default pool and its
// release threshold are left alone; lsamgdd_trim_memory hands the cached memory back.
cudaMemPool_t device_pool();
void trim_device_pool(int device);

// Stream-ordered device buffer (cudaMallocFromPoolAsync on the owner's stream).
template <class T>
class DBuf {
 public:
  DBuf() = default;
  DBuf(size_t n, cudaStream_t s) { alloc(n, s); }
  ~DBuf() { release(); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept { swap(o); }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      release();
      swap(o);
    }
    return *this;
  }
  void alloc(size_t n, cudaStream_t s) {
    release();
    stream_ = s;
    n_ = n;
    if (n) LSB_CUDA(cudaMallocFromPoolAsync(reinterpret_cast<void**>(&p_), n * sizeof(T), device_pool(), s));
  }
  void release() {
    if (p_) cudaFreeAsync(p_, stream_);
    p_ = nullptr;
    n_ = 0;
  }
  void zero(cudaStream_t s) {
    if (n_) LSB_CUDA(cudaMemsetAsync(p_, 0, n_ * sizeof(T), s));
  }
  void upload(const T* h, size_t n, cudaStream_t s) {
    if (n != n_) alloc(n, s);
    if (n) LSB_CUDA(cudaMemcpyAsync(p_, h, n * sizeof(T), cudaMemcpyHostToDevice, s));
  }
  void upload(const std::vector<T>& h, cudaStream_t s) { upload(h.data(), h.size(), s); }
  std::vector<T> download(cudaStream_t s) const {
    std::vector<T> h(n_);
    if (n_) {
      // Wait for the stream first: a copy into pageable memory blocks inside the driver until the
      // stream's earlier kernels finish, and other host threads' CUDA calls queue up behind it.
      LSB_CUDA(cudaStreamSynchronize(s));
      LSB_CUDA(cudaMemcpyAsync(h.data(), p_, n_ * sizeof(T), cudaMemcpyDeviceToHost, s));
      LSB_CUDA(cudaStreamSynchronize(s));
    }
    return h;
  }
  T* get() const { return p_; }
  size_t size() const { return n_; }
  size_t bytes() const { return n_ * sizeof(T); }

 private:
  void swap(DBuf& o) noexcept {
    std::swap(p_, o.p_);
    std::swap(n_, o.n_);
    std::swap(stream_, o.stream_);
  }
  T* p_ = nullptr;
  size_t n_ = 0;
  cudaStream_t stream_ = nullptr;
};

template <class T>
T read_scalar(const T* d, cudaStream_t s) {
  T h{};
  LSB_CUDA(cudaStreamSynchronize(s));  // see DBuf::download
  LSB_CUDA(cudaMemcpyAsync(&h, d, sizeof(T), cudaMemcpyDeviceToHost, s));
  LSB_CUDA(cudaStreamSynchronize(s));
  return h;
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Number of SMs of the current device (148 on B200); grids are sized in
// multiples of it.
int sm_count();

// True the first time it is called for the current device with this flag word
// (one bit per device ordinal): guards per-device one-time settings such as
// cudaFuncSetAttribute without process-wide booleans.
bool first_on_device(std::atomic<uint64_t>& flags);

#ifdef __CUDACC__
// A cooperating group that runs one problem: a warp (lane-parallel,
// __syncwarp) or a whole CTA (__syncthreads). Every batched setup kernel is
// written once against this interface and instantiated for both.
struct WarpTeam {
  __device__ int rank() const { return threadIdx.x & 31; }
  __device__ static constexpr int size() { return 32; }
  __device__ void sync() const { __syncwarp(); }
};
struct BlockTeam {
  __device__ int rank() const { return threadIdx.x; }
  __device__ int size() const { return blockDim.x; }
  __device__ void sync() const { __syncthreads(); }
};
// The leader CTA of a cluster launch: a BlockTeam whose eigensolves all take
// the cluster wavefront path (no single-CTA pipeline, whose static shared
// arrays would not fit beside the wavefront's staging buffers).
struct ClusterLeadTeam : BlockTeam {};
#endif

}  // namespace lsb
