// Host-side helpers shared by the driver and the model code.
#pragma once
#include <algorithm>
#include <stdexcept>
#include <string>

#include <cuda_runtime.h>

namespace simnet {

struct ApiError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// A sub-trace's write queue outgrew its device ring (the reference's queue is
// an unbounded deque): the round loop reruns with a larger ring when the
// caller left write_ring on auto (0).
struct WriteRingOverflow : ApiError {
  uint32_t capacity;
  WriteRingOverflow(const std::string& m, uint32_t cap) : ApiError(m), capacity(cap) {}
};

#define CUDA_OK(expr)                                                                      \
  do {                                                                                     \
    cudaError_t e_ = (expr);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      throw ::simnet::ApiError(std::string("CUDA error: ") + cudaGetErrorString(e_) +      \
                               " at " #expr);                                              \
  } while (0)

// Grow-only device allocation.
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  void* need(size_t b) {
    if (b > bytes) {
      if (p) cudaFree(p);
      p = nullptr;
      bytes = 0;
      const size_t want = std::max<size_t>(b, 256);
      CUDA_OK(cudaMalloc(&p, want));
      bytes = want;
    }
    return p;
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

}  // namespace simnet
