// common.h -- shared host/device utilities of libtnsample (B200, sm_100a).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

namespace tn {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define TN_CUDA(x)                                                                      \
  do {                                                                                  \
    cudaError_t _e = (x);                                                               \
    if (_e != cudaSuccess) {                                                            \
      if (_e == cudaErrorMemoryAllocation)                                              \
        throw ::tn::Error(-4, std::string("CUDA out of memory at ") + __FILE__ + ":" +  \
                                  std::to_string(__LINE__));                            \
      throw ::tn::Error(-5, std::string("CUDA error ") + cudaGetErrorString(_e) + " at " + \
                                __FILE__ + ":" + std::to_string(__LINE__));             \
    }                                                                                   \
  } while (0)

// Count of this library's kernel launches (reported as gpu_launches by bench.py).
extern int64_t g_launches;
inline void note_launch() {
  ++g_launches;
}
#define TN_LAUNCHED()                 \
  do {                                \
    ::tn::note_launch();              \
    TN_CUDA(cudaGetLastError());      \
  } while (0)

// Stream-ordered device buffer (cudaMallocAsync pool; freed on the same stream).
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaStream_t s = nullptr;
  DevBuf() = default;
  DevBuf(size_t n, cudaStream_t st) { alloc(n, st); }
  void alloc(size_t n, cudaStream_t st) {
    release();
    s = st;
    bytes = n;
    if (n) TN_CUDA(cudaMallocAsync(&p, n, st));
  }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    bytes = 0;
  }
  ~DevBuf() { release(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes), s(o.s) { o.p = nullptr; o.bytes = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p; bytes = o.bytes; s = o.s;
      o.p = nullptr; o.bytes = 0;
    }
    return *this;
  }
  template <class T> T* as() const { return reinterpret_cast<T*>(p); }
};

inline int64_t prod(const std::vector<int>& v) {
  int64_t r = 1;
  for (int x : v) r *= x;
  return r;
}

inline unsigned ceil_div(int64_t a, int64_t b) { return (unsigned)((a + b - 1) / b); }

}  // namespace tn
