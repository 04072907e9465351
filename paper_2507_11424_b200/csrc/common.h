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

// Count of this library's kernel launches on the calling thread (reported as gpu_launches by
// bench.py and per call by tn_get_stats). Thread-local: distinct states may be driven from
// distinct threads concurrently.
extern thread_local int64_t g_launches;
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
  // Optional device floats: upper bounds of max |component| over the buffer's complex
  // contents, one per sample of the batch (tail_n = the batch size; 1 for a shared tensor),
  // written by the tensor-core GEMM that produced them (lets a consumer GEMM scale its FP16
  // operand planes without a max pass, per sample, so that a sample's result never depends
  // on which other samples share its batch). They live in `tail` spare bytes allocated after
  // the data (no separate allocation); any in-place write must drop them.
  float* tail = nullptr;
  int tail_n = 0;
  bool amax_valid = false;
  DevBuf() = default;
  DevBuf(size_t n, cudaStream_t st, int tail_floats = 0) { alloc(n, st, tail_floats); }
  void alloc(size_t n, cudaStream_t st, int tail_floats = 0) {
    release();
    s = st;
    bytes = n;
    if (n) {
      const size_t pad = tail_floats > 0 ? ((size_t)tail_floats * sizeof(float) + 255) / 256 * 256 : 0;
      TN_CUDA(cudaMallocAsync(&p, n + pad, st));
      if (tail_floats > 0) {
        tail = reinterpret_cast<float*>(reinterpret_cast<char*>(p) + ((n + 15) / 16) * 16);
        tail_n = tail_floats;
      }
    }
  }
  float* amax() const { return amax_valid ? tail : nullptr; }
  float* make_amax() {  // the producer zeroes the tail_n floats (stream order) before writing
    if (!tail) return nullptr;
    amax_valid = true;
    return tail;
  }
  void drop_amax() { amax_valid = false; }
  void release() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    tail = nullptr;
    tail_n = 0;
    amax_valid = false;
    bytes = 0;
  }
  ~DevBuf() { release(); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept
      : p(o.p), bytes(o.bytes), s(o.s), tail(o.tail), tail_n(o.tail_n), amax_valid(o.amax_valid) {
    o.p = nullptr; o.bytes = 0; o.tail = nullptr; o.tail_n = 0; o.amax_valid = false;
  }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p; bytes = o.bytes; s = o.s; tail = o.tail; tail_n = o.tail_n; amax_valid = o.amax_valid;
      o.p = nullptr; o.bytes = 0; o.tail = nullptr; o.tail_n = 0; o.amax_valid = false;
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
