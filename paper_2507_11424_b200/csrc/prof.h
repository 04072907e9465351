// prof.h -- optional per-phase device-time accounting (CUDA events on the launching stream).
// Enabled with TN_PROFILE=1; read with tn_debug_profile(). Off by default (no events).
#pragma once
#include <cuda_runtime.h>

#include <vector>

namespace tn {

// P_TC_KERNEL (the tcgen05 GEMM kernel alone) nests inside P_GEMM_TC (operand prep + kernel).
enum ProfCat { P_GEMM_TC = 0, P_GEMM_SIMT, P_PERMUTE, P_ORTH, P_TAIL, P_MISC, P_TC_KERNEL, P_NCAT };

struct Prof {
  bool on = false;
  unsigned mask = ~0u;  // categories recorded while on (bit c = ProfCat c)
  struct Rec {
    int cat;
    cudaEvent_t a, b;
  };
  std::vector<Rec> pending;
  std::vector<cudaEvent_t> pool;
  double ms[P_NCAT] = {0};
  long count[P_NCAT] = {0};
  cudaEvent_t get();
  void flush();
};
extern Prof g_prof;

struct ProfScope {
  int cat;
  cudaStream_t s;
  cudaEvent_t a = nullptr;
  ProfScope(int c, cudaStream_t st) : cat(c), s(st) {
    if (g_prof.on && ((g_prof.mask >> c) & 1u)) {
      a = g_prof.get();
      cudaEventRecord(a, s);
    }
  }
  ~ProfScope() {
    if (g_prof.on && a) {
      cudaEvent_t b = g_prof.get();
      cudaEventRecord(b, s);
      g_prof.pending.push_back({cat, a, b});
      if (g_prof.pending.size() > 65536) g_prof.flush();  // rare: a flush synchronises
    }
  }
};

}  // namespace tn
