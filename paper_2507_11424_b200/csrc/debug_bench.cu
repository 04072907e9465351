// debug_bench.cu -- test-only GEMM timing entry point (device-resident operands).
#include <cmath>
#include <vector>

#include "tensor.h"

using namespace tn;

namespace {
__global__ void fill_hash(float2* p, int64_t n, uint64_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = (uint64_t)i * 0x9E3779B97F4A7C15ull + seed;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    p[i] = make_float2((float)(z >> 40) * 0x1.0p-23f - 1.f, (float)((z >> 16) & 0xFFFFFF) * 0x1.0p-23f - 1.f);
  }
}
}  // namespace

extern "C" int tn_debug_gemm_bench(int M, int N, int K, int nb, int mode, int reps, double* out) {
  try {
    Ctx c;
    TN_CUDA(cudaStreamCreate(&c.stream));
    c.nb = nb;
    c.gemm_mode = mode;
    {
      // as tn_load_state: keep freed blocks in the pool (otherwise every synchronisation
      // returns GBs to the OS and the next call re-maps them inside the timed region)
      int dev = 0;
      cudaMemPool_t pool;
      TN_CUDA(cudaGetDevice(&dev));
      TN_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
      uint64_t thr = UINT64_MAX;
      TN_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    }
    double ms = 0, err = 0;
    {
      Tensor A = new_tensor(c, {M, K}, true), B = new_tensor(c, {K, N}, false);
      fill_hash<<<1184, 256, 0, c.stream>>>(A.p, (int64_t)M * K * nb, 1);
      fill_hash<<<1184, 256, 0, c.stream>>>(B.p, (int64_t)K * N, 2);
      Tensor Cw = contract(c, A, "mk", false, B, "kn", false, "mn");  // warm-up
      cudaEvent_t e0, e1;
      TN_CUDA(cudaEventCreate(&e0));
      TN_CUDA(cudaEventCreate(&e1));
      TN_CUDA(cudaEventRecord(e0, c.stream));
      for (int r = 0; r < reps; ++r) Cw = contract(c, A, "mk", false, B, "kn", false, "mn");
      TN_CUDA(cudaEventRecord(e1, c.stream));
      TN_CUDA(cudaEventSynchronize(e1));
      float t = 0;
      TN_CUDA(cudaEventElapsedTime(&t, e0, e1));
      ms = t / reps;
      // fp64 check of a few rows x columns
      int rows = 4, cols = std::min(N, 64);
      std::vector<float2> a((size_t)rows * K), b((size_t)K * N), cc((size_t)rows * N);
      TN_CUDA(cudaMemcpy(a.data(), A.p, sizeof(float2) * a.size(), cudaMemcpyDeviceToHost));
      TN_CUDA(cudaMemcpy(b.data(), B.p, sizeof(float2) * b.size(), cudaMemcpyDeviceToHost));
      TN_CUDA(cudaMemcpy(cc.data(), Cw.p, sizeof(float2) * cc.size(), cudaMemcpyDeviceToHost));
      double num = 0, den = 0;
      for (int i = 0; i < rows; ++i)
        for (int j = 0; j < cols; ++j) {
          double re = 0, im = 0;
          for (int k = 0; k < K; ++k) {
            float2 x = a[(size_t)i * K + k], y = b[(size_t)k * N + j];
            re += (double)x.x * y.x - (double)x.y * y.y;
            im += (double)x.x * y.y + (double)x.y * y.x;
          }
          float2 g = cc[(size_t)i * N + j];
          num += (g.x - re) * (g.x - re) + (g.y - im) * (g.y - im);
          den += re * re + im * im;
        }
      err = std::sqrt(num / std::max(den, 1e-300));
      A = Tensor{};
      B = Tensor{};
      Cw = Tensor{};
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
    }
    TN_CUDA(cudaStreamSynchronize(c.stream));
    cudaStreamDestroy(c.stream);
    out[0] = ms;
    out[1] = err;
    return 0;
  } catch (const std::exception& e) {
    fprintf(stderr, "%s\n", e.what());
    return -1;
  }
}

// Counters for bench.py: [0] complex MACs issued, [1] of which on tcgen05, [2] tcgen05 GEMM
// kernel launches, [3] all kernel launches of this library.
extern "C" int tn_debug_counters(double* out, int reset) {
  out[0] = tn::g_cmacs;
  out[1] = tn::g_cmacs_tc;
  out[2] = (double)tn::g_tc_launches;
  out[3] = (double)tn::g_launches;
  if (reset) {
    tn::g_cmacs = 0;
    tn::g_cmacs_tc = 0;
    tn::g_tc_launches = 0;
  }
  return 0;
}

// Per-row complex MACs of the last sampled batch (all samples of the batch).
extern "C" int tn_debug_row_cmacs(double* out, int n) {
  int m = (int)tn::g_row_cmacs.size();
  for (int i = 0; i < n && i < m; ++i) out[i] = tn::g_row_cmacs[i];
  return m;
}

#include "linalg.h"

// Timing of one batched orthonormalisation (debug/benchmark only): nb random m x n matrices
// (well conditioned), `reps` calls, average ms per call in out[0].
extern "C" int tn_debug_orth_bench(int m, int n, int nb, int reps, int with_c, double* out) {
  try {
    Ctx c;
    TN_CUDA(cudaStreamCreate(&c.stream));
    {
      int dev = 0;
      cudaMemPool_t pool;
      TN_CUDA(cudaGetDevice(&dev));
      TN_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
      uint64_t thr = UINT64_MAX;
      TN_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    }
    size_t sz = (size_t)m * n * nb;
    DevBuf dx(sz * sizeof(float2), c.stream), dq(sz * sizeof(float2), c.stream),
        dc((size_t)n * n * nb * sizeof(float2), c.stream);
    fill_hash<<<1184, 256, 0, c.stream>>>(dx.as<float2>(), (int64_t)sz, 7);
    MatView xv{dx.as<float2>(), (int64_t)m * n, n, 1, false, m, n};
    MatView qv{dq.as<float2>(), (int64_t)m * n, n, 1, false, m, n};
    orthonormalize(c, xv, qv, with_c ? dc.as<float2>() : nullptr, nb);
    cudaEvent_t e0, e1;
    TN_CUDA(cudaEventCreate(&e0));
    TN_CUDA(cudaEventCreate(&e1));
    TN_CUDA(cudaEventRecord(e0, c.stream));
    for (int r = 0; r < reps; ++r) orthonormalize(c, xv, qv, with_c ? dc.as<float2>() : nullptr, nb);
    TN_CUDA(cudaEventRecord(e1, c.stream));
    TN_CUDA(cudaEventSynchronize(e1));
    float t = 0;
    TN_CUDA(cudaEventElapsedTime(&t, e0, e1));
    out[0] = t / reps;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    dx.release();
    dq.release();
    dc.release();
    TN_CUDA(cudaStreamSynchronize(c.stream));
    cudaStreamDestroy(c.stream);
    return 0;
  } catch (const std::exception& e) {
    fprintf(stderr, "%s\n", e.what());
    return -1;
  }
}
