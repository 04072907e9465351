// debug.cu -- test-only entry points exposing single building blocks (contraction engine,
// orthonormalisation) on host buffers, for unit tests against numpy. Not part of the
// public ABI in include/tnsample.h.
#include <cstring>
#include <string>
#include <vector>

#include "linalg.h"
#include "tensor.h"

using namespace tn;

namespace {
thread_local std::string g_dbg_err;
}

extern "C" {

const char* tn_debug_last_error(void) { return g_dbg_err.c_str(); }

// out = contract(A[la], B[lb]) -> lout.  per_A/per_B: operand carries nb samples.
int tn_debug_contract(const char* la, int ra, const int* sa, const float* A, int conjA, int perA, const char* lb,
                      int rb, const int* sb, const float* B, int conjB, int perB, const char* lout, int nb,
                      float* out, int64_t out_elems, int gemm_mode) {
  try {
    Ctx c;
    TN_CUDA(cudaStreamCreate(&c.stream));
    c.nb = nb;
    c.gemm_mode = gemm_mode;
    std::vector<int> shA(sa, sa + ra), shB(sb, sb + rb);
    Tensor tA = new_tensor(c, shA, perA != 0), tB = new_tensor(c, shB, perB != 0);
    TN_CUDA(cudaMemcpy(tA.p, A, sizeof(float2) * tA.size() * (perA ? nb : 1), cudaMemcpyHostToDevice));
    TN_CUDA(cudaMemcpy(tB.p, B, sizeof(float2) * tB.size() * (perB ? nb : 1), cudaMemcpyHostToDevice));
    Tensor o = contract(c, tA, la, conjA != 0, tB, lb, conjB != 0, lout);
    int n = o.bstride ? nb : 1;
    if (o.size() * n != out_elems) throw Error(-1, "out size mismatch " + std::to_string(o.size() * n));
    TN_CUDA(cudaStreamSynchronize(c.stream));
    if (o.bstride && o.bstride != o.size()) throw Error(-1, "non-contiguous batch");
    TN_CUDA(cudaMemcpy(out, o.p, sizeof(float2) * out_elems, cudaMemcpyDeviceToHost));
    o = Tensor{};
    tA = Tensor{};
    tB = Tensor{};
    TN_CUDA(cudaStreamSynchronize(c.stream));
    cudaStreamDestroy(c.stream);
    return 0;
  } catch (const std::exception& e) {
    g_dbg_err = e.what();
    return -1;
  }
}

// Q = orthonormal basis of span(X) (m x n, row-major, nb matrices); C = Q^H X.
// transpose != 0: orthonormalise the ROWS of X (X is n x m row-major, as right_orth).
int tn_debug_orth(int m, int n, int nb, const float* X, float* Q, float* Cout, int transpose) {
  try {
    Ctx c;
    TN_CUDA(cudaStreamCreate(&c.stream));
    size_t sz = (size_t)m * n * nb;
    DevBuf dx(sz * sizeof(float2), c.stream), dq(sz * sizeof(float2), c.stream),
        dc((size_t)n * n * nb * sizeof(float2), c.stream);
    TN_CUDA(cudaMemcpy(dx.p, X, sz * sizeof(float2), cudaMemcpyHostToDevice));
    MatView xv, qv;
    if (!transpose) {
      xv = MatView{dx.as<float2>(), (int64_t)m * n, n, 1, false, m, n};
      qv = MatView{dq.as<float2>(), (int64_t)m * n, n, 1, false, m, n};
    } else {
      xv = MatView{dx.as<float2>(), (int64_t)m * n, 1, m, true, m, n};
      qv = MatView{dq.as<float2>(), (int64_t)m * n, 1, m, true, m, n};
    }
    orthonormalize(c, xv, qv, dc.as<float2>(), nb);
    TN_CUDA(cudaStreamSynchronize(c.stream));
    TN_CUDA(cudaMemcpy(Q, dq.p, sz * sizeof(float2), cudaMemcpyDeviceToHost));
    if (Cout) TN_CUDA(cudaMemcpy(Cout, dc.p, (size_t)n * n * nb * sizeof(float2), cudaMemcpyDeviceToHost));
    dx.release();
    dq.release();
    dc.release();
    TN_CUDA(cudaStreamSynchronize(c.stream));
    cudaStreamDestroy(c.stream);
    return 0;
  } catch (const std::exception& e) {
    g_dbg_err = e.what();
    return -1;
  }
}
}

#include "fit.h"

extern "C" {
// Run one Fit_R on host-provided strip tensors (shared, nb = 1) and return the sites.
// top_shape: 4 ints per column (single: [m,u,n,0]; double: [e,d,D,f]); top_data[j] NULL =
// identity with bond topbond[j]. mat_shape: 5 ints per column (single: [u,p,l,r,0];
// double: [s,u,d,l,r]). Sites are written back to back into out (complex64), their shapes
// (4 ints, trailing 0 for 3-leg sites) into out_shapes; returns K (or -1).
int tn_debug_fit(int dbl, int W, const int* top_shape, const float* const* top_data, const int* topbond,
                 const int* mat_shape, const float* const* mat_data, const int* out_cols, int R, int tag, int b1,
                 int nh, uint64_t seed, float* out, int64_t cap, int* out_shapes, double* logn, int gemm_mode) {
  try {
    Ctx c;
    TN_CUDA(cudaStreamCreate(&c.stream));
    c.nb = 1;
    c.gemm_mode = gemm_mode;
    DStrip s;
    s.dbl = dbl != 0;
    s.per_sample = false;
    s.W = W;
    for (int j = 0; j < W; ++j) {
      Tensor t;
      if (top_data[j]) {
        std::vector<int> sh(top_shape + 4 * j, top_shape + 4 * j + (dbl ? 4 : 3));
        t = new_tensor(c, sh, false);
        TN_CUDA(cudaMemcpy(t.p, top_data[j], sizeof(float2) * t.size(), cudaMemcpyHostToDevice));
      }
      s.tops.push_back(t);
      s.topbond.push_back(topbond[j]);
      std::vector<int> ms(mat_shape + 5 * j, mat_shape + 5 * j + (dbl ? 5 : 4));
      Tensor m = new_tensor(c, ms, false);
      TN_CUDA(cudaMemcpy(m.p, mat_data[j], sizeof(float2) * m.size(), cudaMemcpyHostToDevice));
      s.mats.push_back(m);
      s.out.push_back(out_cols[j] != 0);
    }
    int K = 0;
    {
      DevBuf ln(sizeof(double), c.stream);
      FitResult fr = fit(c, s, R, tag, b1, seed, nh, ln.as<double>(), false);
      TN_CUDA(cudaStreamSynchronize(c.stream));
      int64_t off = 0;
      if (fr.sites.empty()) {
        TN_CUDA(cudaMemcpy(out, fr.scalar.p, sizeof(float2), cudaMemcpyDeviceToHost));
      }
      for (size_t k = 0; k < fr.sites.size(); ++k) {
        const Tensor& t = fr.sites[k];
        if (off + t.size() > cap) throw Error(-1, "debug_fit: output buffer too small");
        TN_CUDA(cudaMemcpy(out + 2 * off, t.p, sizeof(float2) * t.size(), cudaMemcpyDeviceToHost));
        for (int q = 0; q < 4; ++q) out_shapes[4 * k + q] = q < t.rank() ? t.shape[q] : 0;
        off += t.size();
      }
      TN_CUDA(cudaMemcpy(logn, ln.p, sizeof(double), cudaMemcpyDeviceToHost));
      K = (int)fr.sites.size();
      s = DStrip{};
    }
    TN_CUDA(cudaStreamSynchronize(c.stream));
    cudaStreamDestroy(c.stream);
    return K;
  } catch (const std::exception& e) {
    g_dbg_err = e.what();
    return -1;
  }
}
}
