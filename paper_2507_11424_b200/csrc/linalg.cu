// linalg.cu -- CholeskyQR2 with pivoted rank detection, FP64 arithmetic (see linalg.h).
#include <algorithm>
#include <atomic>
#include <complex>
#include <cstdio>
#include <vector>

#include "linalg.h"

namespace tn {
__device__ long long g_chol_clk[8];  // debugging: phase clocks of the last chol_smem_kernel (block 0)
__device__ int g_chol_dbg = 0;       // debugging (timing experiments only): bit 0 skips the Schur update
namespace {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {  // conj(a) * b
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__device__ __forceinline__ double2 ld2(const float2* p, bool cj) {
  float2 v = *p;
  return make_double2((double)v.x, cj ? -(double)v.y : (double)v.y);
}

// ---- cross product  out[b][i][j] = sum_r conj(Y(r,i)) X(r,j)   (fp64 accumulation) ----
// grid: (tiles_j, tiles_i, nb * splits); partial results to part[b][split][i][j].
constexpr int CT = 32;
__global__ void __launch_bounds__(256) cross64_kernel(MatView Y, MatView X, int m, int splits,
                                                      double2* __restrict__ part) {
  __shared__ double2 sy[CT][CT + 1];
  __shared__ double2 sx[CT][CT + 1];
  int b = blockIdx.z / splits, sp = blockIdx.z - b * splits;
  int i0 = blockIdx.y * CT, j0 = blockIdx.x * CT;
  int rows_per = (m + splits - 1) / splits;
  int r_begin = sp * rows_per, r_end = min(m, r_begin + rows_per);
  int t = threadIdx.x;
  int ti = t >> 3, tj = (t & 7) * 4;  // 32 rows of i, 4 consecutive j per thread
  double2 acc[4] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
  const float2* yb = Y.p + b * Y.bs;
  const float2* xb = X.p + b * X.bs;
  for (int r0 = r_begin; r0 < r_end; r0 += CT) {
    for (int e = t; e < CT * CT; e += 256) {
      int rr = e / CT, cc = e - rr * CT;
      int r = r0 + rr;
      bool ok = r < r_end;
      sy[rr][cc] = (ok && i0 + cc < Y.n) ? ld2(yb + r * Y.si + (i0 + cc) * Y.sj, Y.cj) : make_double2(0, 0);
      sx[rr][cc] = (ok && j0 + cc < X.n) ? ld2(xb + r * X.si + (j0 + cc) * X.sj, X.cj) : make_double2(0, 0);
    }
    __syncthreads();
#pragma unroll 4
    for (int rr = 0; rr < CT; ++rr) {
      double2 yv = sy[rr][ti];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        double2 p = cmulc(yv, sx[rr][tj + q]);
        acc[q].x += p.x;
        acc[q].y += p.y;
      }
    }
    __syncthreads();
  }
  int nI = Y.n, nJ = X.n;
  double2* out = part + ((int64_t)b * splits + sp) * nI * nJ;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    int i = i0 + ti, j = j0 + tj + q;
    if (i < nI && j < nJ) out[(int64_t)i * nJ + j] = acc[q];
  }
}

__global__ void reduce_splits(const double2* __restrict__ part, double2* __restrict__ out, int splits,
                              int64_t per, int nb) {
  int64_t tot = per * nb;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = e / per, r = e - b * per;
    double2 s = make_double2(0, 0);
    for (int k = 0; k < splits; ++k) {
      double2 v = part[(b * splits + k) * per + r];
      s.x += v.x;
      s.y += v.y;
    }
    out[e] = s;
  }
}

// G[b] = sum over splits of the Gram partials (fixed order, 4 independent partial sums so the
// loads overlap); herm: lower triangle only; inactive matrices skipped.
__global__ void reduce_gram_kernel(const double2* __restrict__ part, double2* __restrict__ out, int splits, int nI,
                                   int nJ, int nb, int herm, const int* __restrict__ active) {
  const int64_t per = (int64_t)nI * nJ, tot = per * nb;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = e / per, r = e - b * per;
    if (active && !active[b]) continue;
    if (herm && (r % nJ) > (r / nJ)) continue;
    const double2* p = part + b * splits * per + r;
    double2 s0 = make_double2(0, 0), s1 = s0, s2 = s0, s3 = s0;
    int k = 0;
    for (; k + 4 <= splits; k += 4) {
      const double2 v0 = p[(k + 0) * per], v1 = p[(k + 1) * per], v2 = p[(k + 2) * per], v3 = p[(k + 3) * per];
      s0.x += v0.x; s0.y += v0.y;
      s1.x += v1.x; s1.y += v1.y;
      s2.x += v2.x; s2.y += v2.y;
      s3.x += v3.x; s3.y += v3.y;
    }
    for (; k < splits; ++k) {
      const double2 v = p[k * per];
      s0.x += v.x;
      s0.y += v.y;
    }
    out[e] = make_double2((s0.x + s1.x) + (s2.x + s3.x), (s0.y + s1.y) + (s2.y + s3.y));
  }
}

// ---- pivoted Cholesky (rank detection). One CTA per matrix; G (n x n, full Hermitian)
// is overwritten. Outputs perm[b][n], rank[b], dmax[b] (largest initial diagonal).
__global__ void __launch_bounds__(512) pivchol_kernel(double2* __restrict__ Gall, int n, double tol,
                                                      int* __restrict__ perm_all, int* __restrict__ rank_all,
                                                      double* __restrict__ dmax_all) {
  int b = blockIdx.x;
  double2* G = Gall + (int64_t)b * n * n;
  int* perm = perm_all + (int64_t)b * n;
  __shared__ double sval[512];
  __shared__ int sidx[512];
  __shared__ int s_piv;
  __shared__ double s_d0;
  __shared__ int s_rank;
  int t = threadIdx.x, nt = blockDim.x;
  for (int i = t; i < n; i += nt) perm[i] = i;
  // d0 = max diagonal
  double best = 0;
  for (int i = t; i < n; i += nt) best = fmax(best, G[(int64_t)i * n + i].x);
  sval[t] = best;
  __syncthreads();
  for (int s = nt / 2; s > 0; s >>= 1) {
    if (t < s) sval[t] = fmax(sval[t], sval[t + s]);
    __syncthreads();
  }
  if (t == 0) { s_d0 = sval[0]; s_rank = n; }
  __syncthreads();
  double d0 = s_d0;
  for (int k = 0; k < n; ++k) {
    // argmax of the remaining diagonal (lowest index on ties)
    double bv = -1;
    int bi = n;
    for (int i = k + t; i < n; i += nt) {
      double v = G[(int64_t)i * n + i].x;
      if (v > bv) { bv = v; bi = i; }
    }
    sval[t] = bv;
    sidx[t] = bi;
    __syncthreads();
    for (int s = nt / 2; s > 0; s >>= 1) {
      if (t < s) {
        if (sval[t + s] > sval[t] || (sval[t + s] == sval[t] && sidx[t + s] < sidx[t])) {
          sval[t] = sval[t + s];
          sidx[t] = sidx[t + s];
        }
      }
      __syncthreads();
    }
    if (t == 0) s_piv = sidx[0];
    __syncthreads();
    int p = s_piv;
    double dp = sval[0];
    __syncthreads();
    if (!(dp > tol * d0) || d0 <= 0) {
      if (t == 0) s_rank = k;
      break;
    }
    if (p != k) {
      // swap rows p,k then columns p,k
      for (int j = t; j < n; j += nt) {
        double2 a = G[(int64_t)k * n + j], c2 = G[(int64_t)p * n + j];
        G[(int64_t)k * n + j] = c2;
        G[(int64_t)p * n + j] = a;
      }
      __syncthreads();
      for (int i = t; i < n; i += nt) {
        double2 a = G[(int64_t)i * n + k], c2 = G[(int64_t)i * n + p];
        G[(int64_t)i * n + k] = c2;
        G[(int64_t)i * n + p] = a;
      }
      if (t == 0) {
        int tmp = perm[k];
        perm[k] = perm[p];
        perm[p] = tmp;
      }
      __syncthreads();
    }
    double lkk = sqrt(G[(int64_t)k * n + k].x);
    for (int i = k + 1 + t; i < n; i += nt) {
      double2 v = G[(int64_t)i * n + k];
      G[(int64_t)i * n + k] = make_double2(v.x / lkk, v.y / lkk);
    }
    __syncthreads();
    int w = n - k - 1;
    for (int e = t; e < w * w; e += nt) {
      int i = k + 1 + e / w, j = k + 1 + e % w;
      double2 li = G[(int64_t)i * n + k], lj = G[(int64_t)j * n + k];
      double2 pr = cmul(li, make_double2(lj.x, -lj.y));
      double2 g = G[(int64_t)i * n + j];
      G[(int64_t)i * n + j] = make_double2(g.x - pr.x, g.y - pr.y);
    }
    __syncthreads();
  }
  __syncthreads();
  if (t == 0) {
    rank_all[b] = s_rank;
    dmax_all[b] = d0;
  }
}

// ---- Cholesky (no pivoting) and W = R^{-1}, R = L^H. One CTA per matrix.
__global__ void __launch_bounds__(512) cholinv_kernel(double2* __restrict__ Gall, double2* __restrict__ Wall,
                                                      int n, int* __restrict__ bad) {
  int b = blockIdx.x;
  double2* G = Gall + (int64_t)b * n * n;
  double2* W = Wall + (int64_t)b * n * n;
  int t = threadIdx.x, nt = blockDim.x;
  double scale = 0;
  for (int k = 0; k < n; ++k) scale = fmax(scale, G[(int64_t)k * n + k].x);
  for (int k = 0; k < n; ++k) {
    double d = G[(int64_t)k * n + k].x;
    if (!(d > 1e-300 + 1e-30 * scale)) {
      if (t == 0) atomicOr(bad, 1);
      d = 1e-300 + 1e-30 * scale;
    }
    double lkk = sqrt(d);
    __syncthreads();
    if (t == 0) G[(int64_t)k * n + k] = make_double2(lkk, 0);
    for (int i = k + 1 + t; i < n; i += nt) {
      double2 v = G[(int64_t)i * n + k];
      G[(int64_t)i * n + k] = make_double2(v.x / lkk, v.y / lkk);
    }
    __syncthreads();
    int w = n - k - 1;
    for (int e = t; e < w * w; e += nt) {
      int i = k + 1 + e / w, j = k + 1 + e % w;
      if (j > i) continue;  // lower triangle only
      double2 li = G[(int64_t)i * n + k], lj = G[(int64_t)j * n + k];
      double2 pr = cmul(li, make_double2(lj.x, -lj.y));
      double2 g = G[(int64_t)i * n + j];
      G[(int64_t)i * n + j] = make_double2(g.x - pr.x, g.y - pr.y);
    }
    __syncthreads();
  }
  // Linv column j by forward substitution (thread per column); W = Linv^H
  for (int j = t; j < n; j += nt) {
    // y_i for i >= j; reuse W row j as scratch: W[j][i] = conj(y_i) at the end
    for (int i = 0; i < j; ++i) W[(int64_t)i * n + j] = make_double2(0, 0);
    for (int i = j; i < n; ++i) {
      double2 s = make_double2(i == j ? 1.0 : 0.0, 0);
      for (int k = j; k < i; ++k) {
        double2 lik = G[(int64_t)i * n + k];
        double2 yk = W[(int64_t)k * n + j];  // stored unconjugated temporarily
        double2 pr = cmul(lik, yk);
        s.x -= pr.x;
        s.y -= pr.y;
      }
      double lii = G[(int64_t)i * n + i].x;
      W[(int64_t)i * n + j] = make_double2(s.x / lii, s.y / lii);
    }
  }
  __syncthreads();
  // now W holds Linv (lower, column j in W[:, j]); transpose-conjugate in place -> W = Linv^H
  for (int e = t; e < n * n; e += nt) {
    int i = e / n, j = e % n;
    if (j > i) {
      double2 a = W[(int64_t)i * n + j], c2 = W[(int64_t)j * n + i];
      W[(int64_t)i * n + j] = make_double2(c2.x, -c2.y);
      W[(int64_t)j * n + i] = make_double2(a.x, -a.y);
    } else if (i == j) {
      double2 a = W[(int64_t)i * n + i];
      W[(int64_t)i * n + i] = make_double2(a.x, -a.y);
    }
  }
}

__device__ __forceinline__ uint64_t smix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// X' = [X P(:, :r), Y]: completion columns are deterministic pseudo-random, scaled to the
// largest column norm of X (they only have to be linearly independent of span(X)).
__global__ void build_aprime(MatView X, float2* __restrict__ out, const int* __restrict__ perm_all,
                             const int* __restrict__ rank_all, const double* __restrict__ dmax_all, int nb) {
  int m = X.m, n = X.n;
  int64_t per = (int64_t)m * n, tot = per * nb;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = e / per, r = e - b * per;
    int i = (int)(r / n), j = (int)(r - (int64_t)i * n);
    int rank = rank_all[b];
    float2 v;
    if (j < rank) {
      int pj = perm_all[b * n + j];
      v = X.p[b * X.bs + i * X.si + pj * X.sj];
      if (X.cj) v.y = -v.y;
    } else {
      double sc = dmax_all[b] > 0 ? sqrt(dmax_all[b] / (double)m) : 1.0;
      sc = fmax(sc, 1e-30);  // stay in FP32 range
      uint64_t h1 = smix(0xC0FFEEull ^ ((uint64_t)i * 1315423911ull + (uint64_t)j * 2654435761ull));
      uint64_t h2 = smix(h1);
      double re = ((double)(h1 >> 40) * 0x1.0p-23 - 1.0) * sc;
      double im = ((double)(h2 >> 40) * 0x1.0p-23 - 1.0) * sc;
      v = make_float2((float)re, (float)im);
    }
    out[e] = v;
  }
}

// out(i, j) = sum_k A(i, k) W[k][j]  (A contiguous [b][m][n] fp32, W [b][n][n] fp64)
constexpr int AT_M = 32, AT_N = 32, AT_K = 32;
__global__ void __launch_bounds__(256) apply64_kernel(const float2* __restrict__ A, const double2* __restrict__ Wall,
                                                      MatView O, int m, int n) {
  __shared__ double2 sa[AT_M][AT_K + 1];
  __shared__ double2 sw[AT_K][AT_N + 1];
  int b = blockIdx.z;
  int i0 = blockIdx.y * AT_M, j0 = blockIdx.x * AT_N;
  const float2* Ab = A + (int64_t)b * m * n;
  const double2* W = Wall + (int64_t)b * n * n;
  int t = threadIdx.x;
  int tj = t & 31, ti = (t >> 5) * 4;  // 4 rows per thread
  double2 acc[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) acc[q] = make_double2(0, 0);
  for (int k0 = 0; k0 < n; k0 += AT_K) {
    for (int e = t; e < AT_M * AT_K; e += 256) {
      int ii = e / AT_K, kk = e - ii * AT_K;
      int i = i0 + ii, k = k0 + kk;
      sa[ii][kk] = (i < m && k < n) ? ld2(Ab + (int64_t)i * n + k, false) : make_double2(0, 0);
    }
    for (int e = t; e < AT_K * AT_N; e += 256) {
      int kk = e / AT_N, jj = e - kk * AT_N;
      int k = k0 + kk, j = j0 + jj;
      sw[kk][jj] = (k < n && j < n) ? W[(int64_t)k * n + j] : make_double2(0, 0);
    }
    __syncthreads();
    for (int kk = 0; kk < AT_K; ++kk) {
      double2 w = sw[kk][tj];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        double2 p = cmul(sa[ti + q][kk], w);
        acc[q].x += p.x;
        acc[q].y += p.y;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    int i = i0 + ti + q, j = j0 + tj;
    if (i < m && j < n) {
      float2 v = make_float2((float)acc[q].x, (float)(O.cj ? -acc[q].y : acc[q].y));
      O.p[b * O.bs + i * O.si + j * O.sj] = v;
    }
  }
}

__global__ void d2f_kernel(const double2* __restrict__ in, float2* __restrict__ out, int64_t n) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x)
    out[e] = make_float2((float)in[e].x, (float)in[e].y);
}


// ======================================================================================
// Fast path (n <= 128): register-tiled FP64 Gram / apply kernels and a one-CTA-per-matrix
// Cholesky + triangular inverse entirely in shared memory (lower triangle packed, FP64).
// The Gram's split count depends only on the matrix shape (results are bitwise independent
// of the batch size); splits are summed in a fixed order by the Cholesky kernel's load.

constexpr int GT = 64;   // output tile (complex) per CTA, 4 x 4 per thread
constexpr int GK = 16;   // rows (Gram) / k (apply) per smem chunk

__device__ __forceinline__ float2 mv_ld(const MatView& V, int64_t b, int64_t i, int64_t j) {
  float2 v = V.p[b * V.bs + i * V.si + j * V.sj];
  if (V.cj) v.y = -v.y;
  return v;
}

// part[b][sp][i][j] = sum over rows r of split sp of conj(Y(r, i)) X(r, j); herm: skip tiles
// strictly above the diagonal (only the lower triangle i >= j is consumed).
__global__ void __launch_bounds__(256) gram64_kernel(MatView Y, MatView X, int m, int splits, int herm,
                                                     const int* __restrict__ active, double2* __restrict__ part) {
  const int b = blockIdx.z / splits, sp = blockIdx.z - b * splits;
  if (active && !active[b]) return;
  const int i0 = blockIdx.y * GT, j0 = blockIdx.x * GT;
  if (herm && i0 + GT <= j0) return;
  __shared__ double2 sy[GK][GT];
  __shared__ double2 sx[GK][GT];
  const int rows_per = (m + splits - 1) / splits;
  const int r_begin = sp * rows_per, r_end = min(m, r_begin + rows_per);
  const int t = threadIdx.x, ty = t >> 4, tx = t & 15;
  const bool yrow = (Y.si == 1 && Y.sj != 1), xrow = (X.si == 1 && X.sj != 1);
  double2 acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[a][c] = make_double2(0, 0);
  for (int r0 = r_begin; r0 < r_end; r0 += GK) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = t + 256 * q;
      int rr = yrow ? (e & 15) : (e >> 6), cc = yrow ? (e >> 4) : (e & 63);
      int r = r0 + rr;
      float2 v = make_float2(0.f, 0.f);
      if (r < r_end && i0 + cc < Y.n) v = mv_ld(Y, b, r, i0 + cc);
      sy[rr][cc] = make_double2((double)v.x, (double)v.y);
      rr = xrow ? (e & 15) : (e >> 6);
      cc = xrow ? (e >> 4) : (e & 63);
      r = r0 + rr;
      v = make_float2(0.f, 0.f);
      if (r < r_end && j0 + cc < X.n) v = mv_ld(X, b, r, j0 + cc);
      sx[rr][cc] = make_double2((double)v.x, (double)v.y);
    }
    __syncthreads();
#pragma unroll 4
    for (int rr = 0; rr < GK; ++rr) {
      double2 yv[4], xv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) yv[a] = sy[rr][ty * 4 + a];
#pragma unroll
      for (int c = 0; c < 4; ++c) xv[c] = sx[rr][tx + 16 * c];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          // conj(y) * x
          acc[a][c].x = fma(yv[a].x, xv[c].x, fma(yv[a].y, xv[c].y, acc[a][c].x));
          acc[a][c].y = fma(yv[a].x, xv[c].y, fma(-yv[a].y, xv[c].x, acc[a][c].y));
        }
    }
    __syncthreads();
  }
  const int nI = Y.n, nJ = X.n;
  double2* out = part + ((int64_t)b * splits + sp) * nI * nJ;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int i = i0 + ty * 4 + a, j = j0 + tx + 16 * c;
      if (i < nI && j < nJ) out[(int64_t)i * nJ + j] = acc[a][c];
    }
}

// O(i, j) = sum_k X(i, k) W[b][k][j]  (X FP32 view, W FP64 [n][n], O FP32 view)
// active: per-matrix switch (NULL = all); sel: per-matrix output choice (NULL or sel[b] != 0 ->
// O, else O2).
__global__ void __launch_bounds__(256) apply64v_kernel(MatView X, const double2* __restrict__ Wall, MatView O,
                                                       const int* __restrict__ active, const int* __restrict__ sel,
                                                       MatView O2) {
  const int b = blockIdx.z;
  const int m = X.m, n = X.n;
  if (active && !active[b]) return;
  if (sel && !sel[b]) O = O2;
  __shared__ double2 sa[GT][GK + 1];
  __shared__ double2 sw[GK][GT];
  const int i0 = blockIdx.y * GT, j0 = blockIdx.x * GT;
  const double2* W = Wall + (int64_t)b * n * n;
  const int t = threadIdx.x, ty = t >> 4, tx = t & 15;
  const bool xrow = (X.si == 1 && X.sj != 1);
  double2 acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[a][c] = make_double2(0, 0);
  for (int k0 = 0; k0 < n; k0 += GK) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = t + 256 * q;
      const int ii = xrow ? (e & 63) : (e >> 4), kk = xrow ? (e >> 6) : (e & 15);
      const int i = i0 + ii, k = k0 + kk;
      float2 v = make_float2(0.f, 0.f);
      if (i < m && k < n) v = mv_ld(X, b, i, k);
      sa[ii][kk] = make_double2((double)v.x, (double)v.y);
      const int kk2 = e >> 6, jj = e & 63;
      sw[kk2][jj] = (k0 + kk2 < n && j0 + jj < n) ? W[(int64_t)(k0 + kk2) * n + j0 + jj] : make_double2(0, 0);
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < GK; ++kk) {
      double2 av[4], wv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) av[a] = sa[ty * 4 + a][kk];
#pragma unroll
      for (int c = 0; c < 4; ++c) wv[c] = sw[kk][tx + 16 * c];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          acc[a][c].x = fma(av[a].x, wv[c].x, fma(-av[a].y, wv[c].y, acc[a][c].x));
          acc[a][c].y = fma(av[a].x, wv[c].y, fma(av[a].y, wv[c].x, acc[a][c].y));
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int i = i0 + ty * 4 + a, j = j0 + tx + 16 * c;
      if (i < m && j < n) {
        float2 v = make_float2((float)acc[a][c].x, (float)(O.cj ? -acc[a][c].y : acc[a][c].y));
        O.p[b * O.bs + (int64_t)i * O.si + (int64_t)j * O.sj] = v;
      }
    }
}

constexpr int CH_MAXN = 128;
constexpr int CH_THREADS = 1024;
constexpr size_t CH_SMEM = (size_t)CH_MAXN * (CH_MAXN + 1) / 2 * sizeof(double2)  // packed lower G / L
                           + (size_t)(CH_THREADS / 32) * CH_MAXN * sizeof(double2)   // per-warp y columns
                           + (size_t)CH_MAXN * sizeof(double2)                       // l vector
                           + (size_t)CH_MAXN * (sizeof(double) + 2 * sizeof(int)) + 64;

__device__ __forceinline__ int pk(int i, int j) { return i * (i + 1) / 2 + j; }  // i >= j

// Cholesky G = L L^H of each Hermitian n x n matrix (G summed from `splits` Gram partials),
// then W = P L^{-H} so that Q = X W. PIVOT: symmetric pivoting on the largest remaining
// diagonal with rank detection (diag <= tol * max initial diag stops; rank < n matrices get
// no W -- the completion path handles them). Without PIVOT, tiny pivots are clamped and
// flagged in *bad. Everything lives in shared memory (packed lower triangle in FP64).
// PIVOT also writes deficient[b] = (rank < n) and need2[b] = 1 when a second CholeskyQR
// pass is needed: rank deficiency, or a pivot ratio l_11 / l_nn > 1e3 (an estimate of the
// condition number; below it the single pass, with its Gram exact in FP64 for FP32 data,
// is orthogonal to ~kappa^2 1e-16 < FP32 rounding).

template <bool PIVOT>
__global__ void __launch_bounds__(CH_THREADS) chol_smem_kernel(const double2* __restrict__ part, int splits, int n,
                                                               double tol, double2* __restrict__ Wall,
                                                               int* __restrict__ perm_all, int* __restrict__ rank_all,
                                                               double* __restrict__ dmax_all, int* __restrict__ bad,
                                                               const int* __restrict__ active,
                                                               int* __restrict__ deficient, int* __restrict__ need2) {
  extern __shared__ double2 chs[];
  const int b = blockIdx.x;
  if (active && !active[b]) return;
  double2* S = chs;                                       // packed lower, original indices
  double2* Y = S + CH_MAXN * (CH_MAXN + 1) / 2;           // [32 warps][CH_MAXN]
  double2* lv = Y + (CH_THREADS / 32) * CH_MAXN;          // [CH_MAXN]
  double* dg = reinterpret_cast<double*>(lv + CH_MAXN);   // [CH_MAXN] diagonal
  int* alive = reinterpret_cast<int*>(dg + CH_MAXN);      // [CH_MAXN]
  int* perm = alive + CH_MAXN;                            // [CH_MAXN]
  __shared__ int s_piv, s_rank;
  __shared__ double s_dp, s_d0;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const long long clk0 = clock64();
  const int64_t nn = (int64_t)n * n;
  const double2* P0 = part + (int64_t)b * splits * nn;
  // load the lower triangle (sum of the split partials, fixed order)
  for (int i = warp; i < n; i += CH_THREADS / 32)
    for (int j = lane; j <= i; j += 32) {
      double2 s = P0[(int64_t)i * n + j];
      for (int k = 1; k < splits; ++k) {
        double2 v = P0[k * nn + (int64_t)i * n + j];
        s.x += v.x;
        s.y += v.y;
      }
      S[pk(i, j)] = s;
      if (i == j) dg[i] = s.x;
    }
  for (int i = t; i < n; i += CH_THREADS) {
    alive[i] = 1;
    perm[i] = i;
  }
  __syncthreads();
  if (warp == 0) {
    double mx = 0;
    for (int i = lane; i < n; i += 32) mx = fmax(mx, dg[i]);
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) {
      s_d0 = mx;
      s_rank = n;
    }
  }
  __syncthreads();
  const long long clk1 = clock64();
  const double d0 = s_d0;
  const double floor_d = 1e-300 + 1e-30 * d0;
  // Right-looking Cholesky with one-step lookahead and one block barrier per step. Warp 0
  // owns the "column" phase A: for pivot p_k it forms l = G_k(:, p_k) / sqrt(G_k(p_k, p_k)),
  // stores it (in place and in lvb[k & 1]), updates the remaining diagonal, and picks the next
  // pivot p_{k+1} from it. Warps 1.. apply the rank-1 update of step k (phase B) to the
  // strictly lower remaining block except row/column p_{k+1}, while warp 0 already runs phase
  // A of step k+1 -- it corrects column p_{k+1} by step k's rank-1 term itself.
  double2* lvb = Y;  // [2][CH_MAXN] column buffers (the per-warp scratch is free here)
  __shared__ int s_brk, s_next;
  auto phase_a = [&](int k, int p, const double2* lprev, double2* lcur) {
    // warp 0 only: column of pivot p (G_k(:,p) = stored column minus the previous step's term).
    // Lane l owns rows l, l+32, l+64, l+96: all loads are issued first, then the arithmetic,
    // then the stores, and the next pivot is picked from the updated diagonal on the way.
    double dp = dg[p];
    bool brk = false;
    if (PIVOT) {
      brk = !(dp > tol * d0) || d0 <= 0;
    } else if (!(dp > floor_d)) {
      if (lane == 0) atomicOr(bad, 1);
      dp = floor_d;
    }
    int nxt = n;
    if (!brk) {
      const double inv = rsqrt(dp);
      const double lkk = dp * inv;
      const double2 lpp = lprev ? lprev[p] : make_double2(0, 0);
      double bv = -1;
      int bi = n;
#pragma unroll
      for (int q0 = 0; q0 < CH_MAXN / 32; q0 += 2) {  // two rows per lane at a time (64 registers)
        double2 g[2], li[2];
        double dgi[2];
        bool act[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int i = lane + 32 * (q0 + h);
          act[h] = i < n && i != p && alive[i];
          g[h] = make_double2(0, 0);
          li[h] = make_double2(0, 0);
          dgi[h] = 0;
          if (act[h]) {
            g[h] = i > p ? S[pk(i, p)] : S[pk(p, i)];
            if (lprev) li[h] = lprev[i];
            dgi[h] = dg[i];
          }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int i = lane + 32 * (q0 + h);
          if (i >= n) break;
          if (act[h]) {
            double2 gg = g[h];
            if (i < p) gg.y = -gg.y;  // G(i, p) = conj(G(p, i))
            if (lprev) {              // lookahead: step k-1's rank-1 term on column p
              gg.x -= li[h].x * lpp.x + li[h].y * lpp.y;
              gg.y -= li[h].y * lpp.x - li[h].x * lpp.y;
            }
            const double2 l = make_double2(gg.x * inv, gg.y * inv);
            lcur[i] = l;
            if (i > p) S[pk(i, p)] = l;
            else S[pk(p, i)] = make_double2(l.x, -l.y);
            const double d = dgi[h] - (l.x * l.x + l.y * l.y);
            dg[i] = d;
            if (PIVOT && d > bv) {  // increasing i per lane: the first maximum wins ties
              bv = d;
              bi = i;
            }
          } else {
            lcur[i] = make_double2(0, 0);
            if (i == p) S[pk(p, p)] = make_double2(lkk, 0);
          }
        }
      }
      if (lane == 0) {
        alive[p] = 0;
        perm[k] = p;
      }
      // next pivot from the updated diagonal
      if (k + 1 < n) {
        if (PIVOT) {
          for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
            if (ov > bv || (ov == bv && oi < bi)) {
              bv = ov;
              bi = oi;
            }
          }
          nxt = bi < n ? bi : n;  // nothing alive: the rank check of the next step stops
        } else {
          nxt = k + 1;
        }
      }
      __syncwarp();
    }
    if (lane == 0) {
      s_brk = brk ? 1 : 0;
      if (brk) s_rank = k;
      s_next = nxt;
    }
  };
  // first pivot and phase A of step 0
  if (warp == 0) {
    int p0 = 0;
    if (PIVOT) {
      double bv = -1;
      int bi = n;
      for (int i = lane; i < n; i += 32)
        if (dg[i] > bv) {
          bv = dg[i];
          bi = i;
        }
      for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > bv || (ov == bv && oi < bi)) {
          bv = ov;
          bi = oi;
        }
      }
      p0 = bi < n ? bi : 0;
    }
    phase_a(0, p0, nullptr, lvb);
  }
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    if (s_brk) break;
    const int pn = s_next;  // pivot of step k+1 (n if none)
    const double2* lk = lvb + (k & 1) * CH_MAXN;
    if (warp == 0) {
      if (k + 1 < n && pn < n) {
        phase_a(k + 1, pn, lk, lvb + ((k + 1) & 1) * CH_MAXN);
      } else if (k + 1 < n && lane == 0) {  // no pivot left (only for PIVOT): rank k + 1
        s_brk = 1;
        s_rank = k + 1;
      }
    } else if (!(g_chol_dbg & 1)) {
      // phase B of step k, rows/columns of p_{k+1} excluded (warp 0 updates that column)
      for (int i = warp - 1; i < n; i += CH_THREADS / 32 - 1) {
        if (i == pn || !alive[i]) continue;
        const double2 li = lk[i];
        for (int j = lane; j < i; j += 32) {
          if (j == pn || !alive[j]) continue;
          const double2 lj = lk[j];
          double2 g = S[pk(i, j)];
          g.x -= li.x * lj.x + li.y * lj.y;
          g.y -= li.y * lj.x - li.x * lj.y;
          S[pk(i, j)] = g;
        }
      }
    }
    __syncthreads();
  }
  __syncthreads();
  const long long clk2 = clock64();
  const int rank = s_rank;
  if (PIVOT && t == 0) {
    rank_all[b] = rank;
    dmax_all[b] = d0;
    deficient[b] = rank < n ? 1 : 0;
    int nd = 1;
    if (rank == n && n > 0) {
      const double l0 = S[pk(perm[0], perm[0])].x, l1 = S[pk(perm[n - 1], perm[n - 1])].x;
      nd = (l1 > 0 && l0 <= 1e3 * l1) ? 0 : 1;
    }
    need2[b] = nd;
  }
  if (PIVOT) {
    for (int i = t; i < n; i += CH_THREADS) perm_all[(int64_t)b * n + i] = perm[i];
    if (rank < n) return;  // completion path
  }
  // L(i, k) in pivot order = G(perm[i], perm[k]) (i > k); L(k, k) = G(perm[k], perm[k]).
  // Column j of Linv by forward substitution, one warp per column, right-looking: lane l owns
  // rows l, l+32, l+64, l+96 (running sums in registers); once y_k is known (owner lane,
  // multiplied by the stored 1/L(k,k)) it is broadcast and every lane updates its later rows.
  // W = P L^-H: W[perm[j]][k] = conj(Linv(k, j)).
  double* dinv = dg;  // the remaining-diagonal array is free now: 1 / L(k, k) in pivot order
  for (int k = t; k < n; k += CH_THREADS) dinv[k] = 1.0 / S[pk(perm[k], perm[k])].x;
  __syncthreads();
  double2* W = Wall + (int64_t)b * nn;
  int prow[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) prow[q] = (lane + 32 * q < n) ? perm[lane + 32 * q] : 0;
  for (int jj = warp; jj < n; jj += CH_THREADS / 32) {
    // balance: warp w takes columns w, 2*32-1-w, ... (long and short columns)
    const int blk = jj / (CH_THREADS / 32), w = jj % (CH_THREADS / 32);
    const int sz = min(CH_THREADS / 32, n - blk * (CH_THREADS / 32));
    const int j = (blk & 1) ? blk * (CH_THREADS / 32) + (sz - 1 - w) : jj;
    const int pj = perm[j];
    double2* Wrow = W + (int64_t)pj * n;
    double2 acc[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = lane + 32 * q;
      acc[q] = make_double2(i == j ? 1.0 : 0.0, 0.0);
      if (i < j && i < n) Wrow[i] = make_double2(0, 0);
    }
#pragma unroll
    for (int kb = 0; kb < 4; ++kb) {
      if (kb * 32 >= n) break;
      for (int kl = 0; kl < 32; ++kl) {
        const int k = kb * 32 + kl;
        if (k >= n) break;
        if (k < j) continue;
        const double ax = __shfl_sync(0xffffffffu, acc[kb].x, kl);
        const double ay = __shfl_sync(0xffffffffu, acc[kb].y, kl);
        const double dk = dinv[k];
        const double2 yk = make_double2(ax * dk, ay * dk);
        if (lane == kl) Wrow[k] = make_double2(yk.x, -yk.y);
        const int pkk = perm[k];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int i = lane + 32 * q;
          if (q >= kb && i > k && i < n) {
            const int pi = prow[q];
            double2 l = pi > pkk ? S[pk(pi, pkk)] : S[pk(pkk, pi)];
            if (pi < pkk) l.y = -l.y;
            acc[q].x -= l.x * yk.x - l.y * yk.y;
            acc[q].y -= l.x * yk.y + l.y * yk.x;
          }
        }
      }
    }
  }
  __syncthreads();
  if (b == 0 && t == 0) {
    g_chol_clk[0] = clk1 - clk0;
    g_chol_clk[1] = clk2 - clk1;
    g_chol_clk[2] = clock64() - clk2;
  }
}


}  // namespace

// out[b] = Y^H X  (n_Y x n_X), fp64
static void cross64(Ctx& c, const MatView& Y, const MatView& X, int m, int nb, double2* out) {
  int tiles = (int)(ceil_div(Y.n, CT) * ceil_div(X.n, CT));
  int64_t want = 2 * 148;
  int splits = (int)std::max<int64_t>(1, std::min<int64_t>(want / std::max<int64_t>(1, (int64_t)tiles * nb),
                                                           std::max(1, m / 256)));
  splits = std::max(1, std::min(splits, 64));
  int64_t per = (int64_t)Y.n * X.n;
  DevBuf part((size_t)per * nb * splits * sizeof(double2), c.stream);
  dim3 grid(ceil_div(X.n, CT), ceil_div(Y.n, CT), (unsigned)(nb * splits));
  cross64_kernel<<<grid, 256, 0, c.stream>>>(Y, X, m, splits, part.as<double2>());
  TN_LAUNCHED();
  unsigned blocks = (unsigned)std::min<int64_t>((per * nb + 255) / 256, 4096);
  reduce_splits<<<blocks, 256, 0, c.stream>>>(part.as<double2>(), out, splits, per, nb);
  TN_LAUNCHED();
}


static bool getenv_flag(const char* k) {
  const char* v = getenv(k);
  return v && *v && *v != '0';
}

// shape-only split count (determinism across batch sizes)
static int gram_splits(int m, int nI, int nJ) {
  int tiles = (int)(ceil_div(nI, GT) * ceil_div(nJ, GT));
  int want = (2 * 148 + tiles - 1) / tiles;
  return std::max(1, std::min({want, std::max(1, m / 128), 64}));
}

// G[b] = Y^H X (FP64, [nb][nY][nX]; lower triangle only when herm) via split partials and a
// parallel fixed-order reduction. The partials' buffer is reused across calls.
static void gram(Ctx& c, const MatView& Y, const MatView& X, int m, int nb, bool herm, const int* active,
                 DevBuf& part, double2* G) {
  const int splits = gram_splits(m, Y.n, X.n);
  size_t need = (size_t)nb * splits * Y.n * X.n * sizeof(double2);
  if (part.bytes < need) part.alloc(need, c.stream);
  dim3 grid(ceil_div(X.n, GT), ceil_div(Y.n, GT), (unsigned)(nb * splits));
  gram64_kernel<<<grid, 256, 0, c.stream>>>(Y, X, m, splits, herm ? 1 : 0, active, part.as<double2>());
  TN_LAUNCHED();
  const int64_t tot = (int64_t)nb * Y.n * X.n;
  const unsigned blocks = (unsigned)std::min<int64_t>((tot + 255) / 256, 148 * 8);
  reduce_gram_kernel<<<blocks, 256, 0, c.stream>>>(part.as<double2>(), G, splits, Y.n, X.n, nb, herm ? 1 : 0, active);
  TN_LAUNCHED();
}

static void orth_fast(Ctx& c, const MatView& X, const MatView& Q, float2* Cout, int nb) {
  const int m = X.m, n = X.n;
  // kernel attributes are per device context: set once per device ordinal
  static std::atomic<uint64_t> attr_done{0};
  int dev = 0;
  TN_CUDA(cudaGetDevice(&dev));
  const uint64_t dbit = 1ull << (dev & 63);
  if (!(attr_done.load() & dbit)) {
    TN_CUDA(cudaFuncSetAttribute(chol_smem_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CH_SMEM));
    TN_CUDA(cudaFuncSetAttribute(chol_smem_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CH_SMEM));
    attr_done.fetch_or(dbit);
  }
  static const double tol = getenv("TN_ORTH_TOL") ? atof(getenv("TN_ORTH_TOL")) : 1e-13;
  static const bool always2 = getenv_flag("TN_ORTH_ALWAYS2");
  const size_t nn = (size_t)n * n * nb;
  DevBuf part, W(nn * sizeof(double2), c.stream), Gm(nn * sizeof(double2), c.stream);
  DevBuf perm((size_t)n * nb * sizeof(int), c.stream), rank((size_t)nb * sizeof(int), c.stream);
  DevBuf dmax((size_t)nb * sizeof(double), c.stream), bad(sizeof(int), c.stream);
  DevBuf flags((size_t)2 * nb * sizeof(int), c.stream);
  int* deficient = flags.as<int>();
  int* need2 = deficient + nb;
  DevBuf Q1((size_t)m * n * nb * sizeof(float2), c.stream);
  TN_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), c.stream));
  MatView Q1v{Q1.as<float2>(), (int64_t)m * n, n, 1, false, m, n};
  const dim3 agrid(ceil_div(n, GT), ceil_div(m, GT), nb);
  // pass 1: G = X^H X, pivoted Cholesky (rank detection, condition estimate); full rank:
  // Q1 = X P L^-H, written straight to Q when no second pass is needed
  gram(c, X, X, m, nb, true, nullptr, part, Gm.as<double2>());
  chol_smem_kernel<true><<<nb, CH_THREADS, CH_SMEM, c.stream>>>(Gm.as<double2>(), 1, n, tol, W.as<double2>(),
                                                                perm.as<int>(), rank.as<int>(), dmax.as<double>(),
                                                                bad.as<int>(), nullptr, deficient, need2);
  TN_LAUNCHED();
  if (always2) TN_CUDA(cudaMemsetAsync(need2, 0xFF, sizeof(int) * nb, c.stream));  // (-1: every matrix)
  apply64v_kernel<<<agrid, 256, 0, c.stream>>>(X, W.as<double2>(), Q1v, nullptr, need2, Q);
  TN_LAUNCHED();
  // rank-deficient matrices only (every kernel returns at once for the others):
  // X' = [X P(:, :r), Y] -> Cholesky -> Q1 = X' R'^-1 (need2 is set for them)
  {
    DevBuf Ap((size_t)m * n * nb * sizeof(float2), c.stream);
    int64_t tot = (int64_t)m * n * nb;
    unsigned blocks = (unsigned)std::min<int64_t>((tot + 255) / 256, 148 * 16);
    build_aprime<<<blocks, 256, 0, c.stream>>>(X, Ap.as<float2>(), perm.as<int>(), rank.as<int>(),
                                               dmax.as<double>(), nb);
    TN_LAUNCHED();
    MatView Av{Ap.as<float2>(), (int64_t)m * n, n, 1, false, m, n};
    gram(c, Av, Av, m, nb, true, deficient, part, Gm.as<double2>());
    chol_smem_kernel<false><<<nb, CH_THREADS, CH_SMEM, c.stream>>>(Gm.as<double2>(), 1, n, 0.0,
                                                                   W.as<double2>(), nullptr, nullptr, nullptr,
                                                                   bad.as<int>(), deficient, nullptr, nullptr);
    TN_LAUNCHED();
    apply64v_kernel<<<agrid, 256, 0, c.stream>>>(Av, W.as<double2>(), Q1v, deficient, nullptr, Q1v);
    TN_LAUNCHED();
  }
  // pass 2 (re-orthogonalisation) where needed: G2 = Q1^H Q1 -> Q = Q1 R2^-1
  gram(c, Q1v, Q1v, m, nb, true, need2, part, Gm.as<double2>());
  chol_smem_kernel<false><<<nb, CH_THREADS, CH_SMEM, c.stream>>>(Gm.as<double2>(), 1, n, 0.0, W.as<double2>(),
                                                                 nullptr, nullptr, nullptr, bad.as<int>(), need2,
                                                                 nullptr, nullptr);
  TN_LAUNCHED();
  apply64v_kernel<<<agrid, 256, 0, c.stream>>>(Q1v, W.as<double2>(), Q, need2, nullptr, Q);
  TN_LAUNCHED();
  if (Cout) {
    gram(c, Q, X, m, nb, false, nullptr, part, Gm.as<double2>());
    unsigned b2 = (unsigned)std::min<int64_t>(((int64_t)nn + 255) / 256, 4096);
    d2f_kernel<<<b2, 256, 0, c.stream>>>(Gm.as<double2>(), Cout, (int64_t)nn);
    TN_LAUNCHED();
  }
}


// TN_ORTH_CHECK=1 (debugging only): host-side check of Q^H Q = I and X = Q Q^H X.
static void orth_check(Ctx& c, const MatView& X, const MatView& Q, int nb) {
  TN_CUDA(cudaStreamSynchronize(c.stream));
  const int m = X.m, n = X.n;
  auto fetch = [&](const MatView& V, int b, std::vector<std::complex<double>>& out) {
    int64_t lo = INT64_MAX, hi = 0;
    for (int64_t i : {(int64_t)0, (int64_t)m - 1})
      for (int64_t j : {(int64_t)0, (int64_t)n - 1}) {
        int64_t o = b * V.bs + i * V.si + j * V.sj;
        lo = std::min(lo, o);
        hi = std::max(hi, o);
      }
    std::vector<float2> h(hi - lo + 1);
    TN_CUDA(cudaMemcpy(h.data(), V.p + lo, h.size() * sizeof(float2), cudaMemcpyDeviceToHost));
    out.assign((size_t)m * n, 0);
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < n; ++j) {
        float2 v = h[b * V.bs + (int64_t)i * V.si + (int64_t)j * V.sj - lo];
        out[(size_t)i * n + j] = std::complex<double>(v.x, V.cj ? -v.y : v.y);
      }
  };
  for (int b = 0; b < nb; ++b) {
    std::vector<std::complex<double>> x, q;
    fetch(X, b, x);
    fetch(Q, b, q);
    double orth = 0, xn = 0, res = 0;
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        std::complex<double> s = 0;
        for (int r = 0; r < m; ++r) s += std::conj(q[(size_t)r * n + i]) * q[(size_t)r * n + j];
        orth = std::max(orth, std::abs(s - (i == j ? 1.0 : 0.0)));
      }
    std::vector<std::complex<double>> c2((size_t)n * n);
    for (int i = 0; i < n; ++i)
      for (int j = 0; j < n; ++j) {
        std::complex<double> s = 0;
        for (int r = 0; r < m; ++r) s += std::conj(q[(size_t)r * n + i]) * x[(size_t)r * n + j];
        c2[(size_t)i * n + j] = s;
      }
    for (int r = 0; r < m; ++r)
      for (int j = 0; j < n; ++j) {
        std::complex<double> s = 0;
        for (int i = 0; i < n; ++i) s += q[(size_t)r * n + i] * c2[(size_t)i * n + j];
        res += std::norm(x[(size_t)r * n + j] - s);
        xn += std::norm(x[(size_t)r * n + j]);
      }
    double rel = std::sqrt(res / std::max(xn, 1e-300));
    if (orth > 1e-4 || rel > 1e-4 || !std::isfinite(orth) || !std::isfinite(rel))
      fprintf(stderr, "ORTH_CHECK m=%d n=%d b=%d/%d: |QhQ-I|=%.3e |X-QQhX|/|X|=%.3e |X|=%.3e\n", m, n, b, nb, orth, rel,
              std::sqrt(xn));
  }
}

void orthonormalize(Ctx& c, const MatView& X, const MatView& Q, float2* Cout, int nb) {
  int m = X.m, n = X.n;
  if (n == 0 || nb == 0) return;
  if (m < n) throw Error(-1, "orthonormalize: more columns than rows");
  ProfScope ps(P_ORTH, c.stream);
  if (n <= CH_MAXN && !getenv_flag("TN_ORTH_OLD")) {
    orth_fast(c, X, Q, Cout, nb);
    if (getenv_flag("TN_ORTH_CHECK")) orth_check(c, X, Q, nb);
    return;
  }
  size_t nn = (size_t)n * n * nb;
  DevBuf G(nn * sizeof(double2), c.stream), W(nn * sizeof(double2), c.stream);
  DevBuf perm((size_t)n * nb * sizeof(int), c.stream), rank((size_t)nb * sizeof(int), c.stream);
  DevBuf dmax((size_t)nb * sizeof(double), c.stream), bad(sizeof(int), c.stream);
  DevBuf Ap((size_t)m * n * nb * sizeof(float2), c.stream), Q1((size_t)m * n * nb * sizeof(float2), c.stream);
  TN_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), c.stream));
  int thr = n >= 256 ? 512 : 256;
  // pass 0: rank detection
  cross64(c, X, X, m, nb, G.as<double2>());
  pivchol_kernel<<<nb, thr, 0, c.stream>>>(G.as<double2>(), n, 1e-13, perm.as<int>(), rank.as<int>(),
                                           dmax.as<double>());
  TN_LAUNCHED();
  int64_t tot = (int64_t)m * n * nb;
  unsigned blocks = (unsigned)std::min<int64_t>((tot + 255) / 256, 148 * 16);
  build_aprime<<<blocks, 256, 0, c.stream>>>(X, Ap.as<float2>(), perm.as<int>(), rank.as<int>(),
                                             dmax.as<double>(), nb);
  TN_LAUNCHED();
  MatView Av{Ap.as<float2>(), (int64_t)m * n, n, 1, false, m, n};
  MatView Q1v{Q1.as<float2>(), (int64_t)m * n, n, 1, false, m, n};
  // pass 1
  cross64(c, Av, Av, m, nb, G.as<double2>());
  cholinv_kernel<<<nb, thr, 0, c.stream>>>(G.as<double2>(), W.as<double2>(), n, bad.as<int>());
  TN_LAUNCHED();
  dim3 grid(ceil_div(n, AT_N), ceil_div(m, AT_M), nb);
  apply64_kernel<<<grid, 256, 0, c.stream>>>(Ap.as<float2>(), W.as<double2>(), Q1v, m, n);
  TN_LAUNCHED();
  // pass 2 (re-orthogonalisation)
  cross64(c, Q1v, Q1v, m, nb, G.as<double2>());
  cholinv_kernel<<<nb, thr, 0, c.stream>>>(G.as<double2>(), W.as<double2>(), n, bad.as<int>());
  TN_LAUNCHED();
  apply64_kernel<<<grid, 256, 0, c.stream>>>(Q1.as<float2>(), W.as<double2>(), Q, m, n);
  TN_LAUNCHED();
  if (Cout) {
    cross64(c, Q, X, m, nb, G.as<double2>());
    unsigned b2 = (unsigned)std::min<int64_t>(((int64_t)nn + 255) / 256, 4096);
    d2f_kernel<<<b2, 256, 0, c.stream>>>(G.as<double2>(), Cout, (int64_t)nn);
    TN_LAUNCHED();
  }
}

}  // namespace tn

// debugging: clocks of the last chol_smem_kernel's block 0: load, factorisation, inverse
extern "C" int tn_debug_chol_clocks(long long* out) {
  return cudaMemcpyFromSymbol(out, tn::g_chol_clk, 3 * sizeof(long long)) == cudaSuccess ? 0 : -1;
}

extern "C" int tn_debug_chol_flags(int f) {
  return cudaMemcpyToSymbol(tn::g_chol_dbg, &f, sizeof(int)) == cudaSuccess ? 0 : -1;
}
