// linalg.cu -- CholeskyQR2 with pivoted rank detection, FP64 arithmetic (see linalg.h).
#include <algorithm>

#include "linalg.h"

namespace tn {
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

void orthonormalize(Ctx& c, const MatView& X, const MatView& Q, float2* Cout, int nb) {
  int m = X.m, n = X.n;
  if (n == 0 || nb == 0) return;
  if (m < n) throw Error(-1, "orthonormalize: more columns than rows");
  ProfScope ps(P_ORTH, c.stream);
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
