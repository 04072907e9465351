// su.cu -- NEXT-4: tensor-network-state construction on the GPU by belief
// propagation and the BP-gauged simple update, in complex FP64.
//
// The same algorithm as the oracle generator (oracle/generator.py, O7), step by step:
//  * BP (R20): synchronous sweeps over all directed edges; message
//    mu_{v->w} = contraction of A_v, conj(A_v) and every incoming message except the one on
//    the edge, Hermitised and normalised; identity-initialised; stop at residual < tol.
//  * gate on edge e = (v, w): gauge both sites with the square roots of their
//    other incoming messages (eigen-based, relative cutoff 1e-12), reduce each site to its
//    (bond e, physical) factor by an orthonormal decomposition of the rest, contract the two
//    factors with the gate, SVD, keep <= chi singular values (relative cutoff on sigma^2),
//    record eps = discarded sum sigma^2 / sum sigma^2 (Eq. 1), split sqrt(sigma)
//    to both sides, ungauge with the inverse square roots, normalise both tensors, set both
//    messages on e to diag(sigma_kept) normalised (Vidal-gauge equivalence).
// The decompositions (orthonormal factor of a site, SVD of theta, matrix square roots) all use
// one batched FP64 Hermitian Jacobi eigensolver (one CTA per matrix, parallel round-robin
// rotations): orthonormal factor Q = X V L^-1/2 from the Gram X^H X = V L V^H (directions with
// L < 1e-15 L_max dropped), SVD of theta from theta^H theta. Bases differ from numpy's by a
// gauge on the new bond (R7); the represented state and the singular values do not.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/tnsample.h"
#include "common.h"

using namespace tn;

namespace {

thread_local std::string g_su_err;

struct T64 {
  std::shared_ptr<DevBuf> mem;
  double2* p = nullptr;
  std::vector<int> shape;
  int64_t size() const {
    int64_t s = 1;
    for (int x : shape) s *= x;
    return s;
  }
};

T64 new64(cudaStream_t st, const std::vector<int>& shape) {
  T64 t;
  t.shape = shape;
  t.mem = std::make_shared<DevBuf>((size_t)std::max<int64_t>(1, t.size()) * sizeof(double2), st);
  t.p = t.mem->as<double2>();
  return t;
}

unsigned grid1(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)); }

// ------------------------------------------------------------------------- permutation
struct Perm64 {
  int rank;
  int64_t odims[8];
  int64_t istr[8];  // input stride of each output axis
  int conj;
};

__global__ void permute64_kernel(const double2* __restrict__ in, double2* __restrict__ out, int64_t n, Perm64 a) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t rem = i, off = 0;
    for (int d = a.rank - 1; d >= 0; --d) {
      const int64_t q = rem / a.odims[d];
      off += (rem - q * a.odims[d]) * a.istr[d];
      rem = q;
    }
    double2 v = in[off];
    if (a.conj) v.y = -v.y;
    out[i] = v;
  }
}

T64 permute64(cudaStream_t st, const T64& a, const std::vector<int>& perm, bool conj = false) {
  const int r = (int)a.shape.size();
  std::vector<int64_t> str(r);
  int64_t acc = 1;
  for (int i = r - 1; i >= 0; --i) {
    str[i] = acc;
    acc *= a.shape[i];
  }
  std::vector<int> os(r);
  Perm64 p{};
  p.rank = r;
  p.conj = conj ? 1 : 0;
  for (int i = 0; i < r; ++i) {
    os[i] = a.shape[perm[i]];
    p.odims[i] = os[i];
    p.istr[i] = str[perm[i]];
  }
  T64 o = new64(st, os);
  if (r == 0) {
    TN_CUDA(cudaMemcpyAsync(o.p, a.p, sizeof(double2), cudaMemcpyDeviceToDevice, st));
    return o;
  }
  permute64_kernel<<<grid1(o.size()), 256, 0, st>>>(a.p, o.p, o.size(), p);
  TN_LAUNCHED();
  return o;
}

// ------------------------------------------------------------------------- FP64 complex GEMM
// C[M][N] = sum_k op(A)[m][k] op(B)[k][n]; A is [M][K] (or [K][M] when tA, conjugated when cA),
// B is [K][N] (or [N][K] when tB, conjugated when cB); row-major, contiguous.
constexpr int G64 = 32;
__global__ void __launch_bounds__(256) gemm64_kernel(const double2* __restrict__ A, const double2* __restrict__ B,
                                                     double2* __restrict__ C, int M, int N, int K, int tA, int cA,
                                                     int tB, int cB) {
  __shared__ double2 As[G64][G64 + 1];
  __shared__ double2 Bs[G64][G64 + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;  // 16 x 16 threads, 2 x 2 outputs each
  const int m0 = blockIdx.y * G64, n0 = blockIdx.x * G64;
  double2 acc[2][2] = {{{0, 0}, {0, 0}}, {{0, 0}, {0, 0}}};
  for (int k0 = 0; k0 < K; k0 += G64) {
    for (int e = threadIdx.x; e < G64 * G64; e += 256) {
      const int r = e / G64, q = e % G64;
      {  // As[mm][kk]
        const int mm = tA ? q : r, kk = tA ? r : q;
        const int gm = m0 + mm, gk = k0 + kk;
        double2 v = make_double2(0, 0);
        if (gm < M && gk < K) v = tA ? A[(int64_t)gk * M + gm] : A[(int64_t)gm * K + gk];
        if (cA) v.y = -v.y;
        As[mm][kk] = v;
      }
      {  // Bs[kk][nn]
        const int kk = tB ? q : r, nn = tB ? r : q;
        const int gk = k0 + kk, gn = n0 + nn;
        double2 v = make_double2(0, 0);
        if (gk < K && gn < N) v = tB ? B[(int64_t)gn * K + gk] : B[(int64_t)gk * N + gn];
        if (cB) v.y = -v.y;
        Bs[kk][nn] = v;
      }
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < G64; ++kk) {
      double2 a[2], b[2];
      a[0] = As[ty][kk];
      a[1] = As[ty + 16][kk];
      b[0] = Bs[kk][tx];
      b[1] = Bs[kk][tx + 16];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          acc[i][j].x = fma(a[i].x, b[j].x, fma(-a[i].y, b[j].y, acc[i][j].x));
          acc[i][j].y = fma(a[i].x, b[j].y, fma(a[i].y, b[j].x, acc[i][j].y));
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int gm = m0 + ty + 16 * i, gn = n0 + tx + 16 * j;
      if (gm < M && gn < N) C[(int64_t)gm * N + gn] = acc[i][j];
    }
}

void gemm64(cudaStream_t st, const double2* A, const double2* B, double2* C, int M, int N, int K, bool tA, bool cA,
            bool tB, bool cB) {
  if (M <= 0 || N <= 0) return;
  if (K <= 0) {
    TN_CUDA(cudaMemsetAsync(C, 0, sizeof(double2) * (size_t)M * N, st));
    return;
  }
  dim3 grid((N + G64 - 1) / G64, (M + G64 - 1) / G64);
  gemm64_kernel<<<grid, 256, 0, st>>>(A, B, C, M, N, K, tA, cA, tB, cB);
  TN_LAUNCHED();
}

// numpy.tensordot(a, b, (axa, axb)), optionally conj(b): result axes = a's free axes (in
// order) then b's free axes (in order).
T64 tensordot64(cudaStream_t st, const T64& a, const std::vector<int>& axa, const T64& b, const std::vector<int>& axb,
                bool conjb = false) {
  const int ra = (int)a.shape.size(), rb = (int)b.shape.size();
  std::vector<int> fa, fb, pa, pb, oshape;
  int64_t M = 1, N = 1, K = 1;
  for (int i = 0; i < ra; ++i)
    if (std::find(axa.begin(), axa.end(), i) == axa.end()) {
      fa.push_back(i);
      M *= a.shape[i];
      oshape.push_back(a.shape[i]);
    }
  for (int i = 0; i < rb; ++i)
    if (std::find(axb.begin(), axb.end(), i) == axb.end()) {
      fb.push_back(i);
      N *= b.shape[i];
      oshape.push_back(b.shape[i]);
    }
  for (size_t i = 0; i < axa.size(); ++i) {
    if (a.shape[axa[i]] != b.shape[axb[i]]) throw Error(TN_E_ARG, "tensordot64: contracted dims differ");
    K *= a.shape[axa[i]];
  }
  pa = fa;
  pa.insert(pa.end(), axa.begin(), axa.end());
  pb = std::vector<int>(axb.begin(), axb.end());
  pb.insert(pb.end(), fb.begin(), fb.end());
  T64 ap = permute64(st, a, pa);
  T64 bp = permute64(st, b, pb, conjb);
  T64 o = new64(st, oshape);
  gemm64(st, ap.p, bp.p, o.p, (int)M, (int)N, (int)K, false, false, false, false);
  return o;
}

// move axis `from` to position `to` (numpy.moveaxis)
T64 moveaxis64(cudaStream_t st, const T64& a, int from, int to) {
  const int r = (int)a.shape.size();
  std::vector<int> order;
  for (int i = 0; i < r; ++i)
    if (i != from) order.push_back(i);
  order.insert(order.begin() + to, from);
  bool ident = true;
  for (int i = 0; i < r; ++i) ident = ident && order[i] == i;
  return ident ? a : permute64(st, a, order);
}

// ------------------------------------------------------------------------- Jacobi eigensolver
// Hermitian A (n x n, n <= 256, overwritten) = V diag(w) V^H, w sorted descending. One CTA per
// matrix; parallel cyclic Jacobi: each round rotates n/2 disjoint (p, q) pairs (round-robin
// schedule), rows then columns; stop when the off-diagonal weight < (1e-15)^2 of the total.
constexpr int JMAX = 256;
__global__ void __launch_bounds__(256) jacobi_eigh_kernel(double2* __restrict__ A, double2* __restrict__ V,
                                                          double* __restrict__ w, int n, int max_sweeps) {
  __shared__ double cs[JMAX / 2], sn[JMAX / 2];
  __shared__ double2 ph[JMAX / 2];
  __shared__ int pp[JMAX / 2], qq[JMAX / 2];
  __shared__ double red[256];
  __shared__ int order[JMAX];
  const int t = threadIdx.x;
  for (int e = t; e < n * n; e += blockDim.x) V[e] = make_double2((e / n) == (e % n) ? 1.0 : 0.0, 0.0);
  __syncthreads();
  const int m = n + (n & 1);
  const int npair = m / 2;
  for (int sweep = 0; sweep < max_sweeps && n > 1; ++sweep) {
    double off = 0, tot = 0;
    for (int e = t; e < n * n; e += blockDim.x) {
      const double2 v = A[e];
      const double a2 = v.x * v.x + v.y * v.y;
      tot += a2;
      if (e / n != e % n) off += a2;
    }
    red[t] = off;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
      if (t < s) red[t] += red[t + s];
      __syncthreads();
    }
    const double offs = red[0];
    __syncthreads();
    red[t] = tot;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
      if (t < s) red[t] += red[t + s];
      __syncthreads();
    }
    const double tots = red[0];
    __syncthreads();
    if (!(offs > 1e-30 * tots)) break;
    for (int step = 0; step < m - 1; ++step) {
      if (t < npair) {
        int i, j;
        if (t == 0) {
          i = step;
          j = m - 1;
        } else {
          i = (step + t) % (m - 1);
          j = (step - t + (m - 1)) % (m - 1);
        }
        const int p = min(i, j), q = max(i, j);
        pp[t] = p;
        qq[t] = q;
        double c = 1, s = 0;
        double2 e = make_double2(1, 0);
        if (q < n) {
          const double2 b = A[(int64_t)p * n + q];
          const double ab = hypot(b.x, b.y);
          if (ab > 1e-300) {
            const double a = A[(int64_t)p * n + p].x, d = A[(int64_t)q * n + q].x;
            const double tau = (d - a) / (2 * ab);
            const double tt = tau >= 0 ? 1.0 / (tau + sqrt(1 + tau * tau)) : -1.0 / (-tau + sqrt(1 + tau * tau));
            c = 1 / sqrt(1 + tt * tt);
            s = tt * c;
            e = make_double2(b.x / ab, b.y / ab);
          }
        }
        cs[t] = c;
        sn[t] = s;
        ph[t] = e;
      }
      __syncthreads();
      // rows: A1[p][:] = c A[p] - s e A[q];  A1[q][:] = s conj(e) A[p] + c A[q]
      for (int idx = t; idx < npair * n; idx += blockDim.x) {
        const int k = idx / n, col = idx - k * n;
        const int p = pp[k], q = qq[k];
        if (q >= n || sn[k] == 0.0) continue;
        const double c = cs[k], s = sn[k];
        const double2 e = ph[k];
        const double2 ap = A[(int64_t)p * n + col], aq = A[(int64_t)q * n + col];
        const double2 se_aq = make_double2(s * (e.x * aq.x - e.y * aq.y), s * (e.x * aq.y + e.y * aq.x));
        const double2 sce_ap = make_double2(s * (e.x * ap.x + e.y * ap.y), s * (e.x * ap.y - e.y * ap.x));
        A[(int64_t)p * n + col] = make_double2(c * ap.x - se_aq.x, c * ap.y - se_aq.y);
        A[(int64_t)q * n + col] = make_double2(sce_ap.x + c * aq.x, sce_ap.y + c * aq.y);
      }
      __syncthreads();
      // columns of A and V: X[:, p] = c X[:, p] - s conj(e) X[:, q];  X[:, q] = s e X[:, p] + c X[:, q]
      for (int idx = t; idx < 2 * npair * n; idx += blockDim.x) {
        const bool isV = idx >= npair * n;
        const int r = isV ? idx - npair * n : idx;
        const int k = r / n, row = r - k * n;
        const int p = pp[k], q = qq[k];
        if (q >= n || sn[k] == 0.0) continue;
        double2* X = isV ? V : A;
        const double c = cs[k], s = sn[k];
        const double2 e = ph[k];
        const double2 xp = X[(int64_t)row * n + p], xq = X[(int64_t)row * n + q];
        const double2 sce_xq = make_double2(s * (e.x * xq.x + e.y * xq.y), s * (e.x * xq.y - e.y * xq.x));
        const double2 se_xp = make_double2(s * (e.x * xp.x - e.y * xp.y), s * (e.x * xp.y + e.y * xp.x));
        X[(int64_t)row * n + p] = make_double2(c * xp.x - sce_xq.x, c * xp.y - sce_xq.y);
        X[(int64_t)row * n + q] = make_double2(se_xp.x + c * xq.x, se_xp.y + c * xq.y);
      }
      __syncthreads();
    }
  }
  // sort descending (selection of ranks), permute V's columns
  if (t == 0) {
    for (int i = 0; i < n; ++i) order[i] = i;
    for (int i = 0; i < n; ++i) {
      int best = i;
      for (int j = i + 1; j < n; ++j)
        if (A[(int64_t)order[j] * n + order[j]].x > A[(int64_t)order[best] * n + order[best]].x) best = j;
      const int tmp = order[i];
      order[i] = order[best];
      order[best] = tmp;
    }
  }
  __syncthreads();
  for (int i = t; i < n; i += blockDim.x) w[i] = A[(int64_t)order[i] * n + order[i]].x;
  // A is no longer needed: use it as scratch for the sorted V
  for (int e = t; e < n * n; e += blockDim.x) {
    const int row = e / n, col = e - row * n;
    A[e] = V[(int64_t)row * n + order[col]];
  }
  __syncthreads();
  for (int e = t; e < n * n; e += blockDim.x) V[e] = A[e];
}

// Hermitian eigendecomposition of an n x n device matrix (FP64): w (host, descending), V (device).
void eigh64(cudaStream_t st, const double2* H, int n, T64& V, std::vector<double>& w) {
  if (n > JMAX) throw Error(TN_E_ARG, "eigh64: n > 256");
  T64 A = new64(st, {n, n});
  TN_CUDA(cudaMemcpyAsync(A.p, H, sizeof(double2) * (size_t)n * n, cudaMemcpyDeviceToDevice, st));
  V = new64(st, {n, n});
  DevBuf wd(sizeof(double) * n, st);
  jacobi_eigh_kernel<<<1, 256, 0, st>>>(A.p, V.p, wd.as<double>(), n, 60);
  TN_LAUNCHED();
  w.resize(n);
  TN_CUDA(cudaMemcpyAsync(w.data(), wd.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  TN_CUDA(cudaStreamSynchronize(st));
}

// X[:, j] *= s[j] (n columns, m rows)
__global__ void scale_cols64_kernel(double2* X, int64_t m, int n, const double* s) {
  const int64_t tot = m * n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    const double f = s[i % n];
    X[i].x *= f;
    X[i].y *= f;
  }
}

// first k columns of an n x n matrix, scaled: out[r][j] = V[r][j] * s[j], r < n, j < k
T64 cols_scaled(cudaStream_t st, const T64& V, int k, const std::vector<double>& s) {
  const int n = V.shape[0];
  T64 o = new64(st, {n, k});
  TN_CUDA(cudaMemcpy2DAsync(o.p, sizeof(double2) * k, V.p, sizeof(double2) * n, sizeof(double2) * k, n,
                            cudaMemcpyDeviceToDevice, st));
  DevBuf sd(sizeof(double) * k, st);
  TN_CUDA(cudaMemcpyAsync(sd.p, s.data(), sizeof(double) * k, cudaMemcpyHostToDevice, st));
  scale_cols64_kernel<<<grid1((int64_t)n * k), 256, 0, st>>>(o.p, n, k, sd.as<double>());
  TN_LAUNCHED();
  TN_CUDA(cudaStreamSynchronize(st));  // s is a host temporary
  return o;
}

// Frobenius norm^2 of a tensor (FP64, one block)
__global__ void norm2_64_kernel(const double2* __restrict__ x, int64_t n, double* out) {
  __shared__ double red[256];
  double s = 0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += x[i].x * x[i].x + x[i].y * x[i].y;
  red[threadIdx.x] = s;
  __syncthreads();
  for (int k = 128; k > 0; k >>= 1) {
    if (threadIdx.x < k) red[threadIdx.x] += red[threadIdx.x + k];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

__global__ void scale64_kernel(double2* x, int64_t n, const double* nrm2) {
  const double f = *nrm2 > 0 ? 1.0 / sqrt(*nrm2) : 1.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    x[i].x *= f;
    x[i].y *= f;
  }
}

void normalize64(cudaStream_t st, T64& t) {
  DevBuf n2(sizeof(double), st);
  norm2_64_kernel<<<1, 256, 0, st>>>(t.p, t.size(), n2.as<double>());
  TN_LAUNCHED();
  scale64_kernel<<<grid1(t.size()), 256, 0, st>>>(t.p, t.size(), n2.as<double>());
  TN_LAUNCHED();
}

// out = (m + m^H) / 2 for an n x n matrix; and |a - b|^2 accumulated into acc[0]
__global__ void herm64_kernel(const double2* __restrict__ m, double2* __restrict__ out, int n) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n * n; e += gridDim.x * blockDim.x) {
    const int i = e / n, j = e - i * n;
    const double2 a = m[e], b = m[(int64_t)j * n + i];
    out[e] = make_double2(0.5 * (a.x + b.x), 0.5 * (a.y - b.y));
  }
}

__global__ void diff2_64_kernel(const double2* __restrict__ a, const double2* __restrict__ b, int64_t n, double* acc) {
  __shared__ double red[256];
  double s = 0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double dx = a[i].x - b[i].x, dy = a[i].y - b[i].y;
    s += dx * dx + dy * dy;
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int k = 128; k > 0; k >>= 1) {
    if (threadIdx.x < k) red[threadIdx.x] += red[threadIdx.x + k];
    __syncthreads();
  }
  if (threadIdx.x == 0) *acc = red[0];
}

}  // namespace

// ------------------------------------------------------------------------- the engine
struct tn_su {
  int n = 0, device = 0;
  cudaStream_t stream = nullptr;
  std::vector<std::pair<int, int>> edges;
  std::vector<std::vector<int>> inc;
  std::vector<int> dims;
  std::vector<T64> t;
  std::vector<T64> msg;  // msg[2 e + side]: message from edges[e].first (side 0) / .second (side 1) along e
  std::vector<double> eps;
};

namespace {

int leg(const tn_su* s, int v, int e) {
  const auto& in = s->inc[v];
  return 1 + (int)(std::find(in.begin(), in.end(), e) - in.begin());
}
int other(const tn_su* s, int v, int e) { return s->edges[e].first == v ? s->edges[e].second : s->edges[e].first; }
// message from vertex u along edge e
T64& msg_from(tn_su* s, int u, int e) { return s->msg[2 * e + (s->edges[e].first == u ? 0 : 1)]; }

// apply matrix m[k][k'] on leg ax of t: t'[..., k', ...] = sum_k t[..., k, ...] m[k][k']
T64 apply_leg(cudaStream_t st, const T64& t, int ax, const T64& m) {
  T64 x = tensordot64(st, t, {ax}, m, {0});
  return moveaxis64(st, x, (int)x.shape.size() - 1, ax);
}

// BP message update mu_{v -> w} on edge e (oracle TNS._update)
T64 bp_update(tn_su* s, int v, int e, std::vector<T64>& msg) {
  cudaStream_t st = s->stream;
  T64 tt = s->t[v];
  for (int e2 : s->inc[v]) {
    if (e2 == e) continue;
    const int u = other(s, v, e2);
    const T64& m = msg[2 * e2 + (s->edges[e2].first == u ? 0 : 1)];
    tt = apply_leg(st, tt, leg(s, v, e2), m);
  }
  const int ax = leg(s, v, e);
  std::vector<int> others;
  for (int i = 0; i < (int)s->t[v].shape.size(); ++i)
    if (i != ax) others.push_back(i);
  T64 out = tensordot64(st, tt, others, s->t[v], others, true);
  T64 h = new64(st, out.shape);
  const int d = out.shape[0];
  herm64_kernel<<<grid1((int64_t)d * d), 256, 0, st>>>(out.p, h.p, d);
  TN_LAUNCHED();
  normalize64(st, h);
  return h;
}

T64 eye64(cudaStream_t st, int d, double scale) {
  std::vector<double2> h((size_t)d * d, make_double2(0, 0));
  for (int i = 0; i < d; ++i) h[(size_t)i * d + i] = make_double2(scale, 0);
  T64 o = new64(st, {d, d});
  TN_CUDA(cudaMemcpyAsync(o.p, h.data(), sizeof(double2) * h.size(), cudaMemcpyHostToDevice, st));
  TN_CUDA(cudaStreamSynchronize(st));
  return o;
}

// sqrt and pseudo-inverse sqrt of a Hermitian PSD message (oracle TNS._sqrt_pair, cut 1e-12)
void sqrt_pair(cudaStream_t st, const T64& m, T64& sq, T64& isq) {
  const int d = m.shape[0];
  T64 h = new64(st, {d, d});
  herm64_kernel<<<grid1((int64_t)d * d), 256, 0, st>>>(m.p, h.p, d);
  TN_LAUNCHED();
  T64 V;
  std::vector<double> w;
  eigh64(st, h.p, d, V, w);
  const double wmax = std::max(0.0, w[0]);
  std::vector<double> a(d), b(d);
  for (int i = 0; i < d; ++i) {
    const double l = std::max(0.0, w[i]);
    a[i] = std::sqrt(l);
    b[i] = (l > 1e-12 * wmax && l > 0) ? 1.0 / std::sqrt(l) : 0.0;
  }
  T64 Va = cols_scaled(st, V, d, a), Vb = cols_scaled(st, V, d, b);
  sq = new64(st, {d, d});
  isq = new64(st, {d, d});
  gemm64(st, Va.p, V.p, sq.p, d, d, d, false, false, true, true);  // V diag(a) V^H
  gemm64(st, Vb.p, V.p, isq.p, d, d, d, false, false, true, true);
}

}  // namespace

namespace {
template <class F>
int su_guard(F&& f) {
  try {
    f();
    return TN_OK;
  } catch (const Error& e) {
    g_su_err = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_su_err = e.what();
    return TN_E_CUDA;
  }
}
}  // namespace

extern "C" {

const char* tn_su_last_error(void) { return g_su_err.c_str(); }

int tn_su_create(int32_t n_vertices, int32_t n_edges, const int32_t* edges, const uint8_t* bits, tn_su** out) {
  return su_guard([&] {
    if (!out || (!edges && n_edges > 0) || !bits || n_vertices < 1 || n_edges < 0) throw Error(TN_E_ARG, "bad argument");
    *out = nullptr;
    auto s = std::make_unique<tn_su>();
    s->n = n_vertices;
    s->inc.assign(n_vertices, {});
    for (int e = 0; e < n_edges; ++e) {
      int u = edges[2 * e], v = edges[2 * e + 1];
      if (u < 0 || v < 0 || u >= n_vertices || v >= n_vertices || u == v) throw Error(TN_E_GRAPH, "bad edge");
      if (u > v) std::swap(u, v);
      s->edges.push_back({u, v});
      s->inc[u].push_back(e);
      s->inc[v].push_back(e);
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) throw Error(TN_E_CUDA, "no CUDA device");
    TN_CUDA(cudaGetDevice(&s->device));
    TN_CUDA(cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking));
    s->dims.assign(n_edges, 1);
    for (int v = 0; v < n_vertices; ++v) {
      std::vector<int> shape(1 + s->inc[v].size(), 1);
      shape[0] = 2;
      std::vector<double2> h(2, make_double2(0, 0));
      h[bits[v] ? 1 : 0] = make_double2(1, 0);
      T64 t = new64(s->stream, shape);
      TN_CUDA(cudaMemcpyAsync(t.p, h.data(), sizeof(double2) * 2, cudaMemcpyHostToDevice, s->stream));
      s->t.push_back(t);
    }
    s->msg.resize(2 * n_edges);
    for (int e = 0; e < 2 * n_edges; ++e) s->msg[e] = eye64(s->stream, 1, 1.0);
    TN_CUDA(cudaStreamSynchronize(s->stream));
    *out = s.release();
  });
}

int tn_su_bp(tn_su* s, double tol, int32_t max_sweeps, double* out_residual, int32_t* out_sweeps) {
  return su_guard([&] {
    if (!s) throw Error(TN_E_ARG, "NULL state");
    TN_CUDA(cudaSetDevice(s->device));
    cudaStream_t st = s->stream;
    const int ne = (int)s->edges.size();
    std::vector<T64> msg(2 * ne);
    for (int e = 0; e < ne; ++e) {
      const int d = s->dims[e];
      msg[2 * e] = eye64(st, d, 1.0 / std::sqrt((double)d));
      msg[2 * e + 1] = eye64(st, d, 1.0 / std::sqrt((double)d));
    }
    double res = INFINITY;
    int sweeps = 0;
    DevBuf acc(sizeof(double) * std::max(1, 2 * ne), st);
    for (int it = 0; it < max_sweeps && ne > 0; ++it) {
      std::vector<T64> nw(2 * ne);
      for (int e = 0; e < ne; ++e) {
        nw[2 * e] = bp_update(s, s->edges[e].first, e, msg);
        nw[2 * e + 1] = bp_update(s, s->edges[e].second, e, msg);
      }
      for (int k = 0; k < 2 * ne; ++k) {
        diff2_64_kernel<<<1, 256, 0, st>>>(nw[k].p, msg[k].p, nw[k].size(), acc.as<double>() + k);
        TN_LAUNCHED();
      }
      std::vector<double> h(2 * ne);
      TN_CUDA(cudaMemcpyAsync(h.data(), acc.p, sizeof(double) * 2 * ne, cudaMemcpyDeviceToHost, st));
      TN_CUDA(cudaStreamSynchronize(st));
      res = 0;
      for (double x : h) res = std::max(res, std::sqrt(x));
      msg = std::move(nw);
      ++sweeps;
      if (res < tol) break;
    }
    s->msg = std::move(msg);
    if (out_residual) *out_residual = ne > 0 ? res : 0.0;
    if (out_sweeps) *out_sweeps = sweeps;
  });
}

int tn_su_apply2(tn_su* s, int32_t e, const double* gate, int32_t chi, double cutoff, double* out_eps) {
  return su_guard([&] {
    if (!s || !gate) throw Error(TN_E_ARG, "NULL argument");
    if (e < 0 || e >= (int)s->edges.size() || chi < 1) throw Error(TN_E_ARG, "bad edge or chi");
    TN_CUDA(cudaSetDevice(s->device));
    cudaStream_t st = s->stream;
    const int v = s->edges[e].first, w = s->edges[e].second;
    struct Side {
      T64 Q;                 // [m][k] orthonormal columns
      T64 R;                 // [k][2][d_e]
      std::vector<int> others, osh;
      std::vector<std::pair<int, T64>> inv;
      int nd;
    } sd[2];
    for (int side = 0; side < 2; ++side) {
      const int a = side == 0 ? v : w;
      T64 t = s->t[a];
      Side& S = sd[side];
      for (int e2 : s->inc[a]) {
        if (e2 == e) continue;
        const int o = other(s, a, e2);
        T64 sq, isq;
        sqrt_pair(st, msg_from(s, o, e2), sq, isq);
        const int ax = leg(s, a, e2);
        t = apply_leg(st, t, ax, sq);
        S.inv.push_back({ax, isq});
      }
      const int ax_e = leg(s, a, e);
      S.nd = (int)t.shape.size();
      for (int i = 1; i < S.nd; ++i)
        if (i != ax_e) S.others.push_back(i);
      std::vector<int> perm = S.others;
      perm.push_back(0);
      perm.push_back(ax_e);
      T64 tp = permute64(st, t, perm);
      int64_t mrows = 1;
      for (int i : S.others) {
        S.osh.push_back(t.shape[i]);
        mrows *= t.shape[i];
      }
      const int de = t.shape[ax_e];
      const int ncol = 2 * de;
      // orthonormal factor of the rest: Gram -> eigh -> Q = X V L^-1/2, R = L^1/2 V^H
      T64 G = new64(st, {ncol, ncol});
      gemm64(st, tp.p, tp.p, G.p, ncol, ncol, (int)mrows, true, true, false, false);  // X^H X
      T64 V;
      std::vector<double> lam;
      eigh64(st, G.p, ncol, V, lam);
      const double lmax = std::max(lam[0], 0.0);
      int k = 0;
      while (k < ncol && lam[k] > 1e-15 * lmax && lam[k] > 0) ++k;
      k = std::max(k, 1);
      std::vector<double> isl(k), sl(k);
      for (int i = 0; i < k; ++i) {
        sl[i] = std::sqrt(std::max(lam[i], 0.0));
        isl[i] = sl[i] > 0 ? 1.0 / sl[i] : 0.0;
      }
      T64 Vk_is = cols_scaled(st, V, k, isl);  // [ncol][k]
      S.Q = new64(st, {(int)mrows, k});
      gemm64(st, tp.p, Vk_is.p, S.Q.p, (int)mrows, k, ncol, false, false, false, false);
      T64 Vk_s = cols_scaled(st, V, k, sl);  // [ncol][k]
      T64 Rm = new64(st, {k, ncol});
      // R = diag(sl) V_k^H: R[i][c] = conj(V[c][i]) sl[i] -> (Vk_s)^H
      gemm64(st, Vk_s.p, eye64(st, ncol, 1.0).p, Rm.p, k, ncol, ncol, true, true, false, false);
      S.R = Rm;
      S.R.shape = {k, 2, de};
    }
    // theta[a, s, t, b] = sum_x Rv[a, s, x] Rw[b, t, x]; then the gate
    const int qa = sd[0].R.shape[0], qb = sd[1].R.shape[0];
    T64 th = tensordot64(st, sd[0].R, {2}, sd[1].R, {2});  // [a, s, b, t]
    th = permute64(st, th, {0, 1, 3, 2});                   // [a, s, t, b]
    T64 g = new64(st, {2, 2, 2, 2});
    TN_CUDA(cudaMemcpyAsync(g.p, gate, sizeof(double2) * 16, cudaMemcpyHostToDevice, st));
    T64 th2 = tensordot64(st, g, {2, 3}, th, {1, 2});  // [s, t, a, b]
    th2 = permute64(st, th2, {2, 0, 1, 3});             // [a, s, t, b]
    const int M = qa * 2, Nn = 2 * qb;
    // SVD of Theta (M x Nn) via Theta^H Theta = V S^2 V^H
    T64 H = new64(st, {Nn, Nn});
    gemm64(st, th2.p, th2.p, H.p, Nn, Nn, M, true, true, false, false);
    T64 V;
    std::vector<double> lam;
    eigh64(st, H.p, Nn, V, lam);
    std::vector<double> sig(Nn);
    double tot = 0;
    for (int i = 0; i < Nn; ++i) {
      sig[i] = std::sqrt(std::max(lam[i], 0.0));
      tot += sig[i] * sig[i];
    }
    const int rank_max = std::min(M, Nn);
    int cnt = 0;
    for (int i = 0; i < rank_max; ++i)
      if (tot > 0 && sig[i] * sig[i] / tot > cutoff) ++cnt;
    const int keep = std::min(chi, std::max(1, cnt));
    double disc = 0;
    for (int i = keep; i < Nn; ++i) disc += sig[i] * sig[i];
    const double epsv = tot > 0 ? disc / tot : 0.0;
    s->eps.push_back(epsv);
    if (out_eps) *out_eps = epsv;
    // U sqrt(S) = Theta V S^-1/2 ; sqrt(S) V^H
    std::vector<double> isq(keep), ssq(keep);
    for (int i = 0; i < keep; ++i) {
      ssq[i] = std::sqrt(sig[i]);
      isq[i] = sig[i] > 0 ? 1.0 / std::sqrt(sig[i]) : 0.0;
    }
    T64 Vi = cols_scaled(st, V, keep, isq);  // [Nn][keep]
    T64 Us = new64(st, {M, keep});
    gemm64(st, th2.p, Vi.p, Us.p, M, keep, Nn, false, false, false, false);
    T64 Vs = cols_scaled(st, V, keep, ssq);  // [Nn][keep]
    T64 VhS = new64(st, {keep, Nn});          // sqrt(S) V^H
    gemm64(st, Vs.p, eye64(st, Nn, 1.0).p, VhS.p, keep, Nn, Nn, true, true, false, false);
    // new site factors: rv [a, 2, keep]; rw [b, t, keep] from VhS [keep, t, b]
    T64 rv = Us;
    rv.shape = {qa, 2, keep};
    T64 vh3 = VhS;
    vh3.shape = {keep, 2, qb};
    T64 rw = permute64(st, vh3, {2, 1, 0});  // [b, t, keep]
    for (int side = 0; side < 2; ++side) {
      const int a = side == 0 ? v : w;
      Side& S = sd[side];
      T64 rn = side == 0 ? rv : rw;
      const int kk = rn.shape[0];
      T64 tn = new64(st, {S.Q.shape[0], 2 * keep});
      gemm64(st, S.Q.p, rn.p, tn.p, S.Q.shape[0], 2 * keep, kk, false, false, false, false);
      std::vector<int> sh = S.osh;
      sh.push_back(2);
      sh.push_back(keep);
      tn.shape = sh;
      // back to (s, legs in edge-id order): the current axes are others..., 0, ax_e
      const int ax_e = leg(s, a, e);
      std::vector<int> src = S.others;
      src.push_back(0);
      src.push_back(ax_e);
      std::vector<int> inv(src.size());
      for (size_t i = 0; i < src.size(); ++i) inv[src[i]] = (int)i;
      T64 t = permute64(st, tn, inv);
      for (auto& kv : S.inv) t = apply_leg(st, t, kv.first, kv.second);
      normalize64(st, t);
      s->t[a] = t;
    }
    s->dims[e] = keep;
    T64 dm = new64(st, {keep, keep});
    {
      double nn = 0;
      for (int i = 0; i < keep; ++i) nn += sig[i] * sig[i];
      nn = std::sqrt(nn);
      std::vector<double2> h((size_t)keep * keep, make_double2(0, 0));
      for (int i = 0; i < keep; ++i) h[(size_t)i * keep + i] = make_double2(nn > 0 ? sig[i] / nn : 0.0, 0);
      TN_CUDA(cudaMemcpyAsync(dm.p, h.data(), sizeof(double2) * h.size(), cudaMemcpyHostToDevice, st));
      TN_CUDA(cudaStreamSynchronize(st));
    }
    s->msg[2 * e] = dm;
    s->msg[2 * e + 1] = dm;
  });
}

int tn_su_bond_dims(tn_su* s, int32_t* out) {
  return su_guard([&] {
    if (!s || !out) throw Error(TN_E_ARG, "NULL argument");
    for (size_t e = 0; e < s->dims.size(); ++e) out[e] = s->dims[e];
  });
}

int tn_su_export(tn_su* s, double* const* tensors) {
  return su_guard([&] {
    if (!s || !tensors) throw Error(TN_E_ARG, "NULL argument");
    TN_CUDA(cudaSetDevice(s->device));
    for (int v = 0; v < s->n; ++v) {
      if (!tensors[v]) throw Error(TN_E_ARG, "NULL tensor pointer");
      TN_CUDA(cudaMemcpyAsync(tensors[v], s->t[v].p, sizeof(double2) * s->t[v].size(), cudaMemcpyDeviceToHost,
                              s->stream));
    }
    TN_CUDA(cudaStreamSynchronize(s->stream));
  });
}

int tn_su_free(tn_su* s) {
  return su_guard([&] {
    if (!s) return;
    cudaSetDevice(s->device);
    cudaStreamSynchronize(s->stream);
    cudaStream_t st = s->stream;
    delete s;
    cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
  });
}

}  // extern "C"
