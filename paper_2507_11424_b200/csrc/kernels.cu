// kernels.cu -- hash init, normalisation, the conditional/draw tail, selections.
#include <algorithm>
#include <cmath>

#include "kernels.h"

namespace tn {
namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void hash_init_kernel(float2* __restrict__ o, int64_t size, int64_t bs, int nb, uint64_t base) {
  int64_t tot = size * nb;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = e / size, i = e - b * size;
    uint64_t h0 = splitmix64(base + 2ull * (uint64_t)i);
    uint64_t h1 = splitmix64(base + 2ull * (uint64_t)i + 1ull);
    float re = (float)(h0 >> 40) * 0x1.0p-23f - 1.0f;  // exact in FP32
    float im = (float)(h1 >> 40) * 0x1.0p-23f - 1.0f;
    o[b * bs + i] = make_float2(re, im);
  }
}

// per-sample sum of |t|^2 -> partials[b][chunk]
__global__ void sumsq_kernel(const float2* __restrict__ t, int64_t size, int64_t bs, int chunks,
                             double* __restrict__ part) {
  int b = blockIdx.y, ch = blockIdx.x;
  int64_t per = (size + chunks - 1) / chunks;
  int64_t i0 = ch * per, i1 = min(size, i0 + per);
  double s = 0;
  const float2* p = t + b * bs;
  for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    float2 v = p[i];
    s += (double)v.x * v.x + (double)v.y * v.y;
  }
  __shared__ double sh[256];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int k = 128; k > 0; k >>= 1) {
    if (threadIdx.x < k) sh[threadIdx.x] += sh[threadIdx.x + k];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[b * chunks + ch] = sh[0];
}

__global__ void norm_finalize(const double* __restrict__ part, int chunks, int nb, float* __restrict__ inv,
                              double* __restrict__ logn, bool acc) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  double s = 0;
  for (int k = 0; k < chunks; ++k) s += part[b * chunks + k];
  double nrm = sqrt(s);
  inv[b] = nrm > 0 ? (float)(1.0 / nrm) : 1.0f;
  if (logn) {
    double l = nrm > 0 ? log(nrm) : -INFINITY;
    logn[b] = acc ? logn[b] + l : l;
  }
}

__global__ void scale_kernel(float2* __restrict__ t, int64_t size, int64_t bs, int nb, const float* __restrict__ inv) {
  int64_t tot = size * nb;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = e / size, i = e - b * size;
    float s = inv[b];
    float2 v = t[b * bs + i];
    t[b * bs + i] = make_float2(v.x * s, v.y * s);
  }
}

__global__ void sum2_kernel(const float2* __restrict__ t, float2* __restrict__ out, int64_t half, int64_t ibs,
                            int64_t obs, int nb) {
  int64_t tot = half * nb;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = e / half, i = e - b * half;
    float2 a = t[b * ibs + i], c = t[b * ibs + half + i];
    out[b * obs + i] = make_float2(a.x + c.x, a.y + c.y);
  }
}

// tail: partial dots, 2 per sample (s = 0, 1), fp64 accumulation
__global__ void tail_partial(const float2* __restrict__ L, int64_t lbs, const float2* __restrict__ R, int64_t rbs,
                             int64_t size, int chunks, double* __restrict__ part) {
  int b = blockIdx.y, ch = blockIdx.x;
  int64_t per = (size + chunks - 1) / chunks;
  int64_t i0 = ch * per, i1 = min(size, i0 + per);
  const float2* l = L + b * lbs;
  const float2* r0 = R + b * rbs;
  const float2* r1 = r0 + size;
  double s0 = 0, s1 = 0;
  for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    float2 a = l[i], x = r0[i], y = r1[i];
    s0 += (double)a.x * x.x - (double)a.y * x.y;
    s1 += (double)a.x * y.x - (double)a.y * y.y;
  }
  __shared__ double sh0[256], sh1[256];
  sh0[threadIdx.x] = s0;
  sh1[threadIdx.x] = s1;
  __syncthreads();
  for (int k = 128; k > 0; k >>= 1) {
    if (threadIdx.x < k) {
      sh0[threadIdx.x] += sh0[threadIdx.x + k];
      sh1[threadIdx.x] += sh1[threadIdx.x + k];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[(b * chunks + ch) * 2] = sh0[0];
    part[(b * chunks + ch) * 2 + 1] = sh1[0];
  }
}

__global__ void tail_finalize(const double* __restrict__ part, int chunks, int nb, TailOut o) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  double w0 = 0, w1 = 0;
  for (int k = 0; k < chunks; ++k) {
    w0 += part[(b * chunks + k) * 2];
    w1 += part[(b * chunks + k) * 2 + 1];
  }
  uint32_t fl = 0;
  if (!isfinite(w0) || !isfinite(w1)) fl |= 4u;
  if (w0 < 0 || w1 < 0) fl |= 1u;
  w0 = fmax(w0, 0.0);
  w1 = fmax(w1, 0.0);
  double tot = w0 + w1, p0;
  if (tot > 0) {
    p0 = w0 / tot;
  } else {
    fl |= 2u;
    p0 = 0.5;
  }
  double u = o.u[(int64_t)b * o.N + o.vertex];
  int x = (u < p0) ? 0 : 1;
  double px = x == 0 ? p0 : 1.0 - p0;
  o.x[b] = x;
  o.bits[(int64_t)b * o.N + o.vertex] = (uint8_t)x;
  if (o.cond) o.cond[(int64_t)b * o.N + o.vertex] = px;
  o.logq[b] += (fl & 4u) ? NAN : (px > 0 ? log(px) : -INFINITY);
  o.flags[b] |= fl;
}

__global__ void select_kernel(const float2* __restrict__ n, int64_t nbs, float2* __restrict__ out, int64_t obs,
                              int a, int d, int z, const int* __restrict__ x, int nb) {
  int64_t per = (int64_t)a * d * z, tot = per * nb;
  int64_t dz = (int64_t)d * z;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = e / per, r = e - b * per;
    int64_t ia = r / dz, rest = r - ia * dz;
    out[b * obs + r] = n[b * nbs + (ia * 2 + x[b]) * dz + rest];
  }
}

__global__ void gather_bit_kernel(const float2* __restrict__ A, int64_t half, float2* __restrict__ out, int64_t obs,
                                  const uint8_t* __restrict__ bits, int N, int v, int nb) {
  int64_t tot = half * nb;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = e / half, i = e - b * half;
    int s = bits[b * N + v];
    out[b * obs + i] = A[s * half + i];
  }
}

__global__ void fill_kernel(float2* __restrict__ t, int64_t n, float2 v) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) t[e] = v;
}

__global__ void copy_rows_kernel(const float2* __restrict__ src, int64_t sbs, float2* __restrict__ dst, int64_t dbs,
                                 int64_t off, int64_t size, int nb) {
  int64_t tot = size * nb;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = e / size, i = e - b * size;
    dst[b * dbs + off + i] = src[b * sbs + i];
  }
}

__global__ void add_kernel(float2* __restrict__ dst, int64_t dbs, const float2* __restrict__ src, int64_t sbs,
                           int64_t size, int nb) {
  int64_t tot = size * nb;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = e / size, i = e - b * size;
    float2 a = dst[b * dbs + i], s = src[b * sbs + i];
    dst[b * dbs + i] = make_float2(a.x + s.x, a.y + s.y);
  }
}

__global__ void log_add_kernel(double* out, const double* a, const double* b, const double* c, int n, bool acc) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double v = a[i] + (b ? b[i] : 0.0) + (c ? c[i] : 0.0);
  out[i] = acc ? out[i] + v : v;
}

unsigned grid_for(int64_t n) { return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)); }

}  // namespace

void hash_init(Ctx& c, Tensor& o, int nb, uint64_t seed, int tag, int b1, int k) {
  uint64_t base = ((((seed * 31ull + (uint64_t)tag) * 1000003ull + (uint64_t)b1) * 1000003ull + (uint64_t)k) *
                   4294967311ull);
  int64_t size = o.size();
  int n = o.bstride ? nb : 1;
  hash_init_kernel<<<grid_for(size * n), 256, 0, c.stream>>>(o.p, size, o.bstride, n, base);
  TN_LAUNCHED();
}

void normalize(Ctx& c, Tensor& t, int nb, double* logn, bool acc) {
  invalidate_amax(t);
  ProfScope ps(P_MISC, c.stream);
  int n = t.bstride ? nb : 1;
  int64_t size = t.size();
  int chunks = (int)std::max<int64_t>(1, std::min<int64_t>(256, size / 4096));
  DevBuf part((size_t)n * chunks * sizeof(double), c.stream), inv((size_t)n * sizeof(float), c.stream);
  sumsq_kernel<<<dim3(chunks, n), 256, 0, c.stream>>>(t.p, size, t.bstride, chunks, part.as<double>());
  TN_LAUNCHED();
  norm_finalize<<<ceil_div(n, 128), 128, 0, c.stream>>>(part.as<double>(), chunks, n, inv.as<float>(), logn, acc);
  TN_LAUNCHED();
  scale_kernel<<<grid_for(size * n), 256, 0, c.stream>>>(t.p, size, t.bstride, n, inv.as<float>());
  TN_LAUNCHED();
}

Tensor sum2(Ctx& c, const Tensor& t) {
  std::vector<int> sh(t.shape.begin() + 1, t.shape.end());
  int nb = t.bstride ? c.nb : 1;
  Tensor out = new_tensor_n(c, sh, nb);
  if (!t.bstride) out.bstride = 0;
  int64_t half = out.size();
  sum2_kernel<<<grid_for(half * nb), 256, 0, c.stream>>>(t.p, out.p, half, t.bstride, out.bstride, nb);
  TN_LAUNCHED();
  return out;
}

void tail_draw(Ctx& c, const Tensor& L, const Tensor& Rs, int nb, const TailOut& o) {
  ProfScope ps(P_TAIL, c.stream);
  int64_t size = L.size();
  if (Rs.size() != 2 * size) throw Error(-1, "tail_draw: size mismatch");
  int chunks = (int)std::max<int64_t>(1, std::min<int64_t>(512, size / 8192));
  DevBuf part((size_t)nb * chunks * 2 * sizeof(double), c.stream);
  tail_partial<<<dim3(chunks, nb), 256, 0, c.stream>>>(L.p, L.bstride, Rs.p, Rs.bstride, size, chunks,
                                                       part.as<double>());
  TN_LAUNCHED();
  tail_finalize<<<ceil_div(nb, 128), 128, 0, c.stream>>>(part.as<double>(), chunks, nb, o);
  TN_LAUNCHED();
}

Tensor select_s(Ctx& c, const Tensor& n, const int* x, int nb) {
  // n: [a, 2, d, z]
  int a = n.shape[0], d = n.shape[2], z = n.shape[3];
  Tensor out = new_tensor_n(c, {a, d, z}, nb);
  select_kernel<<<grid_for(out.size() * nb), 256, 0, c.stream>>>(n.p, n.bstride, out.p, out.bstride, a, d, z, x, nb);
  TN_LAUNCHED();
  return out;
}

Tensor gather_bit(Ctx& c, const Tensor& A, const uint8_t* bits, int N, int v, int nb) {
  std::vector<int> sh(A.shape.begin() + 1, A.shape.end());
  Tensor out = new_tensor_n(c, sh, nb);
  int64_t half = out.size();
  gather_bit_kernel<<<grid_for(half * nb), 256, 0, c.stream>>>(A.p, half, out.p, out.bstride, bits, N, v, nb);
  TN_LAUNCHED();
  return out;
}

Tensor ones(Ctx& c, const std::vector<int>& shape, int nb) {
  Tensor t = new_tensor_n(c, shape, nb);
  int64_t n = t.size() * std::max(nb, 1);
  fill_kernel<<<grid_for(n), 256, 0, c.stream>>>(t.p, n, make_float2(1.f, 0.f));
  TN_LAUNCHED();
  return t;
}

void copy_rows(Ctx& c, const Tensor& src, Tensor& dst, int64_t x0, int nb) {
  invalidate_amax(dst);
  int64_t rowsz = dst.size() / dst.shape[0];
  int n = src.bstride ? nb : 1;
  int64_t size = src.size();
  copy_rows_kernel<<<grid_for(size * n), 256, 0, c.stream>>>(src.p, src.bstride, dst.p, dst.bstride, x0 * rowsz, size, n);
  TN_LAUNCHED();
}

void add_into(Ctx& c, Tensor& dst, const Tensor& src, int nb) {
  invalidate_amax(dst);
  int n = dst.bstride ? nb : 1;
  int64_t size = dst.size();
  add_kernel<<<grid_for(size * n), 256, 0, c.stream>>>(dst.p, dst.bstride, src.p, src.bstride, size, n);
  TN_LAUNCHED();
}

void log_add(Ctx& c, double* out, const double* a, const double* b, const double* c2, int n, bool acc) {
  log_add_kernel<<<ceil_div(n, 128), 128, 0, c.stream>>>(out, a, b, c2, n, acc);
  TN_LAUNCHED();
}

namespace {
__global__ void scalar_logphase_kernel(const float2* __restrict__ t, int64_t bs, int nb, double* logacc,
                                       double* phase) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  const float2 v = t[b * bs];
  const double a = hypot((double)v.x, (double)v.y);
  logacc[b] += a > 0 ? log(a) : -INFINITY;
  phase[b] = atan2((double)v.y, (double)v.x);
}
}  // namespace

void scalar_logphase(Ctx& c, const Tensor& t, int nb, double* logacc, double* phase) {
  scalar_logphase_kernel<<<ceil_div(nb, 128), 128, 0, c.stream>>>(t.p, t.bstride, nb, logacc, phase);
  TN_LAUNCHED();
}

void scalars_to_host(Ctx& c, const Tensor& t, int nb, std::vector<float2>& out) {
  out.resize(nb);
  int n = t.bstride ? nb : 1;
  std::vector<float2> tmp((size_t)t.size() * n);
  TN_CUDA(cudaMemcpyAsync(tmp.data(), t.p, tmp.size() * sizeof(float2), cudaMemcpyDeviceToHost, c.stream));
  TN_CUDA(cudaStreamSynchronize(c.stream));
  for (int b = 0; b < nb; ++b) out[b] = tmp[(size_t)(t.bstride ? b * t.bstride : 0)];
}

}  // namespace tn

// ---- debugging aid (TN_NAN_CHECK): number of non-finite complex entries of a tensor
namespace tn {
namespace {
__global__ void nonfinite_kernel(const float2* __restrict__ t, int64_t n, unsigned long long* cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    float2 v = t[i];
    if (!isfinite(v.x) || !isfinite(v.y)) atomicAdd(cnt, 1ull);
  }
}
}  // namespace
int64_t count_nonfinite(Ctx& c, const float2* p, int64_t n) {
  DevBuf d(sizeof(unsigned long long), c.stream);
  TN_CUDA(cudaMemsetAsync(d.p, 0, sizeof(unsigned long long), c.stream));
  if (n > 0) nonfinite_kernel<<<1184, 256, 0, c.stream>>>(p, n, d.as<unsigned long long>());
  unsigned long long h = 0;
  TN_CUDA(cudaMemcpyAsync(&h, d.p, sizeof h, cudaMemcpyDeviceToHost, c.stream));
  TN_CUDA(cudaStreamSynchronize(c.stream));
  return (int64_t)h;
}
}  // namespace tn

// ---- sample certification statistics (tn_certify). One CTA, FP64.
namespace tn {
namespace {
__global__ void __launch_bounds__(1024) cert_kernel(const double* __restrict__ lq, const double* __restrict__ lp,
                                                    int64_t n, double log_z, double* __restrict__ out) {
  __shared__ double red[32];
  __shared__ double s_bc;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  auto block_sum = [&](double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[w] = v;
    __syncthreads();
    if (w == 0) {
      double x = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
      for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      if (lane == 0) s_bc = x;
    }
    __syncthreads();
    double r = s_bc;
    __syncthreads();
    return r;
  };
  auto block_max = [&](double v) {
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) red[w] = v;
    __syncthreads();
    if (w == 0) {
      double x = lane < (int)(blockDim.x >> 5) ? red[lane] : -INFINITY;
      for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
      if (lane == 0) s_bc = x;
    }
    __syncthreads();
    double r = s_bc;
    __syncthreads();
    return r;
  };
  double mx = -INFINITY, cnt = 0, dsum = 0;
  for (int64_t k = t; k < n; k += blockDim.x) {
    const double d = lp[k] - lq[k];
    if (isfinite(d)) {
      mx = fmax(mx, d);
      cnt += 1;
      dsum += -d;
    }
  }
  mx = block_max(mx);
  cnt = block_sum(cnt);
  dsum = block_sum(dsum);
  double s1 = 0, s2 = 0;
  for (int64_t k = t; k < n; k += blockDim.x) {
    const double d = lp[k] - lq[k];
    if (isfinite(d)) {
      const double e = exp(d - mx);
      s1 += e;
      s2 += e * e;
    }
  }
  s1 = block_sum(s1);
  s2 = block_sum(s2);
  if (t == 0) {
    const double mean = s1 / cnt;  // in units of e^mx
    const double lne = mx + log(mean);
    double rel = 0;
    if (cnt > 1) {
      const double var = fmax(0.0, (s2 / cnt - mean * mean) * cnt / (cnt - 1));
      rel = sqrt(var / cnt) / mean;
    }
    const double lz = isfinite(log_z) ? log_z : lne;
    out[0] = cnt > 0 ? lne : NAN;
    out[1] = cnt > 0 ? rel : NAN;
    out[2] = cnt > 0 ? dsum / cnt + lz : NAN;
    out[3] = cnt > 0 ? s1 * s1 / s2 : 0;
    out[4] = cnt;
    out[5] = (double)n - cnt;
  }
}
// Importance weights w_k = exp(ln p_k - ln q_k - max) (0 for non-finite ratios) and the
// per-sample sector test: pass[k] = every group g holds target[g] ones (1 if no groups).
__global__ void __launch_bounds__(1024) obs_weights_kernel(const double* __restrict__ lq, const double* __restrict__ lp,
                                                          const uint8_t* __restrict__ bits, int64_t n, int N,
                                                          const int* __restrict__ group_of, int n_groups,
                                                          const int* __restrict__ target, double* __restrict__ w,
                                                          double* __restrict__ pass) {
  __shared__ double red[32];
  __shared__ double s_mx;
  const int t = threadIdx.x, lane = t & 31, wp = t >> 5;
  double mx = -INFINITY;
  for (int64_t k = t; k < n; k += blockDim.x) {
    const double d = lp[k] - lq[k];
    if (isfinite(d)) mx = fmax(mx, d);
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) red[wp] = mx;
  __syncthreads();
  if (t == 0) {
    double x = -INFINITY;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) x = fmax(x, red[i]);
    s_mx = x;
  }
  __syncthreads();
  for (int64_t k = t; k < n; k += blockDim.x) {
    const double d = lp[k] - lq[k];
    w[k] = isfinite(d) ? exp(d - s_mx) : 0.0;
    int cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (group_of)
      for (int v = 0; v < N; ++v) {
        const int g = group_of[v];
        if (g >= 0 && g < 8) cnt[g] += bits[k * N + v];
      }
    bool ok = true;
    for (int g = 0; g < n_groups && g < 8; ++g) ok = ok && cnt[g] == target[g];
    pass[k] = ok ? 1.0 : 0.0;
  }
}

// Block v: fixed-order sums over the samples of w z_v, z_v, w (z = 1 - 2 x_v) and, in block N,
// of pass and w pass (deterministic: per-thread strided partial sums, fixed tree).
__global__ void __launch_bounds__(256) obs_sums_kernel(const uint8_t* __restrict__ bits, const double* __restrict__ w,
                                                      const double* __restrict__ pass, int64_t n, int N,
                                                      double* __restrict__ out) {
  __shared__ double sh[3][256];
  const int v = blockIdx.x, t = threadIdx.x;
  double a = 0, b = 0, c = 0;
  for (int64_t k = t; k < n; k += blockDim.x) {
    if (v < N) {
      const double z = 1.0 - 2.0 * bits[k * N + v];
      a += w[k] * z;
      b += z;
      c += w[k];
    } else {
      a += pass[k];
      b += w[k] * pass[k];
      c += w[k];
    }
  }
  sh[0][t] = a;
  sh[1][t] = b;
  sh[2][t] = c;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (t < s)
      for (int q = 0; q < 3; ++q) sh[q][t] += sh[q][t + s];
    __syncthreads();
  }
  if (t == 0)
    for (int q = 0; q < 3; ++q) out[3 * v + q] = sh[q][0];
}
}  // namespace

void observables(Ctx& c, const uint8_t* bits, const double* logq, const double* logp, int64_t n, int N,
                 const int* group_of, int n_groups, const int* target, double* w, double* pass, double* sums) {
  obs_weights_kernel<<<1, 1024, 0, c.stream>>>(logq, logp, bits, n, N, group_of, n_groups, target, w, pass);
  TN_LAUNCHED();
  obs_sums_kernel<<<N + 1, 256, 0, c.stream>>>(bits, w, pass, n, N, sums);
  TN_LAUNCHED();
}

void cert_stats(Ctx& c, const double* logq, const double* logp, int64_t n, double log_z, double* out) {
  cert_kernel<<<1, 1024, 0, c.stream>>>(logq, logp, n, log_z, out);
  TN_LAUNCHED();
}
}  // namespace tn
