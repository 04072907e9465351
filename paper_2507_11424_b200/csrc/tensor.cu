// tensor.cu -- device tensors, permutation kernel, FP32 SIMT complex GEMM and the
// contraction planner (see tensor.h).
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <map>

#include "tensor.h"

namespace tn {

thread_local int64_t g_launches = 0;
thread_local double g_cmacs = 0.0;
thread_local double g_cmacs_tc = 0.0;
thread_local int64_t g_tc_launches = 0;
thread_local std::vector<double> g_row_cmacs;

// tcgen05 path (gemm_tc.cu); returns false when the shape/layout is not eligible.
bool gemm_tc(Ctx& c, const GemmDesc& g);

Tensor new_tensor_n(Ctx& c, const std::vector<int>& shape, int nb) {
  Tensor t;
  t.shape = shape;
  int64_t sz = prod(shape);
  t.bstride = nb > 1 ? sz : (nb == 1 ? sz : 0);
  size_t bytes = (size_t)std::max<int64_t>(1, sz * std::max(nb, 1)) * sizeof(float2);
  t.mem = std::make_shared<DevBuf>(bytes, c.stream, std::max(nb, 1));
  t.p = t.mem->as<float2>();
  return t;
}

Tensor new_tensor(Ctx& c, const std::vector<int>& shape, bool per_sample) {
  Tensor t = new_tensor_n(c, shape, per_sample ? c.nb : 1);
  if (!per_sample) t.bstride = 0;
  return t;
}

void zero(Ctx& c, Tensor& t, int nb) {
  invalidate_amax(t);
  int64_t n = t.bstride ? t.bstride * nb : t.size();
  TN_CUDA(cudaMemsetAsync(t.p, 0, (size_t)n * sizeof(float2), c.stream));
}

// ----------------------------------------------------------------------------- permute
struct PermArgs {
  int rank;
  int64_t dims[8];      // output dims
  int64_t istride[8];   // input stride of each output axis
  int64_t size;         // elements per sample
  int64_t ibs, obs;     // sample strides
  int nb;
  bool conj;
};

__global__ void permute_kernel(const float2* __restrict__ in, float2* __restrict__ out, PermArgs a) {
  int64_t total = a.size * a.nb;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = i / a.size, r = i - b * a.size;
    int64_t off = 0, rem = r;
#pragma unroll
    for (int d = 7; d >= 0; --d) {
      if (d < a.rank) {
        int64_t q = rem / a.dims[d];
        int64_t idx = rem - q * a.dims[d];
        off += idx * a.istride[d];
        rem = q;
      }
    }
    float2 v = in[b * a.ibs + off];
    if (a.conj) v.y = -v.y;
    out[b * a.obs + r] = v;
  }
}

// Row copy: the innermost output axis is contiguous in the input as well. One warp per output
// row (all axes but the last), lanes across the row: coalesced on both sides.
__global__ void permute_rows_kernel(const float2* __restrict__ in, float2* __restrict__ out, PermArgs a) {
  const int64_t L = a.dims[a.rank - 1];
  const int64_t rows_per = a.size / L, rows = rows_per * a.nb;
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t row = w0; row < rows; row += nw) {
    const int64_t b = row / rows_per;
    int64_t rem = row - b * rows_per, off = 0;
    for (int d = a.rank - 2; d >= 0; --d) {
      const int64_t q = rem / a.dims[d];
      off += (rem - q * a.dims[d]) * a.istride[d];
      rem = q;
    }
    const float2* src = in + b * a.ibs + off;
    float2* dst = out + b * a.obs + (row - b * rows_per) * L;
    for (int64_t l = lane; l < L; l += 32) {
      float2 v = src[l];
      if (a.conj) v.y = -v.y;
      dst[l] = v;
    }
  }
}

// Tiled transpose: output axis `kin` is the input's contiguous axis, the last output axis is
// strided in the input. 32x32 tiles through shared memory; every other axis (and the
// sample) is a batch coordinate of the grid.
struct Perm2 {
  PermArgs a;
  int kin;                 // output axis with input stride 1
  int64_t ostride[8];      // output strides (row-major of the output dims)
  int64_t nother;          // product of the other axes
  int ntk, ntl;            // tiles along kin and along the last axis
};

__global__ void __launch_bounds__(256) permute_tile_kernel(const float2* __restrict__ in, float2* __restrict__ out,
                                                           Perm2 p) {
  __shared__ float2 tile[32][33];
  const PermArgs& a = p.a;
  const int last = a.rank - 1;
  const int64_t dk = a.dims[p.kin], dl = a.dims[last];
  const int t = blockIdx.x, tk = t % p.ntk, tl = t / p.ntk;
  const int64_t bb = blockIdx.y + (int64_t)blockIdx.z * gridDim.y;
  if (bb >= p.nother * a.nb) return;
  const int64_t b = bb / p.nother;
  int64_t rem = bb - b * p.nother, ioff = 0, ooff = 0;
  for (int d = last - 1; d >= 0; --d) {
    if (d == p.kin) continue;
    const int64_t q = rem / a.dims[d];
    const int64_t idx = rem - q * a.dims[d];
    ioff += idx * a.istride[d];
    ooff += idx * p.ostride[d];
    rem = q;
  }
  const float2* src = in + b * a.ibs + ioff;
  float2* dst = out + b * a.obs + ooff;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int j = ty; j < 32; j += 8) {
    const int64_t l = (int64_t)tl * 32 + j, k = (int64_t)tk * 32 + tx;
    if (l < dl && k < dk) tile[j][tx] = src[k + l * a.istride[last]];
  }
  __syncthreads();
  for (int j = ty; j < 32; j += 8) {
    const int64_t k = (int64_t)tk * 32 + j, l = (int64_t)tl * 32 + tx;
    if (l < dl && k < dk) {
      float2 v = tile[tx][j];
      if (a.conj) v.y = -v.y;
      dst[k * p.ostride[p.kin] + l] = v;
    }
  }
}

static std::vector<int64_t> strides_of(const std::vector<int>& shape) {
  std::vector<int64_t> s(shape.size());
  int64_t acc = 1;
  for (int i = (int)shape.size() - 1; i >= 0; --i) {
    s[i] = acc;
    acc *= shape[i];
  }
  return s;
}

Tensor permute(Ctx& c, const Tensor& A, const char* la, const char* lout, bool conj) {
  int r = (int)strlen(la);
  if (r != A.rank() || (int)strlen(lout) != r) throw Error(-1, "permute: label/rank mismatch");
  auto st = strides_of(A.shape);
  std::vector<int> oshape(r);
  PermArgs a{};
  a.rank = 0;
  // drop unit dims, merge nothing (simple)
  std::vector<int64_t> dims, istr;
  for (int i = 0; i < r; ++i) {
    const char* q = strchr(la, lout[i]);
    if (!q) throw Error(-1, "permute: unknown label");
    int j = (int)(q - la);
    oshape[i] = A.shape[j];
    if (A.shape[j] != 1) {
      dims.push_back(A.shape[j]);
      istr.push_back(st[j]);
    }
  }
  // merge output axes that are also adjacent (and in order) in the input
  std::vector<int64_t> md, ms;
  for (size_t i = 0; i < dims.size(); ++i) {
    if (!md.empty() && ms.back() == istr[i] * dims[i]) {
      md.back() *= dims[i];
      ms.back() = istr[i];
    } else {
      md.push_back(dims[i]);
      ms.push_back(istr[i]);
    }
  }
  if (md.size() > 8) throw Error(-1, "permute: rank > 8");
  int nb = A.bstride ? c.nb : 1;
  Tensor out = new_tensor_n(c, oshape, nb);
  if (!A.bstride) out.bstride = 0;
  a.rank = (int)md.size();
  for (int i = 0; i < a.rank; ++i) {
    a.dims[i] = md[i];
    a.istride[i] = ms[i];
  }
  if (a.rank == 0) {
    a.rank = 1;
    a.dims[0] = 1;
    a.istride[0] = 1;
  }
  a.size = A.size();
  a.ibs = A.bstride;
  a.obs = out.bstride;
  a.nb = nb;
  a.conj = conj;
  int64_t total = a.size * nb;
  if (total == 0) return out;
  ProfScope ps(P_PERMUTE, c.stream);
  const int last = a.rank - 1;
  int kin = -1;
  for (int i = 0; i < a.rank; ++i)
    if (a.istride[i] == 1) kin = i;
  if (kin == last && a.dims[last] >= 16) {
    int64_t rows = total / a.dims[last];
    unsigned blocks = (unsigned)std::min<int64_t>((rows + 7) / 8, 148 * 64);
    permute_rows_kernel<<<blocks, 256, 0, c.stream>>>(A.p, out.p, a);
  } else if (kin >= 0 && kin != last && a.dims[last] >= 8 && a.dims[kin] >= 8) {
    Perm2 p;
    p.a = a;
    p.kin = kin;
    int64_t acc = 1;
    for (int i = last; i >= 0; --i) {
      p.ostride[i] = acc;
      acc *= a.dims[i];
    }
    p.nother = a.size / (a.dims[kin] * a.dims[last]);
    p.ntk = (int)((a.dims[kin] + 31) / 32);
    p.ntl = (int)((a.dims[last] + 31) / 32);
    int64_t nbat = p.nother * nb;
    unsigned gy = (unsigned)std::min<int64_t>(nbat, 65535);
    unsigned gz = (unsigned)((nbat + gy - 1) / gy);
    dim3 grid((unsigned)(p.ntk * p.ntl), gy, gz);
    permute_tile_kernel<<<grid, 256, 0, c.stream>>>(A.p, out.p, p);
  } else {
    unsigned blocks = (unsigned)std::min<int64_t>((total + 255) / 256, 148 * 32);
    permute_kernel<<<blocks, 256, 0, c.stream>>>(A.p, out.p, a);
  }
  TN_LAUNCHED();
  return out;
}

// ----------------------------------------------------------------------------- SIMT GEMM
// 64x64 complex tile, BK = 8, 256 threads, 4x4 complex outputs per thread, FP32 FMA.
// Used for shapes the tcgen05 kernel does not take (small or unaligned) and as the
// forced path gemm=1.
namespace {
constexpr int BM = 64, BN = 64, BK = 8, PAD = 2;

__device__ __forceinline__ float2 ld_c(const float2* p, bool cj) {
  float2 v = __ldg(p);
  if (cj) v.y = -v.y;
  return v;
}

// Thin GEMMs (N <= 8, e.g. a physical or unit output leg): one warp per output row, the lanes
// stride over K (coalesced when A's K stride is 1), N running sums per lane, fixed-order warp
// reduction. Memory-bound; the tiled SIMT kernel wastes most of its 64-wide N tile here.
constexpr int THIN_N = 8;
__global__ void __launch_bounds__(256) cgemm_thin(GemmDesc g) {
  const int bz = blockIdx.y;
  const int b1 = bz / g.nb2, b2 = bz - b1 * g.nb2;
  const float2* A = g.A + b1 * g.sa1 + b2 * g.sa2;
  const float2* B = g.B + b1 * g.sb1 + b2 * g.sb2;
  float2* C = g.C + b1 * g.sc1 + b2 * g.sc2;
  const int lane = threadIdx.x & 31;
  const int64_t m = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (m >= g.M) return;
  float2 acc[THIN_N];
#pragma unroll
  for (int n = 0; n < THIN_N; ++n) acc[n] = make_float2(0.f, 0.f);
  for (int k = lane; k < g.K; k += 32) {
    const float2 a = ld_c(A + m * g.am + (int64_t)k * g.ak, g.conjA);
#pragma unroll
    for (int n = 0; n < THIN_N; ++n) {
      if (n < g.N) {
        const float2 b = ld_c(B + (int64_t)k * g.bk + (int64_t)n * g.bn, g.conjB);
        acc[n].x = fmaf(a.x, b.x, fmaf(-a.y, b.y, acc[n].x));
        acc[n].y = fmaf(a.x, b.y, fmaf(a.y, b.x, acc[n].y));
      }
    }
  }
#pragma unroll
  for (int n = 0; n < THIN_N; ++n) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      acc[n].x += __shfl_xor_sync(0xffffffffu, acc[n].x, o);
      acc[n].y += __shfl_xor_sync(0xffffffffu, acc[n].y, o);
    }
  }
  if (lane < g.N) {
    float2 v = acc[0];
#pragma unroll
    for (int n = 1; n < THIN_N; ++n)
      if (lane == n) v = acc[n];
    float2* cp = C + m * g.cm + lane;
    if (g.accumulate) {
      const float2 o = *cp;
      v.x += o.x;
      v.y += o.y;
    }
    *cp = v;
  }
}

__global__ void __launch_bounds__(256) cgemm_simt(GemmDesc g) {
  __shared__ __align__(16) float2 As[BK][BM + PAD];
  __shared__ __align__(16) float2 Bs[BK][BN + PAD];
  int bz = blockIdx.z;
  int b1 = bz / g.nb2, b2 = bz - b1 * g.nb2;
  const float2* A = g.A + b1 * g.sa1 + b2 * g.sa2;
  const float2* B = g.B + b1 * g.sb1 + b2 * g.sb2;
  float2* C = g.C + b1 * g.sc1 + b2 * g.sc2;
  int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  int t = threadIdx.x;
  int tx = t & 15, ty = t >> 4;
  float2 acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = make_float2(0.f, 0.f);
  const bool a_kc = (g.ak == 1);
  const bool b_nc = (g.bn == 1);
  float2 ra[2], rb[2];
  auto load = [&](int k0) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      int e = t + 256 * i;
      int m, k;
      if (a_kc) { m = e >> 3; k = e & 7; } else { m = e & 63; k = e >> 6; }
      int gm = m0 + m, gk = k0 + k;
      ra[i] = (gm < g.M && gk < g.K) ? ld_c(A + gm * g.am + gk * g.ak, g.conjA) : make_float2(0.f, 0.f);
      int n;
      if (b_nc) { n = e & 63; k = e >> 6; } else { n = e >> 3; k = e & 7; }
      int gn = n0 + n;
      gk = k0 + k;
      rb[i] = (gn < g.N && gk < g.K) ? ld_c(B + gk * g.bk + gn * g.bn, g.conjB) : make_float2(0.f, 0.f);
    }
  };
  auto store = [&]() {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      int e = t + 256 * i;
      int m, k;
      if (a_kc) { m = e >> 3; k = e & 7; } else { m = e & 63; k = e >> 6; }
      As[k][m] = ra[i];
      int n;
      if (b_nc) { n = e & 63; k = e >> 6; } else { n = e >> 3; k = e & 7; }
      Bs[k][n] = rb[i];
    }
  };
  load(0);
  for (int k0 = 0; k0 < g.K; k0 += BK) {
    store();
    __syncthreads();
    if (k0 + BK < g.K) load(k0 + BK);
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float4 a01 = *reinterpret_cast<const float4*>(&As[kk][ty * 4]);
      float4 a23 = *reinterpret_cast<const float4*>(&As[kk][ty * 4 + 2]);
      float4 b01 = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
      float4 b23 = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4 + 2]);
      float2 a[4] = {{a01.x, a01.y}, {a01.z, a01.w}, {a23.x, a23.y}, {a23.z, a23.w}};
      float2 b[4] = {{b01.x, b01.y}, {b01.z, b01.w}, {b23.x, b23.y}, {b23.z, b23.w}};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          acc[i][j].x = fmaf(a[i].x, b[j].x, acc[i][j].x);
          acc[i][j].x = fmaf(-a[i].y, b[j].y, acc[i][j].x);
          acc[i][j].y = fmaf(a[i].x, b[j].y, acc[i][j].y);
          acc[i][j].y = fmaf(a[i].y, b[j].x, acc[i][j].y);
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int gm = m0 + ty * 4 + i;
    if (gm >= g.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int gn = n0 + tx * 4 + j;
      if (gn >= g.N) continue;
      float2* cp = C + (int64_t)gm * g.cm + gn;
      if (g.accumulate) {
        float2 o = *cp;
        o.x += acc[i][j].x;
        o.y += acc[i][j].y;
        *cp = o;
      } else {
        *cp = acc[i][j];
      }
    }
  }
}
}  // namespace

// TN_GEMM_LOG: shapes routed to the SIMT GEMM (calls, complex MACs), printed by
// tn_debug_simt_log() -- instrumentation only.
static bool simt_log_on() {
  static int on = -1;
  if (on < 0) on = getenv("TN_GEMM_LOG") ? 1 : 0;
  return on == 1;
}
std::map<std::string, std::pair<double, double>>& simt_tab() {
  static auto* t = new std::map<std::string, std::pair<double, double>>();
  return *t;
}

bool gemm(Ctx& c, const GemmDesc& g) {
  if (g.M <= 0 || g.N <= 0 || g.nb1 <= 0 || g.nb2 <= 0) return false;
  g_cmacs += (double)g.M * g.N * std::max(g.K, 0) * g.nb1 * g.nb2;
  if (g.K <= 0) {
    if (!g.accumulate) {
      // C = 0 (empty contraction): handled by the planner allocating zeroed outputs
    }
    return false;
  }
  {
    ProfScope ps(P_GEMM_TC, c.stream);
    if (c.gemm_mode != 1 && gemm_tc(c, g)) return true;
  }
  ProfScope ps(P_GEMM_SIMT, c.stream);
  if (simt_log_on()) {
    char k[128];
    snprintf(k, sizeof k, "M=%d N=%d K=%d nb1=%d nb2=%d", g.M, g.N, g.K, g.nb1, g.nb2);
    auto& e = simt_tab()[k];
    e.first += 1;
    e.second += (double)g.M * g.N * g.K * g.nb1 * g.nb2;
  }
  int64_t nbz = (int64_t)g.nb1 * g.nb2;
  if (nbz > 65535) {
    // split the outer batch into chunks
    GemmDesc h = g;
    int per = std::max(1, 65535 / g.nb2);
    for (int b0 = 0; b0 < g.nb1; b0 += per) {
      h.nb1 = std::min(per, g.nb1 - b0);
      h.A = g.A + b0 * g.sa1;
      h.B = g.B + b0 * g.sb1;
      h.C = g.C + b0 * g.sc1;
      gemm(c, h);
    }
    g_cmacs -= (double)g.M * g.N * g.K * g.nb1 * g.nb2;
    return false;
  }
  if (g.N <= THIN_N && g.K >= 256) {
    dim3 tgrid(ceil_div(g.M, 8), (unsigned)nbz);
    cgemm_thin<<<tgrid, 256, 0, c.stream>>>(g);
    TN_LAUNCHED();
    return false;
  }
  dim3 grid(ceil_div(g.N, BN), ceil_div(g.M, BM), (unsigned)nbz);
  if (grid.y > 65535) {
    GemmDesc h = g;
    int rows = 65535 * BM;
    for (int m0 = 0; m0 < g.M; m0 += rows) {
      h.M = std::min(rows, g.M - m0);
      h.A = g.A + (int64_t)m0 * g.am;
      h.C = g.C + (int64_t)m0 * g.cm;
      gemm(c, h);
      g_cmacs -= (double)h.M * h.N * h.K * h.nb1 * h.nb2;
    }
    return false;
  }
  cgemm_simt<<<grid, 256, 0, c.stream>>>(g);
  TN_LAUNCHED();
  return false;
}

// ----------------------------------------------------------------------------- planner
namespace {
struct Op {
  const Tensor* t;
  std::string lab;          // labels without unit dims
  std::vector<int> dims;    // matching dims
  std::vector<int64_t> str; // matching strides
  bool conj;
};

Op make_op(const Tensor& t, const char* l, bool cj) {
  Op o{&t, "", {}, {}, cj};
  int r = (int)strlen(l);
  if (r != t.rank()) throw Error(-1, std::string("contract: rank mismatch for labels ") + l);
  auto st = strides_of(t.shape);
  for (int i = 0; i < r; ++i)
    if (t.shape[i] != 1) {
      o.lab.push_back(l[i]);
      o.dims.push_back(t.shape[i]);
      o.str.push_back(st[i]);
    }
  return o;
}

// If the labels `grp` (in this order) occupy consecutive axes of op, return the stride of
// the compound index (stride of the last one); -1 otherwise. Empty group -> 0.
int64_t group_stride(const Op& o, const std::string& grp) {
  if (grp.empty()) return 0;
  size_t p0 = o.lab.find(grp[0]);
  if (p0 == std::string::npos) return -1;
  for (size_t i = 0; i < grp.size(); ++i)
    if (p0 + i >= o.lab.size() || o.lab[p0 + i] != grp[i]) return -1;
  return o.str[p0 + grp.size() - 1];
}

std::string order_in(const std::string& lab, const std::string& set) {
  std::string r;
  for (char ch : lab)
    if (set.find(ch) != std::string::npos) r.push_back(ch);
  return r;
}
}  // namespace

// Plane-output request of contract_planes: the consumer's batch / row / K labels.
struct PlaneReq {
  std::string zl, rl, kl;
};

// The plane-output half of contract_planes: map every output digit of the GEMM g (M digits:
// the folded sample, then Ms; N digits: Ns) to the consumer's planes, allocate them and run g.
thread_local int64_t g_plane_gemms = 0;  // GEMMs run with plane output (tn_debug_plane_gemms)

static Tensor plane_output(Ctx& c, GemmDesc& g, const PlaneReq& rq, std::map<char, int>& dim,
                           const std::string& Ls, const std::string& Ms, const std::string& Ns,
                           const std::string& out, bool per_out, int64_t Msz) {
    const PlaneReq* req = &rq;
    // ---- plane output (contract_planes): C goes straight into the consumer's A planes
    if (!per_out || !Ls.empty() || g.nb2 != 1 || (g.nb1 != 1 && g.nb1 != c.nb) || Ms.empty() || Ns.empty())
      throw Error(-1, "contract_planes: unsupported GEMM form");
    const std::string &zl = req->zl, &rl = req->rl, &kl = req->kl;
    if (zl.size() + rl.size() + kl.size() != out.size() || kl.empty() || rl.empty())
      throw Error(-1, "contract_planes: the consumer labels must partition the output labels");
    auto grp_of = [&](char ch) -> int {
      if (zl.find(ch) != std::string::npos) return 0;
      if (rl.find(ch) != std::string::npos) return 1;
      if (kl.find(ch) != std::string::npos) return 2;
      throw Error(-1, "contract_planes: output label missing from the consumer labels");
    };
    auto prod_of = [&](const std::string& l) {
      int64_t r = 1;
      for (char ch : l) r *= dim[ch];
      return r;
    };
    auto stride_in = [&](const std::string& l, char ch) {
      int64_t r = 1;
      for (size_t i = l.find(ch) + 1; i < l.size(); ++i) r *= dim[l[i]];
      return r;
    };
    const char inner = kl.back();
    const int64_t NZ = prod_of(zl), Mc = prod_of(rl), Kc = prod_of(kl);
    const int64_t Mpc = (Mc + 255) / 256 * 256, Krpc = (2 * Kc + 63) / 64 * 64;
    // Scale-block shape in the producer's tile. Mode 1: the consumer's inner K label (128) is
    // this GEMM's inner row digit -- a block is one column of a CTA's 128 rows. Mode 2: the
    // inner K label (32) is the inner row digit and the next K label, this GEMM's inner column
    // digit, supplies 4 -- a block is a warp's 32 rows x 4 adjacent columns.
    int mode = 0;
    char outer = 0;
    if (dim[inner] % 128 == 0 && Ms.back() == inner) mode = 1;
    else if (dim[inner] == 32 && Ms.back() == inner && kl.size() >= 2 && Ns.back() == kl[kl.size() - 2] &&
             dim[kl[kl.size() - 2]] % 4 == 0) {
      mode = 2;
      outer = kl[kl.size() - 2];
    }
    if (!mode || Mpc != Mc || Krpc != 2 * Kc || Mc <= 128)
      throw Error(-1, "contract_planes: shapes do not allow plane output");
    const int64_t nsb = Kc / 128;
    auto digit = [&](char ch, int64_t& po, int64_t& so) {
      const int gi = grp_of(ch);
      if (gi == 0) {
        const int64_t st = stride_in(zl, ch);
        po = st * Mpc * Krpc;
        so = st * nsb * Mpc;
      } else if (gi == 1) {
        const int64_t st = stride_in(rl, ch);
        po = st * Krpc;
        so = st;
      } else {
        const int64_t st = stride_in(kl, ch);
        po = 2 * st;
        so = (ch == inner) ? 0 : (st / 128) * Mpc;
      }
    };
    PlaneOut pout;
    const bool folded = (g.M == Msz * c.nb) && c.nb > 1;
    if (!folded && g.M != Msz) throw Error(-1, "contract_planes: unexpected GEMM rows");
    auto add = [](PView& v, int d, int64_t po, int64_t so) {
      if (v.rank >= 6) throw Error(-1, "contract_planes: more than six digits");
      v.dims[v.rank] = d;
      v.po[v.rank] = po;
      v.so[v.rank] = so;
      ++v.rank;
    };
    if (folded) add(pout.vm, c.nb, NZ * Mpc * Krpc, NZ * nsb * Mpc);
    else if (g.nb1 > 1) {  // samples on the GEMM's batch index
      pout.zpo = NZ * Mpc * Krpc;
      pout.zso = NZ * nsb * Mpc;
    }
    for (char ch : Ms) {
      int64_t po, so;
      digit(ch, po, so);
      if (mode == 1 && ch == inner && dim[ch] > 128) {  // split: (label / 128: block, label % 128: a tile's rows)
        add(pout.vm, dim[ch] / 128, 2 * 128, Mpc);
        add(pout.vm, 128, 2, 0);
      } else {
        add(pout.vm, dim[ch], po, so);
      }
    }
    for (char ch : Ns) {
      int64_t po, so;
      digit(ch, po, so);
      if (mode == 2 && ch == outer) {  // split: (label / 4: block index, label % 4: inside a block)
        const int64_t st = stride_in(kl, ch);  // = 32
        add(pout.vn, dim[ch] / 4, 2 * st * 4, Mpc);
        add(pout.vn, 4, 2 * st, 0);
      } else {
        add(pout.vn, dim[ch], po, so);
      }
    }
    pout.mode = mode;
    auto P = std::make_shared<Planes>();
    P->lab = zl + rl + kl;
    P->nz = (int)(c.nb * NZ);
    P->Mp = (int)Mpc;
    P->Krp = (int)Krpc;
    P->nsb = (int)nsb;
    const size_t nh = (size_t)P->nz * Mpc * Krpc;
    P->hi = std::make_shared<DevBuf>(nh * 2, c.stream);
    P->lo = std::make_shared<DevBuf>(nh * 2, c.stream);
    P->asc = std::make_shared<DevBuf>((size_t)P->nz * nsb * Mpc * sizeof(float), c.stream);
    pout.hi = P->hi->as<__half>();
    pout.lo = P->lo->as<__half>();
    pout.asc = P->asc->as<float>();
    g.po = &pout;
    g.C = nullptr;
    g.amaxC = nullptr;
    if (!gemm(c, g)) throw Error(-1, "contract_planes: not on the tensor cores");
    ++g_plane_gemms;
    Tensor T;
    T.planes = P;
    for (char ch : P->lab) T.shape.push_back(dim[ch]);
    T.bstride = T.size();
    return T;
}

static Tensor contract_impl(Ctx& c, const Tensor& A0, const char* la0, bool conjA0, const Tensor& B0,
                            const char* lb0, bool conjB0, const char* lout, const PlaneReq* req) {
  // dims of every label
  std::map<char, int> dim;
  auto reg = [&](const Tensor& t, const char* l) {
    int r = (int)strlen(l);
    if (r != t.rank()) throw Error(-1, std::string("contract: rank mismatch ") + l);
    for (int i = 0; i < r; ++i) {
      auto it = dim.find(l[i]);
      if (it != dim.end() && it->second != t.shape[i])
        throw Error(-1, std::string("contract: dim mismatch on label ") + l[i]);
      dim[l[i]] = t.shape[i];
    }
  };
  reg(A0, la0);
  reg(B0, lb0);
  std::vector<int> oshape;
  for (const char* q = lout; *q; ++q) {
    auto it = dim.find(*q);
    if (it == dim.end()) {  // a label absent from both operands is a unit axis
      dim[*q] = 1;
      oshape.push_back(1);
    } else {
      oshape.push_back(it->second);
    }
  }
  // left operand = the per-sample one when the other is shared
  bool swap = (A0.bstride == 0 && B0.bstride != 0);
  const Tensor& X = swap ? B0 : A0;
  const Tensor& Y = swap ? A0 : B0;
  const char* lx = swap ? lb0 : la0;
  const char* ly = swap ? la0 : lb0;
  bool cx = swap ? conjB0 : conjA0, cy = swap ? conjA0 : conjB0;
  Op ox = make_op(X, lx, cx), oy = make_op(Y, ly, cy);
  std::string out;
  for (const char* q = lout; *q; ++q)
    if (dim[*q] != 1) out.push_back(*q);
  std::string Ls, Ms, Ns, Ks;
  for (char ch : out) {
    bool inx = ox.lab.find(ch) != std::string::npos, iny = oy.lab.find(ch) != std::string::npos;
    if (inx && iny) Ls.push_back(ch);
    else if (inx) Ms.push_back(ch);
    else if (iny) Ns.push_back(ch);
    else throw Error(-1, "contract: output label not in operands");
  }
  for (char ch : ox.lab)
    if (out.find(ch) == std::string::npos) {
      if (oy.lab.find(ch) == std::string::npos) throw Error(-1, "contract: label summed in one operand only");
      Ks.push_back(ch);
    }
  for (char ch : oy.lab)
    if (out.find(ch) == std::string::npos && ox.lab.find(ch) == std::string::npos)
      throw Error(-1, "contract: label summed in one operand only");
  int64_t Lsz = 1, Msz = 1, Nsz = 1, Ksz = 1;
  for (char ch : Ls) Lsz *= dim[ch];
  for (char ch : Ms) Msz *= dim[ch];
  for (char ch : Ns) Nsz *= dim[ch];
  for (char ch : Ks) Ksz *= dim[ch];
  bool per_out = X.bstride || Y.bstride;
  if (Y.planes) throw Error(-1, "contract: a planes operand must be the per-sample left operand");
  if (X.planes) {
    // A from the planes its producer wrote: the planes fix the batch, row and K orders
    const Planes& P = *X.planes;
    const std::string Kx = order_in(ox.lab, Ks);
    if (cx || P.lab != std::string(lx) || P.lab != Ls + Ms + Kx || !per_out)
      throw Error(-1, std::string("contract: planes ") + P.lab + " do not fit " + lx);
    GemmDesc g;
    g.M = (int)Msz;
    g.N = (int)Nsz;
    g.K = (int)Ksz;
    g.pa = &P;
    auto mk = [](const Op& o, const std::string& grp, View4& v) {
      std::vector<int64_t> d, st;
      for (char ch : grp) {
        size_t q = o.lab.find(ch);
        int64_t dd = o.dims[q], ss = o.str[q];
        if (!d.empty() && st.back() == ss * dd) {
          d.back() *= dd;
          st.back() = ss;
        } else {
          d.push_back(dd);
          st.push_back(ss);
        }
      }
      if (d.size() > 4) return false;
      if (d.empty()) {
        d.push_back(1);
        st.push_back(0);
      }
      v.rank = (int)d.size();
      for (int i = 0; i < v.rank; ++i) {
        v.dims[i] = (int)d[i];
        v.str[i] = st[i];
      }
      return true;
    };
    if (group_stride(oy, Ls) < 0 || !mk(oy, Kx, g.vbk) || !mk(oy, Ns, g.vbn))
      throw Error(-1, "contract: planes consumer needs a gatherable right operand");
    g.vam.rank = 1;
    g.vam.dims[0] = (int)Msz;
    g.vak.rank = 1;
    g.vak.dims[0] = (int)Ksz;
    g.B = Y.p;
    g.conjB = cy;
    g.nb1 = c.nb;
    g.nb2 = (int)Lsz;
    g.sb1 = Y.bstride;
    g.sb2 = Ls.empty() ? 0 : group_stride(oy, Ls);
    if (P.nz != g.nb1 * g.nb2) throw Error(-1, "contract: planes batch mismatch");
    g.work_per_sample = Msz * Nsz * Ksz * Lsz;
    g.m_per_sample = (int)Msz;
    if (req) return plane_output(c, g, *req, dim, Ls, Ms, Ns, out, per_out, Msz);  // planes in and out
    const std::string gout = Ls + Ms + Ns;
    std::vector<int> gshape;
    for (char ch : gout) gshape.push_back(dim[ch]);
    Tensor C = new_tensor_n(c, gshape, c.nb);
    g.C = C.p;
    g.cm = Nsz;
    g.sc1 = C.bstride;
    g.sc2 = Msz * Nsz;
    g.work_per_sample = Msz * Nsz * Ksz * Lsz;
    g.m_per_sample = (int)Msz;
    if (!gemm(c, g)) throw Error(-1, "contract: planes consumer not on the tensor cores");
    if (gout == out) {
      C.shape = oshape;
      return C;
    }
    std::string dst(lout), src = gout;
    for (char ch : dst)
      if (src.find(ch) == std::string::npos) src.push_back(ch);
    Tensor Ct = C;
    Ct.shape.clear();
    for (char ch : src) Ct.shape.push_back(dim.count(ch) ? dim[ch] : 1);
    return permute(c, Ct, src.c_str(), dst.c_str(), false);
  }

  // choose the K order: keep whichever operand's order avoids a permute, else the larger's
  std::string Kx = order_in(ox.lab, Ks), Ky = order_in(oy.lab, Ks);
  auto x_ok = [&](const std::string& K) {
    return group_stride(ox, Ls) >= 0 && group_stride(ox, Ms) >= 0 && group_stride(ox, K) >= 0;
  };
  auto y_ok = [&](const std::string& K) {
    return group_stride(oy, Ls) >= 0 && group_stride(oy, Ns) >= 0 && group_stride(oy, K) >= 0;
  };
  std::string Kord;
  // per-sample sizes: the K order (hence the summation order) must not depend on the batch
  int64_t szx = X.size(), szy = Y.size();
  if (x_ok(Kx) && y_ok(Kx)) Kord = Kx;
  else if (x_ok(Ky) && y_ok(Ky)) Kord = Ky;
  else if (x_ok(Kx)) Kord = Kx;   // permute Y
  else if (y_ok(Ky)) Kord = Ky;   // permute X
  else Kord = (szx >= szy) ? Kx : Ky;

  // Tensor-core GEMMs gather their operands from any multi-axis layout while splitting them
  // into TF32 planes, so no permute is needed on that path.
  GemmDesc gv;
  bool views = false;
  static const bool no_views = getenv("TN_NOVIEWS") != nullptr;
  if (!no_views && (!x_ok(Kord) || !y_ok(Kord)) && tc_eligible(c, Msz, Nsz, Ksz, Msz * Nsz * Ksz * Lsz) &&
      group_stride(ox, Ls) >= 0 && group_stride(oy, Ls) >= 0) {
    auto mkview = [](const Op& o, const std::string& grp, View4& v) {
      std::vector<int64_t> d, s;
      for (char ch : grp) {
        size_t p = o.lab.find(ch);
        int64_t dd = o.dims[p], ss = o.str[p];
        if (!d.empty() && s.back() == ss * dd) {
          d.back() *= dd;
          s.back() = ss;
        } else {
          d.push_back(dd);
          s.push_back(ss);
        }
      }
      if (d.size() > 4) return false;
      if (d.empty()) {
        d.push_back(1);
        s.push_back(0);
      }
      v.rank = (int)d.size();
      for (int i = 0; i < v.rank; ++i) {
        v.dims[i] = (int)d[i];
        v.str[i] = s[i];
      }
      return true;
    };
    std::string Kv = Kx;
    views = mkview(ox, Ms, gv.vam) && mkview(ox, Kv, gv.vak) && mkview(oy, Kv, gv.vbk) && mkview(oy, Ns, gv.vbn);
  }
  // materialise operands in GEMM-viewable layouts when needed
  Tensor Xp, Yp;
  const Tensor* Xu = &X;
  const Tensor* Yu = &Y;
  std::string lxu = lx, lyu = ly;
  Op oxu = ox, oyu = oy;
  if (views) {
    // gather path: no operand permutes
  } else if (!x_ok(Kord)) {
    std::string full = Ls + Ms + Kord;
    // permute needs all labels incl. unit dims: append unit labels at the end
    std::string src(lx), dst = full;
    for (char ch : src)
      if (dst.find(ch) == std::string::npos) dst.push_back(ch);
    Xp = permute(c, X, lx, dst.c_str(), cx);
    Xu = &Xp;
    lxu = dst;
    oxu = make_op(Xp, dst.c_str(), false);
  }
  if (!views && !y_ok(Kord)) {
    std::string full = Ls + Kord + Ns;
    std::string src(ly), dst = full;
    for (char ch : src)
      if (dst.find(ch) == std::string::npos) dst.push_back(ch);
    Yp = permute(c, Y, ly, dst.c_str(), cy);
    Yu = &Yp;
    lyu = dst;
    oyu = make_op(Yp, dst.c_str(), false);
  }
  // output: GEMM writes [L][M][N]; permute afterwards if lout differs
  std::string gout = Ls + Ms + Ns;
  bool direct = (gout == out);
  Tensor C;
  std::vector<int> gshape;
  for (char ch : gout) gshape.push_back(dim[ch]);
  if (req) {
    // no complex64 output: the epilogue writes the consumer's planes (allocated below)
  } else if (direct) {
    C = new_tensor_n(c, oshape, per_out ? c.nb : 1);
  } else {
    C = new_tensor_n(c, gshape.empty() ? std::vector<int>{1} : gshape, per_out ? c.nb : 1);
  }
  if (!per_out) C.bstride = 0;
  if (req) C.bstride = Msz * Nsz;  // the planes hold the samples back to back, like a dense C

  GemmDesc g;
  g.M = (int)Msz;
  g.N = (int)Nsz;
  g.K = (int)Ksz;
  g.A = Xu->p;
  g.am = group_stride(oxu, Ms);
  g.ak = group_stride(oxu, Kord);
  g.conjA = (Xu == &X) ? cx : false;
  g.B = Yu->p;
  g.bk = group_stride(oyu, Kord);
  g.bn = group_stride(oyu, Ns);
  g.conjB = (Yu == &Y) ? cy : false;
  g.C = C.p;
  g.cm = Nsz;
  if (Ms.empty()) g.am = 0;
  if (Kord.empty()) { g.ak = 0; g.bk = 0; }
  if (Ns.empty()) g.bn = 0;
  int64_t lsx = group_stride(oxu, Ls), lsy = group_stride(oyu, Ls);
  g.nb2 = (int)Lsz;
  g.sa2 = Ls.empty() ? 0 : lsx;
  g.sb2 = Ls.empty() ? 0 : lsy;
  g.sc2 = Msz * Nsz;
  g.nb1 = per_out ? c.nb : 1;
  g.sa1 = Xu->bstride;
  g.sb1 = Yu->bstride;
  g.sc1 = C.bstride;
  g.work_per_sample = Msz * Nsz * Ksz * Lsz;
  g.m_per_sample = (int)Msz;
  if (Ksz == 0 || Msz == 0 || Nsz == 0) { zero(c, C, g.nb1); }
  if (views) {
    g.vam = gv.vam;
    g.vak = gv.vak;
    g.vbk = gv.vbk;
    g.vbn = gv.vbn;
    g.conjA = cx;
    g.conjB = cy;
    // fold the sample batch into M (outermost M axis) when Y is shared
    if (g.nb1 > 1 && Y.bstride == 0 && g.nb2 == 1 && g.vam.rank < 4 && C.bstride == Msz * g.cm) {
      for (int i = g.vam.rank; i > 0; --i) {
        g.vam.dims[i] = g.vam.dims[i - 1];
        g.vam.str[i] = g.vam.str[i - 1];
      }
      g.vam.dims[0] = g.nb1;
      g.vam.str[0] = X.bstride;
      g.vam.rank += 1;
      g.M = (int)(Msz * g.nb1);
      g.nb1 = 1;
    }
  } else if (g.nb1 > 1 && Yu->bstride == 0 && g.nb2 == 1 && (Ms.empty() ? false : Xu->bstride == Msz * g.am) &&
             C.bstride == Msz * g.cm) {
    // fold the sample batch into M when Y is shared
    g.M = (int)(Msz * g.nb1);
    g.nb1 = 1;
  }
  // operand / output magnitude bounds (tensor-core path): A's bound spares its row-max pass
  if (Xu == &X) {
    g.amaxA = tensor_amax(X, &g.amaxA_n);
    if (g.amaxA_n < (X.bstride ? c.nb : 1)) g.amaxA = nullptr;  // bounds of another batch
  }
  if (C.mem && !g.accumulate && tc_bounds_wanted()) {
    g.amaxC = C.mem->make_amax();
    g.amaxC_n = C.mem->tail_n;
  }
  if (req) return plane_output(c, g, *req, dim, Ls, Ms, Ns, out, per_out, Msz);
  const bool tc = gemm(c, g);
  if (!tc && C.mem) C.mem->drop_amax();
  if (direct) return C;
  std::string gl = gout.empty() ? std::string("?") : gout;
  // permute to requested order (including unit dims)
  std::string dst(lout), src = gl;
  for (char ch : dst)
    if (src.find(ch) == std::string::npos && gl != "?") src.push_back(ch);
  Tensor Ct = C;
  Ct.shape.clear();
  for (char ch : src) Ct.shape.push_back(dim.count(ch) ? dim[ch] : 1);
  if (gl == "?") { Ct.shape = oshape; return Ct; }
  Tensor R = permute(c, Ct, src.c_str(), dst.c_str(), false);
  if (C.mem && C.mem->amax() && R.mem && R.mem->tail && R.mem->tail_n >= C.mem->tail_n) {  // same values
    TN_CUDA(cudaMemcpyAsync(R.mem->tail, C.mem->tail, sizeof(float) * C.mem->tail_n, cudaMemcpyDeviceToDevice,
                            c.stream));
    R.mem->make_amax();
  }
  return R;
}

Tensor contract(Ctx& c, const Tensor& A, const char* la, bool conjA, const Tensor& B, const char* lb, bool conjB,
                const char* lout) {
  return contract_impl(c, A, la, conjA, B, lb, conjB, lout, nullptr);
}

Tensor contract_planes(Ctx& c, const Tensor& A, const char* la, bool conjA, const Tensor& B, const char* lb,
                       bool conjB, const char* lout, const char* zl, const char* rl, const char* kl) {
  PlaneReq r{zl, rl, kl};
  return contract_impl(c, A, la, conjA, B, lb, conjB, lout, &r);
}

}  // namespace tn

// Test-only: GEMMs that wrote their consumer's planes since the last reset (this thread).
extern "C" int64_t tn_debug_plane_gemms(int reset) {
  const int64_t n = tn::g_plane_gemms;
  if (reset) tn::g_plane_gemms = 0;
  return n;
}

extern "C" int tn_debug_simt_log(void) {
  std::vector<std::pair<double, std::string>> rows;
  for (auto& kv : tn::simt_tab()) rows.push_back({kv.second.second, kv.first});
  std::sort(rows.rbegin(), rows.rend());
  for (size_t i = 0; i < rows.size() && i < 25; ++i)
    fprintf(stderr, "SIMT %-50s n=%8.0f cmac=%.3e\n", rows[i].second.c_str(), tn::simt_tab()[rows[i].second].first,
            rows[i].first);
  return (int)rows.size();
}
