// tn.cu -- state, row partitions, norm-environment precompute, sampling, amplitudes and the
// C ABI of libtnsample (include/tnsample.h).
//
// Paper map (P:n = PAPER.md line n):
//   a0 validate + layout ........ P:97, P:275 (line partition), R1
//   a1 norm environments ........ P:112, P:279 (M_{b+1->b}, once per state)
//   a2 row product + compression  P:100, P:277, P:289-290 (n_b = Fit_R(m_{b-1} psi_b), R3)
//   a3 right ladder pass ........ P:289 ("one-site reduced density matrix")
//   a4 left pass + draw ......... P:289, P:293 (q = product of the conditionals), R9, R10
//   a5 project + merge .......... P:290, R14
//   a7 amplitude ................ P:85
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <map>
#include <memory>
#include <set>
#include <string>
#include <vector>

#include <nccl.h>

#include "../../include/tnsample.h"
#include "fit.h"
#include "kernels.h"
#include "tensor.h"

using namespace tn;

namespace {

thread_local std::string g_err;

struct VInfo {
  int b = -1, j = -1, up = -1, down = -1, left = -1, right = -1;
};

struct Envs {
  std::vector<std::vector<Tensor>> M;  // M[b]: norm MPS incident on row b from below (sites on down-edge vertices)
  std::vector<double> logs;
  bool ready = false;
};

struct Layout {
  std::vector<std::vector<int>> rows;
  std::vector<VInfo> info;
  std::vector<Tensor> A;   // [s,u,d,l,r] complex64, shared
  std::vector<Tensor> Bn;  // [u, 2*d, l, r] (n-fit column tensor), shared
  std::map<int, Envs> envs;  // by chi_env
};

}  // namespace

struct tn_state {
  int n = 0, n_edges = 0, chi = 0, device = 0;
  std::vector<std::pair<int, int>> edges;
  std::vector<int> bond;
  std::vector<std::vector<int>> inc;  // incident edge ids (increasing)
  std::vector<std::vector<double>> host;  // complex128 tensors (file layout)
  cudaStream_t stream = nullptr;
  Ctx ctx;
  int nh = 2;
  int order = 0;  // 0: compress-then-sample (R3); 1: the paper's literal order (NEXT-3)
  uint64_t seed = 0x2507114240ull;
  int64_t max_batch = 0;
  int64_t chunk_elems = 0;  // double-layer chunk budget override (0 = DStrip default)
  std::map<std::string, std::unique_ptr<Layout>> layouts;
  std::string cur_key;
  int64_t last_launches = 0;
  double last_precompute_s = 0;
};

namespace {

std::string row_key(const int32_t* row_ptr, const int32_t* rv, int n_rows) {
  std::string k;
  k.reserve((size_t)(n_rows + 1 + row_ptr[n_rows]) * 4);
  k.append(reinterpret_cast<const char*>(row_ptr), sizeof(int32_t) * (size_t)(n_rows + 1));
  k.append(reinterpret_cast<const char*>(rv), sizeof(int32_t) * (size_t)row_ptr[n_rows]);
  return k;
}

// R1: grid-layered line partition -- at most one up and one down edge per
// vertex, intra-row edges between consecutive vertices, non-crossing inter-row edges.
void analyse_rows(const tn_state* st, const int32_t* row_ptr, const int32_t* rv, int n_rows, Layout& L) {
  if (!row_ptr || !rv || n_rows < 1) throw Error(TN_E_ARG, "row order: NULL pointer or n_rows < 1");
  if (row_ptr[0] != 0 || row_ptr[n_rows] != st->n) throw Error(TN_E_ROWS, "row_ptr must start at 0 and end at n_vertices");
  L.rows.assign(n_rows, {});
  L.info.assign(st->n, VInfo{});
  std::vector<char> seen(st->n, 0);
  for (int b = 0; b < n_rows; ++b) {
    if (row_ptr[b + 1] <= row_ptr[b]) throw Error(TN_E_ROWS, "empty row");
    for (int i = row_ptr[b]; i < row_ptr[b + 1]; ++i) {
      int v = rv[i];
      if (v < 0 || v >= st->n || seen[v]) throw Error(TN_E_ROWS, "row order is not a permutation of the vertices");
      seen[v] = 1;
      L.info[v].b = b;
      L.info[v].j = i - row_ptr[b];
      L.rows[b].push_back(v);
    }
  }
  for (int e = 0; e < st->n_edges; ++e) {
    int u = st->edges[e].first, v = st->edges[e].second;
    VInfo &iu = L.info[u], &iv = L.info[v];
    if (iu.b == iv.b) {
      if (std::abs(iu.j - iv.j) != 1) throw Error(TN_E_ROWS, "intra-row edge between non-consecutive vertices");
      VInfo& lo = iu.j < iv.j ? iu : iv;
      VInfo& hi = iu.j < iv.j ? iv : iu;
      if (lo.right >= 0 || hi.left >= 0) throw Error(TN_E_ROWS, "duplicate intra-row edge");
      lo.right = e;
      hi.left = e;
    } else if (std::abs(iu.b - iv.b) == 1) {
      VInfo& top = iu.b < iv.b ? iu : iv;
      VInfo& bot = iu.b < iv.b ? iv : iu;
      if (top.down >= 0 || bot.up >= 0) throw Error(TN_E_ROWS, "vertex with more than one up or down edge");
      top.down = e;
      bot.up = e;
    } else {
      throw Error(TN_E_ROWS, "edge skips a row");
    }
  }
  for (int b = 0; b + 1 < n_rows; ++b) {
    int last = -1;
    for (int v : L.rows[b]) {
      int e = L.info[v].down;
      if (e < 0) continue;
      int o = st->edges[e].first == v ? st->edges[e].second : st->edges[e].first;
      if (L.info[o].j <= last) throw Error(TN_E_ROWS, "crossing inter-row edges");
      last = L.info[o].j;
    }
  }
}

// a0: permute the file legs (s, edges by id) to A_v[s,u,d,l,r], complex128 -> complex64.
void build_layout(tn_state* st, Layout& L) {
  Ctx& c = st->ctx;
  c.nb = 1;
  L.A.resize(st->n);
  L.Bn.resize(st->n);
  for (int v = 0; v < st->n; ++v) {
    const VInfo& I = L.info[v];
    int keys[4] = {I.up, I.down, I.left, I.right};
    int dims[5] = {2, 1, 1, 1, 1};
    int64_t fstride[5] = {0, 0, 0, 0, 0};
    const auto& inc = st->inc[v];
    // strides in the file layout (2, d_e1, d_e2, ...)
    std::vector<int64_t> fs(inc.size() + 1);
    int64_t acc = 1;
    for (int i = (int)inc.size(); i >= 1; --i) {
      fs[i] = acc;
      acc *= st->bond[inc[i - 1]];
    }
    fs[0] = acc;
    fstride[0] = fs[0];
    for (int q = 0; q < 4; ++q) {
      if (keys[q] < 0) continue;
      int pos = (int)(std::find(inc.begin(), inc.end(), keys[q]) - inc.begin());
      dims[q + 1] = st->bond[keys[q]];
      fstride[q + 1] = fs[pos + 1];
    }
    int64_t total = 2LL * dims[1] * dims[2] * dims[3] * dims[4];
    std::vector<float2> a(total), bn(total);
    const double* src = st->host[v].data();
    int64_t idx = 0;
    for (int s = 0; s < 2; ++s)
      for (int u = 0; u < dims[1]; ++u)
        for (int d = 0; d < dims[2]; ++d)
          for (int l = 0; l < dims[3]; ++l)
            for (int r = 0; r < dims[4]; ++r, ++idx) {
              int64_t off = s * fstride[0] + u * fstride[1] + d * fstride[2] + l * fstride[3] + r * fstride[4];
              float2 val = make_float2((float)src[2 * off], (float)src[2 * off + 1]);
              a[idx] = val;
              // Bn[u][s*D + d][l][r]
              int64_t bi = (((int64_t)u * (2 * dims[2]) + (s * dims[2] + d)) * dims[3] + l) * dims[4] + r;
              bn[bi] = val;
            }
    L.A[v] = new_tensor(c, {2, dims[1], dims[2], dims[3], dims[4]}, false);
    L.Bn[v] = new_tensor(c, {dims[1], 2 * dims[2], dims[3], dims[4]}, false);
    TN_CUDA(cudaMemcpyAsync(L.A[v].p, a.data(), total * sizeof(float2), cudaMemcpyHostToDevice, c.stream));
    TN_CUDA(cudaMemcpyAsync(L.Bn[v].p, bn.data(), total * sizeof(float2), cudaMemcpyHostToDevice, c.stream));
  }
  TN_CUDA(cudaStreamSynchronize(c.stream));
}

Layout& get_layout(tn_state* st, const int32_t* row_ptr, const int32_t* rv, int n_rows) {
  if (!row_ptr || !rv) throw Error(TN_E_ARG, "row order: NULL pointer");
  if (n_rows < 1) throw Error(TN_E_ARG, "n_rows < 1");
  std::string key = row_key(row_ptr, rv, n_rows);
  auto it = st->layouts.find(key);
  if (it != st->layouts.end()) {
    st->cur_key = key;
    return *it->second;
  }
  auto L = std::make_unique<Layout>();
  analyse_rows(st, row_ptr, rv, n_rows, *L);
  build_layout(st, *L);
  Layout& ref = *L;
  st->layouts[key] = std::move(L);
  st->cur_key = key;
  return ref;
}

bool has(const Layout& L, int v, int key) {
  const VInfo& I = L.info[v];
  return (key == 0 ? I.up : I.down) >= 0;
}

// tops for a row: sites of an incoming MPS on the columns with an edge `key` (0 = up, 1 = down)
void place_tops(const Layout& L, int b, const std::vector<Tensor>* mps, int key, DStrip& s) {
  const auto& row = L.rows[b];
  s.tops.assign(row.size(), Tensor{});
  s.topbond.assign(row.size(), 1);
  int k = 0, bond = 1;
  for (size_t j = 0; j < row.size(); ++j) {
    s.topbond[j] = bond;
    if (mps && has(L, row[j], key)) {
      const Tensor& t = (*mps)[k++];
      s.tops[j] = t;
      bond = t.shape.back();
    }
  }
  if (mps && k != (int)mps->size()) throw Error(TN_E_ROWS, "incoming boundary MPS does not match the row");
}

// a1 / O4: M_{N_b} trivial; M_{b -> b-1} = Fit_R(M_{b+1->b} T_b), b = N_b .. 2
Envs& norm_envs(tn_state* st, Layout& L, int R) {
  auto it = L.envs.find(R);
  if (it != L.envs.end() && it->second.ready) return it->second;
  auto t0 = std::chrono::steady_clock::now();
  Ctx& c = st->ctx;
  c.nb = 1;
  Envs& E = L.envs[R];
  int nbr = (int)L.rows.size();
  E.M.assign(nbr, {});
  E.logs.assign(nbr, 0.0);
  DevBuf logd(sizeof(double) * nbr, c.stream);
  TN_CUDA(cudaMemsetAsync(logd.p, 0, sizeof(double) * nbr, c.stream));
  // TN_PRE_ROWS=k (profiling only): stop after the k bottom-most fits; the environments are
  // then incomplete and not marked ready.
  const char* lim_s = getenv("TN_PRE_ROWS");
  const int lim = lim_s ? std::atoi(lim_s) : -1;
  for (int b = nbr - 1; b >= 1; --b) {
    if (lim >= 0 && nbr - 1 - b >= lim) {
      TN_CUDA(cudaStreamSynchronize(c.stream));
      st->last_precompute_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      return E;
    }
    DStrip s;
    s.dbl = true;
    s.per_sample = false;
    s.W = (int)L.rows[b].size();
    if (st->chunk_elems > 0) s.chunk_elems = st->chunk_elems;
    place_tops(L, b, E.M[b].empty() ? nullptr : &E.M[b], 1, s);
    for (int v : L.rows[b]) {
      s.mats.push_back(L.A[v]);
      s.out.push_back(has(L, v, 0));
    }
    // TN_FAKE_ENVS=1 (profiling the per-sample path at full shapes only): structural shapes,
    // hash values, no fit -- the samples drawn are meaningless.
    static const bool fake = getenv("TN_FAKE_ENVS") && std::atoi(getenv("TN_FAKE_ENVS")) != 0;
    FitResult fr = fake ? fake_fit(c, s, R, 2, b + 1, st->seed)
                        : fit(c, s, R, 2, b + 1, st->seed, st->nh, logd.as<double>() + (b - 1), false);
    E.M[b - 1] = fr.sites;
  }
  TN_CUDA(cudaMemcpyAsync(E.logs.data(), logd.p, sizeof(double) * nbr, cudaMemcpyDeviceToHost, c.stream));
  TN_CUDA(cudaStreamSynchronize(c.stream));
  for (int b = 0; b + 1 < nbr; ++b)
    if (!std::isfinite(E.logs[b])) {
      L.envs.erase(R);
      throw Error(TN_E_NUMERIC, "non-finite norm environment at row " + std::to_string(b + 2));
    }
  E.ready = true;
  st->last_precompute_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return E;
}

Tensor viewt(const Tensor& t, std::vector<int> shape) {
  Tensor v = t;
  v.shape = std::move(shape);
  return v;
}

// per-sample bytes estimate for batch sizing (ladder intermediates dominate)
int64_t per_sample_bytes(const Layout& L, int R, int chi) {
  int64_t worst = 0;
  for (const auto& row : L.rows) {
    int64_t rs = 0, y = 0;
    for (size_t j = 0; j < row.size(); ++j) {
      int64_t D = std::min<int64_t>(R, 4LL * chi * chi);
      int64_t dd = L.A[row[j]].shape[2];
      int64_t f = std::min<int64_t>(R, chi * chi);
      y = std::max(y, D * 2 * dd * f * D);
      rs += 2 * D * f * D;
    }
    worst = std::max(worst, 5 * y + rs);
  }
  return worst * 8 + (64LL << 20);
}

// O5 for one batch of nb samples (device outputs).
// pa_log / pa_phase (optional, device [nb]): ln|a| and arg a of the amplitude carried along
// the sampling path (m_{N_b-1 -> N_b} . X_{N_b}; p(x) = |a|^2 when the fits
// are (near) exact): the n-fits' log-norms, the merge normalisations and the final scalar.
// Whether a ladder GEMM (Y2 = Y1 . M_j or G2 = G1 . M_j) can write its closure's A planes
// directly (contract_planes): rows = rbond x ebond (the closure's M, a whole number of CTA-pair
// tiles), inner K = kbond = whole scale blocks (multiples of 128 complex: a CTA tile's 128 rows
// are one block), a down edge (d > 1), tensor-core GEMMs.
// TN_LADDER_PLANES=0 disables it, =1 keeps only the G2 / Y2 planes, =2 adds G1 (A/B measurements).
bool ladder_planes_ok(const Ctx& c, int rbond, int ebond, int d, int kbond) {
  static const bool off = getenv("TN_LADDER_PLANES") && std::atoi(getenv("TN_LADDER_PLANES")) == 0;
  if (off || c.gemm_mode == 1 || ebond <= 1 || d <= 1 || kbond % 128 != 0) return false;
  const int64_t rows = (int64_t)rbond * ebond;
  return rows % 256 == 0 && rows > 128 && ((int64_t)ebond * d) % 128 == 0 &&
         tc_eligible(c, (int64_t)rbond * 2 * kbond, (int64_t)ebond * d, (int64_t)d * ebond,
                     (int64_t)rbond * 2 * kbond * ebond * d * d * ebond);
}

// Whether Y1 = n_j . R (M = (a, s, d), N = (Z, f), K = z) can write Y2's A planes (rows (a, s, Z),
// K = (f, d)): d = 32 is a warp's rows, 4 adjacent f complete a scale block (plane mode 2).
bool y1_planes_ok(const Ctx& c, int a, int d, int f, int Z) {
  static const bool off = getenv("TN_LADDER_PLANES") && std::atoi(getenv("TN_LADDER_PLANES")) < 3;
  if (off || c.gemm_mode == 1 || d != 32 || f % 4 != 0 || a <= 1) return false;
  const int64_t rows = (int64_t)a * 2 * Z;
  return rows % 256 == 0 && ((int64_t)a * 2 * d) % 256 == 0 && ((int64_t)Z * f) % 128 == 0;
}

// Whether G1 = Lx . n_j[x] (M = (A, e), N = (d, z), K = a) can write G2's A planes (rows (z, A),
// K = (d, e)): e is whole scale blocks, whole CTA-pair tiles, a down edge.
bool g1_planes_ok(const Ctx& c, int e, int A, int d, int z) {
  static const bool off = getenv("TN_LADDER_PLANES") && std::atoi(getenv("TN_LADDER_PLANES")) < 2;
  if (off || c.gemm_mode == 1 || e % 128 != 0 || d <= 1 || A <= 1) return false;
  const int64_t rows = (int64_t)z * A;
  return rows % 256 == 0 && ((int64_t)A * e) % 256 == 0 && ((int64_t)d * z) % 128 == 0;
}

void sample_batch(tn_state* st, Layout& L, Envs& E, int R, int nb, const double* u_dev, uint8_t* bits_dev,
                  double* logq_dev, double* cond_dev, uint32_t* flags_dev, double* pa_log = nullptr,
                  double* pa_phase = nullptr) {
  Ctx& c = st->ctx;
  c.nb = nb;
  int N = st->n;
  TN_CUDA(cudaMemsetAsync(logq_dev, 0, sizeof(double) * nb, c.stream));
  TN_CUDA(cudaMemsetAsync(flags_dev, 0, sizeof(uint32_t) * nb, c.stream));
  DevBuf xbuf(sizeof(int) * nb, c.stream);
  if (pa_log) {
    TN_CUDA(cudaMemsetAsync(pa_log, 0, sizeof(double) * nb, c.stream));
    TN_CUDA(cudaMemsetAsync(pa_phase, 0, sizeof(double) * nb, c.stream));
  }
  std::vector<Tensor> m_prev;
  bool have_prev = false;
  g_row_cmacs.assign(L.rows.size(), 0.0);
  for (int b = 0; b < (int)L.rows.size(); ++b) {
    const double cm0 = g_cmacs;
    struct RowCount {
      int b;
      double c0;
      ~RowCount() { g_row_cmacs[b] = g_cmacs - c0; }
    } row_count{b, cm0};
    const auto& row = L.rows[b];
    int W = (int)row.size();
    // a2: n_b = Fit_R(m_{b-1} psi_b), (s, d) open at every vertex
    DStrip s;
    s.dbl = false;
    s.per_sample = true;
    s.W = W;
    place_tops(L, b, have_prev ? &m_prev : nullptr, 0, s);
    for (int v : row) {
      s.mats.push_back(L.Bn[v]);
      s.out.push_back(true);
    }
    FitResult fr = fit(c, s, R, 1, b + 1, st->seed, st->nh, pa_log, pa_log != nullptr);
    for (int j = 0; j < W; ++j) nan_check(c, ("n site row " + std::to_string(b) + " j " + std::to_string(j)).c_str(), fr.sites[j], nb);
    std::vector<Tensor> n(W);
    for (int j = 0; j < W; ++j) {
      const Tensor& o = fr.sites[j];
      int dd = L.A[row[j]].shape[2];
      n[j] = viewt(o, {o.shape[0], 2, dd, o.shape[2]});
    }
    // M sites for this row (norm MPS from below), identity where no down edge
    DStrip ms;
    place_tops(L, b, E.M[b].empty() ? nullptr : &E.M[b], 1, ms);
    // a3: right pass
    std::vector<Tensor> Rs(W);
    Tensor Rr = ones(c, {1, 1, 1}, nb);
    for (int j = W - 1; j >= 0; --j) {
      if (ladder_planes_ok(c, n[j].shape[0], ms.tops[j].p ? ms.tops[j].shape[0] : 0, n[j].shape[2], n[j].shape[3]) &&
          y1_planes_ok(c, n[j].shape[0], n[j].shape[2], Rr.shape[1], Rr.shape[2])) {
        // Y1 = n_j . R writes Y2's A planes (rows (a, s, Z), K = (f, d): blocks of a warp's 32 d
        // x 4 f), Y2 = Y1 . M_j (planes in) writes the closure's (rows (a, e) per (sample, s),
        // K = (D, Z)): the right pass has no complex64 ladder intermediate and no operand prep
        Tensor Y1p = contract_planes(c, n[j], "asdz", false, Rr, "zfZ", false, "asdZf", "", "asZ", "fd");
        Tensor Y2p = contract_planes(c, Y1p, "asZfd", false, ms.tops[j], "edDf", false, "asZeD", "s", "ae", "DZ");
        Rs[j] = contract(c, Y2p, "saeDZ", false, n[j], "AsDZ", true, "saeA");
      } else if (ladder_planes_ok(c, n[j].shape[0], ms.tops[j].p ? ms.tops[j].shape[0] : 0, n[j].shape[2],
                                  n[j].shape[3])) {
        // Y2 = Y1 . M_j written by its GEMM straight into the FP16 A planes of the closure
        // Rs = Y2 . conj(n_j) (rows (a, e) per (sample, s), K = (D, Z)): no complex64 Y2 and no
        // operand prep for the closure
        Tensor Y1 = contract(c, n[j], "asdz", false, Rr, "zfZ", false, "asdfZ");
        Tensor Y2p = contract_planes(c, Y1, "asdfZ", false, ms.tops[j], "edDf", false, "asZeD", "s", "ae", "DZ");
        Rs[j] = contract(c, Y2p, "saeDZ", false, n[j], "AsDZ", true, "saeA");
      } else {
        Tensor Y1 = contract(c, n[j], "asdz", false, Rr, "zfZ", false, "asdfZ");
        Tensor Y2;
        if (ms.tops[j].p) Y2 = contract(c, Y1, "asdfZ", false, ms.tops[j], "edDf", false, "asZeD");
        else Y2 = permute(c, Y1, "asdfZ", "asZfd");  // identity: e = f, d = D = 1
        Rs[j] = contract(c, Y2, "asZeD", false, n[j], "AsDZ", true, "saeA");
      }
      nan_check(c, ("Rs row " + std::to_string(b) + " j " + std::to_string(j)).c_str(), Rs[j], nb);
      if (j > 0) {
        Rr = sum2(c, Rs[j]);
        normalize(c, Rr, nb, nullptr, false);  // any positive rescale (R13)
      }
    }
    // a4: left pass + draw
    Tensor Lx = ones(c, {1, 1, 1}, nb);
    std::vector<Tensor> proj(W);
    for (int j = 0; j < W; ++j) {
      int v = row[j];
      TailOut to{xbuf.as<int>(), bits_dev, logq_dev, cond_dev, flags_dev, u_dev, N, v};
      tail_draw(c, Lx, Rs[j], nb, to);
      Rs[j] = Tensor{};
      Tensor nx = select_s(c, n[j], xbuf.as<int>(), nb);
      proj[j] = nx;
      if (j + 1 < W) {
        if (ladder_planes_ok(c, nx.shape[2], ms.tops[j].p ? ms.tops[j].shape[3] : 0, nx.shape[1], nx.shape[0]) &&
            g1_planes_ok(c, Lx.shape[1], Lx.shape[2], nx.shape[1], nx.shape[2])) {
          // G1 = Lx . n_j[x] into the A planes of G2 (rows (z, A), K = (d, e)), G2 = G1 . M_j
          // into the A planes of Lx = G2 . conj(n_j[x]) (rows (z, f), K = (D, A)): neither
          // intermediate exists in complex64 and neither GEMM preps its A operand
          Tensor G1p = contract_planes(c, Lx, "aeA", false, nx, "adz", false, "Aedz", "", "zA", "de");
          Tensor G2p = contract_planes(c, G1p, "zAde", false, ms.tops[j], "edDf", false, "zADf", "", "zf", "DA");
          Lx = contract(c, G2p, "zfDA", false, nx, "ADZ", true, "zfZ");
        } else if (ladder_planes_ok(c, nx.shape[2], ms.tops[j].p ? ms.tops[j].shape[3] : 0, nx.shape[1],
                                    nx.shape[0])) {
          // G2 = G1 . M_j straight into the A planes of Lx = G2 . conj(n_j[x]) (rows (z, f),
          // K = (D, A))
          Tensor G1 = contract(c, Lx, "aeA", false, nx, "adz", false, "eAdz");
          Tensor G2p = contract_planes(c, G1, "eAdz", false, ms.tops[j], "edDf", false, "zADf", "", "zf", "DA");
          Lx = contract(c, G2p, "zfDA", false, nx, "ADZ", true, "zfZ");
        } else {
          Tensor G1 = contract(c, Lx, "aeA", false, nx, "adz", false, "eAdz");
          Tensor G2;
          if (ms.tops[j].p) G2 = contract(c, G1, "eAdz", false, ms.tops[j], "edDf", false, "AzDf");
          else G2 = permute(c, G1, "eAdz", "Azde");  // identity: f = e, d = D = 1
          Lx = contract(c, G2, "AzDf", false, nx, "ADZ", true, "zfZ");
        }
        nan_check(c, ("Lx pre-norm row " + std::to_string(b) + " j " + std::to_string(j)).c_str(), Lx, nb);
        normalize(c, Lx, nb, nullptr, false);
        nan_check(c, ("Lx row " + std::to_string(b) + " j " + std::to_string(j)).c_str(), Lx, nb);
      }
    }
    // a5: m_b = merge(n_b[x_b]) -- vertices without a down edge are multiplied into the
    // nearest down-edge site to the right, else to the left (R14); normalise.
    std::vector<int> downs;
    for (int j = 0; j < W; ++j)
      if (has(L, row[j], 1)) downs.push_back(j);
    m_prev.clear();
    have_prev = !downs.empty();
    if (downs.empty() && pa_log) {  // the boundary contraction ends in a scalar
      Tensor t = viewt(proj[0], {proj[0].shape[0], proj[0].shape[2]});
      for (int i = 1; i < W; ++i) {
        Tensor mat = viewt(proj[i], {proj[i].shape[0], proj[i].shape[2]});
        t = contract(c, t, "ab", false, mat, "bc", false, "ac");
      }
      scalar_logphase(c, t, nb, pa_log, pa_phase);
    }
    int prev = -1;
    for (size_t k = 0; k < downs.size(); ++k) {
      int j = downs[k];
      Tensor t = proj[j];
      for (int i = j - 1; i > prev; --i) {
        Tensor mat = viewt(proj[i], {proj[i].shape[0], proj[i].shape[2]});
        t = contract(c, mat, "ab", false, t, "bdz", false, "adz");
      }
      if (k + 1 == downs.size())
        for (int i = j + 1; i < W; ++i) {
          Tensor mat = viewt(proj[i], {proj[i].shape[0], proj[i].shape[2]});
          t = contract(c, t, "adz", false, mat, "zy", false, "ady");
        }
      normalize(c, t, nb, pa_log, pa_log != nullptr);
      m_prev.push_back(t);
      prev = j;
    }
  }
}

// Identity "top" for a column without an incoming MPS site: [bond, 1, bond] (single layer)
// or [bond, 1, 1, bond] (double layer), shared by all samples.
Tensor identity_top(Ctx& c, int bond, bool dbl) {
  std::vector<float2> h((size_t)bond * bond, make_float2(0.f, 0.f));
  for (int i = 0; i < bond; ++i) h[(size_t)i * bond + i] = make_float2(1.f, 0.f);
  Tensor t = new_tensor(c, dbl ? std::vector<int>{bond, 1, 1, bond} : std::vector<int>{bond, 1, bond}, false);
  TN_CUDA(cudaMemcpyAsync(t.p, h.data(), h.size() * sizeof(float2), cudaMemcpyHostToDevice, c.stream));
  TN_CUDA(cudaStreamSynchronize(c.stream));  // h is a host temporary
  return t;
}

// NEXT-3 for one batch (oracle sample_literal): the paper's literal order
// (PAPER.md:289-290). Row b is sampled from the five-layer ladder m_{b-1}.psi_b.conj(psi_b).
// conj(m_{b-1}).M_{b+1->b} (right env [b, r, R, B, f]: m bond, ket / bra row bond, conj(m)
// bond, M bond), then m_b = Fit_R(m_{b-1}.X_b), X_b = x_b.psi_b with the down legs open
// (tag 4). Same tail (draw, clamp, ln q) as O5. Feasible where R <= chi (the paper's runs):
// the environment has R_x^2 R_n chi^2 entries.
void sample_batch_literal(tn_state* st, Layout& L, Envs& E, int R, int nb, const double* u_dev, uint8_t* bits_dev,
                          double* logq_dev, double* cond_dev, uint32_t* flags_dev) {
  Ctx& c = st->ctx;
  c.nb = nb;
  int N = st->n;
  TN_CUDA(cudaMemsetAsync(logq_dev, 0, sizeof(double) * nb, c.stream));
  TN_CUDA(cudaMemsetAsync(flags_dev, 0, sizeof(uint32_t) * nb, c.stream));
  DevBuf xbuf(sizeof(int) * nb, c.stream);
  std::vector<Tensor> m_prev;
  bool have_prev = false;
  for (int b = 0; b < (int)L.rows.size(); ++b) {
    const auto& row = L.rows[b];
    const int W = (int)row.size();
    DStrip ms, Ms;
    place_tops(L, b, have_prev ? &m_prev : nullptr, 0, ms);
    place_tops(L, b, E.M[b].empty() ? nullptr : &E.M[b], 1, Ms);
    std::vector<Tensor> mj(W), Mj(W);
    for (int j = 0; j < W; ++j) {
      mj[j] = ms.tops[j].p ? ms.tops[j] : identity_top(c, ms.topbond[j], false);
      Mj[j] = Ms.tops[j].p ? Ms.tops[j] : identity_top(c, Ms.topbond[j], true);
    }
    // right pass: Rs[j][s, a, l, L, A, e]
    std::vector<Tensor> Rs(W);
    Tensor Rr = ones(c, {1, 1, 1, 1, 1}, nb);
    for (int j = W - 1; j >= 0; --j) {
      const Tensor& A = L.A[row[j]];
      Tensor T1 = contract(c, Rr, "brRBf", false, mj[j], "aub", false, "rRBfau");
      Tensor T2 = contract(c, T1, "rRBfau", false, A, "sudlr", false, "RBfasdl");
      Tensor T3 = contract(c, T2, "RBfasdl", false, Mj[j], "edDf", false, "RBasleD");
      Tensor T4 = contract(c, T3, "RBasleD", false, A, "sUDLR", true, "sBaleUL");
      Rs[j] = contract(c, T4, "sBaleUL", false, mj[j], "AUB", true, "salLAe");
      if (j > 0) {
        Rr = sum2(c, Rs[j]);
        normalize(c, Rr, nb, nullptr, false);
      }
    }
    // left pass + draw
    Tensor Lx = ones(c, {1, 1, 1, 1, 1}, nb);
    std::vector<Tensor> Ax(W);
    for (int j = 0; j < W; ++j) {
      const int v = row[j];
      TailOut to{xbuf.as<int>(), bits_dev, logq_dev, cond_dev, flags_dev, u_dev, N, v};
      tail_draw(c, Lx, Rs[j], nb, to);
      Rs[j] = Tensor{};
      Ax[j] = gather_bit(c, L.A[v], bits_dev, N, v, nb);  // A_v[x_v] = [u, d, l, r] per sample
      if (j + 1 < W) {
        Tensor G1 = contract(c, Lx, "alLAe", false, mj[j], "aub", false, "lLAeub");
        Tensor G2 = contract(c, G1, "lLAeub", false, Ax[j], "udlr", false, "LAebdr");
        Tensor G3 = contract(c, G2, "LAebdr", false, Mj[j], "edDf", false, "LAbrDf");
        Tensor G4 = contract(c, G3, "LAbrDf", false, Ax[j], "UDLR", true, "AbrfUR");
        Lx = contract(c, G4, "AbrfUR", false, mj[j], "AUB", true, "brRBf");
        normalize(c, Lx, nb, nullptr, false);
      }
    }
    // m_b = Fit_R(m_{b-1} . X_b), down legs open
    if (b + 1 < (int)L.rows.size()) {
      DStrip s;
      s.dbl = false;
      s.per_sample = true;
      s.W = W;
      place_tops(L, b, have_prev ? &m_prev : nullptr, 0, s);
      for (int j = 0; j < W; ++j) {
        s.mats.push_back(Ax[j]);
        s.out.push_back(has(L, row[j], 1));
      }
      FitResult fr = fit(c, s, R, 4, b + 1, st->seed, st->nh, nullptr, false);
      m_prev = fr.sites;
      have_prev = !m_prev.empty();
    }
  }
}

// O6 for one batch: ln|<x|psi>| and phase.
void amplitude_batch(tn_state* st, Layout& L, int R, int nb, const uint8_t* bits_dev, double* logabs,
                     double* phase) {
  Ctx& c = st->ctx;
  c.nb = nb;
  DevBuf logn(sizeof(double) * nb, c.stream);
  TN_CUDA(cudaMemsetAsync(logn.p, 0, sizeof(double) * nb, c.stream));
  std::vector<Tensor> m_prev;
  bool have_prev = false;
  for (int b = 0; b < (int)L.rows.size(); ++b) {
    const auto& row = L.rows[b];
    DStrip s;
    s.dbl = false;
    s.per_sample = true;
    s.W = (int)row.size();
    place_tops(L, b, have_prev ? &m_prev : nullptr, 0, s);
    for (int v : row) {
      s.mats.push_back(gather_bit(c, L.A[v], bits_dev, st->n, v, nb));  // A_v[x_v] = [u,d,l,r]
      s.out.push_back(has(L, v, 1));
    }
    FitResult fr = fit(c, s, R, 3, b + 1, st->seed, st->nh, logn.as<double>(), true);
    if (fr.sites.empty()) {
      std::vector<float2> sc;
      scalars_to_host(c, fr.scalar, nb, sc);
      std::vector<double> ln(nb), sl(nb);
      TN_CUDA(cudaMemcpyAsync(ln.data(), logn.p, sizeof(double) * nb, cudaMemcpyDeviceToHost, c.stream));
      TN_CUDA(cudaMemcpyAsync(sl.data(), fr.scalar_log->p, sizeof(double) * nb, cudaMemcpyDeviceToHost, c.stream));
      TN_CUDA(cudaStreamSynchronize(c.stream));
      for (int k = 0; k < nb; ++k) {
        double a = std::hypot((double)sc[k].x, (double)sc[k].y);
        logabs[k] = a > 0 ? ln[k] + sl[k] + std::log(a) : -INFINITY;
        phase[k] = std::atan2((double)sc[k].y, (double)sc[k].x);
      }
      return;
    }
    m_prev = fr.sites;
    have_prev = true;
  }
  throw Error(TN_E_ROWS, "last row has down edges");
}

int choose_batch(tn_state* st, Layout& L, int R, int64_t n) {
  if (st->max_batch > 0) return (int)std::min<int64_t>(n, st->max_batch);
  size_t fr = 0, tot = 0;
  TN_CUDA(cudaMemGetInfo(&fr, &tot));
  int64_t per = per_sample_bytes(L, R, st->chi);
  int64_t nbmax = std::max<int64_t>(1, (int64_t)(0.6 * (double)fr) / per);
  return (int)std::min<int64_t>({n, nbmax, 65535});
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return TN_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "host out of memory";
    return TN_E_NOMEM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return TN_E_CUDA;
  }
}

void use_device(tn_state* st) { TN_CUDA(cudaSetDevice(st->device)); }

void sample_common(tn_state* st, const int32_t* row_ptr, const int32_t* rv, int32_t n_rows, int32_t chi_env,
                   int64_t n_samples, const double* u, bool u_on_device, uint8_t* bits, double* logp, double* cond,
                   uint32_t* flags, bool out_on_device, cudaStream_t user_stream, double* pa_log = nullptr,
                   double* pa_phase = nullptr) {
  if (!st) throw Error(TN_E_ARG, "state is NULL");
  if (n_samples <= 0) throw Error(TN_E_ARG, "n_samples must be > 0");
  if (chi_env < 1) throw Error(TN_E_ARG, "chi_env must be >= 1");
  if (!u || !bits || !logp) throw Error(TN_E_ARG, "NULL uniforms or output pointer");
  use_device(st);
  int N = st->n;
  if (!u_on_device) {
    for (int64_t i = 0; i < n_samples * N; ++i)
      if (!(u[i] >= 0.0 && u[i] < 1.0)) throw Error(TN_E_ARG, "uniform not finite or outside [0,1)");
  }
  int64_t l0 = g_launches;
  Layout& L = get_layout(st, row_ptr, rv, n_rows);
  Envs& E = norm_envs(st, L, chi_env);
  cudaStream_t saved = st->ctx.stream;
  if (user_stream) st->ctx.stream = user_stream;
  Ctx& c = st->ctx;
  try {
    int64_t done = 0;
    while (done < n_samples) {
      int nb = choose_batch(st, L, chi_env, n_samples - done);
      DevBuf ub, bb, lb, cb, fb;
      const double* ud;
      uint8_t* bd;
      double *ld, *cd;
      uint32_t* fd;
      if (u_on_device) {
        ud = u + done * N;
      } else {
        ub.alloc(sizeof(double) * nb * N, c.stream);
        TN_CUDA(cudaMemcpyAsync(ub.p, u + done * N, sizeof(double) * nb * N, cudaMemcpyHostToDevice, c.stream));
        ud = ub.as<double>();
      }
      if (out_on_device) {
        bd = bits + done * N;
        ld = logp + done;
        cd = cond ? cond + done * N : nullptr;
        if (flags) {
          fd = flags + done;
        } else {
          fb.alloc(sizeof(uint32_t) * nb, c.stream);
          fd = fb.as<uint32_t>();
        }
      } else {
        bb.alloc((size_t)nb * N, c.stream);
        lb.alloc(sizeof(double) * nb, c.stream);
        fb.alloc(sizeof(uint32_t) * nb, c.stream);
        if (cond) cb.alloc(sizeof(double) * nb * N, c.stream);
        bd = bb.as<uint8_t>();
        ld = lb.as<double>();
        fd = fb.as<uint32_t>();
        cd = cond ? cb.as<double>() : nullptr;
      }
      DevBuf pal, pap;  // path amplitudes (host outputs only)
      if (pa_log) {
        if (out_on_device || st->order == 1) throw Error(TN_E_ARG, "path amplitudes: host outputs, order 0 only");
        pal.alloc(sizeof(double) * nb, c.stream);
        pap.alloc(sizeof(double) * nb, c.stream);
      }
      if (st->order == 1) sample_batch_literal(st, L, E, chi_env, nb, ud, bd, ld, cd, fd);
      else sample_batch(st, L, E, chi_env, nb, ud, bd, ld, cd, fd, pa_log ? pal.as<double>() : nullptr,
                        pa_log ? pap.as<double>() : nullptr);
      if (pa_log) {
        TN_CUDA(cudaMemcpyAsync(pa_log + done, pal.p, sizeof(double) * nb, cudaMemcpyDeviceToHost, c.stream));
        TN_CUDA(cudaMemcpyAsync(pa_phase + done, pap.p, sizeof(double) * nb, cudaMemcpyDeviceToHost, c.stream));
      }
      if (!out_on_device) {
        TN_CUDA(cudaMemcpyAsync(bits + done * N, bd, (size_t)nb * N, cudaMemcpyDeviceToHost, c.stream));
        TN_CUDA(cudaMemcpyAsync(logp + done, ld, sizeof(double) * nb, cudaMemcpyDeviceToHost, c.stream));
        if (flags) TN_CUDA(cudaMemcpyAsync(flags + done, fd, sizeof(uint32_t) * nb, cudaMemcpyDeviceToHost, c.stream));
        if (cond) TN_CUDA(cudaMemcpyAsync(cond + done * N, cd, sizeof(double) * nb * N, cudaMemcpyDeviceToHost, c.stream));
        TN_CUDA(cudaStreamSynchronize(c.stream));
      }
      done += nb;
    }
  } catch (...) {
    st->ctx.stream = saved;
    throw;
  }
  st->ctx.stream = saved;
  if (user_stream && user_stream != st->stream) {
    // the library frees its cached buffers (environments, layouts) on st->stream: order those
    // frees after the kernels just queued on the caller's stream
    cudaEvent_t ev;
    TN_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    TN_CUDA(cudaEventRecord(ev, user_stream));
    TN_CUDA(cudaStreamWaitEvent(st->stream, ev, 0));
    TN_CUDA(cudaEventDestroy(ev));
  }
  st->last_launches = g_launches - l0;
}

}  // namespace

extern "C" {

const char* tn_last_error(void) { return g_err.c_str(); }

int tn_load_state(const tn_graph* g, const double* const* tensors, int32_t chi, tn_state** out) {
  return guarded([&] {
    if (!g || !tensors || !out) throw Error(TN_E_ARG, "NULL argument");
    *out = nullptr;
    if (g->n_vertices < 1 || g->n_edges < 0) throw Error(TN_E_ARG, "n_vertices must be >= 1");
    if (g->n_edges > 0 && (!g->edges || !g->bond_dims)) throw Error(TN_E_ARG, "NULL edges / bond_dims");
    if (chi < 1) throw Error(TN_E_ARG, "chi must be >= 1");
    auto st = std::make_unique<tn_state>();
    st->n = g->n_vertices;
    st->n_edges = g->n_edges;
    st->chi = chi;
    st->inc.assign(st->n, {});
    std::set<std::pair<int, int>> seen;
    for (int e = 0; e < g->n_edges; ++e) {
      int u = g->edges[2 * e], v = g->edges[2 * e + 1];
      if (u < 0 || v < 0 || u >= st->n || v >= st->n) throw Error(TN_E_GRAPH, "edge vertex id out of range");
      if (u == v) throw Error(TN_E_GRAPH, "self-loop");
      auto key = std::make_pair(std::min(u, v), std::max(u, v));
      if (!seen.insert(key).second) throw Error(TN_E_GRAPH, "duplicate edge");
      int d = g->bond_dims[e];
      if (d < 1 || d > chi) throw Error(TN_E_GRAPH, "bond dimension outside [1, chi]");
      st->edges.push_back({u, v});
      st->bond.push_back(d);
      st->inc[u].push_back(e);
      st->inc[v].push_back(e);
    }
    st->host.resize(st->n);
    for (int v = 0; v < st->n; ++v) {
      if (!tensors[v]) throw Error(TN_E_ARG, "NULL tensor pointer");
      int64_t sz = 2;
      for (int e : st->inc[v]) sz *= st->bond[e];
      st->host[v].assign(tensors[v], tensors[v] + 2 * sz);
    }
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) throw Error(TN_E_CUDA, "no CUDA device");
    TN_CUDA(cudaGetDevice(&st->device));
    {
      // keep freed blocks in the stream-ordered pool across synchronisations (the default
      // release threshold of 0 returns GBs of intermediates to the OS at every sync)
      cudaMemPool_t pool;
      TN_CUDA(cudaDeviceGetDefaultMemPool(&pool, st->device));
      uint64_t thr = UINT64_MAX;
      TN_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    }
    TN_CUDA(cudaStreamCreateWithFlags(&st->stream, cudaStreamNonBlocking));
    st->ctx.stream = st->stream;
    st->ctx.guess_cache = std::make_shared<std::map<std::string, std::vector<Tensor>>>();
    if (const char* gm = getenv("TN_GEMM")) st->ctx.gemm_mode = std::atoi(gm);  // debugging override
    *out = st.release();
  });
}

int tn_comm_unique_id(uint8_t* out_id) {
  return guarded([&] {
    if (!out_id) throw Error(TN_E_ARG, "NULL argument");
    static_assert(sizeof(ncclUniqueId) == TN_COMM_ID_BYTES, "NCCL unique id size");
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) throw Error(TN_E_NCCL, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
    std::memcpy(out_id, &id, sizeof id);
  });
}

int tn_set_comm(tn_state* st, const uint8_t* id, int32_t rank, int32_t world) {
  return guarded([&] {
    if (!st || !id) throw Error(TN_E_ARG, "NULL argument");
    if (world < 1 || rank < 0 || rank >= world) throw Error(TN_E_ARG, "rank must be in [0, world)");
    use_device(st);
    if (st->ctx.comm) {
      ncclCommDestroy(reinterpret_cast<ncclComm_t>(st->ctx.comm));
      st->ctx.comm = nullptr;
    }
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof uid);
    ncclComm_t comm;
    ncclResult_t r = ncclCommInitRank(&comm, world, uid, rank);
    if (r != ncclSuccess) throw Error(TN_E_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    st->ctx.comm = comm;
    st->ctx.rank = rank;
    st->ctx.world = world;
  });
}

int tn_free_state(tn_state* st) {
  return guarded([&] {
    if (!st) return;
    cudaSetDevice(st->device);
    cudaStreamSynchronize(st->stream);
    if (st->ctx.comm) ncclCommDestroy(reinterpret_cast<ncclComm_t>(st->ctx.comm));
    st->layouts.clear();
    if (st->ctx.guess_cache) {  // built on whatever stream sampled first: free on the state's own
      cudaDeviceSynchronize();
      for (auto& kv : *st->ctx.guess_cache)
        for (auto& t : kv.second)
          if (t.mem) t.mem->s = st->stream;
      st->ctx.guess_cache->clear();
    }
    cudaStreamSynchronize(st->stream);
    cudaStreamDestroy(st->stream);
    delete st;
  });
}

int tn_set_option(tn_state* st, const char* name, int64_t value) {
  return guarded([&] {
    if (!st || !name) throw Error(TN_E_ARG, "NULL argument");
    std::string k(name);
    if (k == "fit_half_sweeps") {
      if (value < 1) throw Error(TN_E_ARG, "fit_half_sweeps must be >= 1");
      st->nh = (int)value;
    } else if (k == "init_seed") {
      st->seed = (uint64_t)value;
    } else if (k == "gemm") {
      if (value < 0 || value > 2) throw Error(TN_E_ARG, "gemm must be 0, 1 or 2");
      st->ctx.gemm_mode = (int)value;
    } else if (k == "order") {
      if (value < 0 || value > 1) throw Error(TN_E_ARG, "order must be 0 (compress-then-sample) or 1 (literal)");
      st->order = (int)value;
      return;
    } else if (k == "max_batch") {
      st->max_batch = value;
      return;
    } else if (k == "chunk_elems") {
      if (value < 0) throw Error(TN_E_ARG, "chunk_elems must be >= 0");
      st->chunk_elems = value;
    } else {
      throw Error(TN_E_ARG, "unknown option " + k);
    }
    for (auto& kv : st->layouts) kv.second->envs.clear();
  });
}

int tn_prepare(tn_state* st, const int32_t* row_ptr, const int32_t* row_vertices, int32_t n_rows, int32_t chi_env) {
  return guarded([&] {
    if (!st) throw Error(TN_E_ARG, "state is NULL");
    if (chi_env < 1) throw Error(TN_E_ARG, "chi_env must be >= 1");
    use_device(st);
    int64_t l0 = g_launches;
    Layout& L = get_layout(st, row_ptr, row_vertices, n_rows);
    norm_envs(st, L, chi_env);
    st->last_launches = g_launches - l0;
  });
}

int tn_sample(tn_state* st, const int32_t* row_ptr, const int32_t* row_vertices, int32_t n_rows, int32_t chi_env,
              int64_t n_samples, const double* uniforms, uint8_t* out_bits, double* out_logp) {
  return guarded([&] {
    sample_common(st, row_ptr, row_vertices, n_rows, chi_env, n_samples, uniforms, false, out_bits, out_logp,
                  nullptr, nullptr, false, nullptr);
  });
}

int tn_sample_ex(tn_state* st, const int32_t* row_ptr, const int32_t* row_vertices, int32_t n_rows, int32_t chi_env,
                 int64_t n_samples, int64_t sample_offset, const double* uniforms, uint8_t* out_bits,
                 double* out_logp, double* out_cond, uint32_t* out_flags) {
  (void)sample_offset;
  return guarded([&] {
    if (sample_offset < 0) throw Error(TN_E_ARG, "sample_offset < 0");
    sample_common(st, row_ptr, row_vertices, n_rows, chi_env, n_samples, uniforms, false, out_bits, out_logp,
                  out_cond, out_flags, false, nullptr);
  });
}

int tn_sample_path(tn_state* st, const int32_t* row_ptr, const int32_t* row_vertices, int32_t n_rows,
                   int32_t chi_env, int64_t n_samples, const double* uniforms, uint8_t* out_bits, double* out_logq,
                   double* out_logabs, double* out_phase) {
  return guarded([&] {
    if (!out_logabs || !out_phase) throw Error(TN_E_ARG, "NULL path-amplitude output");
    sample_common(st, row_ptr, row_vertices, n_rows, chi_env, n_samples, uniforms, false, out_bits, out_logq,
                  nullptr, nullptr, false, nullptr, out_logabs, out_phase);
  });
}

int tn_sample_dev(tn_state* st, const int32_t* row_ptr, const int32_t* row_vertices, int32_t n_rows, int32_t chi_env,
                  int64_t n_samples, const double* uniforms_dev, uint8_t* out_bits_dev, double* out_logp_dev,
                  double* out_cond_dev, uint32_t* out_flags_dev, void* stream) {
  return guarded([&] {
    if (!st) throw Error(TN_E_ARG, "state is NULL");
    Layout* L = nullptr;
    {
      std::string key = (row_ptr && row_vertices && n_rows >= 1) ? row_key(row_ptr, row_vertices, n_rows) : "";
      auto it = st->layouts.find(key);
      if (it == st->layouts.end()) throw Error(TN_E_ROWS, "tn_sample_dev requires tn_prepare for this row order");
      L = it->second.get();
      auto e = L->envs.find(chi_env);
      if (e == L->envs.end() || !e->second.ready) throw Error(TN_E_ROWS, "tn_sample_dev requires tn_prepare for chi_env");
    }
    sample_common(st, row_ptr, row_vertices, n_rows, chi_env, n_samples, uniforms_dev, true, out_bits_dev,
                  out_logp_dev, out_cond_dev, out_flags_dev, true, (cudaStream_t)stream);
  });
}

int tn_amplitude(tn_state* st, const uint8_t* bits, int64_t n, int32_t chi_env, double* out_logabs, double* out_phase) {
  return guarded([&] {
    if (!st || !bits || !out_logabs || !out_phase) throw Error(TN_E_ARG, "NULL argument");
    if (n <= 0) throw Error(TN_E_ARG, "n must be > 0");
    if (chi_env < 1) throw Error(TN_E_ARG, "chi_env must be >= 1");
    auto it = st->layouts.find(st->cur_key);
    if (st->cur_key.empty() || it == st->layouts.end()) throw Error(TN_E_ROWS, "no row order prepared");
    for (int64_t i = 0; i < n * st->n; ++i)
      if (bits[i] > 1) throw Error(TN_E_ARG, "bits must be 0 or 1");
    use_device(st);
    int64_t l0 = g_launches;
    Layout& L = *it->second;
    Ctx& c = st->ctx;
    int64_t done = 0;
    while (done < n) {
      int nb = choose_batch(st, L, chi_env, n - done);
      DevBuf bd((size_t)nb * st->n, c.stream);
      TN_CUDA(cudaMemcpyAsync(bd.p, bits + done * st->n, (size_t)nb * st->n, cudaMemcpyHostToDevice, c.stream));
      amplitude_batch(st, L, chi_env, nb, bd.as<uint8_t>(), out_logabs + done, out_phase + done);
      done += nb;
    }
    st->last_launches = g_launches - l0;
  });
}

int tn_log_norm(tn_state* st, int32_t chi_env, double* out_lognorm) {
  return guarded([&] {
    if (!st || !out_lognorm) throw Error(TN_E_ARG, "NULL argument");
    auto it = st->layouts.find(st->cur_key);
    if (st->cur_key.empty() || it == st->layouts.end()) throw Error(TN_E_ROWS, "no row order prepared");
    use_device(st);
    Layout& L = *it->second;
    Envs& E = norm_envs(st, L, chi_env);
    Ctx& c = st->ctx;
    c.nb = 1;
    DStrip s;
    s.dbl = true;
    s.per_sample = false;
    s.W = (int)L.rows[0].size();
    place_tops(L, 0, E.M[0].empty() ? nullptr : &E.M[0], 1, s);
    for (int v : L.rows[0]) {
      s.mats.push_back(L.A[v]);
      s.out.push_back(false);
    }
    FitResult fr = fit(c, s, 1, 2, 1, st->seed, st->nh, nullptr, false);
    std::vector<float2> sc;
    scalars_to_host(c, fr.scalar, 1, sc);
    double sl = 0;
    TN_CUDA(cudaMemcpy(&sl, fr.scalar_log->p, sizeof(double), cudaMemcpyDeviceToHost));
    double tot = sl;
    for (double x : E.logs) tot += x;
    *out_lognorm = std::log(std::hypot((double)sc[0].x, (double)sc[0].y)) + tot;
  });
}

int tn_certify(tn_state* st, const uint8_t* bits, const double* logq, int64_t n, int32_t chi_env_verify,
               double log_z, double* out_logp, tn_cert_stats* out) {
  return guarded([&] {
    if (!st || !bits || !logq || !out) throw Error(TN_E_ARG, "NULL argument");
    if (n <= 0) throw Error(TN_E_ARG, "n must be > 0");
    std::vector<double> la(n), ph(n), lp(n);
    int rc = tn_amplitude(st, bits, n, chi_env_verify, la.data(), ph.data());
    if (rc != TN_OK) throw Error(rc, g_err);
    for (int64_t k = 0; k < n; ++k) lp[k] = 2.0 * la[k];
    Ctx& c = st->ctx;
    DevBuf dq(sizeof(double) * n, c.stream), dp(sizeof(double) * n, c.stream), ds(sizeof(double) * 8, c.stream);
    TN_CUDA(cudaMemcpyAsync(dq.p, logq, sizeof(double) * n, cudaMemcpyHostToDevice, c.stream));
    TN_CUDA(cudaMemcpyAsync(dp.p, lp.data(), sizeof(double) * n, cudaMemcpyHostToDevice, c.stream));
    cert_stats(c, dq.as<double>(), dp.as<double>(), n, log_z, ds.as<double>());
    double h[8];
    TN_CUDA(cudaMemcpyAsync(h, ds.p, sizeof h, cudaMemcpyDeviceToHost, c.stream));
    TN_CUDA(cudaStreamSynchronize(c.stream));
    out->log_norm_estimate = h[0];
    out->norm_rel_stderr = h[1];
    out->kld = h[2];
    out->ess = h[3];
    out->n_used = (int64_t)h[4];
    out->n_excluded = (int64_t)h[5];
    if (out_logp) std::copy(lp.begin(), lp.end(), out_logp);
  });
}

int tn_observables(const uint8_t* bits, const double* logq, const double* logp, int64_t n, int32_t n_vertices,
                   const int32_t* group_of, int32_t n_groups, const int32_t* target_ones, double* out_z_weighted,
                   double* out_z_plain, double* out_pass_rate, double* out_pass_rate_weighted) {
  return guarded([&] {
    if (!bits || !logq || !logp || !out_z_weighted || !out_z_plain || !out_pass_rate)
      throw Error(TN_E_ARG, "NULL argument");
    if (n <= 0 || n_vertices < 1) throw Error(TN_E_ARG, "n and n_vertices must be > 0");
    if (n_groups < 0 || n_groups > 8 || (n_groups > 0 && (!group_of || !target_ones)))
      throw Error(TN_E_ARG, "n_groups must be in [0, 8] with group_of and target_ones given");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) throw Error(TN_E_CUDA, "no CUDA device");
    Ctx c;
    TN_CUDA(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
    struct StreamGuard {
      cudaStream_t s;
      ~StreamGuard() { cudaStreamDestroy(s); }
    } sg{c.stream};
    const int N = n_vertices;
    {
      DevBuf db((size_t)n * N, c.stream), dq(sizeof(double) * n, c.stream), dp(sizeof(double) * n, c.stream);
      DevBuf dw(sizeof(double) * n, c.stream), dpass(sizeof(double) * n, c.stream);
      DevBuf ds(sizeof(double) * 3 * (N + 1), c.stream), dg(sizeof(int) * N, c.stream), dt(sizeof(int) * 8, c.stream);
      TN_CUDA(cudaMemcpyAsync(db.p, bits, (size_t)n * N, cudaMemcpyHostToDevice, c.stream));
      TN_CUDA(cudaMemcpyAsync(dq.p, logq, sizeof(double) * n, cudaMemcpyHostToDevice, c.stream));
      TN_CUDA(cudaMemcpyAsync(dp.p, logp, sizeof(double) * n, cudaMemcpyHostToDevice, c.stream));
      if (n_groups > 0) {
        TN_CUDA(cudaMemcpyAsync(dg.p, group_of, sizeof(int) * N, cudaMemcpyHostToDevice, c.stream));
        TN_CUDA(cudaMemcpyAsync(dt.p, target_ones, sizeof(int) * n_groups, cudaMemcpyHostToDevice, c.stream));
      }
      observables(c, db.as<uint8_t>(), dq.as<double>(), dp.as<double>(), n, N, n_groups ? dg.as<int>() : nullptr,
                  n_groups, dt.as<int>(), dw.as<double>(), dpass.as<double>(), ds.as<double>());
      std::vector<double> h(3 * (N + 1));
      TN_CUDA(cudaMemcpyAsync(h.data(), ds.p, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, c.stream));
      TN_CUDA(cudaStreamSynchronize(c.stream));
      for (int v = 0; v < N; ++v) {
        out_z_weighted[v] = h[3 * v + 2] > 0 ? h[3 * v] / h[3 * v + 2] : NAN;
        out_z_plain[v] = h[3 * v + 1] / (double)n;
      }
      *out_pass_rate = h[3 * N] / (double)n;
      if (out_pass_rate_weighted) *out_pass_rate_weighted = h[3 * N + 2] > 0 ? h[3 * N + 1] / h[3 * N + 2] : NAN;
    }
    TN_CUDA(cudaStreamSynchronize(c.stream));
  });
}

int tn_get_stats(tn_state* st, int64_t* out_launches, double* out_precompute_s) {
  return guarded([&] {
    if (!st) throw Error(TN_E_ARG, "state is NULL");
    if (out_launches) *out_launches = st->last_launches;
    if (out_precompute_s) *out_precompute_s = st->last_precompute_s;
  });
}

}  // extern "C"
