// fit.cu -- one-site MPS-MPO fitting on the device (see fit.h).
//
// Follows O3 step by step (restated in DESIGN.md): hash init (R4), right-
// orthonormalisation as a true gauge transformation, right environments, nh alternating
// half-sweeps replacing each site by the derivative of <o|T> and
// re-orthonormalising it (exact D_k columns, R6/R7), the turning site not recomputed,
// final centre normalised.
#include <algorithm>
#include <cstdio>

#include <nccl.h>

#include "fit.h"
#include "kernels.h"
#include "linalg.h"

namespace tn {
namespace {

Tensor view(const Tensor& t, std::vector<int> shape) {
  Tensor v = t;
  v.shape = std::move(shape);
  return v;
}

Tensor slice_rows(const Tensor& t, int x0, int x1) {
  Tensor v = t;
  int64_t row = t.size() / t.shape[0];
  v.p = t.p + x0 * row;
  v.shape[0] = x1 - x0;
  return v;
}

int row_bond(const DStrip& s, int j) { return s.dbl ? s.mats[j].shape[3] : s.mats[j].shape[2]; }

int p_dim(const DStrip& s, int j) {
  if (s.dbl) return s.mats[j].shape[1] * s.mats[j].shape[1];
  return s.mats[j].shape[1];
}

std::vector<int> o_shape(const DStrip& s, int j, int dl, int dr) {
  if (s.dbl) return {dl, s.mats[j].shape[1], s.mats[j].shape[1], dr};
  return {dl, s.mats[j].shape[1], dr};
}

struct Ops {
  Ctx& c;
  const DStrip& s;
  int nb() const { return s.per_sample ? c.nb : 1; }
  Tensor trivial() {
    Tensor t = ones(c, s.dbl ? std::vector<int>{1, 1, 1, 1} : std::vector<int>{1, 1, 1}, nb());
    if (!s.per_sample) t.bstride = 0;  // shared: every derived tensor stays shared
    return t;
  }

  // ---------------- single layer
  // mid1(L, j) is needed twice in a left-to-right sweep step (the derivative at k, then the
  // new left environment from the orthonormalised site): the last result is kept, keyed by
  // L's memory (held alive, so the address cannot be recycled meanwhile) and the column.
  Tensor mid1_X;
  std::shared_ptr<DevBuf> mid1_Lmem;
  const float2* mid1_Lp = nullptr;
  int mid1_j = -1;
  Tensor mid1(const Tensor& L, int j) {
    if (mid1_Lmem && L.mem == mid1_Lmem && L.p == mid1_Lp && j == mid1_j) return mid1_X;
    mid1_X = mid1_compute(L, j);
    mid1_Lmem = L.mem;
    mid1_Lp = L.p;
    mid1_j = j;
    return mid1_X;
  }
  Tensor mid1_compute(const Tensor& L, int j) {
    const Tensor& B = s.mats[j];
    if (s.tops[j].p) {
      Tensor X1 = contract(c, L, "xmy", false, s.tops[j], "mun", false, "xyun");
      return contract(c, X1, "xyun", false, B, "upyr", false, "xnpr");
    }
    return contract(c, L, "xny", false, B, "upyr", false, "xnpr");
  }

  // rmid1(F, j) = F . (column j): the right-hand mirror of mid1, [z, m, p, y]. In a
  // right-to-left half-sweep it serves both the derivative at j (L . Z) and, after the
  // orthonormalisation, the new right environment (Z . conj(o)), so the column is
  // contracted once per site instead of twice (mid1 for the derivative, then the chain of
  // absorb_right).
  Tensor rmid1_Z;
  std::shared_ptr<DevBuf> rmid1_Fmem;
  const float2* rmid1_Fp = nullptr;
  int rmid1_j = -1;
  Tensor rmid1(const Tensor& F, int j) {
    if (rmid1_Fmem && F.mem == rmid1_Fmem && F.p == rmid1_Fp && j == rmid1_j) return rmid1_Z;
    const Tensor& B = s.mats[j];
    if (s.tops[j].p) {
      Tensor Z1 = contract(c, F, "znr", false, s.tops[j], "mun", false, "zrmu");
      rmid1_Z = contract(c, Z1, "zrmu", false, B, "upyr", false, "zmpy");
    } else {
      rmid1_Z = contract(c, F, "zmr", false, B, "upyr", false, "zmpy");  // identity top: n = m, u = 1
    }
    rmid1_Fmem = F.mem;
    rmid1_Fp = F.p;
    rmid1_j = j;
    return rmid1_Z;
  }
  bool rmid1_cached(const Tensor& F, int j) const {
    return rmid1_Fmem && F.mem == rmid1_Fmem && F.p == rmid1_Fp && j == rmid1_j;
  }

  // ---------------- double layer, rows [x0,x1) of the output-bond index
  Tensor mid2(const Tensor& L, int j, int x0, int x1) {
    const Tensor& A = s.mats[j];
    Tensor Lc = slice_rows(L, x0, x1);
    Tensor X2;
    if (s.tops[j].p) {
      Tensor X1 = contract(c, Lc, "xeab", false, s.tops[j], "edDf", false, "xabdDf");
      X2 = contract(c, X1, "xabdDf", false, A, "sudar", false, "xbDfsur");
    } else {
      X2 = contract(c, Lc, "xfab", false, A, "sudar", false, "xbDfsur");
    }
    return contract(c, X2, "xbDfsur", false, A, "sUDbR", true, "xfurUR");
  }

  // Double-layer chunk loops. fn(x0, x1) returns the part of chunk
  // [x0, x1). concat: the parts are rows x0..x1-1 of a tensor of shape `shape`; else the result
  // is the sum of the parts (shape `shape`) in chunk order. With a communicator (Ctx::comm)
  // chunk ci is computed by rank ci % world only and broadcast from it; every rank then
  // assembles the same bits in the same order as one GPU does (no reduction across ranks).
  template <class Fn>
  Tensor chunked(int nx, int step, bool concat, const std::vector<int>& shape, Fn fn) {
    const int nch = (nx + step - 1) / step;
    ncclComm_t comm = reinterpret_cast<ncclComm_t>(c.comm);
    if (!comm) {  // one GPU
      Tensor out;
      for (int x0 = 0; x0 < nx; x0 += step) {
        const int x1 = std::min(nx, x0 + step);
        Tensor part = fn(x0, x1);
        if (concat) {
          if (nch == 1) return part;
          if (!out.p) out = new_tensor(c, shape, false);
          copy_rows(c, part, out, x0, 1);
        } else {
          if (!out.p) out = part;
          else add_into(c, out, part, 1);
        }
      }
      return out;
    }
    auto nccl = [](ncclResult_t r) {
      if (r != ncclSuccess) throw Error(-6, std::string("NCCL: ") + ncclGetErrorString(r));
    };
    if (concat) {
      Tensor out = new_tensor(c, shape, false);
      const int64_t row = out.size() / shape[0];
      for (int ci = 0; ci < nch; ++ci) {
        const int x0 = ci * step, x1 = std::min(nx, x0 + step);
        if (ci % c.world == c.rank) copy_rows(c, fn(x0, x1), out, x0, 1);
      }
      invalidate_amax(out);
      nccl(ncclGroupStart());
      for (int ci = 0; ci < nch; ++ci) {
        const int x0 = ci * step, x1 = std::min(nx, x0 + step);
        float* p = reinterpret_cast<float*>(out.p + (int64_t)x0 * row);
        nccl(ncclBroadcast(p, p, (size_t)(x1 - x0) * row * 2, ncclFloat, ci % c.world, comm, c.stream));
      }
      nccl(ncclGroupEnd());
      return out;
    }
    std::vector<Tensor> parts(nch);
    for (int ci = 0; ci < nch; ++ci) {
      const int x0 = ci * step, x1 = std::min(nx, x0 + step);
      if (ci % c.world == c.rank) parts[ci] = fn(x0, x1);
      else parts[ci] = new_tensor(c, shape, false);
      invalidate_amax(parts[ci]);
    }
    nccl(ncclGroupStart());
    for (int ci = 0; ci < nch; ++ci) {
      float* p = reinterpret_cast<float*>(parts[ci].p);
      nccl(ncclBroadcast(p, p, (size_t)parts[ci].size() * 2, ncclFloat, ci % c.world, comm, c.stream));
    }
    nccl(ncclGroupEnd());
    Tensor out = parts[0];
    for (int ci = 1; ci < nch; ++ci) add_into(c, out, parts[ci], 1);
    return out;
  }

  int chunk_rows(int j, int nx) {
    const Tensor& A = s.mats[j];
    int64_t u = A.shape[1], d = A.shape[2], l = A.shape[3], r = A.shape[4];
    int64_t f = s.tops[j].p ? s.tops[j].shape[3] : s.topbond[j];
    int64_t per = std::max({l * l * d * d * f, 2 * l * d * f * u * r, f * u * u * r * r, f * r * r * u * u});
    int64_t rows = std::max<int64_t>(1, s.chunk_elems / std::max<int64_t>(1, per));
    return (int)std::min<int64_t>(rows, nx);
  }

  Tensor absorb_left(const Tensor& L, int j, const Tensor* o) {
    if (!s.dbl) {
      if (!o) {  // the result becomes an environment that is rescaled in place: not cached
        Tensor X = mid1_compute(L, j);
        return view(X, {X.shape[0], X.shape[1], X.shape[3]});
      }
      Tensor X = mid1(L, j);
      return contract(c, X, "xnpr", false, *o, "xpz", true, "znr");
    }
    const int nx = L.shape[0];
    const int step = chunk_rows(j, nx);
    const int f = s.tops[j].p ? s.tops[j].shape[3] : L.shape[1];
    const int r = s.mats[j].shape[4];
    if (!o)  // non-output column: u = U = 1, rows x of [x, f, r, R]
      return chunked(nx, step, true, {nx, f, r, r}, [&](int x0, int x1) {
        Tensor X = mid2(L, j, x0, x1);
        return view(X, {X.shape[0], X.shape[1], X.shape[3], X.shape[5]});
      });
    return chunked(nx, step, false, {o->shape[3], f, r, r}, [&](int x0, int x1) {
      Tensor X = mid2(L, j, x0, x1);
      Tensor oc = slice_rows(*o, x0, x1);
      return contract(c, X, "xfurUR", false, oc, "xuUz", true, "zfrR");
    });
  }

  // d = d<o|T>/d conj(o_j) = L . (column j) . F, contracted from the left
  // (mid1 / mid2).
  Tensor derivative(const Tensor& L, int j, const Tensor& F) {
    if (!s.dbl) {
      Tensor X = mid1(L, j);
      return contract(c, X, "xnpr", false, F, "znr", false, "xpz");
    }
    const int nx = L.shape[0];
    const int step = chunk_rows(j, nx);
    const int u = s.mats[j].shape[1];
    return chunked(nx, step, true, {nx, u, u, F.shape[0]}, [&](int x0, int x1) {
      Tensor X = mid2(L, j, x0, x1);
      return contract(c, X, "xfurUR", false, F, "zfrR", false, "xuUz");
    });
  }

  // The single-layer derivative contracted from the right (rmid1), for right-to-left
  // half-sweeps: the same Z then gives the new right environment (absorb_right).
  Tensor derivative_right(const Tensor& L, int j, const Tensor& F) {
    Tensor Z = rmid1(F, j);
    // Z (the large operand, produced by a tensor-core GEMM with its scale bounds) as the A side
    return contract(c, Z, "zmpy", false, L, "xmy", false, "xpz");
  }

  Tensor absorb_right(const Tensor& F, int j, const Tensor* o) {
    if (!s.dbl) {
      if (o && rmid1_cached(F, j)) return contract(c, rmid1_Z, "zmpy", false, *o, "xpz", true, "xmy");
      const Tensor& B = s.mats[j];
      Tensor Y2;
      if (o) {
        Tensor Y1 = contract(c, F, "znr", false, *o, "xpz", true, "nrxp");
        Y2 = contract(c, Y1, "nrxp", false, B, "upyr", false, "nxuy");
      } else {
        Y2 = contract(c, F, "xnr", false, B, "upyr", false, "nxuy");
      }
      if (s.tops[j].p) return contract(c, Y2, "nxuy", false, s.tops[j], "mun", false, "xmy");
      Tensor Y2v = view(Y2, {Y2.shape[0], Y2.shape[1], Y2.shape[3]});
      return permute(c, Y2v, "nxy", "xny");
    }
    const Tensor& A = s.mats[j];
    const int nx = o ? o->shape[0] : F.shape[0];
    const int step = chunk_rows(j, nx);
    const int e = s.tops[j].p ? s.tops[j].shape[0] : F.shape[1];
    const int l = A.shape[3];
    return chunked(nx, step, true, {nx, e, l, l}, [&](int x0, int x1) {
      Tensor Y2;
      if (o) {
        Tensor oc = slice_rows(*o, x0, x1);
        Tensor Y1 = contract(c, F, "zfrR", false, oc, "xuUz", true, "frRxuU");
        Y2 = contract(c, Y1, "frRxuU", false, A, "sudar", false, "fRxUsda");
      } else {
        Tensor Fc = slice_rows(F, x0, x1);  // non-output column: u = U = 1
        Y2 = contract(c, Fc, "xfrR", false, A, "sudar", false, "fRxUsda");
      }
      Tensor Y3 = contract(c, Y2, "fRxUsda", false, A, "sUDbR", true, "fxdaDb");
      if (s.tops[j].p) return contract(c, Y3, "fxdaDb", false, s.tops[j], "edDf", false, "xeab");
      Tensor Y3v = view(Y3, {Y3.shape[0], Y3.shape[1], Y3.shape[3], Y3.shape[5]});
      return permute(c, Y3v, "fxab", "xfab");
    });
  }
};

}  // namespace
bool nan_check_on() {
  static int on = -1;
  if (on < 0) on = getenv("TN_NAN_CHECK") ? 1 : 0;
  return on == 1;
}
void nan_check(Ctx& c, const char* what, const Tensor& t, int nb) {
  if (!nan_check_on()) return;
  int n = t.bstride ? nb : 1;
  for (int b = 0; b < n; ++b) {
    int64_t k = count_nonfinite(c, t.p + b * t.bstride, t.size());
    if (k) fprintf(stderr, "NAN_CHECK %s: sample %d/%d has %lld non-finite of %lld\n", what, b, n, (long long)k,
                   (long long)t.size());
  }
}

namespace {
// column span of o reshaped (prod(shape[:-1])) x shape[-1]
Tensor left_orth(Ctx& c, const Tensor& o, int nb) {
  Tensor q = new_tensor_n(c, o.shape, nb);
  if (!o.bstride) q.bstride = 0;
  int n = o.shape.back();
  int m = (int)(o.size() / n);
  MatView X{o.p, o.bstride, n, 1, false, m, n};
  MatView Q{q.p, q.bstride, n, 1, false, m, n};
  nan_check(c, "left_orth in", o, nb);
  orthonormalize(c, X, Q, nullptr, o.bstride ? nb : 1);
  nan_check(c, "left_orth out", q, nb);
  return q;
}

// row span of o reshaped shape[0] x (rest); optional C with o = C^H-factor (see linalg.h)
Tensor right_orth(Ctx& c, const Tensor& o, int nb, Tensor* Cout) {
  Tensor q = new_tensor_n(c, o.shape, nb);
  if (!o.bstride) q.bstride = 0;
  int dl = o.shape[0];
  int rest = (int)(o.size() / dl);
  MatView X{o.p, o.bstride, 1, rest, true, rest, dl};
  MatView Q{q.p, q.bstride, 1, rest, true, rest, dl};
  float2* cp = nullptr;
  if (Cout) {
    *Cout = new_tensor_n(c, {dl, dl}, nb);
    if (!o.bstride) Cout->bstride = 0;
    cp = Cout->p;
  }
  nan_check(c, "right_orth in", o, nb);
  orthonormalize(c, X, Q, cp, o.bstride ? nb : 1);
  nan_check(c, "right_orth out", q, nb);
  if (Cout) nan_check(c, "right_orth C", *Cout, nb);
  return q;
}

}  // namespace

std::vector<int> fit_bonds(const DStrip& s, int R) {
  std::vector<int> cols;
  for (int j = 0; j < s.W; ++j)
    if (s.out[j]) cols.push_back(j);
  int K = (int)cols.size();
  std::vector<int64_t> D(K + 1, 1);
  for (int k = 1; k < K; ++k) {
    int64_t cut = INT64_MAX;
    for (int j = cols[k - 1] + 1; j <= cols[k]; ++j) {
      int64_t r = row_bond(s, j);
      int64_t cd = (int64_t)s.topbond[j] * (s.dbl ? r * r : r);
      cut = std::min(cut, cd);
    }
    D[k] = std::min<int64_t>(R, cut);
  }
  std::vector<int64_t> p(K);
  for (int k = 0; k < K; ++k) p[k] = p_dim(s, cols[k]);
  for (int k = 1; k < K; ++k) D[k] = std::min(D[k], D[k - 1] * p[k - 1]);
  for (int k = K - 1; k >= 1; --k) D[k] = std::min(D[k], p[k] * D[k + 1]);
  return std::vector<int>(D.begin(), D.end());
}

// Profiling aid only (TN_FAKE_ENVS): the output sites of the fit with their structural shapes,
// filled with the hash initial guess and normalised, without fitting.
FitResult fake_fit(Ctx& c, const DStrip& s, int R, int tag, int b1, uint64_t seed) {
  FitResult res;
  std::vector<int> cols;
  for (int j = 0; j < s.W; ++j)
    if (s.out[j]) cols.push_back(j);
  std::vector<int> D = fit_bonds(s, R);
  for (size_t k = 0; k < cols.size(); ++k) {
    Tensor o = new_tensor_n(c, o_shape(s, cols[k], D[k], D[k + 1]), 1);
    o.bstride = 0;
    hash_init(c, o, 1, seed, tag, b1, (int)k);
    normalize(c, o, 1, nullptr, false);
    res.sites.push_back(o);
  }
  return res;
}

FitResult fit(Ctx& c, const DStrip& s, int R, int tag, int b1, uint64_t seed, int nh, double* logn,
              bool accumulate) {
  Ops ops{c, s};
  int nb = ops.nb();
  FitResult res;
  std::vector<int> cols;
  for (int j = 0; j < s.W; ++j)
    if (s.out[j]) cols.push_back(j);
  int K = (int)cols.size();
  // Environments are rescaled to unit norm after every absorbed column (any positive rescale
  // is allowed, R13); their accumulated ln-scales (per sample) keep the returned log-norms
  // exact. This keeps long double-layer rows inside the FP32 range.
  struct Env {
    Tensor t;
    std::shared_ptr<DevBuf> lg;  // double[nb]
  };
  auto fresh_log = [&]() {
    auto p = std::make_shared<DevBuf>(sizeof(double) * nb, c.stream);
    TN_CUDA(cudaMemsetAsync(p->p, 0, sizeof(double) * nb, c.stream));
    return p;
  };
  auto rescaled = [&](Tensor t, const Env& parent) {
    Env e;
    e.t = t;
    e.lg = std::make_shared<DevBuf>(sizeof(double) * nb, c.stream);
    TN_CUDA(cudaMemcpyAsync(e.lg->p, parent.lg->p, sizeof(double) * nb, cudaMemcpyDeviceToDevice, c.stream));
    normalize(c, e.t, nb, e.lg->as<double>(), true);
    return e;
  };
  auto trivial_env = [&]() { return Env{ops.trivial(), fresh_log()}; };
  if (K == 0) {
    Env L = trivial_env();
    for (int j = 0; j < s.W; ++j) L = rescaled(ops.absorb_left(L.t, j, nullptr), L);
    res.scalar = L.t;
    res.scalar_log = L.lg;
    return res;
  }
  std::vector<int> D = fit_bonds(s, R);
  std::vector<Tensor> o(K);
  // the shared initial guess of a single-layer fit, right-orthonormalised, from the state's
  // cache when an earlier batch already built it (bitwise the same tensors)
  std::string gkey;
  bool guess_done = false;
  if (!s.dbl && c.guess_cache) {
    gkey = std::to_string(seed) + "/" + std::to_string(tag) + "/" + std::to_string(b1);
    for (int k = 0; k < K; ++k)
      for (int d : o_shape(s, cols[k], D[k], D[k + 1])) gkey += "," + std::to_string(d);
    auto it = c.guess_cache->find(gkey);
    if (it != c.guess_cache->end()) {
      o = it->second;
      guess_done = true;
    }
  }
  for (int k = 0; k < K && !guess_done; ++k) {
    // the initial guess does not depend on the sample (R4: the hash key is (seed, tag, b,
    // k, i)): one shared copy, right-orthonormalised once for the whole batch below
    o[k] = new_tensor_n(c, o_shape(s, cols[k], D[k], D[k + 1]), 1);
    o[k].bstride = 0;
    hash_init(c, o[k], 1, seed, tag, b1, k);
  }
  // right-orthonormalise as a true gauge transformation (absorb the factor to the left)
  for (int k = K - 1; k >= 1 && !guess_done; --k) {
    Tensor C;
    Tensor q = right_orth(c, o[k], nb, &C);
    o[k] = q;
    // o_{k-1}[..., b] <- sum_q o_{k-1}[..., q] conj(C[b, q])
    const Tensor& prev = o[k - 1];
    std::vector<int> sh2 = {(int)(prev.size() / prev.shape.back()), prev.shape.back()};
    Tensor pv = view(prev, sh2);
    Tensor np = contract(c, pv, "aq", false, C, "bq", true, "ab");
    o[k - 1] = view(np, prev.shape);
  }
  if (!gkey.empty() && !guess_done) {
    (*c.guess_cache)[gkey] = o;  // read-only from here on: the sweeps replace every site
    TN_CUDA(cudaStreamSynchronize(c.stream));  // later batches may run on other streams
  }
  auto env_left = [&](const Env& Lk, int k) {
    Env L = rescaled(ops.absorb_left(Lk.t, cols[k], &o[k]), Lk);
    int end = (k + 1 < K) ? cols[k + 1] : s.W;
    for (int j = cols[k] + 1; j < end; ++j) L = rescaled(ops.absorb_left(L.t, j, nullptr), L);
    return L;
  };
  auto env_right = [&](const Env& Fk, int k) {
    Env F = rescaled(ops.absorb_right(Fk.t, cols[k], &o[k]), Fk);
    int start = (k >= 1) ? cols[k - 1] : -1;
    for (int j = cols[k] - 1; j > start; --j) F = rescaled(ops.absorb_right(F.t, j, nullptr), F);
    return F;
  };
  std::vector<Env> Lk(K), Fk(K);
  {
    Env L = trivial_env();
    for (int j = 0; j < cols[0]; ++j) L = rescaled(ops.absorb_left(L.t, j, nullptr), L);
    Lk[0] = L;
    Env F = trivial_env();
    for (int j = s.W - 1; j > cols[K - 1]; --j) F = rescaled(ops.absorb_right(F.t, j, nullptr), F);
    Fk[K - 1] = F;
  }
  for (int k = K - 1; k >= 1; --k) Fk[k - 1] = env_right(Fk[k], k);
  // environments the current centre was computed with (for its true scale)
  Env cl = Lk[0], cf = Fk[0];
  // Single layer: right-to-left half-sweeps contract each column once (rmid1 gives both the
  // derivative and the new right environment); the double layer keeps the mid contraction
  // from the left (its right-hand mirror has the same cost and cannot be reused: the
  // environment needs the orthonormalised site, i.e. all of d, and the double-layer mid is
  // too large to keep -- 137 GB per site at the metric shapes).
  for (int h = 0; h < nh; ++h) {
    if (h % 2 == 0) {
      for (int k = 0; k < K; ++k) {
        if (!(h > 0 && k == 0)) {
          Tensor d = ops.derivative(Lk[k].t, cols[k], Fk[k].t);
          o[k] = view(d, o[k].shape);
          cl = Lk[k];
          cf = Fk[k];
          nan_check(c, "L env", Lk[k].t, nb);
          nan_check(c, "F env", Fk[k].t, nb);
        }
        if (k < K - 1) {
          o[k] = left_orth(c, o[k], nb);
          Lk[k + 1] = env_left(Lk[k], k);
        }
      }
    } else {
      for (int k = K - 1; k >= 0; --k) {
        if (k != K - 1) {
          Tensor d = s.dbl ? ops.derivative(Lk[k].t, cols[k], Fk[k].t)
                           : ops.derivative_right(Lk[k].t, cols[k], Fk[k].t);
          o[k] = view(d, o[k].shape);
          cl = Lk[k];
          cf = Fk[k];
        }
        if (k > 0) {
          o[k] = right_orth(c, o[k], nb, nullptr);
          Fk[k - 1] = env_right(Fk[k], k);
        }
      }
    }
  }
  int centre = (nh % 2 == 1) ? K - 1 : 0;
  DevBuf lc(sizeof(double) * nb, c.stream);
  normalize(c, o[centre], nb, lc.as<double>(), false);
  if (logn) log_add(c, logn, lc.as<double>(), cl.lg->as<double>(), cf.lg->as<double>(), nb, accumulate);
  res.sites = std::move(o);
  return res;
}

}  // namespace tn
