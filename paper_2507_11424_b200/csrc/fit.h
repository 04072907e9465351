// fit.h -- the one-site variational MPS-MPO fit on the device (A12).
#pragma once
#include <vector>

#include "tensor.h"

namespace tn {

// One row of the network between an incoming boundary MPS ("tops") and the fitted MPS.
//  single layer: column j = top_j[m,u,n] x B_j[u,p,l,r], p open at output columns
//  double layer: column j = top_j[e,d,D,f] x A_j[s,u,d,l,r] x conj(A_j), (u,U) open
// A top with p == nullptr is the identity on the incoming bond (no edge at that column).
struct DStrip {
  bool dbl = false;
  int W = 0;
  std::vector<Tensor> tops;
  std::vector<int> topbond;  // incoming-MPS bond at the left of column j
  std::vector<Tensor> mats;
  std::vector<bool> out;
  bool per_sample = true;  // environments / outputs carry the sample batch
  int64_t chunk_elems = (int64_t)1 << 30;  // budget (elements) for double-layer intermediates
};

struct FitResult {
  std::vector<Tensor> sites;  // output MPS (empty when the strip has no output column)
  Tensor scalar;              // [1] per sample: exact contraction when no output column
  std::shared_ptr<DevBuf> scalar_log;  // double[nb]: the scalar's true value is scalar * exp(scalar_log)
};

// Output bonds D_0..D_K by SURVEY R6 (+ neighbour consistency), identical to the oracle.
std::vector<int> fit_bonds(const DStrip& s, int R);

// Fit_R of O3: hash-initialised, gauge-preserving right-orthonormalisation, nh alternating
// half-sweeps (L->R first), centre site normalised; ln of its norm is written (or added,
// when accumulate) to logn[b] (device, per sample) if non-null.
// TN_NAN_CHECK debugging aid (synchronises; no-op unless the variable is set)
void nan_check(Ctx& c, const char* what, const Tensor& t, int nb);

FitResult fake_fit(Ctx& c, const DStrip& s, int R, int tag, int b1, uint64_t seed);  // profiling only

FitResult fit(Ctx& c, const DStrip& s, int R, int tag, int b1, uint64_t seed, int nh, double* logn,
              bool accumulate);

}  // namespace tn
