// kernels.h -- elementwise / reduction kernels of the sampling path (K3, K4).
#pragma once
#include "tensor.h"

namespace tn {

// SplitMix64 initial guess of a fit site (R4/O3), replicated over nb samples.
void hash_init(Ctx& c, Tensor& o, int nb, uint64_t seed, int tag, int b1, int k);

// Per-sample Frobenius norm: t <- t / ||t||, logn[b] (+)= ln ||t|| when logn != nullptr.
// tn_certify statistics: out[0..5] = ln mean(p/q), rel. stderr, KLD, ESS, n used, n excluded
void cert_stats(Ctx& c, const double* logq, const double* logp, int64_t n, double log_z, double* out);
// tn_observables: importance weights w [n] (relative, max 1), sector indicators pass [n] and
// sums [3 (N+1)]: for v < N (sum w z_v, sum z_v, sum w), then (sum pass, sum w pass, sum w).
void observables(Ctx& c, const uint8_t* bits, const double* logq, const double* logp, int64_t n, int N,
                 const int* group_of, int n_groups, const int* target, double* w, double* pass, double* sums);
int64_t count_nonfinite(Ctx& c, const float2* p, int64_t n);  // debugging (synchronises)
void normalize(Ctx& c, Tensor& t, int nb, double* logn, bool accumulate_log);

// out[b][i] = t[b][0][i] + t[b][1][i]  (sum over a leading axis of size 2)
Tensor sum2(Ctx& c, const Tensor& t);

// Conditional / draw / log-q tail (a4, R9, R10): per sample b,
// w_s = Re sum_i L[b][i] Rs[b][s][i]; clamp; P0; x = (u < P0) ? 0 : 1; logq += ln P(x).
struct TailOut {
  int* x;            // [nb] drawn bit (device)
  uint8_t* bits;     // [nb][N] by vertex id
  double* logq;      // [nb]
  double* cond;      // [nb][N] or nullptr
  uint32_t* flags;   // [nb]
  const double* u;   // [nb][N] uniforms
  int N;
  int vertex;
};
void tail_draw(Ctx& c, const Tensor& L, const Tensor& Rs, int nb, const TailOut& o);

// out[b] = n[b][:, x_b] for n of shape [a, 2, d, z] (per sample)
Tensor select_s(Ctx& c, const Tensor& n, const int* x, int nb);

// out[b] = A[bits[b][v]] for shared A of shape [2, ...] (amplitude rows)
Tensor gather_bit(Ctx& c, const Tensor& A, const uint8_t* bits, int N, int v, int nb);

// t[b] = 1 (all elements), per-sample
Tensor ones(Ctx& c, const std::vector<int>& shape, int nb);

// Copy a tensor slice (rows [x0, x1) of axis 0) into dst at the same rows.
void copy_rows(Ctx& c, const Tensor& src, Tensor& dst, int64_t x0, int nb);

// dst += src (elementwise, same size)
void add_into(Ctx& c, Tensor& dst, const Tensor& src, int nb);

// out[i] = (acc ? out[i] : 0) + a[i] + (b ? b[i] : 0) + (c ? c[i] : 0), i < n (device arrays)
void log_add(Ctx& c, double* out, const double* a, const double* b, const double* c2, int n, bool acc);

// Per-sample scalar t[b][0]: logacc[b] += ln|t|, phase[b] = arg t (device arrays).
void scalar_logphase(Ctx& c, const Tensor& t, int nb, double* logacc, double* phase);

// out[b] = per-sample scalar t[b][0] -> host (complex) helper
void scalars_to_host(Ctx& c, const Tensor& t, int nb, std::vector<float2>& out);

}  // namespace tn
