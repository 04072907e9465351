// linalg.h -- batched orthonormal bases for the one-site fit's gauge moves (K2).
//
// The fit needs "an orthonormal basis of the column (or row) span" of the new site with
// exactly D_k vectors. On the GPU this is CholeskyQR2 in FP64
// arithmetic on FP32 data, with a pivoted first Cholesky that detects numerically
// rank-deficient inputs and completes them with deterministic pseudo-random directions
// (harmless: they are orthogonal to the strip's support, R7):
//   G = X^H X (fp64) -> pivoted Cholesky -> rank r, permutation P
//   X' = [X P(:, :r), Y(:, :n-r)]  -> G' = X'^H X' -> R' (Cholesky) -> Q1 = X' R'^-1
//   G2 = Q1^H Q1 -> R2 -> Q = Q1 R2^-1
#pragma once
#include "tensor.h"

namespace tn {

// Strided complex FP32 matrix view of batch element b: X(i, j) = p[b*bs + i*si + j*sj],
// conjugated on access when cj.
struct MatView {
  float2* p = nullptr;
  int64_t bs = 0, si = 0, sj = 0;
  bool cj = false;
  int m = 0, n = 0;
};

// Q(:, :) <- orthonormal basis of span(X) (n = X.n columns, requires X.m >= X.n), nb
// matrices. If Cout is non-null it receives C = Q^H X as [b][n][n] complex FP32 (so that
// X = Q C whenever span(X) is in span(Q)).
void orthonormalize(Ctx& c, const MatView& X, const MatView& Q, float2* Cout, int nb);

}  // namespace tn
