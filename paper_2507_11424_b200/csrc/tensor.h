// tensor.h -- batched complex tensors on the device and the pairwise contraction engine.
//
// Every contraction of the method is expressed as one call of
// contract(): operands are permuted (only when their layout does not already match a
// GEMM view) and multiplied by a batched complex GEMM (gemm.cu: tcgen05 TF32x3 on
// sm_100a for large tiles, FP32 SIMT otherwise). The leading "sample" batch of per-sample
// operands is folded into the GEMM M dimension when the other operand is shared across
// samples (A_v, the norm environment M), so one launch covers the whole batch.
#pragma once
#include <map>
#include <memory>
#include <string>
#include <vector>

#include <cuda_fp16.h>

#include "common.h"
#include "prof.h"

namespace tn {

// FP16 hi/lo planes of a GEMM's A operand (K-major [z][Mp][Krp] halves, element (r, 2k + c)) and
// their per-(row, SB_K block) scales [z][nsb][Mp] (1/s), written directly by the epilogue of the
// GEMM that produces the operand (contract_planes) and consumed by contract() with no prep pass.
struct Planes {
  std::shared_ptr<DevBuf> hi, lo, asc;
  std::string lab;  // logical labels of the operand: batch labels, row labels, K labels (outer -> inner)
  int nz = 0, Mp = 0, Krp = 0, nsb = 0;
};

struct Tensor {
  std::shared_ptr<DevBuf> mem;
  float2* p = nullptr;
  std::vector<int> shape;
  int64_t bstride = 0;  // elements between consecutive samples; 0 = shared by all samples
  std::shared_ptr<Planes> planes;  // set (and p null) for a tensor held only as GEMM A planes
  int64_t size() const { return prod(shape); }
  int rank() const { return (int)shape.size(); }
};

// max |component| bounds of a tensor's memory, one per sample (nullptr if unknown; *n = their
// count: the batch size of a per-sample tensor, 1 for a shared one), and their invalidation,
// to be called by every in-place write (see DevBuf::amax).
inline const float* tensor_amax(const Tensor& t, int* n = nullptr) {
  if (n) *n = t.mem ? t.mem->tail_n : 0;
  return t.mem ? t.mem->amax() : nullptr;
}
inline void invalidate_amax(const Tensor& t) {
  if (t.mem) t.mem->drop_amax();
}

struct Ctx {
  cudaStream_t stream = nullptr;
  int gemm_mode = 0;  // 0 auto, 1 SIMT only, 2 tcgen05 whenever legal
  int nb = 1;         // number of samples in the current batch
  // NEXT-2: an NCCL communicator (ncclComm_t) over the ranks that share the
  // norm-environment precompute; the double-layer fits split their chunk loops across them.
  void* comm = nullptr;
  int rank = 0, world = 1;
  // The single-layer fits' right-orthonormalised initial guesses, by (seed, tag, row, output
  // shapes): they do not depend on the samples (R4), so every sampling step after the first
  // reuses them (owned by the state; see fit.cu).
  std::shared_ptr<std::map<std::string, std::vector<Tensor>>> guess_cache;
};

// Allocate a tensor: per-sample (nb copies) when per_sample, else shared.
Tensor new_tensor(Ctx& c, const std::vector<int>& shape, bool per_sample);
Tensor new_tensor_n(Ctx& c, const std::vector<int>& shape, int nb);  // explicit batch
void zero(Ctx& c, Tensor& t, int nb);

// out[labels_out] = sum over shared labels of opA(A[la]) * opB(B[lb]); labels are single
// characters; labels present in A, B and out are element-wise (batched) labels. conj
// flags conjugate the operand. Per-sample/shared status follows the operands' bstride.
Tensor contract(Ctx& c, const Tensor& A, const char* la, bool conjA, const Tensor& B,
                const char* lb, bool conjB, const char* lout);

// As contract(), but the result is written straight into the A-operand planes of the next
// contraction instead of complex64 memory: zl / rl / kl are that contraction's batch, row and
// K labels (a partition of lout's labels; kl's innermost label must be the innermost row label
// of this GEMM, of dimension SB_K). The returned tensor (labels zl rl kl) can only be passed as
// the first operand of contract() with exactly those labels. Tensor-core path only; throws
// TN_E_ARG where the shapes do not allow it (callers check planes_ok first).
Tensor contract_planes(Ctx& c, const Tensor& A, const char* la, bool conjA, const Tensor& B, const char* lb,
                       bool conjB, const char* lout, const char* zl, const char* rl, const char* kl);

// Reorder the axes: out labels are a permutation of in labels.
Tensor permute(Ctx& c, const Tensor& A, const char* la, const char* lout, bool conj = false);

// Compound index of up to 4 axes (outer -> inner) with arbitrary element strides.
struct View4 {
  int rank = 0;
  int dims[4] = {1, 1, 1, 1};
  int64_t str[4] = {0, 0, 0, 0};
};

// Plain batched GEMM on strided complex views (row-major C with unit column stride):
// C[m, n] (+)= sum_k A(m, k) B(k, n), A(m,k) = A[m*am + k*ak], B(k,n) = B[k*bk + n*bn].
// When the v* views are set (rank > 0) they replace the single strides (tensor-core path
// only): the operand preparation gathers straight from the multi-axis layout.
// Plane output of a GEMM (contract_planes): element (m, n) of C goes to plane offset
// po(m) + po(n) (halves) and its scale block to so(m) + so(n); each side decomposes its index
// into up to six digits (outer -> inner) with a plane stride and a scale stride per digit.
struct PView {
  int rank = 0;
  int dims[6] = {1, 1, 1, 1, 1, 1};
  int64_t po[6] = {0, 0, 0, 0, 0, 0};
  int64_t so[6] = {0, 0, 0, 0, 0, 0};
};
struct PlaneOut {
  __half* hi = nullptr;
  __half* lo = nullptr;
  float* asc = nullptr;
  PView vm, vn;
  int64_t zpo = 0, zso = 0;  // plane / scale stride of the GEMM's batch index (unfolded samples)
  int mode = 1;              // scale block: 1 = a tile column of 128 rows, 2 = a warp's 32 rows x 4 columns
};

struct GemmDesc {
  View4 vam, vak, vbk, vbn;
  const Planes* pa = nullptr;   // A given as planes (no prep)
  const PlaneOut* po = nullptr; // C written as the next GEMM's A planes
  int M = 0, N = 0, K = 0;
  const float2* A = nullptr;
  int64_t am = 0, ak = 0;
  bool conjA = false;
  const float2* B = nullptr;
  int64_t bk = 0, bn = 0;
  bool conjB = false;
  float2* C = nullptr;
  int64_t cm = 0;
  int nb1 = 1, nb2 = 1;
  int64_t sa1 = 0, sb1 = 0, sc1 = 0, sa2 = 0, sb2 = 0, sc2 = 0;
  bool accumulate = false;
  int64_t work_per_sample = 0;  // complex MACs of one sample (kernel choice must not depend on batch)
  int m_per_sample = 0;         // M before the sample batch was folded into it
  // Per-sample max |component| bounds (the sample of an M-side row is row / m_per_sample when
  // the batch is folded into M, else the outer batch index b1; a count of 1 = one bound for all).
  const float* amaxA = nullptr;  // bounds of A (skip A's row-max pass)
  int amaxA_n = 0;
  float* amaxC = nullptr;        // if set: receives the bounds of C (tensor-core path only)
  int amaxC_n = 0;
};
// Returns true when the tensor-core path ran (and filled g.amaxC if set).
bool gemm(Ctx& c, const GemmDesc& g);
// Whether the tensor-core path uses producers' output bounds (the 3M path only).
bool tc_bounds_wanted();
// Whether gemm() will route a GEMM of this per-sample shape to the tensor cores.
bool tc_eligible(const Ctx& c, int64_t M, int64_t N, int64_t K, int64_t work_per_sample);

// Flop accounting of the GEMMs issued (complex MACs), for the roofline report.
// Thread-local (see g_launches).
extern thread_local double g_cmacs;
extern thread_local double g_cmacs_tc;      // the part issued to the tcgen05 kernel
extern thread_local int64_t g_tc_launches;  // tcgen05 GEMM kernel launches
extern thread_local std::vector<double> g_row_cmacs;  // per-row complex MACs of the last sampled batch

}  // namespace tn
