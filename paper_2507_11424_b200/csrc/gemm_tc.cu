// gemm_tc.cu -- complex GEMM on the 5th-generation tensor cores (tcgen05, sm_100a),
// FP32-accurate through an FP16x3 split with exact power-of-two block scaling (K1 of
// SURVEY 2.4).
//
// Complex C = A B is one real GEMM  C_r[M][2N] = A_r[M][2K] . B_r[2K][2N]:
//   A_r = A viewed as interleaved (re, im) along K; C_r = C viewed the same way along N;
//   B_r^T row 2n = (Re b_kn, -Im b_kn) over k, row 2n+1 = (Im b_kn, Re b_kn)  (K-major).
// Every (row m of A, block of SB_K = 128 complex K) and (column n of B, block) is scaled by an
// exact power of two s so that the block's largest |component| lies in [1/2, 1); every scaled
// value x is split into FP16 x = h + l (h = fp16_rn(x), l = fp16_rn(x - h); 22 significant
// bits), and D = A_h B_h + A_h B_l + A_l B_h accumulates in FP32 over one block in TMEM; the
// epilogue promotes each block into FP32 registers multiplied by 1/(s_A s_B). FP16 MMAs run at
// twice the TF32 rate and halve the operand bytes per K.
//
// Data flow: one prep pass gathers each operand straight from its multi-axis layout (View4)
// into packed, zero-padded, K-major FP16 hi/lo planes in HBM, taking each block's scale from
// the tile it converts -- or the producing GEMM's epilogue writes them (plane output, see
// tc_gemm2_kernel<true>); the CTA-pair kernel streams FP16 tiles with TMA (SWIZZLE_128B)
// through a 3-stage mbarrier ring; one elected thread issues tcgen05.mma (cta_group::2,
// M=256, N=256, K=16, kind::f16, FP32 accumulate) into one of two TMEM accumulators; every
// scale block is promoted by eight epilogue warps into FP32 registers (which also bounds the
// tensor core's truncating FP32 accumulation) while the MMA fills the other accumulator.
// Long-K/small-MN GEMMs are split along K (deterministic reduction). The 1-CTA kernel serves
// GEMMs of <= 128 rows; the 3M kernel (off by default) keeps per-row scales.
#include <cuda.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>

#include "tensor.h"

namespace tn {
namespace {

constexpr int TC_BM = 128;        // rows per CTA (UMMA M)
constexpr int TC_BN = 256;        // real columns per CTA (UMMA N) = 128 complex columns
constexpr int TC_BK = 64;         // real K per stage (one 128-byte swizzle atom of FP16)
constexpr int TC_UK = 16;         // K per kind::f16 MMA
constexpr int TC_STAGES = 2;
constexpr int A_TILE = TC_BM * TC_BK * 2;               // 16 KB
constexpr int B_TILE = TC_BN * TC_BK * 2;               // 32 KB
constexpr int STAGE_BYTES = 2 * A_TILE + 2 * B_TILE;    // 96 KB
constexpr int SMEM_BYTES = TC_STAGES * STAGE_BYTES + 1024 + 256;
constexpr uint32_t TMEM_COLS = 512;   // two 128x256 FP32 accumulators (ping-pong over K chunks)
constexpr int TC_KC = 16;             // split-K granularity in k-blocks (16 x 64 real K)
// A is scaled per (row, block of SB_K complex K): one exact power of two per row and block puts
// the block's largest |component| in [1/2, 1), so every element keeps the FP16x3 split's 22
// significant bits relative to its own block instead of to the whole row (or sample). The
// tensor core accumulates one block per TMEM chunk; the epilogue promotes the chunk into FP32
// registers multiplied by the block's 1/s (FFMA), so scale blocks = promotion chunks.
constexpr int SB_KB = 4;              // k-blocks per scale block / promoted chunk
constexpr int SB_K = SB_KB * TC_BK / 2;  // 128 complex K
constexpr int TC_THREADS = 320;       // warp 0 TMA, warp 1 MMA, warps 2..9 epilogue

struct TcParams {
  int M, N;          // complex extents (epilogue bounds)
  int kblocks;       // padded real K / TC_BK
  int ksplit;        // K splits (grid.z = nz * ksplit); > 1 writes partials to ws
  int kb_per_split;  // k-blocks per split (multiple of TC_KC)
  float2* ws;        // [split][z][M][N] partial sums when ksplit > 1
  int64_t ws_split;  // elements per split slice
  int b_batched;     // B planes carry the batch index
  const float* amax; // [z][Mp] row maxima of A (scales)
  const float* bmax; // [zb][Np] column maxima of B
  int Mp, Np;
  float2* C;
  int64_t cm;
  int nb2;
  int64_t sc1, sc2;
  int z0;
  int accumulate;
  const float* amax_sample;   // non-null: one scale per sample for the rows of A (producer's bound)
  int amax_sample_n;          // its count (1: one bound for every row)
  float* amax_out;            // non-null: atomicMax of max |component| of the stored C values, per sample
  int amax_out_n;             // its count
  int rows_per_sample;        // > 0: sample of row m = m / rows_per_sample (batch folded into M);
                              // 0: sample = (z0 + z) / nb2 (outer batch index)
  const float* ascale;        // 4M kernels: [z][nsb][Mp] 1/s of A's (row, scale block) exponents
  const float* bscale;        // 4M kernels: [zb][nsb][Np] 1/s of B's (column, scale block)
  int nsb;                    // scale blocks (SB_KB k-blocks = SB_K complex K each) along K
  // plane output (pair kernel, ksplit 1): C is written as the next GEMM's FP16 A planes with
  // per-(row, block) scales; a CTA's 128 rows are exactly one scale block of that operand
  int pout;
  PView pvm, pvn;
  int64_t pzpo, pzso;
  int pmode;  // 1: scale block = a tile column of 128 rows; 2: a warp's 32 rows x 4 columns
  __half* pho;
  __half* plo;
  float* psc;
};

__device__ __forceinline__ void pview_off(const PView& v, int64_t idx, int64_t& po, int64_t& so) {
  po = 0;
  so = 0;
#pragma unroll
  for (int d = 5; d >= 0; --d) {
    if (d < v.rank) {
      const int64_t q = idx / v.dims[d];
      const int64_t r = idx - q * v.dims[d];
      po += r * v.po[d];
      so += r * v.so[d];
      idx = q;
    }
  }
}

// Max of |components| of 32 complex columns (acc[2 c0 .. 2 c0 + 63]) over the warp's 32 rows:
// five halving exchanges (16 + 8 + 4 + 2 + 1 shuffles); lane l returns column c0 + l.
__device__ __forceinline__ float warp_colmax32(const float* acc, int c0, int lane) {
  float r16[16];
  const bool b16 = lane & 16;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const float mj = fmaxf(fabsf(acc[2 * (c0 + j)]), fabsf(acc[2 * (c0 + j) + 1]));
    const float mk = fmaxf(fabsf(acc[2 * (c0 + j + 16)]), fabsf(acc[2 * (c0 + j + 16) + 1]));
    r16[j] = fmaxf(b16 ? mk : mj, __shfl_xor_sync(0xffffffffu, b16 ? mj : mk, 16));
  }
  float r8[8];
  const bool b8 = lane & 8;
#pragma unroll
  for (int j = 0; j < 8; ++j)
    r8[j] = fmaxf(b8 ? r16[j + 8] : r16[j], __shfl_xor_sync(0xffffffffu, b8 ? r16[j] : r16[j + 8], 8));
  float r4[4];
  const bool b4 = lane & 4;
#pragma unroll
  for (int j = 0; j < 4; ++j)
    r4[j] = fmaxf(b4 ? r8[j + 4] : r8[j], __shfl_xor_sync(0xffffffffu, b4 ? r8[j] : r8[j + 4], 4));
  float r2[2];
  const bool b2 = lane & 2;
#pragma unroll
  for (int j = 0; j < 2; ++j)
    r2[j] = fmaxf(b2 ? r4[j + 2] : r4[j], __shfl_xor_sync(0xffffffffu, b2 ? r4[j] : r4[j + 2], 2));
  const bool b1 = lane & 1;
  return fmaxf(b1 ? r2[1] : r2[0], __shfl_xor_sync(0xffffffffu, b1 ? r2[0] : r2[1], 1));
}

// Sample of an M-side row (A's rows and C's rows share the mapping), for bounds of count n.
__device__ __forceinline__ int sample_of(int rows_per_sample, int z0, int z, int nb2, int row, int n) {
  if (n <= 1) return 0;
  const int s = rows_per_sample > 0 ? row / rows_per_sample : (z0 + z) / nb2;
  return min(s, n - 1);
}

__device__ __forceinline__ void split16(float x, __half& h, __half& l) {
  h = __float2half_rn(x);
  l = __float2half_rn(x - __half2float(h));
}

__device__ __forceinline__ void split16x2(float x, float y, __half2& h, __half2& l) {
  __half hx, lx, hy, ly;
  split16(x, hx, lx);
  split16(y, hy, ly);
  h = __halves2half2(hx, hy);
  l = __halves2half2(lx, ly);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// UMMA shared-memory descriptor: K-major, SWIZZLE_128B, 8-row atoms 1024 B apart (SBO),
// version 1 (sm_100), start address >> 4.
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)(0) << 16;                     // LBO (unused for swizzled K-major)
  d |= (uint64_t)((1024 >> 4) & 0x3FFF) << 32;  // SBO
  d |= (uint64_t)1 << 46;                       // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                       // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// Scale exponent of a row or column maximum mx: mx = f 2^e, f in [1/2, 1). Clamped to
// [-125, 125] so that both s = 2^-e (prep) and 1/s (epilogue) stay finite FP32 numbers: a
// row of magnitude < 2^-126 (numerical noise, e.g. a null direction of a rank-deficient
// basis) would otherwise get s = inf and turn the whole output into NaN.
__device__ __forceinline__ int scale_exp(float mx) {
  int e;
  frexpf(mx, &e);
  return max(-125, min(125, e));
}

// 1 / s for a row or column maximum mx.
__device__ __forceinline__ float inv_scale(float mx) {
  if (!(mx > 0.f)) return 1.f;
  return ldexpf(1.f, scale_exp(mx));
}

// Many warps update one address: read first and only issue the atomic when it would raise
// the value (same-address atomics serialise in L2).
__device__ __forceinline__ void atomic_max_nonneg(float* p, float v) {
  if (v > 0.f && v > *reinterpret_cast<volatile float*>(p))
    atomicMax(reinterpret_cast<unsigned int*>(p), __float_as_uint(v));
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ float row_amax(const TcParams& p, int z, int row) {
  if (p.amax_sample) return p.amax_sample[sample_of(p.rows_per_sample, p.z0, z, p.nb2, row, p.amax_sample_n)];
  return p.amax[(int64_t)z * p.Mp + row];
}

// Per-sample output bound of a warp whose lanes hold rows rows0..rows0+31 (1-CTA kernel: lane =
// row): one atomic when the warp's rows belong to one sample, else one per lane.
__device__ __forceinline__ void amax_out_rows(const TcParams& p, int z, int row, float lmax) {
  const int s = sample_of(p.rows_per_sample, p.z0, z, p.nb2, row, p.amax_out_n);
  const int s0 = __shfl_sync(0xffffffffu, s, 0);
  if (__all_sync(0xffffffffu, s == s0)) {
    lmax = warp_max(lmax);
    if ((threadIdx.x & 31) == 0) atomic_max_nonneg(p.amax_out + s0, lmax);
  } else {
    atomic_max_nonneg(p.amax_out + s, lmax);
  }
}

// Grouped rasterisation: linear tile id -> (m, n), groups of RASTER_GM m-tiles swept with m
// fastest, so a wave of CTAs shares a few A strips and B strips in L2 instead of streaming
// one operand strip per CTA from HBM (a full-K strip is 4-8 MB of FP16 planes).
__device__ int g_raster_gm = 16;  // group height in pair-tiles (4: +2%, 32: +4% step time); tn_debug_raster
__device__ __forceinline__ void raster(int lin, int nm, int nn, int& m, int& n) {
  const int GM = g_raster_gm;
  const int per_group = GM * nn;
  const int g = lin / per_group, r = lin - g * per_group;
  const int m0 = g * GM;
  const int gm = min(GM, nm - m0);
  m = m0 + r % gm;
  n = r / gm;
}

__global__ void __launch_bounds__(TC_THREADS, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap mAhi, const __grid_constant__ CUtensorMap mAlo,
                   const __grid_constant__ CUtensorMap mBhi, const __grid_constant__ CUtensorMap mBlo, TcParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + TC_STAGES * STAGE_BYTES);
  uint64_t* empty = full + TC_STAGES;
  uint64_t* acc_full = empty + TC_STAGES;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < TC_STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 8);  // one arrival per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mAhi)));
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mBhi)));
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;

  const int nblk = blockIdx.x, mblk = blockIdx.y;  // (used for M <= 128 per batch element)
  const int z = blockIdx.z / p.ksplit, split = blockIdx.z - z * p.ksplit;
  const int kb0 = split * p.kb_per_split;
  const int kb1 = min(p.kblocks, kb0 + p.kb_per_split);
  const int nkb = kb1 - kb0;
  const int bz = p.b_batched ? z : 0;
  if (warp == 0) {
    if (lane == 0) {  // TMA producer
      for (int i = 0; i < nkb; ++i) {
        const int kb = kb0 + i;
        const int s = i % TC_STAGES;
        const uint32_t ph = (i / TC_STAGES) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* st = smem + s * STAGE_BYTES;
        mbar_expect_tx(&full[s], STAGE_BYTES);
        tma_load_3d(st, &mAhi, kb * TC_BK, mblk * TC_BM, z, &full[s]);
        tma_load_3d(st + A_TILE, &mAlo, kb * TC_BK, mblk * TC_BM, z, &full[s]);
        tma_load_3d(st + 2 * A_TILE, &mBhi, kb * TC_BK, nblk * TC_BN, bz, &full[s]);
        tma_load_3d(st + 2 * A_TILE + B_TILE, &mBlo, kb * TC_BK, nblk * TC_BN, bz, &full[s]);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      // kind::f16 instruction descriptor: D f32, A/B f16, K-major both, N=256, M=128
      const uint32_t idesc = (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(TC_BN >> 3) << 17) |
                             ((uint32_t)(TC_BM >> 4) << 24);
      for (int i = 0; i < nkb; ++i) {
        const int c = i / SB_KB, buf = c & 1, kin = i - c * SB_KB;
        if (kin == 0) {  // chunk c accumulates into TMEM buffer c&1 once the epilogue drained it
          mbar_wait(&acc_empty[buf], ((c >> 1) & 1) ^ 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
        }
        const uint32_t dacc = tmem + (uint32_t)(buf * TC_BN);
        const int s = i % TC_STAGES;
        const uint32_t ph = (i / TC_STAGES) & 1;
        mbar_wait(&full[s], ph);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t base = smem_u32(smem + s * STAGE_BYTES);
        const uint64_t ahi = smem_desc(base), alo = smem_desc(base + A_TILE);
        const uint64_t bhi = smem_desc(base + 2 * A_TILE), blo = smem_desc(base + 2 * A_TILE + B_TILE);
#pragma unroll
        for (int k = 0; k < TC_BK / TC_UK; ++k) {
          const uint64_t adv = (uint64_t)((k * TC_UK * 2) >> 4);  // 16 halves = 32 bytes along K
          mma_f16(dacc, ahi + adv, bhi + adv, idesc, (kin | k) != 0);
          mma_f16(dacc, ahi + adv, blo + adv, idesc, 1u);
          mma_f16(dacc, alo + adv, bhi + adv, idesc, 1u);
        }
        mma_commit(&empty[s]);
        if (kin == SB_KB - 1 || i == nkb - 1) mma_commit(&acc_full[buf]);
      }
    }
    __syncwarp();
  } else {
    // epilogue: warps 2..9; warp w drains TMEM lanes 32*(w%4)..+31 (its rows) and columns
    // [128*h, 128*h + 128), h = (w-2)/4. Each K chunk's partial sum is promoted from TMEM
    // into FP32 registers (round-to-nearest adds).
    const int lg = warp & 3;
    const int half = (warp - 2) >> 2;
    const int row = mblk * TC_BM + lg * 32 + lane;
    float acc[128];
#pragma unroll
    for (int i = 0; i < 128; ++i) acc[i] = 0.f;
    const int nchunks = (nkb + SB_KB - 1) / SB_KB;
    const float* ascr = p.ascale + ((int64_t)z * p.nsb + kb0 / SB_KB) * p.Mp + row;  // row < Mp
    const float* bscr = p.bscale + ((int64_t)bz * p.nsb + kb0 / SB_KB) * p.Np + ((nblk * TC_BN + half * 128) >> 1);
    for (int c = 0; c < nchunks; ++c) {
      const int buf = c & 1;
      const float f = ascr[(int64_t)c * p.Mp];  // 1/s of this row's scale block
      const float* fb = bscr + (int64_t)c * p.Np;  // 1/s of the block's 64 columns (< Np)
      mbar_wait(&acc_full[buf], (c >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
      for (int cc = 0; cc < 128; cc += 16) {
        uint32_t v[16];
        const uint32_t taddr = tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)(buf * TC_BN + half * 128 + cc);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int i = 0; i < 16; i += 2) {
          const float g = f * __ldg(fb + ((cc + i) >> 1));
          acc[cc + i] = fmaf(__uint_as_float(v[i]), g, acc[cc + i]);
          acc[cc + i + 1] = fmaf(__uint_as_float(v[i + 1]), g, acc[cc + i + 1]);
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[buf]);
    }
    float lmax = 0.f;
    if (row < p.M) {  // (A's and B's scales were applied per block during the promotion)
      const int n0 = (nblk * TC_BN + half * 128) >> 1;
      if (p.ksplit > 1) {  // partial sum of this K split -> workspace
        float2* W = p.ws + split * p.ws_split + ((int64_t)z * p.M + row) * p.N;
#pragma unroll
        for (int q = 0; q < 64; ++q) {
          const int n = n0 + q;
          if (n < p.N) {
            W[n] = make_float2(acc[2 * q], acc[2 * q + 1]);
          }
        }
      } else {
        const int b1 = (p.z0 + z) / p.nb2, b2 = (p.z0 + z) - b1 * p.nb2;
        float2* Crow = p.C + b1 * p.sc1 + b2 * p.sc2 + (int64_t)row * p.cm;
#pragma unroll
        for (int q = 0; q < 64; ++q) {
          const int n = n0 + q;
          if (n < p.N) {
            float2 val = make_float2(acc[2 * q], acc[2 * q + 1]);
            if (p.accumulate) {
              float2 o = Crow[n];
              val.x += o.x;
              val.y += o.y;
            }
            Crow[n] = val;
            lmax = fmaxf(lmax, fmaxf(fabsf(val.x), fabsf(val.y)));
          }
        }
      }
    }
    if (p.amax_out && p.ksplit == 1) amax_out_rows(p, z, row, lmax);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

// ---------------------------------------------------------------------------------------
// CTA-pair variant (cta_group::2): a cluster of two CTAs on one TPC computes a 256 x 256
// (real) tile with tcgen05.mma M=256. CTA r loads its own 128 rows of A and rows
// [128 r, 128 r + 128) of the B^T tile into its shared memory; the leader's single MMA thread
// reads both CTAs' operands, so each SM streams half of B per MMA -- the shared-memory read
// traffic per MAC drops by a third against the 1-CTA 128 x 256 tile (the FP16x3 split reads
// every operand tile twice per k-step, which made the 1-CTA kernel shared-memory bound).
// Accumulators: each CTA's TMEM holds its 128 rows x 256 columns (two ping-pong buffers).
constexpr int T2_STAGES = 3;
constexpr int A2_TILE = 128 * TC_BK * 2;                 // 16 KB per CTA
constexpr int B2_TILE = 128 * TC_BK * 2;                 // 16 KB per CTA (half of the B tile)
constexpr int STAGE2_BYTES = 2 * A2_TILE + 2 * B2_TILE;  // 64 KB
constexpr int EPI_Q = 8;  // complex columns per staged store step (the fast path stores 4 lanes x 2 per row)
constexpr int EPI_STAGE_BYTES = 8 * 32 * (EPI_Q + 1) * 8;  // per-warp 32 x (8+1) float2 (8 warps)
constexpr int EPI_COLSC_BYTES = 8 * 64 * 4;                 // per-warp column scales of a tile
constexpr int SMEM2_BYTES = T2_STAGES * STAGE2_BYTES + EPI_STAGE_BYTES + EPI_COLSC_BYTES + 1024 + 256;

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ uint32_t map_to_rank(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// TMA load into this CTA's shared memory, completion counted on the leader CTA's mbarrier
// (bar_cluster = shared::cluster address of that barrier).
__device__ __forceinline__ void tma_load_3d_pair(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                                 uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
      "%4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar_cluster)
      : "memory");
}

__device__ __forceinline__ void mma_f16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// arrive (once per CTA of the pair) on the barrier at the same offset in both CTAs
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}

// Persistent: a grid of at most 74 CTA pairs walks the tile space (batch element, K split,
// M pair-tile, N tile) with a static stride; the TMA ring, the MMA's TMEM ping-pong and the
// epilogue run continuously across tiles, so one tile's epilogue overlaps the next tile's
// main loop and the prologue (barrier init, TMEM allocation) is paid once per CTA.
struct PairTile {
  int z, split, mblk0, nblk, kb0, nkb;
};

__device__ __forceinline__ PairTile pair_tile(const TcParams& p, int t, int npm, int nn) {
  PairTile r;
  const int per_z = npm * nn;
  const int zs = t / per_z, rem = t - zs * per_z;
  r.z = zs / p.ksplit;
  r.split = zs - r.z * p.ksplit;
  int mpair;
  raster(rem, npm, nn, mpair, r.nblk);
  r.mblk0 = 2 * mpair;
  r.kb0 = r.split * p.kb_per_split;
  r.nkb = min(p.kblocks, r.kb0 + p.kb_per_split) - r.kb0;
  return r;
}

template <bool POUT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(TC_THREADS, 1)
    tc_gemm2_kernel(const __grid_constant__ CUtensorMap mAhi, const __grid_constant__ CUtensorMap mAlo,
                    const __grid_constant__ CUtensorMap mBhi, const __grid_constant__ CUtensorMap mBlo, TcParams p,
                    int npm, int nn, int ntiles) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + T2_STAGES * STAGE2_BYTES);
  uint64_t* empty = full + T2_STAGES;
  uint64_t* acc_full = empty + T2_STAGES;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  float2* epi_stage = reinterpret_cast<float2*>(smem + T2_STAGES * STAGE2_BYTES + 256);
  float* epi_colsc = reinterpret_cast<float*>(smem + T2_STAGES * STAGE2_BYTES + 256 + EPI_STAGE_BYTES);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < T2_STAGES; ++i) {
      mbar_init(&full[i], 1);   // leader: its producer's arrive.expect_tx (both CTAs' bytes)
      mbar_init(&empty[i], 1);  // one multicast MMA commit
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc_full[i], 1);
      mbar_init(&acc_empty[i], 16);  // leader: 8 epilogue warps of each CTA
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mAhi)));
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mBhi)));
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster_sync_all();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer (both CTAs)
      const uint32_t full0 = map_to_rank(smem_u32(&full[0]), 0);
      int i = 0;  // running stage counter
      for (int t = cluster; t < ntiles; t += nclusters) {
        const PairTile tl = pair_tile(p, t, npm, nn);
        const int mrow = (tl.mblk0 + (int)rank) * 128;
        const int brow = tl.nblk * TC_BN + (int)rank * 128;
        const int bz = p.b_batched ? tl.z : 0;
        for (int q = 0; q < tl.nkb; ++q, ++i) {
          const int kb = tl.kb0 + q;
          const int s = i % T2_STAGES;
          const uint32_t ph = (i / T2_STAGES) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t* st = smem + s * STAGE2_BYTES;
          if (rank == 0) mbar_expect_tx(&full[s], 2 * STAGE2_BYTES);
          const uint32_t fb = full0 + (uint32_t)(s * sizeof(uint64_t));
          tma_load_3d_pair(st, &mAhi, kb * TC_BK, mrow, tl.z, fb);
          tma_load_3d_pair(st + A2_TILE, &mAlo, kb * TC_BK, mrow, tl.z, fb);
          tma_load_3d_pair(st + 2 * A2_TILE, &mBhi, kb * TC_BK, brow, bz, fb);
          tma_load_3d_pair(st + 2 * A2_TILE + B2_TILE, &mBlo, kb * TC_BK, brow, bz, fb);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {  // MMA issuer (leader CTA only)
      // kind::f16 instruction descriptor: D f32, A/B f16, K-major both, N=256, M=256
      const uint32_t idesc = (1u << 4) | ((uint32_t)(TC_BN >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
      int i = 0, c = 0;  // running stage and chunk counters
      for (int t = cluster; t < ntiles; t += nclusters) {
        const PairTile tl = pair_tile(p, t, npm, nn);
        for (int q = 0; q < tl.nkb; ++q, ++i) {
          const int kin = q % SB_KB, buf = c & 1;
          if (kin == 0) {
            mbar_wait(&acc_empty[buf], ((c >> 1) & 1) ^ 1);
            asm volatile("tcgen05.fence::after_thread_sync;");
          }
          const uint32_t dacc = tmem + (uint32_t)(buf * TC_BN);
          const int s = i % T2_STAGES;
          const uint32_t ph = (i / T2_STAGES) & 1;
          mbar_wait(&full[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t base = smem_u32(smem + s * STAGE2_BYTES);
          const uint64_t ahi = smem_desc(base), alo = smem_desc(base + A2_TILE);
          const uint64_t bhi = smem_desc(base + 2 * A2_TILE), blo = smem_desc(base + 2 * A2_TILE + B2_TILE);
#pragma unroll
          for (int k = 0; k < TC_BK / TC_UK; ++k) {
            const uint64_t adv = (uint64_t)((k * TC_UK * 2) >> 4);
            mma_f16_pair(dacc, ahi + adv, bhi + adv, idesc, (kin | k) != 0);
            mma_f16_pair(dacc, ahi + adv, blo + adv, idesc, 1u);
            mma_f16_pair(dacc, alo + adv, bhi + adv, idesc, 1u);
          }
          mma_commit_pair(&empty[s]);
          if (kin == SB_KB - 1 || q == tl.nkb - 1) {
            mma_commit_pair(&acc_full[buf]);
            ++c;
          }
        }
      }
    }
    __syncwarp();
  } else {
    // epilogue (both CTAs): warp w drains TMEM lanes 32*(w%4)..+31 (this CTA's rows) and
    // columns [128*h, 128*h + 128), h = (w-2)/4; chunks are promoted into FP32 registers.
    const int lg = warp & 3;
    const int half = (warp - 2) >> 2;
    const uint32_t acc_empty0 = map_to_rank(smem_u32(&acc_empty[0]), 0);
    int c = 0;  // running chunk counter
    for (int t = cluster; t < ntiles; t += nclusters) {
      const PairTile tl = pair_tile(p, t, npm, nn);
      const int row = (tl.mblk0 + (int)rank) * 128 + lg * 32 + lane;
      float acc[128];
#pragma unroll
      for (int i = 0; i < 128; ++i) acc[i] = 0.f;
      const int nchunks = (tl.nkb + SB_KB - 1) / SB_KB;
      // scale indices as 32-bit element offsets (the scale arrays hold < 2^32 floats; fewer
      // live registers next to the 128 accumulators)
      uint32_t ai = (uint32_t)((tl.z * p.nsb + tl.kb0 / SB_KB) * p.Mp + row);  // row < Mp
      uint32_t bi = (uint32_t)(((p.b_batched ? tl.z : 0) * p.nsb + tl.kb0 / SB_KB) * p.Np +
                               ((tl.nblk * TC_BN + half * 128) >> 1) + lane);
      float* fcol = epi_colsc + (warp - 2) * 64;  // this warp's 64 column factors of the chunk
      for (int cc0 = 0; cc0 < nchunks; ++cc0, ++c, ai += p.Mp, bi += p.Np) {
        const int buf = c & 1;
        const float f = p.ascale[ai];  // 1/s of this row's scale block
        __syncwarp();
        fcol[lane] = p.bscale[bi];  // columns < Np
        fcol[lane + 32] = p.bscale[bi + 32];
        __syncwarp();
        mbar_wait(&acc_full[buf], (c >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;");
#pragma unroll
        for (int cc = 0; cc < 128; cc += 8) {
          uint32_t v[8];
          const uint32_t taddr = tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)(buf * TC_BN + half * 128 + cc);
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                       : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                       : "r"(taddr));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int i = 0; i < 8; i += 2) {
            const float g = f * fcol[(cc + i) >> 1];
            acc[cc + i] = fmaf(__uint_as_float(v[i]), g, acc[cc + i]);
            acc[cc + i + 1] = fmaf(__uint_as_float(v[i + 1]), g, acc[cc + i + 1]);
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(acc_empty0 + (uint32_t)(buf * sizeof(uint64_t)));
      }
      if (POUT && p.pmode == 2) {
        // Plane output, blocks of a warp's 32 rows x 4 adjacent columns (16 per warp): group
        // maxima by four halving exchanges (8 + 4 + 2 + 1 shuffles: lane l holds group l / 2)
        // and one more across the lane pair; no shared memory.
        const int n0 = (tl.nblk * TC_BN + half * 128) >> 1;
        const int64_t mrow = (int64_t)(tl.mblk0 + (int)rank) * 128 + lg * 32 + lane;
        float g8[8];
        const bool b16 = lane & 16;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float lo4 = 0.f, hi4 = 0.f;
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const int qa = 4 * j + t, qb = 4 * (j + 8) + t;
            lo4 = fmaxf(lo4, fmaxf(fabsf(acc[2 * qa]), fabsf(acc[2 * qa + 1])));
            hi4 = fmaxf(hi4, fmaxf(fabsf(acc[2 * qb]), fabsf(acc[2 * qb + 1])));
          }
          g8[j] = fmaxf(b16 ? hi4 : lo4, __shfl_xor_sync(0xffffffffu, b16 ? lo4 : hi4, 16));
        }
        float g4[4], g2[2];
        const bool b8 = lane & 8, b4 = lane & 4, b2 = lane & 2;
#pragma unroll
        for (int j = 0; j < 4; ++j)
          g4[j] = fmaxf(b8 ? g8[j + 4] : g8[j], __shfl_xor_sync(0xffffffffu, b8 ? g8[j] : g8[j + 4], 8));
#pragma unroll
        for (int j = 0; j < 2; ++j)
          g2[j] = fmaxf(b4 ? g4[j + 2] : g4[j], __shfl_xor_sync(0xffffffffu, b4 ? g4[j] : g4[j + 2], 4));
        float g1 = fmaxf(b2 ? g2[1] : g2[0], __shfl_xor_sync(0xffffffffu, b2 ? g2[0] : g2[1], 2));
        g1 = fmaxf(g1, __shfl_xor_sync(0xffffffffu, g1, 1));
        const float sg = g1 > 0.f ? ldexpf(1.f, -scale_exp(g1)) : 1.f;
        int64_t pm, sm, pnA, snA, pnB, snB;
        pview_off(p.pvm, mrow, pm, sm);
        pm += (int64_t)(p.z0 + tl.z) * p.pzpo;
        sm += (int64_t)(p.z0 + tl.z) * p.pzso;
        pview_off(p.pvn, n0 + lane, pnA, snA);
        pview_off(p.pvn, n0 + lane + 32, pnB, snB);
        if ((lane & 1) == 0) {  // group lane / 2: columns n0 + 4 (lane / 2) .. + 3 (sm: same for the warp)
          int64_t pq, sq;
          pview_off(p.pvn, n0 + 2 * lane, pq, sq);
          p.psc[sm + sq] = g1 > 0.f ? inv_scale(g1) : 1.f;
        }
        __half2* hi = reinterpret_cast<__half2*>(p.pho);
        __half2* lo = reinterpret_cast<__half2*>(p.plo);
#pragma unroll
        for (int q = 0; q < 64; ++q) {
          const float sc = __shfl_sync(0xffffffffu, sg, (q >> 2) << 1);
          const int64_t pn = __shfl_sync(0xffffffffu, q < 32 ? pnA : pnB, q & 31);
          __half2 h, l;
          split16x2(acc[2 * q] * sc, acc[2 * q + 1] * sc, h, l);
          const int64_t off = (pm + pn) >> 1;  // half2 index: the warp's 32 rows are 32 adjacent k
          hi[off] = h;
          lo[off] = l;
        }
        continue;
      }
      if (POUT) {
        // Plane output: the CTA's 128 rows x this half's 64 complex columns; column q of the
        // tile is one scale block (row of the consumer's A, block of 128 consumer K). Block
        // maxima: warp column maxima, then the four warps of this half combine them in shared
        // memory (named barrier 1 + half, 128 threads).
        const int n0 = (tl.nblk * TC_BN + half * 128) >> 1;
        const int64_t mrow = (int64_t)(tl.mblk0 + (int)rank) * 128 + lg * 32 + lane;
        float* slot = epi_colsc + (warp - 2) * 64;
        const float cA = warp_colmax32(acc, 0, lane), cB = warp_colmax32(acc, 32, lane);
        __syncwarp();
        slot[lane] = cA;
        slot[lane + 32] = cB;
        asm volatile("bar.sync %0, 128;" ::"r"(1 + half) : "memory");
        float mA = 0.f, mB = 0.f;
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const float* o = epi_colsc + (half * 4 + w) * 64;
          mA = fmaxf(mA, o[lane]);
          mB = fmaxf(mB, o[lane + 32]);
        }
        asm volatile("bar.sync %0, 128;" ::"r"(1 + half) : "memory");
        const float sA = mA > 0.f ? ldexpf(1.f, -scale_exp(mA)) : 1.f;
        const float sB = mB > 0.f ? ldexpf(1.f, -scale_exp(mB)) : 1.f;
        int64_t pm, sm, pnA, snA, pnB, snB;
        pview_off(p.pvm, mrow, pm, sm);
        pm += (int64_t)(p.z0 + tl.z) * p.pzpo;
        sm += (int64_t)(p.z0 + tl.z) * p.pzso;
        pview_off(p.pvn, n0 + lane, pnA, snA);
        pview_off(p.pvn, n0 + lane + 32, pnB, snB);
        if (lg == 0) {  // one writer per block: sm is the same for the CTA's 128 rows
          p.psc[sm + snA] = mA > 0.f ? inv_scale(mA) : 1.f;
          p.psc[sm + snB] = mB > 0.f ? inv_scale(mB) : 1.f;
        }
        __half2* hi = reinterpret_cast<__half2*>(p.pho);
        __half2* lo = reinterpret_cast<__half2*>(p.plo);
        // the innermost N digit runs over >= 32 aligned columns: a column's plane offset is that
        // of the first column of its 32-group plus a multiple of the digit's stride
        const bool lin = p.pvn.dims[p.pvn.rank - 1] % 32 == 0;
        const int64_t pst = p.pvn.po[p.pvn.rank - 1];
        const int64_t pg0 = __shfl_sync(0xffffffffu, pnA, 0), pg1 = __shfl_sync(0xffffffffu, pnB, 0);
#pragma unroll
        for (int q = 0; q < 64; ++q) {
          const float sc = __shfl_sync(0xffffffffu, q < 32 ? sA : sB, q & 31);
          const int64_t pn = lin ? (q < 32 ? pg0 : pg1) + (q & 31) * pst
                                 : __shfl_sync(0xffffffffu, q < 32 ? pnA : pnB, q & 31);
          __half2 h, l;
          split16x2(acc[2 * q] * sc, acc[2 * q + 1] * sc, h, l);
          const int64_t off = (pm + pn) >> 1;  // half2 index (complex element)
          hi[off] = h;
          lo[off] = l;
        }
        continue;
      }
      // Coalesced output: each warp stages 32 rows x 8 complex columns in shared memory
      // (padded rows), then writes 4 rows per store instruction (8 lanes x 8 B = 64 B each),
      // instead of 32 scattered rows per instruction.
      {
        const int z = tl.z;
        const int row0 = (tl.mblk0 + (int)rank) * 128 + lg * 32;
        const float rs = (row < p.M) ? 1.f : 0.f;  // A's scales: applied per block in the promotion
        float lmax = 0.f;
        const int n0 = (tl.nblk * TC_BN + half * 128) >> 1;
        float2* base;
        int64_t ld;
        bool acc_out = false;
        if (p.ksplit > 1) {
          base = p.ws + tl.split * p.ws_split + (int64_t)z * p.M * p.N;
          ld = p.N;
        } else {
          const int b1 = (p.z0 + z) / p.nb2, b2 = (p.z0 + z) - b1 * p.nb2;
          base = p.C + b1 * p.sc1 + b2 * p.sc2;
          ld = p.cm;
          acc_out = p.accumulate != 0;
        }
        float2* stg = epi_stage + (warp - 2) * 32 * (EPI_Q + 1);

        const int sub = lane >> 3, col = lane & 7;
        // per-sample output bounds: one per warp when its 32 rows belong to one sample (always,
        // unless a sample's row count is not a multiple of 32), else one atomic per element
        const int s_lo = sample_of(p.rows_per_sample, p.z0, z, p.nb2, row0, p.amax_out_n);
        const bool s_mixed = p.amax_out && p.ksplit == 1 &&
                             sample_of(p.rows_per_sample, p.z0, z, p.nb2, min(row0 + 31, p.M - 1), p.amax_out_n) != s_lo;
        // Interior fast path (warp-uniform): the warp's 32 rows and 64 columns all in range, no
        // read-modify-write, one output bound per warp. Each lane then stores two adjacent
        // complex values (16 B) of rows row0 + 8 r + lane / 4 with no per-element predicates or
        // index arithmetic -- the general loop below costs ~60 instructions per output, which
        // made the K = 128 GEMMs (one accumulation chunk per tile) epilogue-bound.
        const bool fast = !acc_out && !s_mixed && row0 + 32 <= p.M && n0 + 64 <= p.N && (ld & 1) == 0 &&
                          ((reinterpret_cast<uintptr_t>(base) & 15) == 0);
#pragma unroll
        for (int q0 = 0; q0 < 64; q0 += EPI_Q) {
#pragma unroll
          for (int q = 0; q < EPI_Q; ++q) {
            stg[lane * (EPI_Q + 1) + q] = make_float2(acc[2 * (q0 + q)] * rs, acc[2 * (q0 + q) + 1] * rs);
          }
          __syncwarp();
          if (fast) {
            const int fr = lane >> 2, fc = (lane & 3) * 2;  // row within an 8-row group, column pair
            float2* fdst = base + (int64_t)(row0 + fr) * ld + (n0 + q0 + fc);
#pragma unroll
            for (int r = 0; r < 4; ++r) {
              const float2* src = stg + (r * 8 + fr) * (EPI_Q + 1) + fc;
              const float2 a = src[0], b = src[1];
              *reinterpret_cast<float4*>(fdst + (int64_t)(8 * r) * ld) = make_float4(a.x, a.y, b.x, b.y);
              lmax = fmaxf(lmax, fmaxf(fmaxf(fabsf(a.x), fabsf(a.y)), fmaxf(fabsf(b.x), fabsf(b.y))));
            }
          } else {
            const int n = n0 + q0 + col;
#pragma unroll 4
            for (int r = 0; r < 32; r += 4) {
              const int rr = r + sub, grow = row0 + rr;
              if (grow < p.M && n < p.N) {
                float2 val = stg[rr * (EPI_Q + 1) + col];
                float2* dst = base + (int64_t)grow * ld + n;
                if (acc_out) {
                  const float2 o = *dst;
                  val.x += o.x;
                  val.y += o.y;
                }
                *dst = val;
                const float mv = fmaxf(fabsf(val.x), fabsf(val.y));
                if (s_mixed)
                  atomic_max_nonneg(p.amax_out + sample_of(p.rows_per_sample, p.z0, z, p.nb2, grow, p.amax_out_n), mv);
                lmax = fmaxf(lmax, mv);
              }
            }
          }
          __syncwarp();
        }
        if (p.amax_out && p.ksplit == 1 && !s_mixed) {
          lmax = warp_max(lmax);
          if (lane == 0) atomic_max_nonneg(p.amax_out + s_lo, lmax);
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster_sync_all();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

// Deterministic split-K reduction: C (+)= sum over splits in a fixed order.
// One block per output row (z, row): its N complex values, summed over the splits in order.
__global__ void __launch_bounds__(128) splitk_reduce_kernel(const float2* __restrict__ ws, int ksplit,
                                                            int64_t ws_split, int nz, int M, int N, float2* C,
                                                            int64_t cm, int nb2, int64_t sc1, int64_t sc2, int z0,
                                                            int accumulate, float* amax_out, int amax_out_n,
                                                            int rows_per_sample) {
  const int64_t line = blockIdx.x;  // zz * M + row
  const int zz = (int)(line / M), row = (int)(line - (int64_t)zz * M);
  const int z = z0 + zz;
  const int b1 = z / nb2, b2 = z - b1 * nb2;
  const float2* w = ws + line * N;
  float2* cp = C + b1 * sc1 + b2 * sc2 + (int64_t)row * cm;
  float lmax = 0.f;
  for (int n = threadIdx.x; n < N; n += blockDim.x) {
    float2 s = w[n];
    for (int k = 1; k < ksplit; ++k) {
      const float2 v = w[k * ws_split + n];
      s.x += v.x;
      s.y += v.y;
    }
    if (accumulate) {
      const float2 o = cp[n];
      s.x += o.x;
      s.y += o.y;
    }
    cp[n] = s;
    lmax = fmaxf(lmax, fmaxf(fabsf(s.x), fabsf(s.y)));
  }
  if (amax_out) {  // output bounds (only the 3M path's consumers use them)
    lmax = warp_max(lmax);
    if ((threadIdx.x & 31) == 0)
      atomic_max_nonneg(amax_out + sample_of(rows_per_sample, z0, zz, nb2, row, amax_out_n), lmax);
  }
}

__device__ __forceinline__ int64_t view_off(const View4& v, int64_t idx) {
  int64_t off = 0;
#pragma unroll
  for (int d = 3; d >= 0; --d) {
    if (d < v.rank) {
      const int64_t q = idx / v.dims[d];
      off += (idx - q * v.dims[d]) * v.str[d];
      idx = q;
    }
  }
  return off;
}

// Operand X(r, k) (r = row index: M for A, N for B; k = K index; both compound, View4).
// Tiles of 32 rows x 32 complex k through shared memory: loads run along whichever side is
// contiguous in memory (k_fast), stores along the plane's K axis.
struct PrepArgs {
  const float2* X;
  View4 vr, vk;
  int conj, nb2;
  int64_t s1, s2;
  int z0, R, K, Rrows, Krp;  // Rrows: padded plane rows (A: Mp; B: Nrp)
  int k_fast;
  float* mx;                 // [z][Rp] row maxima (max pass writes, prep reads)
  const float* mx_sample;    // non-null: one maximum per sample for its rows (no max pass)
  int mx_sample_n;           // count of mx_sample (1: one maximum for every row)
  int rows_per_sample;       // sample of row r: r / rows_per_sample, or (z0 + z) / nb2 when 0
  int Rp;                    // row count of mx per z (complex rows)
  __half* hi;
  __half* lo;
  float* asc;                // 4M planes: [z][nsb][Rp] 1/s per (row of A / complex column of B, scale block)
  int nsb;
};

// A CTA covers 32 rows x PK_K complex k (PK_K / 32 sub-tiles of 32 x 32 through shared
// memory): the row offsets are computed once per CTA and the grid is PK_K / 32 times smaller
// than one CTA per sub-tile.
constexpr int PK_K = 128;
static_assert(PK_K == SB_K, "a prep tile spans exactly one scale block of A");

__device__ __forceinline__ void prep_offsets(const PrepArgs& a, int64_t* roff, int64_t* koff, int r0, int k0) {
  const int t = threadIdx.x;
  if (t < PK_K) koff[t] = (k0 + t < a.K) ? view_off(a.vk, k0 + t) : -1;
  else if (t < PK_K + 32) roff[t - PK_K] = (r0 + t - PK_K < a.R) ? view_off(a.vr, r0 + t - PK_K) : -1;
  __syncthreads();
}

__device__ __forceinline__ void load_sub(const PrepArgs& a, const float2* base, float2 (*tile)[33],
                                         const int64_t* roff, const int64_t* koff) {
  const int t = threadIdx.x, tx = t & 31, ty = t >> 5;
#pragma unroll
  for (int j = ty; j < 32; j += 8) {
    const int rr = a.k_fast ? j : tx, kk = a.k_fast ? tx : j;
    const int64_t ro = roff[rr], ko = koff[kk];
    float2 v = make_float2(0.f, 0.f);
    if (ro >= 0 && ko >= 0) v = base[ro + ko];
    if (a.conj) v.y = -v.y;
    tile[rr][kk] = v;
  }
}

__device__ __forceinline__ float prep_rowmax(const PrepArgs& a, int zz, int r) {
  if (a.mx_sample) return a.mx_sample[sample_of(a.rows_per_sample, a.z0, zz, a.nb2, r, a.mx_sample_n)];
  return a.mx[(int64_t)zz * a.Rp + r];
}

__device__ __forceinline__ const float2* prep_base(const PrepArgs& a, int zz) {
  const int z = a.z0 + zz;
  const int b1 = z / a.nb2, b2 = z - b1 * a.nb2;
  return a.X + b1 * a.s1 + b2 * a.s2;
}

// Pass 1: max |component| of every row over K (atomicMax on the IEEE bits of a non-negative
// float is order-independent, hence deterministic).
__global__ void __launch_bounds__(256) rowmax_kernel(PrepArgs a) {
  __shared__ float2 tile[32][33];
  __shared__ int64_t roff[32], koff[PK_K];
  const int r0 = blockIdx.x * 32, k0 = blockIdx.y * PK_K, zz = blockIdx.z;  // rows on x (2^31 limit)
  prep_offsets(a, roff, koff, r0, k0);
  const float2* base = prep_base(a, zz);
  const int t = threadIdx.x, tx = t & 31, ty = t >> 5;
  float m = 0.f;  // thread (ty, tx): row tx... reduced below
  __shared__ float part[8][32];
  for (int sub = 0; sub < PK_K / 32 && k0 + sub * 32 < a.K; ++sub) {
    load_sub(a, base, tile, roff, koff + sub * 32);
    __syncthreads();
    // warp ty scans 4 k columns of every row tx
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float2 v = tile[tx][ty * 4 + q];
      m = fmaxf(m, fmaxf(fabsf(v.x), fabsf(v.y)));
    }
    __syncthreads();
  }
  part[ty][tx] = m;
  __syncthreads();
  if (t < 32 && r0 + t < a.R) {
    float mm = part[0][t];
#pragma unroll
    for (int q = 1; q < 8; ++q) mm = fmaxf(mm, part[q][t]);
    if (mm > 0.f) atomicMax(reinterpret_cast<unsigned int*>(a.mx + (int64_t)zz * a.Rp + r0 + t), __float_as_uint(mm));
  }
}

// rowmax_kernel with the whole 32 x PK_K tile loaded before the scan (see prep_wide_kernel).
__global__ void __launch_bounds__(256, 4) rowmax_wide_kernel(PrepArgs a) {
  __shared__ float tile[32][PK_K + 1];
  __shared__ int64_t roff[32], koff[PK_K];
  __shared__ float part[8][32];
  const int r0 = blockIdx.x * 32, k0 = blockIdx.y * PK_K, zz = blockIdx.z;  // rows on x (2^31 limit)
  prep_offsets(a, roff, koff, r0, k0);
  const float2* base = prep_base(a, zz);
  const int t = threadIdx.x, tx = t & 31, ty = t >> 5;
  float2 v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int rr = a.k_fast ? ty + 8 * (i & 3) : tx;
    const int kk = a.k_fast ? (i >> 2) * 32 + tx : ty + 8 * i;
    const int64_t ro = roff[rr], ko = koff[kk];
    v[i] = make_float2(0.f, 0.f);
    if (ro >= 0 && ko >= 0) v[i] = base[ro + ko];
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int rr = a.k_fast ? ty + 8 * (i & 3) : tx;
    const int kk = a.k_fast ? (i >> 2) * 32 + tx : ty + 8 * i;
    tile[rr][kk] = fmaxf(fabsf(v[i].x), fabsf(v[i].y));
  }
  __syncthreads();
  float m = 0.f;  // warp ty scans 16 k columns of row tx
#pragma unroll
  for (int q = 0; q < 16; ++q) m = fmaxf(m, tile[tx][ty * 16 + q]);
  part[ty][tx] = m;
  __syncthreads();
  if (t < 32 && r0 + t < a.R) {
    float mm = part[0][t];
#pragma unroll
    for (int q = 1; q < 8; ++q) mm = fmaxf(mm, part[q][t]);
    if (mm > 0.f) atomicMax(reinterpret_cast<unsigned int*>(a.mx + (int64_t)zz * a.Rp + r0 + t), __float_as_uint(mm));
  }
}


// Pass 2: scaled FP16 hi/lo planes. KIND 0: A planes [z][Rrows][Krp], element (r, 2k+c) =
// (Re, Im)[c]. KIND 1: B_r^T planes [z][Rrows][Krp], rows 2r = (Re b, -Im b), 2r+1 = (Im b, Re b).
// Each thread converts one complex element per row and stores half2 pairs (128 B per warp).
template <int KIND>
__global__ void __launch_bounds__(256) prep_tiled_kernel(PrepArgs a) {
  __shared__ float2 tile[32][33];
  __shared__ int64_t roff[32], koff[PK_K];
  __shared__ float scl[32];
  const int r0 = blockIdx.x * 32, k0 = blockIdx.y * PK_K, zz = blockIdx.z;  // rows on x
  const int t = threadIdx.x, tx = t & 31, ty = t >> 5;
  prep_offsets(a, roff, koff, r0, k0);
  const float2* base = prep_base(a, zz);
  const int64_t plane = (int64_t)a.Rrows * a.Krp;
  __half2* hi = reinterpret_cast<__half2*>(a.hi + zz * plane);
  __half2* lo = reinterpret_cast<__half2*>(a.lo + zz * plane);
  const int kp = a.Krp >> 1;  // half2 per plane row
  for (int sub = 0; sub < PK_K / 32; ++sub) {
    const int kb = k0 + sub * 32;
    if (2 * kb >= a.Krp) break;
    load_sub(a, base, tile, roff, koff + sub * 32);
    __syncthreads();
    const int kc = kb + tx;  // complex k of this thread
    if (2 * kc < a.Krp) {
      if (KIND == 0) {
#pragma unroll
        for (int j = ty; j < 32; j += 8) {
          const int r = r0 + j;
          if (r >= a.Rrows) continue;
          const float2 v = tile[j][tx];
          const float sc = scl[j];
          __half2 h, l;
          split16x2(v.x * sc, v.y * sc, h, l);
          hi[(int64_t)r * kp + kc] = h;
          lo[(int64_t)r * kp + kc] = l;
        }
      } else {
#pragma unroll
        for (int j = ty; j < 32; j += 8) {
          const int row = 2 * (r0 + j);
          if (row >= a.Rrows) continue;
          const float2 b = tile[j][tx];
          const float sc = scl[j];
          __half2 h, l;
          split16x2(b.x * sc, -b.y * sc, h, l);
          hi[(int64_t)row * kp + kc] = h;
          lo[(int64_t)row * kp + kc] = l;
          split16x2(b.y * sc, b.x * sc, h, l);
          hi[(int64_t)(row + 1) * kp + kc] = h;
          lo[(int64_t)(row + 1) * kp + kc] = l;
        }
      }
    }
    __syncthreads();
  }
}

// Same planes as prep_tiled_kernel, but the whole 32 x PK_K tile is loaded before any store:
// 16 independent 8-byte loads per thread in flight instead of 4 per barrier-separated
// sub-tile (the sub-tile version is memory-latency bound at ~55 % of HBM bandwidth on the
// large double-layer operands).
template <int KIND>
__global__ void __launch_bounds__(256, 4) prep_wide_kernel(PrepArgs a) {
  __shared__ float2 tile[32][PK_K + 1];
  __shared__ int64_t roff[32], koff[PK_K];
  __shared__ float scl[32];
  const int r0 = blockIdx.x * 32, k0 = blockIdx.y * PK_K, zz = blockIdx.z;  // rows on x
  const int t = threadIdx.x, tx = t & 31, ty = t >> 5;
  prep_offsets(a, roff, koff, r0, k0);
  const float2* base = prep_base(a, zz);
  float2 v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int rr = a.k_fast ? ty + 8 * (i & 3) : tx;
    const int kk = a.k_fast ? (i >> 2) * 32 + tx : ty + 8 * i;
    const int64_t ro = roff[rr], ko = koff[kk];
    v[i] = make_float2(0.f, 0.f);
    if (ro >= 0 && ko >= 0) v[i] = base[ro + ko];
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int rr = a.k_fast ? ty + 8 * (i & 3) : tx;
    const int kk = a.k_fast ? (i >> 2) * 32 + tx : ty + 8 * i;
    float2 w = v[i];
    if (a.conj) w.y = -w.y;
    tile[rr][kk] = w;
  }
  __syncthreads();
  {  // this tile is one scale block of 32 rows (A) / complex columns (B); 8 threads per row
    const int j = t >> 3, q = t & 7;
    float m = 0.f;
#pragma unroll
    for (int i = 0; i < PK_K / 8; ++i) {
      const float2 w = tile[j][q + 8 * i];
      m = fmaxf(m, fmaxf(fabsf(w.x), fabsf(w.y)));
    }
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (q == 0) {
      const bool pos = m > 0.f;
      scl[j] = pos ? ldexpf(1.f, -scale_exp(m)) : 1.f;
      if (r0 + j < a.Rp) a.asc[((int64_t)zz * a.nsb + blockIdx.y) * a.Rp + r0 + j] = pos ? inv_scale(m) : 1.f;
    }
    __syncthreads();
  }
  const int64_t plane = (int64_t)a.Rrows * a.Krp;
  __half2* hi = reinterpret_cast<__half2*>(a.hi + zz * plane);
  __half2* lo = reinterpret_cast<__half2*>(a.lo + zz * plane);
  const int kp = a.Krp >> 1;  // half2 per plane row
#pragma unroll
  for (int sub = 0; sub < PK_K / 32; ++sub) {
    const int kc = k0 + sub * 32 + tx;  // complex k of this thread
    if (2 * kc >= a.Krp) break;
    if (KIND == 0) {
#pragma unroll
      for (int j = ty; j < 32; j += 8) {
        const int r = r0 + j;
        if (r >= a.Rrows) continue;
        const float2 w = tile[j][sub * 32 + tx];
        const float sc = scl[j];
        __half2 h, l;
        split16x2(w.x * sc, w.y * sc, h, l);
        hi[(int64_t)r * kp + kc] = h;
        lo[(int64_t)r * kp + kc] = l;
      }
    } else {
#pragma unroll
      for (int j = ty; j < 32; j += 8) {
        const int row = 2 * (r0 + j);
        if (row >= a.Rrows) continue;
        const float2 b = tile[j][sub * 32 + tx];
        const float sc = scl[j];
        __half2 h, l;
        split16x2(b.x * sc, -b.y * sc, h, l);
        hi[(int64_t)row * kp + kc] = h;
        lo[(int64_t)row * kp + kc] = l;
        split16x2(b.y * sc, b.x * sc, h, l);
        hi[(int64_t)(row + 1) * kp + kc] = h;
        lo[(int64_t)(row + 1) * kp + kc] = l;
      }
    }
  }
}

// A planes when K is the contiguous axis of the operand (innermost K view stride 1, even
// extent): no shared-memory transpose -- each thread streams 2 consecutive complex k of one
// row (one 16-byte load) into one half2x2 (8-byte) store per plane, 8 rows per CTA.
constexpr int PKF_ROWS = 8;
constexpr int PKF_PAIRS = 256;  // k pairs per CTA (= threads)
__global__ void __launch_bounds__(256) prep_kfast_kernel(PrepArgs a) {
  // a CTA covers 8 rows x 512 complex k = four scale blocks; warp w holds complex k
  // [64 w, 64 w + 64) of the CTA, so a scale block is warps (2b, 2b + 1)
  static_assert(PKF_PAIRS * 2 == 4 * SB_K, "kfast CTA = four scale blocks");
  __shared__ int64_t roff[PKF_ROWS];
  __shared__ float wmax[8][PKF_ROWS];
  const int r0 = blockIdx.x * PKF_ROWS, zz = blockIdx.z;  // rows on x (2^31 limit)
  const int t = threadIdx.x, w = t >> 5, lane = t & 31;
  if (t < PKF_ROWS) {
    const int r = r0 + t;
    roff[t] = (r < a.R) ? view_off(a.vr, r) : -1;
  }
  const int kpair = blockIdx.y * PKF_PAIRS + t;  // complex k = 2 kpair, 2 kpair + 1
  const int k = 2 * kpair;
  const bool in_plane = 2 * k < a.Krp;           // plane columns 2k .. 2k+3
  const bool in_k = k < a.K;                      // K even on this path: k + 1 < K too
  const int64_t ko = in_k ? view_off(a.vk, k) : 0;
  __syncthreads();
  const float2* base = prep_base(a, zz);
  float4 v[PKF_ROWS];
  float m8[PKF_ROWS];
#pragma unroll
  for (int j = 0; j < PKF_ROWS; ++j) {
    v[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (in_k && roff[j] >= 0) v[j] = *reinterpret_cast<const float4*>(base + roff[j] + ko);
    if (a.conj) {
      v[j].y = -v[j].y;
      v[j].w = -v[j].w;
    }
    m8[j] = fmaxf(fmaxf(fabsf(v[j].x), fabsf(v[j].y)), fmaxf(fabsf(v[j].z), fabsf(v[j].w)));
  }
  // warp max of the 8 rows in 9 shuffles: halve the rows per lane while doubling the lanes
  // covered (offsets 16, 8, 4), then reduce the remaining row over 4 lanes
  static_assert(PKF_ROWS == 8, "row-halving reduction assumes 8 rows");
  const bool u16 = lane & 16, u8 = lane & 8, u4 = lane & 4;
  float m4[4], m2[2];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float send = u16 ? m8[i] : m8[i + 4];
    const float keep = u16 ? m8[i + 4] : m8[i];
    m4[i] = fmaxf(keep, __shfl_xor_sync(0xffffffffu, send, 16));
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const float send = u8 ? m4[i] : m4[i + 2];
    const float keep = u8 ? m4[i + 2] : m4[i];
    m2[i] = fmaxf(keep, __shfl_xor_sync(0xffffffffu, send, 8));
  }
  float m1 = fmaxf(u4 ? m2[1] : m2[0], __shfl_xor_sync(0xffffffffu, u4 ? m2[0] : m2[1], 4));
  m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, 2));
  m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, 1));
  if ((lane & 3) == 0) wmax[w][(u16 ? 4 : 0) + (u8 ? 2 : 0) + (u4 ? 1 : 0)] = m1;
  __syncthreads();
  const int sb = blockIdx.y * 4 + (w >> 1);  // scale block of this warp
  if (!in_plane) return;
  const int64_t plane = (int64_t)a.Rrows * a.Krp;
  uint2* hi = reinterpret_cast<uint2*>(a.hi + zz * plane);
  uint2* lo = reinterpret_cast<uint2*>(a.lo + zz * plane);
  const int kq = a.Krp >> 2;  // uint2 (4 halves) per plane row
#pragma unroll
  for (int j = 0; j < PKF_ROWS; ++j) {
    const int r = r0 + j;
    if (r >= a.Rrows) break;
    const float m = fmaxf(wmax[w & ~1][j], wmax[w | 1][j]);
    const bool pos = m > 0.f;
    const float sc = pos ? ldexpf(1.f, -scale_exp(m)) : 1.f;
    if (lane == 0 && (w & 1) == 0) a.asc[((int64_t)zz * a.nsb + sb) * a.Rp + r] = pos ? inv_scale(m) : 1.f;
    __half2 h0, l0, h1, l1;
    split16x2(v[j].x * sc, v[j].y * sc, h0, l0);
    split16x2(v[j].z * sc, v[j].w * sc, h1, l1);
    uint2 hv, lv;
    hv.x = *reinterpret_cast<uint32_t*>(&h0);
    hv.y = *reinterpret_cast<uint32_t*>(&h1);
    lv.x = *reinterpret_cast<uint32_t*>(&l0);
    lv.y = *reinterpret_cast<uint32_t*>(&l1);
    hi[(int64_t)r * kq + kpair] = hv;
    lo[(int64_t)r * kq + kpair] = lv;
  }
}


// 3M operand planes: six K-major FP16 planes [z][Rrows][Krp] (Krp = padded complex K) at
// stride pstride elements: (Xr, Xi, Xr + Xi) x (hi, lo) of the row-scaled operand (conj
// applied first). Same gather as prep_wide_kernel (whole 32 x PK_K tile loaded first); each
// thread then writes two consecutive k of one row as half2 into every plane.
__global__ void __launch_bounds__(256, 4) prep3m_wide_kernel(PrepArgs a, int64_t pstride) {
  __shared__ float2 tile[32][PK_K + 1];
  __shared__ int64_t roff[32], koff[PK_K];
  __shared__ float scl[32];
  const int r0 = blockIdx.x * 32, k0 = blockIdx.y * PK_K, zz = blockIdx.z;
  const int t = threadIdx.x, tx = t & 31, ty = t >> 5;
  if (t >= 224) {
    const int i = t - 224;
    const float m = (r0 + i < a.R) ? prep_rowmax(a, zz, r0 + i) : 0.f;
    scl[i] = (m > 0.f) ? ldexpf(1.f, -scale_exp(m)) : 1.f;
  }
  prep_offsets(a, roff, koff, r0, k0);
  const float2* base = prep_base(a, zz);
  float2 v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int rr = a.k_fast ? ty + 8 * (i & 3) : tx;
    const int kk = a.k_fast ? (i >> 2) * 32 + tx : ty + 8 * i;
    const int64_t ro = roff[rr], ko = koff[kk];
    v[i] = make_float2(0.f, 0.f);
    if (ro >= 0 && ko >= 0) v[i] = base[ro + ko];
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int rr = a.k_fast ? ty + 8 * (i & 3) : tx;
    const int kk = a.k_fast ? (i >> 2) * 32 + tx : ty + 8 * i;
    float2 w = v[i];
    if (a.conj) w.y = -w.y;
    tile[rr][kk] = w;
  }
  __syncthreads();
  const int64_t plane = (int64_t)a.Rrows * a.Krp;
  const int kp = a.Krp >> 1;  // half2 per plane row
#pragma unroll
  for (int it = 0; it < 8; ++it) {
    const int item = t + 256 * it;  // (row, k pair): 32 x 64
    const int r = item >> 6, kq = item & 63;
    const int row = r0 + r, kc = (k0 >> 1) + kq;  // half2 index within the plane row
    if (row >= a.Rrows || 2 * kc >= a.Krp) continue;
    const float2 x0 = tile[r][2 * kq], x1 = tile[r][2 * kq + 1];
    const float sc = scl[r];
    const float re0 = x0.x * sc, im0 = x0.y * sc, re1 = x1.x * sc, im1 = x1.y * sc;
    __half2 h, l;
    __half2* P = reinterpret_cast<__half2*>(a.hi + zz * plane) + (int64_t)row * kp + kc;
    split16x2(re0, re1, h, l);
    P[0] = h;
    P[pstride >> 1] = l;
    split16x2(im0, im1, h, l);
    P[2 * (pstride >> 1)] = h;
    P[3 * (pstride >> 1)] = l;
    split16x2(re0 + im0, re1 + im1, h, l);
    P[4 * (pstride >> 1)] = h;
    P[5 * (pstride >> 1)] = l;
  }
}

// 3M planes of a K-contiguous operand (no transpose): 8 rows per CTA, each thread two
// consecutive complex k (one 16-byte load) -> one half2 per plane.
__global__ void __launch_bounds__(256) prep3m_kfast_kernel(PrepArgs a, int64_t pstride) {
  __shared__ int64_t roff[PKF_ROWS];
  __shared__ float scl[PKF_ROWS];
  const int r0 = blockIdx.x * PKF_ROWS, zz = blockIdx.z;
  const int t = threadIdx.x;
  if (t < PKF_ROWS) {
    const int r = r0 + t;
    roff[t] = (r < a.R) ? view_off(a.vr, r) : -1;
    const float m = (r < a.R) ? prep_rowmax(a, zz, r) : 0.f;
    scl[t] = (m > 0.f) ? ldexpf(1.f, -scale_exp(m)) : 1.f;
  }
  const int kpair = blockIdx.y * PKF_PAIRS + t;  // complex k = 2 kpair, 2 kpair + 1
  const int k = 2 * kpair;
  const bool in_plane = k < a.Krp;
  const bool in_k = k < a.K;
  const int64_t ko = in_k ? view_off(a.vk, k) : 0;
  __syncthreads();
  if (!in_plane) return;
  const float2* base = prep_base(a, zz);
  const int64_t plane = (int64_t)a.Rrows * a.Krp;
  const int kp = a.Krp >> 1;
#pragma unroll
  for (int j = 0; j < PKF_ROWS; ++j) {
    const int r = r0 + j;
    if (r >= a.Rrows) break;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (in_k && roff[j] >= 0) v = *reinterpret_cast<const float4*>(base + roff[j] + ko);
    if (a.conj) {
      v.y = -v.y;
      v.w = -v.w;
    }
    const float sc = scl[j];
    const float re0 = v.x * sc, im0 = v.y * sc, re1 = v.z * sc, im1 = v.w * sc;
    __half2 h, l;
    __half2* P = reinterpret_cast<__half2*>(a.hi + zz * plane) + (int64_t)r * kp + kpair;
    split16x2(re0, re1, h, l);
    P[0] = h;
    P[pstride >> 1] = l;
    split16x2(im0, im1, h, l);
    P[2 * (pstride >> 1)] = h;
    P[3 * (pstride >> 1)] = l;
    split16x2(re0 + im0, re1 + im1, h, l);
    P[4 * (pstride >> 1)] = h;
    P[5 * (pstride >> 1)] = l;
  }
}

// ---------------------------------------------------------------------------------------
// 3M (Gauss) complex GEMM on the CTA pair. C = A B is formed from three real products
//   T1 = Ar Br,  T2 = Ai Bi,  T3 = (Ar + Ai)(Br + Bi);   Cr = T1 - T2,  Ci = T3 - T1 - T2
// instead of the four real products of the [Re -Im; Im Re] embedding: with the FP16x3 split
// (hi.hi + hi.lo + lo.hi per product) a complex MAC issues 9 FP16 MACs instead of 12.
// Operands are six FP16 planes each (Xr, Xi, Xr + Xi as hi/lo, K-major [rows][K], K = the
// complex K, exact power-of-two row / column scales as in the 4M path), streamed by TMA in
// 16-wide K blocks (SWIZZLE_32B rows) through a 5-stage ring.
// Accumulators: the three products need three 128-column FP32 accumulators in TMEM; the
// fourth 128-column slot rotates so that the chunk promotion (the tensor core's FP32
// accumulation truncates, so partial sums are moved into FP32 registers every 1024 complex
// K) never stalls the MMA: the products restart their accumulation segments staggered by a
// third of a chunk (product j at k-steps (j+1) C/3 + m C), so exactly one segment ends at a
// time, segment i ending when segment i + 3 starts; segment i lives in slot i mod 4 and is
// drained by the epilogue warps (Cr/Ci registers, signs per product) while the next ones run.
constexpr int M3_BK = 16;                              // complex K per stage (32-byte rows)
constexpr int M3_STAGES = 5;
constexpr int M3_NC = 128;                             // complex columns per tile (MMA N = 128)
constexpr int M3_APLANE = 128 * M3_BK * 2;             // 4 KB: 128 rows of one A plane (per CTA)
constexpr int M3_BPLANE = 64 * M3_BK * 2;              // 2 KB: 64 rows of one B plane (per CTA)
constexpr int M3_STAGE = 6 * M3_APLANE + 6 * M3_BPLANE;  // 36 KB
constexpr int M3_SMEM = M3_STAGES * M3_STAGE + EPI_STAGE_BYTES + EPI_COLSC_BYTES + 1024 + 512;
constexpr int M3_C = 64;                               // k-steps (16 complex K) per segment: 1024 K

struct Maps12 {
  CUtensorMap m[12];  // A planes 0..5 (Ar hi/lo, Ai hi/lo, As hi/lo), then B planes 0..5
};

__device__ __forceinline__ uint64_t smem_desc64(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((256 >> 4) & 0x3FFF) << 32;  // SBO: 8-row atoms of 32 B
  d |= (uint64_t)1 << 46;                      // descriptor version (sm_100)
  d |= (uint64_t)6 << 61;                      // SWIZZLE_32B
  return d;
}

// product j starts a new accumulation segment at k-step q
__device__ __forceinline__ bool m3_start(int j, int q) {
  if (q == 0) return true;
  const int off = ((j + 1) * M3_C) / 3;
  return q >= off && ((q - off) % M3_C) == 0;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(TC_THREADS, 1)
    tc_gemm3m_kernel(const __grid_constant__ Maps12 maps, TcParams p, int npm, int nn, int ntiles) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + M3_STAGES * M3_STAGE);
  uint64_t* empty = full + M3_STAGES;
  uint64_t* slot_full = empty + M3_STAGES;
  uint64_t* slot_empty = slot_full + 4;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(slot_empty + 4);
  float2* epi_stage = reinterpret_cast<float2*>(smem + M3_STAGES * M3_STAGE + 512);
  float* epi_colsc = reinterpret_cast<float*>(smem + M3_STAGES * M3_STAGE + 512 + EPI_STAGE_BYTES);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const int cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < M3_STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(&slot_full[i], 1);
      mbar_init(&slot_empty[i], 16);  // leader: 8 epilogue warps of each CTA
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int i = 0; i < 12; ++i) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&maps.m[i])));
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster_sync_all();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer (both CTAs)
      const uint32_t full0 = map_to_rank(smem_u32(&full[0]), 0);
      int i = 0;
      for (int t = cluster; t < ntiles; t += nclusters) {
        const PairTile tl = pair_tile(p, t, npm, nn);
        const int mrow = (tl.mblk0 + (int)rank) * 128;
        const int brow = tl.nblk * M3_NC + (int)rank * 64;
        const int bz = p.b_batched ? tl.z : 0;
        for (int q = 0; q < tl.nkb; ++q, ++i) {
          const int kb = tl.kb0 + q;
          const int s = i % M3_STAGES;
          const uint32_t ph = (i / M3_STAGES) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t* st = smem + s * M3_STAGE;
          if (rank == 0) mbar_expect_tx(&full[s], 2 * M3_STAGE);
          const uint32_t fb = full0 + (uint32_t)(s * sizeof(uint64_t));
#pragma unroll
          for (int pl = 0; pl < 6; ++pl) tma_load_3d_pair(st + pl * M3_APLANE, &maps.m[pl], kb * M3_BK, mrow, tl.z, fb);
#pragma unroll
          for (int pl = 0; pl < 6; ++pl)
            tma_load_3d_pair(st + 6 * M3_APLANE + pl * M3_BPLANE, &maps.m[6 + pl], kb * M3_BK, brow, bz, fb);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {  // MMA issuer (leader CTA only)
      // kind::f16 instruction descriptor: D f32, A/B f16, K-major both, N=128, M=256
      const uint32_t idesc = (1u << 4) | ((uint32_t)(M3_NC >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
      int i = 0, seg = 0;
      int slot_of[3] = {0, 0, 0};
      for (int t = cluster; t < ntiles; t += nclusters) {
        const PairTile tl = pair_tile(p, t, npm, nn);
        for (int qb = 0; qb < tl.nkb; ++qb, ++i) {
          const int s = i % M3_STAGES;
          mbar_wait(&full[s], (i / M3_STAGES) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t base = smem_u32(smem + s * M3_STAGE);
#pragma unroll
          for (int kk = 0; kk < M3_BK / TC_UK; ++kk) {
            const int q = qb * (M3_BK / TC_UK) + kk;
            const uint64_t adv = (uint64_t)((kk * TC_UK * 2) >> 4);
#pragma unroll
            for (int j = 0; j < 3; ++j) {
              uint32_t acc = 1u;
              if (m3_start(j, q)) {
                if (q > 0) mma_commit_pair(&slot_full[slot_of[j]]);  // product j's segment is complete
                const int sl = seg & 3;
                mbar_wait(&slot_empty[sl], ((seg >> 2) & 1) ^ 1);
                asm volatile("tcgen05.fence::after_thread_sync;");
                slot_of[j] = sl;
                ++seg;
                acc = 0u;
              }
              const uint32_t dacc = tmem + (uint32_t)(slot_of[j] * M3_NC);
              const uint64_t ahi = smem_desc64(base + (2 * j) * M3_APLANE) + adv;
              const uint64_t alo = smem_desc64(base + (2 * j + 1) * M3_APLANE) + adv;
              const uint64_t bhi = smem_desc64(base + 6 * M3_APLANE + (2 * j) * M3_BPLANE) + adv;
              const uint64_t blo = smem_desc64(base + 6 * M3_APLANE + (2 * j + 1) * M3_BPLANE) + adv;
              mma_f16_pair(dacc, ahi, bhi, idesc, acc);
              mma_f16_pair(dacc, ahi, blo, idesc, 1u);
              mma_f16_pair(dacc, alo, bhi, idesc, 1u);
            }
          }
          mma_commit_pair(&empty[s]);
        }
        // tile end: the three live segments, in segment-index order (= start order j0, j1, j2
        // cyclically; the latest-started product is the last)
        const int T = tl.nkb * (M3_BK / TC_UK);
        int last_j = 2;  // product of the most recently started segment
        for (int q = T - 1; q >= 0; --q) {
          bool found = false;
          for (int j = 2; j >= 0 && !found; --j)
            if (m3_start(j, q)) {
              last_j = j;
              found = true;
            }
          if (found) break;
        }
        for (int r = 1; r <= 3; ++r) mma_commit_pair(&slot_full[slot_of[(last_j + r) % 3]]);
      }
    }
    __syncwarp();
  } else {
    // epilogue (both CTAs): warp w drains TMEM lanes 32*(w%4).. (its rows) and complex
    // columns [64 h, 64 h + 64) of each segment's slot, h = (w-2)/4, into Cr / Ci registers
    const int lg = warp & 3;
    const int half = (warp - 2) >> 2;
    const uint32_t slot_empty0 = map_to_rank(smem_u32(&slot_empty[0]), 0);
    int seg = 0;
    for (int t = cluster; t < ntiles; t += nclusters) {
      const PairTile tl = pair_tile(p, t, npm, nn);
      const int row = (tl.mblk0 + (int)rank) * 128 + lg * 32 + lane;
      float acc[128];  // acc[2c] = Cr, acc[2c+1] = Ci of complex column c of this warp's half
#pragma unroll
      for (int i = 0; i < 128; ++i) acc[i] = 0.f;
      const int T = tl.nkb * (M3_BK / TC_UK);
      for (int q = 0; q < T; ++q) {
        for (int j = 0; j < 3; ++j) {
          if (!m3_start(j, q)) continue;
          const int sl = seg & 3;
          mbar_wait(&slot_full[sl], (seg >> 2) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          // segment seg = the seg-th start event (this one): product j, drained in index order
#pragma unroll
          for (int cc = 0; cc < 64; cc += 16) {
            uint32_t v[16];
            const uint32_t taddr = tmem + ((uint32_t)(lg * 32) << 16) + (uint32_t)(sl * M3_NC + half * 64 + cc);
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
                "[%16];"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                  "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                  "=r"(v[15])
                : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            const int jp = j;
#pragma unroll
            for (int i2 = 0; i2 < 16; ++i2) {
              const float x = __uint_as_float(v[i2]);
              const int c = cc + i2;
              if (jp == 0) {
                acc[2 * c] += x;
                acc[2 * c + 1] -= x;
              } else if (jp == 1) {
                acc[2 * c] -= x;
                acc[2 * c + 1] -= x;
              } else {
                acc[2 * c + 1] += x;
              }
            }
          }
          asm volatile("tcgen05.fence::before_thread_sync;");
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(slot_empty0 + (uint32_t)(sl * sizeof(uint64_t)));
          ++seg;
        }
      }
      // Coalesced output: each warp stages 32 rows x 8 complex columns in shared memory
      // (padded rows), then writes 4 rows per store instruction (8 lanes x 8 B = 64 B each),
      // instead of 32 scattered rows per instruction.
      {
        const int z = tl.z, bz = p.b_batched ? z : 0;
        const int row0 = (tl.mblk0 + (int)rank) * 128 + lg * 32;
        const float rs = (row < p.M) ? inv_scale(row_amax(p, z, row)) : 0.f;
        float lmax = 0.f;
        const float* bmx = p.bmax + (int64_t)bz * p.Np;
        const int n0 = tl.nblk * M3_NC + half * 64;
        float2* base;
        int64_t ld;
        bool acc_out = false;
        if (p.ksplit > 1) {
          base = p.ws + tl.split * p.ws_split + (int64_t)z * p.M * p.N;
          ld = p.N;
        } else {
          const int b1 = (p.z0 + z) / p.nb2, b2 = (p.z0 + z) - b1 * p.nb2;
          base = p.C + b1 * p.sc1 + b2 * p.sc2;
          ld = p.cm;
          acc_out = p.accumulate != 0;
        }
        float2* stg = epi_stage + (warp - 2) * 32 * (EPI_Q + 1);
        // the tile's 64 column scales, once per warp (all lanes share the columns)
        float* csc = epi_colsc + (warp - 2) * 64;
        {
          const int na = n0 + lane, nb = n0 + lane + 32;
          csc[lane] = (na < p.N) ? inv_scale(bmx[na]) : 0.f;
          csc[lane + 32] = (nb < p.N) ? inv_scale(bmx[nb]) : 0.f;
        }
        __syncwarp();
        const int sub = lane >> 3, col = lane & 7;
        // per-sample output bounds: one per warp when its 32 rows belong to one sample (always,
        // unless a sample's row count is not a multiple of 32), else one atomic per element
        const int s_lo = sample_of(p.rows_per_sample, p.z0, z, p.nb2, row0, p.amax_out_n);
        const bool s_mixed = p.amax_out && p.ksplit == 1 &&
                             sample_of(p.rows_per_sample, p.z0, z, p.nb2, min(row0 + 31, p.M - 1), p.amax_out_n) != s_lo;
#pragma unroll
        for (int q0 = 0; q0 < 64; q0 += EPI_Q) {
#pragma unroll
          for (int q = 0; q < EPI_Q; ++q) {
            const float sc = rs * csc[q0 + q];
            stg[lane * (EPI_Q + 1) + q] = make_float2(acc[2 * (q0 + q)] * sc, acc[2 * (q0 + q) + 1] * sc);
          }
          __syncwarp();
          const int n = n0 + q0 + col;
#pragma unroll 4
          for (int r = 0; r < 32; r += 4) {
            const int rr = r + sub, grow = row0 + rr;
            if (grow < p.M && n < p.N) {
              float2 val = stg[rr * (EPI_Q + 1) + col];
              float2* dst = base + (int64_t)grow * ld + n;
              if (acc_out) {
                const float2 o = *dst;
                val.x += o.x;
                val.y += o.y;
              }
              *dst = val;
              const float mv = fmaxf(fabsf(val.x), fabsf(val.y));
              if (s_mixed)
                atomic_max_nonneg(p.amax_out + sample_of(p.rows_per_sample, p.z0, z, p.nb2, grow, p.amax_out_n), mv);
              lmax = fmaxf(lmax, mv);
            }
          }
          __syncwarp();
        }
        if (p.amax_out && p.ksplit == 1 && !s_mixed) {
          lmax = warp_max(lmax);
          if (lane == 0) atomic_max_nonneg(p.amax_out + s_lo, lmax);
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  cluster_sync_all();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

// TN_PREP_WIDE=0 selects the sub-tile prep kernel (A/B measurement only)
bool prep_wide_on() {
  static const bool on = !(getenv("TN_PREP_WIDE") && std::atoi(getenv("TN_PREP_WIDE")) == 0);
  return on;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    TN_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess) throw Error(-5, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

CUtensorMap make_map(__half* base, int inner, int rows, int nz, int box_rows) {
  CUtensorMap m;
  cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)rows, (cuuint64_t)nz};
  cuuint64_t strides[2] = {(cuuint64_t)inner * 2, (cuuint64_t)inner * rows * 2};
  cuuint32_t box[3] = {(cuuint32_t)TC_BK, (cuuint32_t)box_rows, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, base, dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(-5, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return m;
}

// 3M planes: K-major FP16 rows of M3_BK = 16 elements (32 B), SWIZZLE_32B
CUtensorMap make_map64(__half* base, int inner, int rows, int nz, int box_rows) {
  CUtensorMap m;
  cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)rows, (cuuint64_t)nz};
  cuuint64_t strides[2] = {(cuuint64_t)inner * 2, (cuuint64_t)inner * rows * 2};
  cuuint32_t box[3] = {(cuuint32_t)M3_BK, (cuuint32_t)box_rows, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, base, dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(-5, "cuTensorMapEncodeTiled (64B) failed: " + std::to_string((int)r));
  return m;
}

inline int rup(int x, int m) { return (x + m - 1) / m * m; }

// TN_GEMM_LOG=1: per-shape device time of the tensor-core GEMMs (prep + kernel), printed by
// tn_debug_gemm_log() -- instrumentation for tuning only.
struct ShapeRec {
  std::string key;
  cudaEvent_t a, b, c;  // a: before prep, b: before kernel, c: after
  double cm;
};
std::vector<ShapeRec> g_shape_pending;
std::map<std::string, std::array<double, 4>> g_shape_tab;  // count, prep ms, kernel ms, cmacs
bool shape_log_on() {
  static int on = -1;
  if (on < 0) on = getenv("TN_GEMM_LOG") ? 1 : 0;
  return on == 1;
}
void shape_flush() {
  for (auto& r : g_shape_pending) {
    cudaEventSynchronize(r.c);
    float t1 = 0, t2 = 0;
    cudaEventElapsedTime(&t1, r.a, r.b);
    cudaEventElapsedTime(&t2, r.b, r.c);
    auto& e = g_shape_tab[r.key];
    e[0] += 1;
    e[1] += t1;
    e[2] += t2;
    e[3] += r.cm;
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
    cudaEventDestroy(r.c);
  }
  g_shape_pending.clear();
}

}  // namespace

// Per-sample work (complex MACs) above which the tensor-core path is used. The decision
// depends on per-sample shapes only, so results do not depend on the batch size.
static const double kTcMinWork = 1 << 20;

}  // namespace tn

extern "C" int tn_debug_gemm_log(void) {
  tn::shape_flush();
  std::vector<std::pair<double, std::string>> rows;
  for (auto& kv : tn::g_shape_tab) rows.push_back({kv.second[1] + kv.second[2], kv.first});
  std::sort(rows.rbegin(), rows.rend());
  for (size_t i = 0; i < rows.size() && i < 40; ++i) {
    auto& e = tn::g_shape_tab[rows[i].second];
    fprintf(stderr, "%-60s n=%6.0f prep=%9.1f ms kern=%9.1f ms  %.1f TF alg\n", rows[i].second.c_str(), e[0], e[1],
            e[2], e[2] > 0 ? 8.0 * e[3] / (e[2] * 1e-3) / 1e12 : 0.0);
  }
  return (int)rows.size();
}

namespace tn {

int g_zc_max = 0;  // > 0: at most this many batch elements per A-plane chunk (tn_debug_set_zc)
int g_m3_override = -1;  // >= 0: overrides TN_3M (tn_debug_set_3m; tests)

bool tc_eligible(const Ctx& c, int64_t M, int64_t N, int64_t K, int64_t work_per_sample) {
  if (c.gemm_mode == 1) return false;
  if (M <= 0 || N <= 0 || K <= 0) return false;
  if (c.gemm_mode == 2) return true;
  double work = work_per_sample > 0 ? (double)work_per_sample : (double)M * N * K;
  return work >= kTcMinWork && N >= 32 && K >= 8;
}

// Co-resident CTA pairs of a cluster kernel (a persistent grid larger than this would run its
// surplus clusters as a serial second wave), per device.
template <class K>
int coresident_pairs(K kernel, int smem, std::atomic<int>* cache, int dev) {
  int n = cache[dev & 63].load();
  if (n) return n;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148, 1, 1);
  cfg.blockDim = dim3(TC_THREADS, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at;
  at.id = cudaLaunchAttributeClusterDimension;
  at.val.clusterDim.x = 2;
  at.val.clusterDim.y = 1;
  at.val.clusterDim.z = 1;
  cfg.attrs = &at;
  cfg.numAttrs = 1;
  if (cudaOccupancyMaxActiveClusters(&n, (void*)kernel, &cfg) != cudaSuccess || n < 1) {
    cudaGetLastError();
    n = 64;
  }
  n = std::min(n, 74);
  cache[dev & 63].store(n);
  if (getenv("TN_GEMM_LOG")) fprintf(stderr, "coresident CTA pairs: %d\n", n);
  return n;
}

// The 3M (Gauss) path: six FP16 planes per operand, tc_gemm3m_kernel (see above).
void gemm_tc3m(Ctx& c, const GemmDesc& g, int dev, cudaEvent_t ev_kernel) {
  static std::atomic<uint64_t> attr_done{0};
  const uint64_t dbit = 1ull << (dev & 63);
  if (!(attr_done.load() & dbit)) {
    TN_CUDA(cudaFuncSetAttribute(tc_gemm3m_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, M3_SMEM));
    attr_done.fetch_or(dbit);
  }
  const int Kp = rup(g.K, M3_BK);
  const int Mp = rup(g.M, 2 * TC_BM);
  const int Np = rup(g.N, M3_NC);
  const int nbz = g.nb1 * g.nb2;
  const bool b_batched = (g.sb1 != 0 && g.nb1 > 1) || (g.sb2 != 0 && g.nb2 > 1);
  auto simple = [](int64_t dim, int64_t stride) {
    View4 v;
    v.rank = 1;
    v.dims[0] = (int)dim;
    v.str[0] = stride;
    return v;
  };
  auto inner_unit = [](const View4& v) { return v.rank > 0 && v.str[v.rank - 1] == 1; };
  const int rows_per_sample = g.nb1 > 1 ? 0 : (g.m_per_sample > 0 ? g.m_per_sample : g.M);
  // ---- B planes [6][nzb][Np][Kp]
  const int nzb = b_batched ? nbz : 1;
  const int64_t bstride = (int64_t)nzb * Np * Kp;
  DevBuf b3((size_t)6 * bstride * 2, c.stream);
  DevBuf bmx((size_t)nzb * Np * sizeof(float), c.stream);
  TN_CUDA(cudaMemsetAsync(bmx.p, 0, (size_t)nzb * Np * sizeof(float), c.stream));
  if (g.amaxC) TN_CUDA(cudaMemsetAsync(g.amaxC, 0, sizeof(float) * std::max(1, g.amaxC_n), c.stream));
  for (int zb0 = 0; zb0 < nzb; zb0 += 65535) {
    const int nzc = std::min(65535, nzb - zb0);
    PrepArgs a;
    a.X = g.B;
    a.vr = g.vbn.rank ? g.vbn : simple(g.N, g.bn);
    a.vk = g.vbk.rank ? g.vbk : simple(g.K, g.bk);
    a.conj = g.conjB;
    a.nb2 = g.nb2;
    a.s1 = b_batched ? g.sb1 : 0;
    a.s2 = b_batched ? g.sb2 : 0;
    a.z0 = zb0;
    a.R = g.N;
    a.K = g.K;
    a.Rrows = Np;
    a.Krp = Kp;
    a.k_fast = inner_unit(a.vk) || !inner_unit(a.vr);
    a.mx = bmx.as<float>() + (int64_t)zb0 * Np;
    a.mx_sample = nullptr;
    a.mx_sample_n = 0;
    a.rows_per_sample = 0;
    a.Rp = Np;
    a.hi = b3.as<__half>() + (int64_t)zb0 * Np * Kp;
    a.lo = nullptr;
    dim3 gmax(ceil_div(g.N, 32), ceil_div(g.K, PK_K), nzc);
    rowmax_wide_kernel<<<gmax, 256, 0, c.stream>>>(a);
    TN_LAUNCHED();
    dim3 grid(Np / 32, ceil_div(Kp, PK_K), nzc);
    prep3m_wide_kernel<<<grid, 256, 0, c.stream>>>(a, bstride);
    TN_LAUNCHED();
  }
  // ---- split-K from per-sample shapes only; splits are whole segments (1024 complex K)
  const int kblocks = Kp / M3_BK;
  const int seg_blocks = M3_C * TC_UK / M3_BK;
  const int mps = g.m_per_sample > 0 ? g.m_per_sample : g.M;
  const int64_t tiles_ps = (int64_t)((mps + TC_BM - 1) / TC_BM) * (Np / M3_NC) * g.nb2;
  int ksplit = 1, kbps = kblocks;
  if (tiles_ps < 148 && kblocks >= 2 * seg_blocks) {
    int want = (int)std::min<int64_t>(32, (2 * 148 + tiles_ps - 1) / tiles_ps);
    int maxs = kblocks / seg_blocks;
    ksplit = std::max(1, std::min(want, maxs));
    kbps = ((kblocks + ksplit - 1) / ksplit + seg_blocks - 1) / seg_blocks * seg_blocks;
    ksplit = (kblocks + kbps - 1) / kbps;
  }
  static const bool uniform_off = getenv("TN_ROWSCALE") && std::atoi(getenv("TN_ROWSCALE")) != 0;
  const bool use_uniform = g.amaxA != nullptr && !uniform_off;
  // ---- A planes [6][zc][Mp][Kp], chunked over the batch (<= ~1.5 GB of planes per chunk)
  const int64_t per_z = (int64_t)Mp * Kp;
  const int zc0 = (int)std::max<int64_t>(
      1, std::min<int64_t>({(int64_t)nbz, (int64_t)(65535 / ksplit), (int64_t)(1ll << 27) / std::max<int64_t>(1, per_z)}));
  const int zc = g_zc_max > 0 ? std::min(zc0, g_zc_max) : zc0;
  const int64_t astride = (int64_t)zc * per_z;
  DevBuf a3((size_t)6 * astride * 2, c.stream);
  DevBuf amx((size_t)zc * Mp * sizeof(float), c.stream);
  DevBuf ws;
  const int64_t ws_split = (int64_t)zc * g.M * g.N;
  if (ksplit > 1) ws.alloc((size_t)ksplit * ws_split * sizeof(float2), c.stream);
  const int nclusters_max = [&] {
    static std::atomic<int> cache[64];
    return coresident_pairs(tc_gemm3m_kernel, M3_SMEM, cache, dev);
  }();
  for (int z0 = 0; z0 < nbz; z0 += zc) {
    const int nz = std::min(zc, nbz - z0);
    PrepArgs a;
    a.X = g.A;
    a.vr = g.vam.rank ? g.vam : simple(g.M, g.am);
    a.vk = g.vak.rank ? g.vak : simple(g.K, g.ak);
    a.conj = g.conjA;
    a.nb2 = g.nb2;
    a.s1 = g.sa1;
    a.s2 = g.sa2;
    a.z0 = z0;
    a.R = g.M;
    a.K = g.K;
    a.Rrows = Mp;
    a.Krp = Kp;
    a.k_fast = inner_unit(a.vk) || !inner_unit(a.vr);
    a.mx = amx.as<float>();
    a.mx_sample = use_uniform ? g.amaxA : nullptr;
    a.mx_sample_n = std::max(1, g.amaxA_n);
    a.rows_per_sample = rows_per_sample;
    a.Rp = Mp;
    a.hi = a3.as<__half>();
    a.lo = nullptr;
    if (!use_uniform) {
      TN_CUDA(cudaMemsetAsync(amx.p, 0, (size_t)nz * Mp * sizeof(float), c.stream));
      dim3 gmax(ceil_div(g.M, 32), ceil_div(g.K, PK_K), nz);
      rowmax_wide_kernel<<<gmax, 256, 0, c.stream>>>(a);
      TN_LAUNCHED();
    }
    const View4& vk = a.vk;
    bool kfast = vk.rank > 0 && vk.str[vk.rank - 1] == 1 && vk.dims[vk.rank - 1] % 2 == 0 && g.K % 2 == 0 &&
                 (reinterpret_cast<uintptr_t>(g.A) & 15) == 0 && a.s1 % 2 == 0 && a.s2 % 2 == 0;
    for (int d = 0; d < vk.rank - 1 && kfast; ++d) kfast = vk.str[d] % 2 == 0;
    for (int d = 0; d < a.vr.rank && kfast; ++d) kfast = a.vr.str[d] % 2 == 0 || a.vr.dims[d] == 1;
    if (kfast) {
      dim3 grid(ceil_div(Mp, PKF_ROWS), ceil_div(Kp / 2, PKF_PAIRS), nz);
      prep3m_kfast_kernel<<<grid, 256, 0, c.stream>>>(a, astride);
    } else {
      dim3 grid(Mp / 32, ceil_div(Kp, PK_K), nz);
      prep3m_wide_kernel<<<grid, 256, 0, c.stream>>>(a, astride);
    }
    TN_LAUNCHED();
    Maps12 maps;
    for (int pl = 0; pl < 6; ++pl) {
      maps.m[pl] = make_map64(a3.as<__half>() + pl * astride, Kp, Mp, nz, 128);
      maps.m[6 + pl] = make_map64(b3.as<__half>() + pl * bstride + (b_batched ? (int64_t)z0 * Np * Kp : 0), Kp,
                                  Np, b_batched ? nz : 1, 64);
    }
    TcParams p;
    p.M = g.M;
    p.N = g.N;
    p.kblocks = kblocks;
    p.ksplit = ksplit;
    p.kb_per_split = kbps;
    p.ws = ws.as<float2>();
    p.ws_split = ws_split;
    p.b_batched = b_batched ? 1 : 0;
    p.amax = amx.as<float>();
    p.bmax = bmx.as<float>() + (b_batched ? (int64_t)z0 * Np : 0);
    p.Mp = Mp;
    p.Np = Np;
    p.C = g.C;
    p.cm = g.cm;
    p.nb2 = g.nb2;
    p.sc1 = g.sc1;
    p.sc2 = g.sc2;
    p.z0 = z0;
    p.accumulate = g.accumulate ? 1 : 0;
    p.amax_sample = use_uniform ? g.amaxA : nullptr;
    p.amax_sample_n = std::max(1, g.amaxA_n);
    p.amax_out = g.amaxC;
    p.amax_out_n = std::max(1, g.amaxC_n);
    p.rows_per_sample = rows_per_sample;
    p.pout = 0;
    if (ev_kernel && z0 == 0) cudaEventRecord(ev_kernel, c.stream);
    {
      ProfScope ps(P_TC_KERNEL, c.stream);
      ++g_tc_launches;
      const int npm = Mp / (2 * TC_BM), nn = Np / M3_NC;
      const int ntiles = nz * ksplit * npm * nn;
      const int nclusters = std::min(ntiles, nclusters_max);
      tc_gemm3m_kernel<<<2 * nclusters, TC_THREADS, M3_SMEM, c.stream>>>(maps, p, npm, nn, ntiles);
      TN_LAUNCHED();
    }
    if (ksplit > 1) {
      const unsigned blocks = (unsigned)((int64_t)nz * g.M);
      splitk_reduce_kernel<<<blocks, 128, 0, c.stream>>>(p.ws, ksplit, ws_split, nz, g.M, g.N, g.C, g.cm, g.nb2,
                                                         g.sc1, g.sc2, z0, p.accumulate, g.amaxC, p.amax_out_n,
                                                         rows_per_sample);
      TN_LAUNCHED();
    }
  }
}

// 3M path selection. OFF by default: measured on B200 (profiles/r02_ncu_gemm_3m_vs_4m.json)
// the 3M kernel is bound by shared-memory bandwidth (l1tex 92 %, tensor pipe 42 % active vs
// 50 % / 93 % for the 4M kernel at M=16384, N=K=4096): N = 128 per product (three
// accumulators + a rotating slot in 512 TMEM columns) and six planes per operand make its
// operand tiles per MMA cycle 1.5x larger, and the TMA fills share the port. TN_3M=1 enables
// it for pair GEMMs with K >= 512 (complex), TN_3M=2 for every pair GEMM (tests).
int m3_mode() {
  static const int m = getenv("TN_3M") ? std::atoi(getenv("TN_3M")) : 0;
  return m;
}

// Output bounds (GemmDesc::amaxC) feed only the 3M path's per-sample A scales; the 4M path
// scales A per (row, block) from the data itself.
bool tc_bounds_wanted() { return (g_m3_override >= 0 ? g_m3_override : m3_mode()) != 0; }

bool gemm_tc(Ctx& c, const GemmDesc& g) {
  if (!tc_eligible(c, g.M, g.N, g.K, g.work_per_sample)) return false;
  g_cmacs_tc += (double)g.M * g.N * g.K * g.nb1 * g.nb2;
  ShapeRec srec;
  const bool slog = shape_log_on();
  if (slog) {
    char buf[160];
    snprintf(buf, sizeof buf, "M=%d N=%d K=%d nb1=%d nb2=%d views=%d%d", g.M, g.N, g.K, g.nb1, g.nb2,
             g.vam.rank > 0 ? 1 : 0, g.vbk.rank > 0 ? 1 : 0);
    srec.key = buf;
    srec.cm = (double)g.M * g.N * g.K * g.nb1 * g.nb2;
    cudaEventCreate(&srec.a);
    cudaEventCreate(&srec.b);
    cudaEventCreate(&srec.c);
    cudaEventRecord(srec.a, c.stream);
  }
  struct SlogEnd {
    bool on;
    ShapeRec& r;
    cudaStream_t s;
    ~SlogEnd() {
      if (on) {
        cudaEventRecord(r.c, s);
        g_shape_pending.push_back(r);
        if (g_shape_pending.size() > 2000) shape_flush();
      }
    }
  } slog_end{slog, srec, c.stream};
  // kernel attributes are per device context: set once per device ordinal
  static std::atomic<uint64_t> attr_done{0};
  int dev = 0;
  TN_CUDA(cudaGetDevice(&dev));
  const uint64_t dbit = 1ull << (dev & 63);
  if (!(attr_done.load() & dbit)) {
    TN_CUDA(cudaFuncSetAttribute(tc_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
    TN_CUDA(cudaFuncSetAttribute(tc_gemm2_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM2_BYTES));
    TN_CUDA(cudaFuncSetAttribute(tc_gemm2_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM2_BYTES));
    attr_done.fetch_or(dbit);
  }
  // CTA pairs (M = 256 per cluster) whenever one batch element has more than 128 rows
  static const bool pair_off = getenv("TN_TC2") && std::atoi(getenv("TN_TC2")) == 0;
  const bool pair = !pair_off && g.M > TC_BM;
  const int mm = g_m3_override >= 0 ? g_m3_override : m3_mode();
  if ((g.po || g.pa) && (!pair || mm != 0))
    throw Error(-1, "gemm: plane operands need the 4M CTA-pair path");
  if (pair && mm != 0 && (g.K >= 512 || mm == 2)) {
    gemm_tc3m(c, g, dev, slog ? srec.b : nullptr);
    return true;
  }
  const int Krp = rup(2 * g.K, TC_BK);
  const int Mp = rup(g.M, pair ? 2 * TC_BM : TC_BM);
  const int Nrp = rup(2 * g.N, TC_BN);
  const int Np = Nrp / 2;
  const int nbz = g.nb1 * g.nb2;
  const bool b_batched = (g.sb1 != 0 && g.nb1 > 1) || (g.sb2 != 0 && g.nb2 > 1);
  auto simple = [](int64_t dim, int64_t stride) {
    View4 v;
    v.rank = 1;
    v.dims[0] = (int)dim;
    v.str[0] = stride;
    return v;
  };
  auto inner_unit = [](const View4& v) { return v.rank > 0 && v.str[v.rank - 1] == 1; };
  // ---- B planes (once, or per batch element); scales per (complex column, scale block)
  const int nsb = ceil_div(Krp, 2 * SB_K);
  const int nzb = b_batched ? nbz : 1;
  DevBuf bh((size_t)nzb * Nrp * Krp * 2, c.stream), bl((size_t)nzb * Nrp * Krp * 2, c.stream);
  DevBuf bsc((size_t)nzb * nsb * Np * sizeof(float), c.stream);
  if (g.amaxC) TN_CUDA(cudaMemsetAsync(g.amaxC, 0, sizeof(float) * std::max(1, g.amaxC_n), c.stream));
  // grid.z <= 65535: per-sample B planes are prepared in chunks of batch elements
  for (int zb0 = 0; zb0 < nzb; zb0 += 65535) {
    const int nzc = std::min(65535, nzb - zb0);
    PrepArgs a;
    a.X = g.B;
    a.vr = g.vbn.rank ? g.vbn : simple(g.N, g.bn);
    a.vk = g.vbk.rank ? g.vbk : simple(g.K, g.bk);
    a.conj = g.conjB;
    a.nb2 = g.nb2;
    a.s1 = b_batched ? g.sb1 : 0;
    a.s2 = b_batched ? g.sb2 : 0;
    a.z0 = zb0;
    a.R = g.N;
    a.K = g.K;
    a.Rrows = Nrp;
    a.Krp = Krp;
    a.k_fast = inner_unit(a.vk) || !inner_unit(a.vr);
    a.mx = nullptr;
    a.mx_sample = nullptr;
    a.mx_sample_n = 0;
    a.rows_per_sample = 0;
    a.Rp = Np;
    a.hi = bh.as<__half>() + (int64_t)zb0 * Nrp * Krp;
    a.lo = bl.as<__half>() + (int64_t)zb0 * Nrp * Krp;
    a.asc = bsc.as<float>() + (int64_t)zb0 * nsb * Np;
    a.nsb = nsb;
    dim3 grid(Nrp / 64, ceil_div(Krp / 2, PK_K), nzc);
    prep_wide_kernel<1><<<grid, 256, 0, c.stream>>>(a);
    TN_LAUNCHED();
  }
  const int bbox = pair ? TC_BN / 2 : TC_BN;
  CUtensorMap mbh = make_map(bh.as<__half>(), Krp, Nrp, nzb, bbox);
  CUtensorMap mbl = make_map(bl.as<__half>(), Krp, Nrp, nzb, bbox);
  // ---- split-K when one sample's output has too few tiles to fill the SMs (long-K,
  // small-MN GEMMs such as the fit derivatives). Chosen from per-sample shapes only
  // (bitwise-identical results for any batch size); splits are whole promotion chunks.
  const int kblocks = Krp / TC_BK;
  const int mps = g.m_per_sample > 0 ? g.m_per_sample : g.M;
  const int64_t tiles_ps = (int64_t)((mps + TC_BM - 1) / TC_BM) * (Nrp / TC_BN) * g.nb2;
  int ksplit = 1, kbps = kblocks;
  if (tiles_ps < 148 && kblocks >= 2 * TC_KC) {
    int want = (int)std::min<int64_t>(32, (2 * 148 + tiles_ps - 1) / tiles_ps);
    int maxs = kblocks / TC_KC;
    ksplit = std::max(1, std::min(want, maxs));
    kbps = ((kblocks + ksplit - 1) / ksplit + TC_KC - 1) / TC_KC * TC_KC;
    ksplit = (kblocks + kbps - 1) / kbps;
  }
  // A's scales: one exponent per (row, SB_K complex K) block, found by the prep kernel from the
  // tile it converts (no max pass); rows map to samples as row / m_per_sample when the batch is
  // folded into M, else by the outer batch index (output bounds only).
  const int rows_per_sample = g.nb1 > 1 ? 0 : (g.m_per_sample > 0 ? g.m_per_sample : g.M);
  // ---- A planes, chunked over the batch to bound the workspace (<= ~1 GB per plane)
  const int64_t per_z = (int64_t)Mp * Krp;
  const int zc0 = (int)std::max<int64_t>(
      1, std::min<int64_t>({(int64_t)nbz, (int64_t)(65535 / ksplit), (int64_t)(1ll << 29) / std::max<int64_t>(1, per_z)}));
  int zc = g_zc_max > 0 ? std::min(zc0, g_zc_max) : zc0;  // tn_debug_set_zc: force chunking (tests)
  if (g.pa) {  // A planes written by the producing GEMM (contract_planes)
    if (g.pa->Mp != Mp || g.pa->Krp != Krp || g.pa->nsb != nsb || g.pa->nz != nbz)
      throw Error(-1, "gemm: A planes do not match the GEMM");
    zc = nbz;
  }
  if (g.po && (ksplit != 1 || g.M % (2 * TC_BM) != 0 || g.N % 128 != 0 || g.nb2 != 1 || (g.pa == nullptr && zc < nbz)))
    throw Error(-1, "gemm: plane output needs whole tiles and no split-K");
  DevBuf ah(g.pa ? 0 : (size_t)zc * per_z * 2, c.stream), al(g.pa ? 0 : (size_t)zc * per_z * 2, c.stream);
  DevBuf asc(g.pa ? 0 : (size_t)zc * nsb * Mp * sizeof(float), c.stream);
  DevBuf ws;
  const int64_t ws_split = (int64_t)zc * g.M * g.N;
  if (ksplit > 1) ws.alloc((size_t)ksplit * ws_split * sizeof(float2), c.stream);
  for (int z0 = 0; z0 < nbz; z0 += zc) {
    const int nz = std::min(zc, nbz - z0);
    __half* pah = g.pa ? g.pa->hi->as<__half>() : ah.as<__half>();
    __half* pal = g.pa ? g.pa->lo->as<__half>() : al.as<__half>();
    const float* pasc = g.pa ? g.pa->asc->as<float>() : asc.as<float>();
    if (!g.pa) {
      PrepArgs a;
      a.X = g.A;
      a.vr = g.vam.rank ? g.vam : simple(g.M, g.am);
      a.vk = g.vak.rank ? g.vak : simple(g.K, g.ak);
      a.conj = g.conjA;
      a.nb2 = g.nb2;
      a.s1 = g.sa1;
      a.s2 = g.sa2;
      a.z0 = z0;
      a.R = g.M;
      a.K = g.K;
      a.Rrows = Mp;
      a.Krp = Krp;
      a.k_fast = inner_unit(a.vk) || !inner_unit(a.vr);
      a.mx = nullptr;
      a.mx_sample = nullptr;
      a.mx_sample_n = 0;
      a.rows_per_sample = rows_per_sample;
      a.Rp = Mp;
      a.hi = ah.as<__half>();
      a.lo = al.as<__half>();
      a.asc = asc.as<float>();
      a.nsb = nsb;
      // K-contiguous operands (innermost K stride 1, even length, 16-byte aligned base and
      // row/batch offsets) take the transpose-free kernel
      const View4& vk = a.vk;
      bool kfast = vk.rank > 0 && vk.str[vk.rank - 1] == 1 && vk.dims[vk.rank - 1] % 2 == 0 && g.K % 2 == 0 &&
                   (reinterpret_cast<uintptr_t>(g.A) & 15) == 0 && a.s1 % 2 == 0 && a.s2 % 2 == 0;
      for (int d = 0; d < vk.rank - 1 && kfast; ++d) kfast = vk.str[d] % 2 == 0;
      for (int d = 0; d < a.vr.rank && kfast; ++d) kfast = a.vr.str[d] % 2 == 0 || a.vr.dims[d] == 1;
      static const bool kfast_off = getenv("TN_PREP_KFAST") && std::atoi(getenv("TN_PREP_KFAST")) == 0;
      if (kfast && !kfast_off) {
        dim3 grid(ceil_div(Mp, PKF_ROWS), ceil_div(Krp / 4, PKF_PAIRS), nz);
        prep_kfast_kernel<<<grid, 256, 0, c.stream>>>(a);
      } else {
        dim3 grid(Mp / 32, ceil_div(Krp / 2, PK_K), nz);
        prep_wide_kernel<0><<<grid, 256, 0, c.stream>>>(a);
      }
      TN_LAUNCHED();
    }
    CUtensorMap mah = make_map(pah, Krp, Mp, nz, TC_BM);
    CUtensorMap mal = make_map(pal, Krp, Mp, nz, TC_BM);
    TcParams p;
    p.M = g.M;
    p.N = g.N;
    p.kblocks = kblocks;
    p.ksplit = ksplit;
    p.kb_per_split = kbps;
    p.ws = ws.as<float2>();
    p.ws_split = ws_split;
    p.b_batched = b_batched ? 1 : 0;
    p.amax = nullptr;
    p.ascale = pasc;
    p.nsb = nsb;
    p.pout = 0;
    p.pmode = 0;
    if (g.po) {
      p.pout = 1;
      p.pvm = g.po->vm;
      p.pvn = g.po->vn;
      p.pzpo = g.po->zpo;
      p.pzso = g.po->zso;
      p.pmode = g.po->mode;
      p.pho = g.po->hi;
      p.plo = g.po->lo;
      p.psc = g.po->asc;
    }
    p.bmax = nullptr;
    p.bscale = bsc.as<float>() + (b_batched ? (int64_t)z0 * nsb * Np : 0);
    p.Mp = Mp;
    p.Np = Np;
    p.C = g.C;
    p.cm = g.cm;
    p.nb2 = g.nb2;
    p.sc1 = g.sc1;
    p.sc2 = g.sc2;
    p.z0 = z0;
    p.accumulate = g.accumulate ? 1 : 0;
    p.amax_sample = nullptr;
    p.amax_sample_n = 1;
    p.amax_out = g.amaxC;
    p.amax_out_n = std::max(1, g.amaxC_n);
    p.rows_per_sample = rows_per_sample;
    if (slog && z0 == 0) cudaEventRecord(srec.b, c.stream);
    {
      ProfScope ps(P_TC_KERNEL, c.stream);
      ++g_tc_launches;
      CUtensorMap mb_hi = mbh, mb_lo = mbl;
      if (b_batched) {
        // B planes are indexed by the chunk-relative z: rebuild maps at the chunk's base
        mb_hi = make_map(bh.as<__half>() + (int64_t)z0 * Nrp * Krp, Krp, Nrp, nz, bbox);
        mb_lo = make_map(bl.as<__half>() + (int64_t)z0 * Nrp * Krp, Krp, Nrp, nz, bbox);
      }
      if (pair) {
        // persistent CTA pairs over all (z, split, m pair, n) tiles
        const int npm = Mp / (2 * TC_BM), nn = Nrp / TC_BN;
        const int ntiles = nz * ksplit * npm * nn;
        static std::atomic<int> max_clusters_dev[64];
        int max_clusters = max_clusters_dev[dev & 63].load();
        if (!max_clusters) {
          // clusters that can be co-resident (a persistent grid larger than this would run
          // its surplus clusters as a serial second wave)
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3(148, 1, 1);
          cfg.blockDim = dim3(TC_THREADS, 1, 1);
          cfg.dynamicSmemBytes = SMEM2_BYTES;
          cudaLaunchAttribute at;
          at.id = cudaLaunchAttributeClusterDimension;
          at.val.clusterDim.x = 2;
          at.val.clusterDim.y = 1;
          at.val.clusterDim.z = 1;
          cfg.attrs = &at;
          cfg.numAttrs = 1;
          int n = 0;
          if (cudaOccupancyMaxActiveClusters(&n, (void*)tc_gemm2_kernel<false>, &cfg) != cudaSuccess || n < 1) {
            cudaGetLastError();
            n = 64;
          }
          max_clusters = std::min(n, 74);
          max_clusters_dev[dev & 63].store(max_clusters);
          if (getenv("TN_GEMM_LOG")) fprintf(stderr, "tc_gemm2: %d co-resident CTA pairs\n", max_clusters);
        }
        static const bool persist = !(getenv("TN_PERSIST") && std::atoi(getenv("TN_PERSIST")) == 0);
        const int nclusters = persist ? std::min(ntiles, max_clusters) : ntiles;
        if (p.pout)
          tc_gemm2_kernel<true><<<2 * nclusters, TC_THREADS, SMEM2_BYTES, c.stream>>>(mah, mal, mb_hi, mb_lo, p, npm,
                                                                                    nn, ntiles);
        else
          tc_gemm2_kernel<false><<<2 * nclusters, TC_THREADS, SMEM2_BYTES, c.stream>>>(mah, mal, mb_hi, mb_lo, p, npm,
                                                                                     nn, ntiles);
      } else {
        dim3 grid(Nrp / TC_BN, Mp / TC_BM, nz * ksplit);
        tc_gemm_kernel<<<grid, TC_THREADS, SMEM_BYTES, c.stream>>>(mah, mal, mb_hi, mb_lo, p);
      }
      TN_LAUNCHED();
    }
    if (ksplit > 1) {
      const unsigned blocks = (unsigned)((int64_t)nz * g.M);
      splitk_reduce_kernel<<<blocks, 128, 0, c.stream>>>(p.ws, ksplit, ws_split, nz, g.M, g.N, g.C, g.cm, g.nb2,
                                                         g.sc1, g.sc2, z0, p.accumulate, g.amaxC, p.amax_out_n,
                                                         rows_per_sample);
      TN_LAUNCHED();
    }
  }
  return true;
}

}  // namespace tn

extern "C" int tn_debug_raster(int gm) {
  return cudaMemcpyToSymbol(tn::g_raster_gm, &gm, sizeof(int)) == cudaSuccess ? 0 : -1;
}

extern "C" int tn_debug_set_3m(int mode) {
  tn::g_m3_override = mode;
  return 0;
}

extern "C" int tn_debug_set_zc(int zc) {
  tn::g_zc_max = zc;
  return 0;
}

