// gemm_tc.cu -- complex GEMM on the 5th-generation tensor cores (tcgen05, sm_100a),
// FP32-accurate through the TF32x3 split (K1 of SURVEY 2.4).
//
// Complex C = A B is one real GEMM  C_r[M][2N] = A_r[M][2K] . B_r[2K][2N]:
//   A_r = A viewed as interleaved (re, im) along K; C_r = C viewed the same way along N;
//   B_r^T row 2n   = (Re b_kn, -Im b_kn) over k,  row 2n+1 = (Im b_kn, Re b_kn)  (K-major).
// Every real operand x is split x = hi + lo with hi = x truncated to TF32 (exact split), and
// D = A_hi B_hi + A_hi B_lo + A_lo B_hi accumulates in FP32 in tensor memory (TMEM).
//
// Data flow: prep kernels write packed, zero-padded, K-major hi/lo planes to HBM; the GEMM
// kernel streams 128x32 (A) and 256x32 (B) FP32 tiles with TMA (SWIZZLE_128B) through a
// 2-stage mbarrier pipeline; one elected thread issues tcgen05.mma (M=128, N=256, K=8,
// kind::tf32) into a 128x256 FP32 TMEM accumulator; four epilogue warps drain TMEM with
// tcgen05.ld and write complex64 results.
#include <cuda.h>

#include <algorithm>
#include <cstring>

#include "tensor.h"

namespace tn {
namespace {

constexpr int TC_BM = 128;        // rows per CTA (UMMA M)
constexpr int TC_BN = 256;        // real columns per CTA (UMMA N) = 128 complex columns
constexpr int TC_BK = 32;         // real K per stage (one 128-byte swizzle atom of FP32)
constexpr int TC_STAGES = 2;
constexpr int A_TILE = TC_BM * TC_BK * 4;               // 16 KB
constexpr int B_TILE = TC_BN * TC_BK * 4;               // 32 KB
constexpr int STAGE_BYTES = 2 * A_TILE + 2 * B_TILE;    // 96 KB
constexpr int SMEM_BYTES = TC_STAGES * STAGE_BYTES + 1024 + 256;
constexpr uint32_t TMEM_COLS = 512;   // two 128x256 FP32 accumulators (ping-pong over K chunks)
constexpr int TC_KC = 16;             // k-blocks (16 x 32 real K) per promoted chunk
constexpr int TC_THREADS = 320;       // warp 0 TMA, warp 1 MMA, warps 2..9 epilogue

struct TcParams {
  int M, N;          // complex extents (epilogue bounds)
  int kblocks;       // padded real K / TC_BK
  int b_batched;     // B planes carry the batch index
  float2* C;
  int64_t cm;
  int nb2;
  int64_t sc1, sc2;
  int z0;
  int accumulate;
};

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
  d |= (uint64_t)(0) << 16;                   // LBO (unused for swizzled K-major)
  d |= (uint64_t)((1024 >> 4) & 0x3FFF) << 32;  // SBO
  d |= (uint64_t)1 << 46;                     // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                     // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
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

  const int nblk = blockIdx.x, mblk = blockIdx.y, z = blockIdx.z;
  if (warp == 0) {
    if (lane == 0) {  // TMA producer
      const int bz = p.b_batched ? z : 0;
      for (int kb = 0; kb < p.kblocks; ++kb) {
        const int s = kb % TC_STAGES;
        const uint32_t ph = (kb / TC_STAGES) & 1;
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
      // kind::tf32 instruction descriptor: D f32, A/B tf32, K-major both, N=256, M=128
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TC_BN >> 3) << 17) |
                             ((uint32_t)(TC_BM >> 4) << 24);
      for (int kb = 0; kb < p.kblocks; ++kb) {
        const int c = kb / TC_KC, buf = c & 1, kin = kb - c * TC_KC;
        if (kin == 0) {  // chunk c accumulates into TMEM buffer c&1 once the epilogue drained it
          mbar_wait(&acc_empty[buf], ((c >> 1) & 1) ^ 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
        }
        const uint32_t dacc = tmem + (uint32_t)(buf * TC_BN);
        const int s = kb % TC_STAGES;
        const uint32_t ph = (kb / TC_STAGES) & 1;
        mbar_wait(&full[s], ph);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t base = smem_u32(smem + s * STAGE_BYTES);
        const uint64_t ahi = smem_desc(base), alo = smem_desc(base + A_TILE);
        const uint64_t bhi = smem_desc(base + 2 * A_TILE), blo = smem_desc(base + 2 * A_TILE + B_TILE);
#pragma unroll
        for (int k = 0; k < TC_BK / 8; ++k) {
          const uint64_t adv = (uint64_t)((k * 32) >> 4);  // 8 tf32 = 32 bytes along K
          mma_tf32(dacc, ahi + adv, bhi + adv, idesc, (kin | k) != 0);
          mma_tf32(dacc, ahi + adv, blo + adv, idesc, 1u);
          mma_tf32(dacc, alo + adv, bhi + adv, idesc, 1u);
        }
        mma_commit(&empty[s]);
        if (kin == TC_KC - 1 || kb == p.kblocks - 1) mma_commit(&acc_full[buf]);
      }
    }
    __syncwarp();
  } else {
    // epilogue: warps 2..9; warp w drains TMEM lanes 32*(w%4)..+31 (its rows) and columns
    // [128*h, 128*h + 128), h = (w-2)/4. Each K chunk's partial sum is promoted from TMEM
    // into FP32 registers (round-to-nearest adds), which bounds the error of the tensor
    // core's truncating accumulation to one chunk.
    const int lg = warp & 3;
    const int half = (warp - 2) >> 2;
    const int row = mblk * TC_BM + lg * 32 + lane;
    float acc[128];
#pragma unroll
    for (int i = 0; i < 128; ++i) acc[i] = 0.f;
    const int nchunks = (p.kblocks + TC_KC - 1) / TC_KC;
    for (int c = 0; c < nchunks; ++c) {
      const int buf = c & 1;
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
        for (int i = 0; i < 16; ++i) acc[cc + i] += __uint_as_float(v[i]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[buf]);
    }
    if (row < p.M) {
      const int b1 = (p.z0 + z) / p.nb2, b2 = (p.z0 + z) - b1 * p.nb2;
      float2* Crow = p.C + b1 * p.sc1 + b2 * p.sc2 + (int64_t)row * p.cm;
      const int n0 = (nblk * TC_BN + half * 128) >> 1;
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
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

__device__ __forceinline__ float tf32_trunc(float x) { return __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }

// A_r hi/lo planes: [z][Mp][Krp], element (m, kr) = Re/Im of A(m, kr/2)
__global__ void prep_a_kernel(const float2* __restrict__ A, int64_t am, int64_t ak, int conj, int nb2, int64_t sa1,
                              int64_t sa2, int z0, int M, int K, int Mp, int Krp, float* __restrict__ hi,
                              float* __restrict__ lo, int nz) {
  const int64_t per = (int64_t)Mp * Krp, tot = per * nz;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t zz = e / per, r = e - zz * per;
    const int m = (int)(r / Krp), kr = (int)(r - (int64_t)m * Krp);
    const int k = kr >> 1;
    float x = 0.f;
    if (m < M && k < K) {
      const int z = z0 + (int)zz;
      const int b1 = z / nb2, b2 = z - b1 * nb2;
      const float2 a = A[b1 * sa1 + b2 * sa2 + m * am + k * ak];
      x = (kr & 1) ? (conj ? -a.y : a.y) : a.x;
    }
    const float h = tf32_trunc(x);
    hi[e] = h;
    lo[e] = x - h;
  }
}

// B_r^T hi/lo planes: [z][Nrp][Krp]; row 2n = (Re b, -Im b), row 2n+1 = (Im b, Re b)
__global__ void prep_b_kernel(const float2* __restrict__ B, int64_t bk, int64_t bn, int conj, int nb2, int64_t sb1,
                              int64_t sb2, int z0, int N, int K, int Nrp, int Krp, float* __restrict__ hi,
                              float* __restrict__ lo, int nz) {
  const int64_t per = (int64_t)Nrp * Krp, tot = per * nz;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t zz = e / per, r = e - zz * per;
    const int nr = (int)(r / Krp), kr = (int)(r - (int64_t)nr * Krp);
    const int n = nr >> 1, k = kr >> 1;
    float x = 0.f;
    if (n < N && k < K) {
      const int z = z0 + (int)zz;
      const int b1 = z / nb2, b2 = z - b1 * nb2;
      float2 b = B[b1 * sb1 + b2 * sb2 + k * bk + n * bn];
      if (conj) b.y = -b.y;
      const int sel = ((nr & 1) << 1) | (kr & 1);
      x = sel == 0 ? b.x : (sel == 1 ? -b.y : (sel == 2 ? b.y : b.x));
    }
    const float h = tf32_trunc(x);
    hi[e] = h;
    lo[e] = x - h;
  }
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

CUtensorMap make_map(float* base, int inner, int rows, int nz, int box_rows) {
  CUtensorMap m;
  cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)rows, (cuuint64_t)nz};
  cuuint64_t strides[2] = {(cuuint64_t)inner * 4, (cuuint64_t)inner * rows * 4};
  cuuint32_t box[3] = {(cuuint32_t)TC_BK, (cuuint32_t)box_rows, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base, dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(-5, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return m;
}

inline int rup(int x, int m) { return (x + m - 1) / m * m; }

}  // namespace

// Per-sample work (complex MACs) above which the tensor-core path is used. The decision
// depends on per-sample shapes only, so results do not depend on the batch size.
static const double kTcMinWork = 1 << 20;

bool gemm_tc(Ctx& c, const GemmDesc& g) {
  if (c.gemm_mode == 1) return false;
  double work = g.work_per_sample > 0 ? (double)g.work_per_sample : (double)g.M * g.N * g.K;
  if (c.gemm_mode != 2 && (work < kTcMinWork || g.N < 32 || g.K < 8)) return false;
  static bool attr = false;
  if (!attr) {
    TN_CUDA(cudaFuncSetAttribute(tc_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
    attr = true;
  }
  const int Krp = rup(2 * g.K, TC_BK);
  const int Mp = rup(g.M, TC_BM);
  const int Nrp = rup(2 * g.N, TC_BN);
  const int nbz = g.nb1 * g.nb2;
  const bool b_batched = (g.sb1 != 0 && g.nb1 > 1) || (g.sb2 != 0 && g.nb2 > 1);
  // B planes (once, or per batch element)
  const int nzb = b_batched ? nbz : 1;
  DevBuf bh((size_t)nzb * Nrp * Krp * 4, c.stream), bl((size_t)nzb * Nrp * Krp * 4, c.stream);
  {
    int64_t tot = (int64_t)nzb * Nrp * Krp;
    unsigned blocks = (unsigned)std::min<int64_t>((tot + 255) / 256, 148 * 32);
    prep_b_kernel<<<blocks, 256, 0, c.stream>>>(g.B, g.bk, g.bn, g.conjB, g.nb2, g.sb1, g.sb2, 0, g.N, g.K, Nrp, Krp,
                                                bh.as<float>(), bl.as<float>(), nzb);
    TN_LAUNCHED();
  }
  CUtensorMap mbh = make_map(bh.as<float>(), Krp, Nrp, nzb, TC_BN);
  CUtensorMap mbl = make_map(bl.as<float>(), Krp, Nrp, nzb, TC_BN);
  // A planes, chunked over the batch to bound the workspace (<= ~2 GB per plane)
  const int64_t per_z = (int64_t)Mp * Krp;
  const int zc = (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)nbz, (int64_t)65535, (int64_t)(1ll << 29) / std::max<int64_t>(1, per_z)}));
  DevBuf ah((size_t)zc * per_z * 4, c.stream), al((size_t)zc * per_z * 4, c.stream);
  for (int z0 = 0; z0 < nbz; z0 += zc) {
    const int nz = std::min(zc, nbz - z0);
    int64_t tot = (int64_t)nz * per_z;
    unsigned blocks = (unsigned)std::min<int64_t>((tot + 255) / 256, 148 * 32);
    prep_a_kernel<<<blocks, 256, 0, c.stream>>>(g.A, g.am, g.ak, g.conjA, g.nb2, g.sa1, g.sa2, z0, g.M, g.K, Mp, Krp,
                                                ah.as<float>(), al.as<float>(), nz);
    TN_LAUNCHED();
    CUtensorMap mah = make_map(ah.as<float>(), Krp, Mp, nz, TC_BM);
    CUtensorMap mal = make_map(al.as<float>(), Krp, Mp, nz, TC_BM);
    TcParams p;
    p.M = g.M;
    p.N = g.N;
    p.kblocks = Krp / TC_BK;
    p.b_batched = b_batched ? 1 : 0;
    p.C = g.C;
    p.cm = g.cm;
    p.nb2 = g.nb2;
    p.sc1 = g.sc1;
    p.sc2 = g.sc2;
    p.z0 = z0;
    p.accumulate = g.accumulate ? 1 : 0;
    if (b_batched && z0 != 0) {
      // B planes are indexed by the absolute z; the maps cover all nbz elements
    }
    dim3 grid(Nrp / TC_BN, Mp / TC_BM, nz);
    if (b_batched) {
      // shift B coordinates by z0: rebuild maps at the chunk's base
      CUtensorMap mbh2 = make_map(bh.as<float>() + (int64_t)z0 * Nrp * Krp, Krp, Nrp, nz, TC_BN);
      CUtensorMap mbl2 = make_map(bl.as<float>() + (int64_t)z0 * Nrp * Krp, Krp, Nrp, nz, TC_BN);
      tc_gemm_kernel<<<grid, TC_THREADS, SMEM_BYTES, c.stream>>>(mah, mal, mbh2, mbl2, p);
    } else {
      tc_gemm_kernel<<<grid, TC_THREADS, SMEM_BYTES, c.stream>>>(mah, mal, mbh, mbl, p);
    }
    TN_LAUNCHED();
  }
  return true;
}

}  // namespace tn
