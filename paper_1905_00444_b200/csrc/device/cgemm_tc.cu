// K2 tensor-core path: the contraction GEMM of contract_ttgt
// (include/qsim/contraction.hpp:208-214) on the 5th-generation tensor cores.
//
// Complex -> real embedding.  A complex row-major A[m][k] IS a real matrix
// A_r[m][2k] (re/im interleaved along K), and with
//   B_r^T[2j  ][2p..2p+1] = ( Re b_pj, -Im b_pj )
//   B_r^T[2j+1][2p..2p+1] = ( Im b_pj,  Re b_pj )
// the real product C_r[m][2n] = A_r * B_r is exactly the complex row-major
// C[m][n] (C_r row = re/im interleaved).  So the large operand A and the
// output C are consumed/produced in place, K-major, with no repacking; only
// the (small) B operand is expanded once per GEMM by tc_prep_b_kernel.  The
// real GEMM does 4 real MACs per complex MAC = the 8 flops of Eq.(1).
//
// FP32 accuracy from TF32 tensor cores (3xTF32): x = hi + lo with
// hi = rna_tf32(x), lo = x - hi (exact), and
//   A*B ~= A_hi*B_hi + A_hi*B_lo + A_lo*B_hi      (FP32 accumulate in TMEM),
// leaving only the lo*lo term (~2^-22 relative).  B is split in the prep
// kernel; A is split in shared memory by converter warps as each stage
// lands (no extra HBM traffic or footprint for the big operand).
//
// Accumulation: the tensor core's FP32 accumulator truncates, so its error
// grows linearly with K (measured 9e-4 at K=65536).  Partial sums are
// therefore promoted every 4 k-blocks (64 complex K; measured error
// ~1e-6 up to K=65536, vs 6.5e-6 for FP32 FFMA) from a
// double-buffered TMEM accumulator into round-to-nearest FP32 registers,
// overlapping the MMA of the next chunk (cf. DeepSeek-V3's FP8 promotion).
//
// Kernel anatomy (one CTA per 128 x BN output tile, 10 warps):
//   warp 0     TMA producer: A tile [128 x 32 fp32] and B_hi/B_lo tiles
//              [BN x 32] per stage, SWIZZLE_128B, mbarrier complete_tx;
//   warp 1     TMEM allocator + single-thread tcgen05.mma issuer
//              (kind::tf32, M=128, N=BN, K=8) into TMEM chunk buffer c&1,
//              tcgen05.commit -> smem-stage and chunk barriers;
//   warps 2-9  workers: convert A (A -> A_hi in place, A_lo alongside,
//              fence.proxy.async), drain finished TMEM chunks (tcgen05.ld)
//              into register accumulators (row = lane quadrant, half the
//              columns each), and the epilogue: apply the operands' pending
//              power-of-two renormalisation, max|c|^2 -> TMeta, store C.
#include <cuda.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "kernels_tc.hpp"

namespace qsg::dev {

__device__ __forceinline__ int tc_pending_shift(const TMeta* m, bool norm) {
  if (!norm || m == nullptr) return 0;
  const unsigned bits = m->maxsq_bits;
  if (bits == 0) return 0;
  const double mx = sqrt(static_cast<double>(__uint_as_float(bits)));
  int e = 0;
  const double fr = frexp(mx, &e);
  return fr == 0.5 ? e - 1 : e;
}

namespace {

constexpr int BM = 128;
constexpr int BK = 32;  // fp32 elements of K_real per stage (= one 128-byte swizzle row)
constexpr int kWorkers = 256;            // warps 2..9
constexpr int kThreads = 64 + kWorkers;   // + producer warp + MMA warp
// k-blocks (32 real K each) accumulated in TMEM before promotion to
// registers: the tensor core's FP32 accumulator truncates, so its error
// grows linearly with the reduction length (measured ~1.4e-8 * k); 32
// complex K per chunk keeps it at the 3xTF32 floor (~5e-7).
constexpr int kChunkDefault = 4;  // QSG_TC_CHUNK overrides (experiments)
constexpr int kShortKChunks = 2;  // promotion chunks of a k <= 256 tile (QSG_TC_SHORTK_CHUNKS; 1 = fastest, see DESIGN 2)
constexpr int A_BYTES = BM * BK * 4;

template <int BN>
struct TcCfg {
  static constexpr int B_BYTES = BN * BK * 4;
  static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr int STAGES = BN >= 256 ? 2 : 3;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr int TMEM_COLS = 2 * BN;  // double-buffered chunk accumulator (power of two)
};

struct TcParams {
  float* c;  // complex64 C[m][n] as fp32 [m][2n]
  long long m, n2;  // rows, real columns (2n)
  int kblocks;
  int n_tiles;  // output tiles along N; blockIdx.x = m_tile * n_tiles + n_tile
  const TMeta* meta_a;
  const TMeta* meta_b;
  TMeta* meta_c;
  int norm_a, norm_b;
  int chunk;   // k-blocks per TMEM promotion chunk
  int group_m;    // m-pairs per rasterization group (fp16 kernel)
  unsigned int* sync;  // fp16 kernel: K-sync arrival counters per checkpoint of the persistent run (null: off)
  int sync_every;      // k-blocks between checkpoints
  int a_presplit;      // fp16 kernel: A stored split (TMeta::split_exp), see GemmArgs
  int c_split;         // fp16 kernel: write C split
  int log2k;           // ceil(log2(k)): the split output's bound exponent
  long long c_total;   // complex elements of C (offset of the lo plane / 4 bytes)
  int stream_store;    // fp16 kernel: evict-first (st.global.cs) output stores
  int lane_store;      // host only: launch the kLane instantiation (split output, lane = row STG.256)
  int half_tail;  // fp16 kernel: the last k-block has only its first 32 real K (2k % 64 == 32)
  int passes;         // fp16 kernel: 3 (hi.hi + hi.lo + lo.hi); 2 = power-model experiment only (QSG_TC_PASSES)
  unsigned long long* prof;  // fp16 pair kernel, QSG_TC_PROF=1: per-CTA role wait / busy cycle counters
  int prefetch;       // fp16 kernel, pre-split A: L2-prefetch the A boxes this many k-blocks ahead
  int convert_ahead;  // fp16 kernel, raw A: convert a chunk's stages before the previous chunk's epilogue (A/B knob)
  int store_perm, nrow_bits, ncol_bits;  // fused output permutation (see GemmArgs)
  unsigned char row_pos[48];
  unsigned char col_pos[24];
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
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// Non-blocking probe of an mbarrier phase (true once `parity` completed).
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}

// CTA-pair TMA: data lands in this CTA's smem, complete_tx goes to the
// barrier at shared::cluster address `bar` (the leader's).
__device__ __forceinline__ void tma_load_2d_pair(const CUtensorMap* map, uint32_t bar, void* dst, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(bar), "r"(x), "r"(y)
      : "memory");
}

// L2 prefetch of a tensor-map box (no shared memory, no barrier).
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int x, int y) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(map), "r"(x), "r"(y)
               : "memory");
}

// K-major, SWIZZLE_128B smem matrix descriptor (rows of 128 B, 8-row atoms
// of 1024 B; SBO = 1024 B; version 1; layout type 2 = SWIZZLE_128B).
// One 32-byte (full sector) store per lane: STG.256 (sm_100), evict-first or not.
__device__ __forceinline__ void st_global_v8(void* g, const uint32_t* v, bool evict_first) {
  if (evict_first)
    asm volatile("st.global.cs.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(g), "r"(v[0]), "r"(v[1]),
                 "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
  else
    asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(g), "r"(v[0]), "r"(v[1]), "r"(v[2]),
                 "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}

__device__ __forceinline__ uint64_t kmajor_sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(1) << 16;              // LBO (unused for swizzled K-major)
  d |= static_cast<uint64_t>(1024 >> 4) << 32;      // SBO
  d |= static_cast<uint64_t>(1) << 46;              // version (Blackwell)
  d |= static_cast<uint64_t>(2) << 61;              // SWIZZLE_128B
  return d;
}

// Instruction descriptor: kind::tf32, D fp32, A/B tf32 K-major, M=128, N=BN.
template <int BN>
__host__ __device__ constexpr uint32_t tf32_idesc() {
  return (1u << 4)               // D format F32
         | (2u << 7)             // A format TF32
         | (2u << 10)            // B format TF32
         | (0u << 15) | (0u << 16)  // K-major A and B
         | (static_cast<uint32_t>(BN >> 3) << 17) | (static_cast<uint32_t>(BM >> 4) << 24);
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t u;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(u) : "f"(x));
  return __uint_as_float(u);
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// 16 columns TMEM -> registers without the trailing wait (issue several,
// then one tcgen05.wait::ld before reading any of them).
__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, float* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]),
        "=f"(v[8]), "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]), "=f"(v[14]), "=f"(v[15])
      : "r"(taddr));
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
    cgemm_tc_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_bhi,
                    const __grid_constant__ CUtensorMap map_blo, const TcParams p) {
  using Cfg = TcCfg<BN>;
  constexpr int HALF = BN / 2;  // accumulator columns owned by one worker thread
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // 1 KiB aligned, still __shared__
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
  uint64_t* conv = full + Cfg::STAGES;
  uint64_t* empty = conv + Cfg::STAGES;
  uint64_t* acc_full = empty + Cfg::STAGES;   // [2] TMEM chunk buffer ready
  uint64_t* acc_empty = acc_full + 2;          // [2] TMEM chunk buffer drained
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n_tile = static_cast<int>(blockIdx.x % p.n_tiles);
  const long long m_tile = blockIdx.x / p.n_tiles;

  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], kWorkers);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], kWorkers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_a) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_bhi) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_blo) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_base_slot)),
                 "n"(Cfg::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_base_slot;
  const int kblocks = p.kblocks;
  const int nchunks = (kblocks + p.chunk - 1) / p.chunk;

  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < kblocks; ++kb) {
        const int s = kb % Cfg::STAGES;
        const uint32_t ph = (kb / Cfg::STAGES) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* st = smem + s * Cfg::STAGE_BYTES;
        mbar_expect_tx(&full[s], A_BYTES + 2 * Cfg::B_BYTES);
        tma_load_2d(&map_a, &full[s], st, kb * BK, static_cast<int>(m_tile * BM));
        tma_load_2d(&map_bhi, &full[s], st + 2 * A_BYTES, kb * BK, n_tile * BN);
        tma_load_2d(&map_blo, &full[s], st + 2 * A_BYTES + Cfg::B_BYTES, kb * BK, n_tile * BN);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = tf32_idesc<BN>();
      for (int c = 0; c < nchunks; ++c) {
        const int buf = c & 1;
        mbar_wait(&acc_empty[buf], ((c >> 1) & 1) ^ 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + static_cast<uint32_t>(buf * BN);
        const int kb_end = min(kblocks, (c + 1) * p.chunk);
        for (int kb = c * p.chunk; kb < kb_end; ++kb) {
          const int s = kb % Cfg::STAGES;
          const uint32_t ph = (kb / Cfg::STAGES) & 1;
          mbar_wait(&conv[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          uint8_t* st = smem + s * Cfg::STAGE_BYTES;
          const uint64_t a_hi = kmajor_sw128_desc(smem_u32(st));
          const uint64_t a_lo = kmajor_sw128_desc(smem_u32(st + A_BYTES));
          const uint64_t b_hi = kmajor_sw128_desc(smem_u32(st + 2 * A_BYTES));
          const uint64_t b_lo = kmajor_sw128_desc(smem_u32(st + 2 * A_BYTES + Cfg::B_BYTES));
          const bool first = kb == c * p.chunk;
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {
            const uint64_t adv = static_cast<uint64_t>(kk * 32 >> 4);  // 8 tf32 = 32 bytes along the swizzled row
            umma_tf32(d, a_hi + adv, b_hi + adv, idesc, (first && kk == 0) ? 0u : 1u);
            umma_tf32(d, a_hi + adv, b_lo + adv, idesc, 1u);
            umma_tf32(d, a_lo + adv, b_hi + adv, idesc, 1u);
          }
          umma_commit(&empty[s]);
        }
        umma_commit(&acc_full[buf]);
      }
    }
    __syncwarp();
  } else {
    // ---- workers (8 warps): convert A per stage; promote each finished
    // TMEM chunk into round-to-nearest FP32 register accumulators; epilogue.
    const int wt = threadIdx.x - 64;          // 0..255
    const int quad = warp & 3;                // TMEM lane quadrant this warp may access
    const int half = (warp - 2) >> 2;         // which half of the BN columns
    float acc[HALF];
#pragma unroll
    for (int i = 0; i < HALF; ++i) acc[i] = 0.f;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(quad * 32) << 16) + static_cast<uint32_t>(half * HALF);
    // Chunk c's stages are converted first; then chunk c-1 (complete by
    // then) is drained, freeing its TMEM buffer before the MMA needs it for
    // chunk c+1.  One drain site keeps `acc` in registers.
    for (int c = 0; c <= nchunks; ++c) {
      if (c < nchunks) {
        const int kb_end = min(kblocks, (c + 1) * p.chunk);
        for (int kb = c * p.chunk; kb < kb_end; ++kb) {
          const int s = kb % Cfg::STAGES;
          const uint32_t ph = (kb / Cfg::STAGES) & 1;
          mbar_wait(&full[s], ph);
          float4* a = reinterpret_cast<float4*>(smem + s * Cfg::STAGE_BYTES);
          float4* alo = reinterpret_cast<float4*>(smem + s * Cfg::STAGE_BYTES + A_BYTES);
#pragma unroll
          for (int i = 0; i < A_BYTES / 16 / kWorkers; ++i) {
            const int idx = i * kWorkers + wt;
            const float4 x = a[idx];
            float4 h, l;
            h.x = tf32_rna(x.x); l.x = x.x - h.x;
            h.y = tf32_rna(x.y); l.y = x.y - h.y;
            h.z = tf32_rna(x.z); l.z = x.z - h.z;
            h.w = tf32_rna(x.w); l.w = x.w - h.w;
            a[idx] = h;
            alo[idx] = l;
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          mbar_arrive(&conv[s]);
        }
      }
      if (c >= 1) {
        const int buf = (c - 1) & 1;
        mbar_wait(&acc_full[buf], ((c - 1) >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
        for (int j = 0; j < HALF / 16; ++j) {
          float v[16];
          tmem_ld16(lane_base + static_cast<uint32_t>(buf * BN + 16 * j), v);
#pragma unroll
          for (int i = 0; i < 16; ++i) acc[16 * j + i] += v[i];
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        mbar_arrive(&acc_empty[buf]);
      }
    }

    // ---- epilogue ----
    const int row = quad * 32 + lane;
    const long long gm = m_tile * BM + row;
    const int sa = tc_pending_shift(p.meta_a, p.norm_a), sb = tc_pending_shift(p.meta_b, p.norm_b);
    const int shift = sa + sb;
    float local = 0.f;
#pragma unroll
    for (int i = 0; i < HALF; ++i) acc[i] = scalbnf(acc[i], -shift);
#pragma unroll
    for (int i = 0; i < HALF; i += 2) local = fmaxf(local, acc[i] * acc[i] + acc[i + 1] * acc[i + 1]);
    float4* dst = reinterpret_cast<float4*>(p.c + gm * p.n2 + static_cast<long long>(n_tile) * BN + half * HALF);
#pragma unroll
    for (int i = 0; i < HALF / 4; ++i) dst[i] = make_float4(acc[4 * i], acc[4 * i + 1], acc[4 * i + 2], acc[4 * i + 3]);
    if (p.meta_c) {
      for (int o = 16; o > 0; o >>= 1) local = fmaxf(local, __shfl_xor_sync(0xffffffffu, local, o));
      if (lane == 0 && local > 0.f) atomicMax(&p.meta_c->maxsq_bits, __float_as_uint(local));
      if (blockIdx.x == 0 && threadIdx.x == 64)
        p.meta_c->log_scale = (p.meta_a ? p.meta_a->log_scale : 0.0) + (p.meta_b ? p.meta_b->log_scale : 0.0) + shift;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(Cfg::TMEM_COLS));
  }
}

// ---------------------------------------------------------------------------
// 2-CTA variant (cta_group::2): a CTA pair computes a 256 x 256 (real) output
// tile with M=256 UMMAs issued by the leader.  Each CTA stages ITS 128 rows
// of A and ITS half (128 rows of B_r^T) of B, so per-SM shared-memory and
// L2 traffic per MMA drop by a third/half against the 1-CTA kernel and a
// third pipeline stage fits (64 KiB per stage).  Each CTA's TMEM holds its
// 128 output rows x 256 columns (x2 chunk buffers = 512 columns).
// Barriers: full[] and the TMEM-chunk acc_full[] are per CTA; conv[] and
// acc_empty[] live in the leader and collect arrivals from both CTAs'
// workers (remote mbarrier arrive over the cluster); the leader's
// tcgen05.commit multicasts to both CTAs.
// Real output columns per CTA pair: 256 for wide GEMMs; 128/64/32 for the
// narrow-N (GEMV-like, HBM-bound) contraction steps.
constexpr int kGroupM = 8;    // m-pairs per rasterization group
template <int BN>
struct Tc2Cfg {
  static constexpr int A_B = BM * BK * 4;            // this CTA's 128 rows of A
  static constexpr int B_B = (BN / 2) * BK * 4;      // this CTA's half of B_r^T
  static constexpr int STAGE_BYTES = 2 * A_B + 2 * B_B;
  // Epilogue staging: per worker warp a 32-row x 16-float chunk, pitch 20
  // floats (conflict-free 16-byte writes), so global stores are 64-byte row
  // segments instead of one 16-byte piece of 32 different rows.
  static constexpr int EPI_PITCH = 20;
  static constexpr int EPI_BYTES = (kWorkers / 32) * 32 * EPI_PITCH * 4;
  static constexpr int STAGES =
      ((224 * 1024 - EPI_BYTES) / STAGE_BYTES) > 6 ? 6 : ((224 * 1024 - EPI_BYTES) / STAGE_BYTES);
  static constexpr int SMEM = STAGES * STAGE_BYTES + EPI_BYTES + 1024 + 256;
  static constexpr int TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;  // power of two >= 32
};

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Arrive on the barrier at the same smem offset in cluster CTA `cta`.
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* bar, uint32_t cta) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(bar)), "r"(cta));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
}

// Warp-aggregated arrival on the leader's barrier: the leader's own warps
// arrive locally (CTA scope), the peer's remotely (release.cluster).
__device__ __forceinline__ void arrive_leader(uint64_t* bar, uint32_t rank) {
  if (rank == 0) mbar_arrive(bar);
  else mbar_arrive_remote(bar, 0);
}

__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAITC_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void umma2_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma2_commit_both(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(static_cast<uint16_t>(0x3))
      : "memory");
}

template <int BN>
__host__ __device__ constexpr uint32_t tf32_idesc_pair() {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(BN >> 3) << 17) |
         (static_cast<uint32_t>(256 >> 4) << 24);
}

// Grouped rasterization of pair tiles: pairs running concurrently cover a
// kGroupM x (clusters/kGroupM) block of (m, n) tiles, so the A rows and the
// expanded-B columns they stream are shared through L2 (n-fastest order
// re-read all of B_r^T from HBM per wave of m tiles: 1.2 TB per s026 launch).
__device__ __forceinline__ void pair_tile_coords(long long t, long long m_pairs, int n_tiles, long long& m_pair,
                                                 int& n_tile, int group_m = kGroupM) {
  // 32-bit divisions (64-bit ones cost ~3x on the workers' per-tile path):
  // a launch has < 2^31 tiles (C would be > 2^47 bytes otherwise).
  const unsigned span = static_cast<unsigned>(group_m) * static_cast<unsigned>(n_tiles), tt = static_cast<unsigned>(t);
  const unsigned first_m = (tt / span) * static_cast<unsigned>(group_m);
  const unsigned gsize = min(static_cast<unsigned>(group_m), static_cast<unsigned>(m_pairs) - first_m);
  const unsigned within = tt % span;
  m_pair = first_m + within % gsize;
  n_tile = static_cast<int>(within / gsize);
}

// Persistent: each CTA pair walks tiles t = cluster, cluster + nclusters, ...
// with pipeline counters that run across tile boundaries, so TMA prefetch,
// conversion and MMA of the next tile overlap the epilogue of the previous
// one and the per-tile setup (barriers, TMEM allocation) is paid once.
template <int kPairBN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    cgemm_tc2_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_bhi,
                     const __grid_constant__ CUtensorMap map_blo, const TcParams p) {
  using Cfg = Tc2Cfg<kPairBN>;
  constexpr int HALF = kPairBN / 2;  // accumulator columns per worker thread
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // 1 KiB aligned, still __shared__
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
  uint64_t* conv = full + Cfg::STAGES;
  uint64_t* empty = conv + Cfg::STAGES;
  uint64_t* acc_full = empty + Cfg::STAGES;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  float* epi_stage = reinterpret_cast<float*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES + 256);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const long long cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
  const long long m_pairs = p.m / 256;
  const long long total = m_pairs * p.n_tiles;
  const long long my_tiles = cluster < total ? (total - 1 - cluster) / nclusters + 1 : 0;

  if (threadIdx.x == 0) {
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], 2);  // one (aggregated) arrival per CTA
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], 2);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_a) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_bhi) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_blo) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_base_slot)),
                 "n"(Cfg::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_base_slot;
  const int kblocks = p.kblocks;
  const int nchunks = (kblocks + p.chunk - 1) / p.chunk;
  const long long total_chunks = my_tiles * nchunks;

  if (warp == 0) {
    if (lane == 0) {
      int s = 0;  // stage ring position / phase, continuous across tiles
      uint32_t ph = 0;
      for (long long ti = 0; ti < my_tiles; ++ti) {
        long long m_pair;
        int n_tile;
        pair_tile_coords(cluster + ti * nclusters, m_pairs, p.n_tiles, m_pair, n_tile);
        const int row0 = static_cast<int>(m_pair * 256 + static_cast<long long>(rank) * BM);
        const int brow0 = n_tile * kPairBN + static_cast<int>(rank) * (kPairBN / 2);
        for (int kb = 0; kb < kblocks; ++kb) {
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t* st = smem + s * Cfg::STAGE_BYTES;
          mbar_expect_tx(&full[s], Cfg::A_B + 2 * Cfg::B_B);
          tma_load_2d(&map_a, &full[s], st, kb * BK, row0);
          tma_load_2d(&map_bhi, &full[s], st + 2 * Cfg::A_B, kb * BK, brow0);
          tma_load_2d(&map_blo, &full[s], st + 2 * Cfg::A_B + Cfg::B_B, kb * BK, brow0);
          if (++s == Cfg::STAGES) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      constexpr uint32_t idesc = tf32_idesc_pair<kPairBN>();
      int s = 0;
      uint32_t ph = 0;
      for (long long q = 0; q < total_chunks; ++q) {
        const int c = static_cast<int>(q % nchunks);
        const int buf = static_cast<int>(q & 1);
        mbar_wait_cluster(&acc_empty[buf], static_cast<uint32_t>(((q >> 1) & 1) ^ 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + static_cast<uint32_t>(buf * kPairBN);
        const int kb_end = min(kblocks, (c + 1) * p.chunk);
        for (int kb = c * p.chunk; kb < kb_end; ++kb) {
          mbar_wait_cluster(&conv[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          uint8_t* st = smem + s * Cfg::STAGE_BYTES;
          const uint64_t a_hi = kmajor_sw128_desc(smem_u32(st));
          const uint64_t a_lo = kmajor_sw128_desc(smem_u32(st + Cfg::A_B));
          const uint64_t b_hi = kmajor_sw128_desc(smem_u32(st + 2 * Cfg::A_B));
          const uint64_t b_lo = kmajor_sw128_desc(smem_u32(st + 2 * Cfg::A_B + Cfg::B_B));
          const bool first = kb == c * p.chunk;
#pragma unroll
          for (int kk = 0; kk < BK / 8; ++kk) {
            const uint64_t adv = static_cast<uint64_t>(kk * 32 >> 4);
            umma2_tf32(d, a_hi + adv, b_hi + adv, idesc, (first && kk == 0) ? 0u : 1u);
            umma2_tf32(d, a_hi + adv, b_lo + adv, idesc, 1u);
            umma2_tf32(d, a_lo + adv, b_hi + adv, idesc, 1u);
          }
          umma2_commit_both(&empty[s]);
          if (++s == Cfg::STAGES) { s = 0; ph ^= 1; }
        }
        umma2_commit_both(&acc_full[buf]);
      }
    }
    __syncwarp();
  } else {
    const int wt = threadIdx.x - 64;
    const int quad = warp & 3;
    const int half = (warp - 2) >> 2;
    float acc[HALF];
#pragma unroll
    for (int i = 0; i < HALF; ++i) acc[i] = 0.f;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(quad * 32) << 16) + static_cast<uint32_t>(half * HALF);
    const int sa = tc_pending_shift(p.meta_a, p.norm_a), sb = tc_pending_shift(p.meta_b, p.norm_b);
    const int shift = sa + sb;
    float local = 0.f;
    int s = 0;
    uint32_t ph = 0;
    // Flat software pipeline over this pair's chunks: convert chunk q, then
    // promote chunk q-1 (complete by then), and after a tile's last chunk
    // write its epilogue -- the MMA meanwhile works on the next tile.
    for (long long q = 0; q <= total_chunks; ++q) {
      if (q < total_chunks) {
        const int c = static_cast<int>(q % nchunks);
        const int kb_end = min(kblocks, (c + 1) * p.chunk);
        for (int kb = c * p.chunk; kb < kb_end; ++kb) {
          mbar_wait(&full[s], ph);
          float4* a = reinterpret_cast<float4*>(smem + s * Cfg::STAGE_BYTES);
          float4* alo = reinterpret_cast<float4*>(smem + s * Cfg::STAGE_BYTES + Cfg::A_B);
#pragma unroll
          for (int i = 0; i < Cfg::A_B / 16 / kWorkers; ++i) {
            const int idx = i * kWorkers + wt;
            const float4 x = a[idx];
            float4 h, l;
            h.x = tf32_rna(x.x); l.x = x.x - h.x;
            h.y = tf32_rna(x.y); l.y = x.y - h.y;
            h.z = tf32_rna(x.z); l.z = x.z - h.z;
            h.w = tf32_rna(x.w); l.w = x.w - h.w;
            a[idx] = h;
            alo[idx] = l;
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          // One cluster-scope arrival per CTA (it costs a GPU-scope membar).
          asm volatile("bar.sync 1, %0;" ::"n"(kWorkers) : "memory");
          if (wt == 0) arrive_leader(&conv[s], rank);
          if (++s == Cfg::STAGES) { s = 0; ph ^= 1; }
        }
      }
      if (q >= 1) {
        const long long qq = q - 1;
        const int buf = static_cast<int>(qq & 1);
        mbar_wait(&acc_full[buf], static_cast<uint32_t>((qq >> 1) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
        for (int j = 0; j < HALF / 16; ++j) {
          float v[16];
          tmem_ld16(lane_base + static_cast<uint32_t>(buf * kPairBN + 16 * j), v);
#pragma unroll
          for (int i = 0; i < 16; ++i) acc[16 * j + i] += v[i];
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        asm volatile("bar.sync 1, %0;" ::"n"(kWorkers) : "memory");
        if (wt == 0) arrive_leader(&acc_empty[buf], rank);
        if (qq % nchunks == nchunks - 1) {  // tile complete: epilogue
          long long m_pair;
          int n_tile;
          pair_tile_coords(cluster + (qq / nchunks) * nclusters, m_pairs, p.n_tiles, m_pair, n_tile);
          // Rows quad*32 .. +31 of this CTA, columns half*HALF .. +HALF.
          const long long row_base = m_pair * 256 + static_cast<long long>(rank) * BM + quad * 32;
          float* base = p.c + row_base * p.n2 + static_cast<long long>(n_tile) * kPairBN + half * HALF;
          float* stg = epi_stage + (warp - 2) * 32 * Cfg::EPI_PITCH;
          // Fused output permutation: complex offset of (own row, tile's first column).
          long long my_row_off = 0, col_tile_off = 0;
          if (p.store_perm) {
            const long long grow = row_base + lane;
            for (int b = 0; b < p.nrow_bits; ++b)
              if ((grow >> b) & 1) my_row_off += 1ll << p.row_pos[b];
            const long long gcol = (static_cast<long long>(n_tile) * kPairBN + half * HALF) / 2;
            for (int b = 0; b < p.ncol_bits; ++b)
              if ((gcol >> b) & 1) col_tile_off += 1ll << p.col_pos[b];
          }
#pragma unroll
          for (int c0 = 0; c0 < HALF; c0 += 16) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float4 v = make_float4(scalbnf(acc[c0 + 4 * i], -shift), scalbnf(acc[c0 + 4 * i + 1], -shift),
                                           scalbnf(acc[c0 + 4 * i + 2], -shift), scalbnf(acc[c0 + 4 * i + 3], -shift));
              local = fmaxf(local, fmaxf(v.x * v.x + v.y * v.y, v.z * v.z + v.w * v.w));
              *reinterpret_cast<float4*>(stg + lane * Cfg::EPI_PITCH + 4 * i) = v;
            }
            __syncwarp();
            long long jc_off = 0;  // complex column offset of this lane's float4 within the chunk
            if (p.store_perm) {
              const int jloc = (c0 >> 1) + 2 * (lane & 3);  // complex column within the tile half
              for (int b = 0; b < 7 && b < p.ncol_bits; ++b)
                if ((jloc >> b) & 1) jc_off += 1ll << p.col_pos[b];
            }
#pragma unroll
            for (int it = 0; it < 4; ++it) {
              const int r = it * 8 + (lane >> 2), c4 = lane & 3;
              const float4 v = *reinterpret_cast<const float4*>(stg + r * Cfg::EPI_PITCH + 4 * c4);
              if (p.store_perm) {
                const long long ro = __shfl_sync(0xffffffffu, my_row_off, r);
                *reinterpret_cast<float4*>(p.c + 2 * (ro + col_tile_off + jc_off)) = v;
              } else {
                *reinterpret_cast<float4*>(base + static_cast<long long>(r) * p.n2 + c0 + 4 * c4) = v;
              }
            }
            __syncwarp();
          }
#pragma unroll
          for (int i = 0; i < HALF; ++i) acc[i] = 0.f;
        }
      }
    }
    if (p.meta_c) {
      for (int o = 16; o > 0; o >>= 1) local = fmaxf(local, __shfl_xor_sync(0xffffffffu, local, o));
      if (lane == 0 && local > 0.f) atomicMax(&p.meta_c->maxsq_bits, __float_as_uint(local));
      if (blockIdx.x == 0 && threadIdx.x == 64)
        p.meta_c->log_scale = (p.meta_a ? p.meta_a->log_scale : 0.0) + (p.meta_b ? p.meta_b->log_scale : 0.0) + shift;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(Cfg::TMEM_COLS));
  }
}

// ---------------------------------------------------------------------------
// 3xFP16 CTA-pair kernel (default for CTA-pair shapes with 2k % 64 == 0).
// Same persistent pipeline as cgemm_tc2_kernel, but each operand is split
// as x * 2^e = hi + lo with hi, lo fp16 and e a per-operand power of two
// that puts max|x| just below 2^15 (from the operand's device max |z|^2).
// hi and lo carry 11 + 11 significand bits (as 3xTF32 does) and the
// products run at the f16 tensor-core rate, twice the tf32 rate; the
// epilogue removes 2^-(ea+eb) exactly.  Elements more than 2^16 below the
// operand's max lose relative precision in lo gradually (subnormal fp16),
// i.e. their absolute error stays below 2^-39 max|x| -- far under FP32's
// normwise error for these sums.
// Stage layout (per CTA): raw A fp32 [128 rows x 64] as two SW128 TMA boxes
// of 32 columns, each converted IN PLACE to interleaved hi / lo SW64 atoms
// (32 fp16 = 64 B per row), then the pre-expanded B_r^T hi / lo fp16
// planes (SW128, 64 fp16 per row).
constexpr int BK16 = 64;  // real K per stage of the fp16 kernel
constexpr std::int64_t kF16Scratch = 256;  // workspace head: two TMeta operand-maximum slots

__device__ __forceinline__ int f16_exp(const TMeta* m) {
  if (m == nullptr) return 0;
  const unsigned bits = m->maxsq_bits;
  if (bits == 0 || bits >= 0x7f800000u) return 0;
  int e = 0;
  frexpf(sqrtf(__uint_as_float(bits)), &e);  // max|z| = f * 2^e, f in [0.5, 1)
  return 15 - e;
}

// Exponent e with max|z| < 2^e from the meta's max |z|^2 (-1000: all zero).
__device__ __forceinline__ int max_exp(const TMeta* m) {
  if (m == nullptr || m->maxsq_bits == 0 || m->maxsq_bits >= 0x7f800000u) return -1000;
  int e = 0;
  frexpf(sqrtf(__uint_as_float(m->maxsq_bits)), &e);
  return e;
}

// K-major, SWIZZLE_64B descriptor (rows of 64 B, 8-row atoms of 512 B at a
// 1 KiB stride: the hi and lo atoms of one 8-row group are interleaved).
__device__ __forceinline__ uint64_t kmajor_sw64_desc(uint32_t saddr, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(1) << 16;
  d |= static_cast<uint64_t>(sbo >> 4) << 32;  // stride between 8-row atoms
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(4) << 61;           // SWIZZLE_64B
  return d;
}

template <int BN>
__host__ __device__ constexpr uint32_t f16_idesc_pair() {
  return (1u << 4)                 // D format F32
         | (0u << 7) | (0u << 10)  // A, B format F16
         | (static_cast<uint32_t>(BN >> 3) << 17) | (static_cast<uint32_t>(256 >> 4) << 24);
}

__device__ __forceinline__ uint32_t elect_one() {
  uint32_t pred;
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, e;\n\t}"
      : "=r"(pred));
  return pred;
}

// Issued only by the lane with do_it != 0 (operands warp-uniform).
__device__ __forceinline__ void umma2_f16_if(uint32_t do_it, uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                             uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 e, %5, 0;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(do_it));
}

__device__ __forceinline__ void umma2_commit_both_if(uint32_t do_it, uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "setp.ne.b32 e, %2, 0;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
          smem_u32(bar)),
      "h"(static_cast<uint16_t>(0x3)), "r"(do_it)
      : "memory");
}

__device__ __forceinline__ uint32_t h2_bits(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }

// 8 fp32 (scaled by s) -> 8 fp16 hi + 8 fp16 lo, x*s = hi + lo (+ O(2^-22)).
__device__ __forceinline__ void split_f16x8(const float4& a, const float4& b, float s, uint4& hi, uint4& lo) {
  const float x[8] = {a.x * s, a.y * s, a.z * s, a.w * s, b.x * s, b.y * s, b.z * s, b.w * s};
  uint32_t h[4], l[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const __half2 hh = __floats2half2_rn(x[2 * j], x[2 * j + 1]);
    const float2 hf = __half22float2(hh);
    h[j] = h2_bits(hh);
    l[j] = h2_bits(__floats2half2_rn(x[2 * j] - hf.x, x[2 * j + 1] - hf.y));
  }
  hi = make_uint4(h[0], h[1], h[2], h[3]);
  lo = make_uint4(l[0], l[1], l[2], l[3]);
}

template <int BN, int KB = BK16>
struct Tc5Cfg {
  static constexpr int A_B = BM * KB * 4;        // raw fp32 A tile (= A hi + lo fp16 planes)
  static constexpr int B_B = (BN / 2) * KB * 2;  // one fp16 plane of this CTA's half of B_r^T
  static constexpr int STAGE_BYTES = A_B + 2 * B_B;
  static constexpr int EPI_PITCH = 20;  // fp32 / narrow path: 16-column slabs, padded rows
  // Per worker warp: a 32 x 32-float staging slab (split path: XOR-swizzled
  // 16-byte chunks, no padding) + a 32-entry table of its rows' permuted
  // offsets (32-bit, in units of 8 complex: rows never land on output bits 0..2).
  static constexpr int EPI_WARP_FLOATS = 32 * 32;
  static constexpr int EPI_BYTES = (kWorkers / 32) * (EPI_WARP_FLOATS * 4 + 32 * 4);
  static constexpr int BAR_BYTES = 512;  // mbarriers + TMEM slot
  static constexpr int SMEM_CAP = 232448 - 1024 - BAR_BYTES;  // 227 KiB opt-in minus alignment slack and barriers
  static constexpr int STAGES =
      ((SMEM_CAP - EPI_BYTES) / STAGE_BYTES) > 6 ? 6 : ((SMEM_CAP - EPI_BYTES) / STAGE_BYTES);
  static constexpr int SMEM = STAGES * STAGE_BYTES + EPI_BYTES + 1024 + BAR_BYTES;
  // TMEM accumulator buffers: two for 256-column tiles; narrow tiles (the
  // HBM-bound n <= 64 steps, one k-block per tile) keep up to 8 tiles in
  // flight so the MMA runs ahead of the per-tile epilogue / relay latency.
  static constexpr int NBUF = BN >= 256 ? 2 : (512 / BN > 8 ? 8 : 512 / BN);
  static constexpr int TMEM_COLS = NBUF * BN < 32 ? 32 : NBUF * BN;
  static_assert(3 * STAGES * 8 + 2 * NBUF * 8 + 8 <= BAR_BYTES, "barrier area");
  static_assert(STAGES >= 2, "shared memory budget");
};

// kSplitA: A arrives pre-split (fp16 hi / lo planes, tc_prep_a_f16_kernel or
// a producer epilogue), so the stage is TMA -> MMA with no worker pass:
// both CTAs' TMA loads complete on the leader's full[s] (cta_group::2) and
// the worker warps only promote and store.  map_a is then the A_hi plane
// and map_alo the A_lo plane (64 or 32 fp16 per row per stage: SW128 or SW64).
// kDirect: single-chunk tiles (k <= 64): no promotion registers; the
// epilogue reads each 16-column slab straight from TMEM and frees the
// accumulator buffer after the tile's stores (the MMA meanwhile fills the
// other buffer).  Without the 128 promoted floats per thread the worker
// warps run spill-free.
template <int kPairBN, bool kSplitA, int kBK = BK16, int kDirect = 0, bool kLane = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    cgemm_f16_pair_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_alo,
                          const __grid_constant__ CUtensorMap map_bhi, const __grid_constant__ CUtensorMap map_blo,
                          const TcParams p) {
  using Cfg = Tc5Cfg<kPairBN, kBK>;
  static_assert(kSplitA || kBK == kBK, "in-kernel A conversion uses 64-K stages");
  static_assert(kBK == 64 || kBK == 32, "stage K");
  constexpr int HALF = kPairBN / 2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // 1 KiB aligned, still __shared__
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
  uint64_t* conv = full + Cfg::STAGES;
  uint64_t* empty = conv + Cfg::STAGES;
  uint64_t* acc_full = empty + Cfg::STAGES;
  uint64_t* acc_empty = acc_full + Cfg::NBUF;
  uint32_t* tmem_base_slot = reinterpret_cast<uint32_t*>(acc_empty + Cfg::NBUF);
  float* epi_stage = reinterpret_cast<float*>(smem + Cfg::STAGES * Cfg::STAGE_BYTES + Cfg::BAR_BYTES);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const long long cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
  const long long m_pairs = p.m / 256;
  const long long total = m_pairs * p.n_tiles;
  const long long my_tiles = cluster < total ? (total - 1 - cluster) / nclusters + 1 : 0;

  if (threadIdx.x == 0) {
    // conv / acc_empty: one arrival per worker warp; the leader's also
    // count the peer's relayed arrival.
    const uint32_t cnt = kWorkers / 32 + (rank == 0 ? 1 : 0);
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], cnt);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < Cfg::NBUF; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], cnt);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_a) : "memory");
    if (kSplitA) asm volatile("prefetch.tensormap [%0];" ::"l"(&map_alo) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_bhi) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&map_blo) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_base_slot)),
                 "n"(Cfg::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_base_slot;
  // QSG_TC_PROF counters (lane 0 of each role): [0] producer waiting for a
  // free stage, [1] MMA waiting for a TMEM buffer, [2] MMA waiting for a
  // landed stage, [3] workers waiting for a full accumulator, [4] workers
  // promoting, [5] workers in the epilogue, [6] kernel cycles.
  unsigned long long prof_t0 = clock64(), prof_acc = 0;
  auto tick = [&]() { return p.prof ? clock64() : 0ull; };
  const int kblocks = p.kblocks;
  const int nchunks = (kblocks + p.chunk - 1) / p.chunk;
  const long long total_chunks = my_tiles * nchunks;

  if (warp == 0) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      bool sync_wait = true;
      for (long long ti = 0; ti < my_tiles; ++ti) {
        long long m_pair;
        int n_tile;
        pair_tile_coords(cluster + ti * nclusters, m_pairs, p.n_tiles, m_pair, n_tile, p.group_m);
        const int row0 = static_cast<int>(m_pair * 256 + static_cast<long long>(rank) * BM);
        const int brow0 = n_tile * kPairBN + static_cast<int>(rank) * (kPairBN / 2);
        // K-sync: the producers stay within two checkpoints of each other,
        // counted in k-blocks over the whole persistent run (tile ti of
        // every pair belongs to the same wave), so the A / B k-slabs that
        // concurrently running pairs share are still in L2 when the last of
        // them reads them.  Unsynchronised pairs drift apart by more than L2
        // holds and re-stream from HBM (long-K tiles: within a tile; short-K
        // tiles: across tiles).
        const long long gk0 = ti * kblocks;
        for (int kb = 0; kb < kblocks; ++kb) {
          const long long gk = gk0 + kb;
          if (p.sync && gk % p.sync_every == 0) {
            const long long c = gk / p.sync_every;
            atomicAdd(p.sync + c, 1u);
            if (c >= 1 && sync_wait) {
              // pairs whose run reaches k-block (c-1)*every: all with base
              // tiles if it falls inside those, else the `extra` ones.
              const long long kprev = (c - 1) * p.sync_every;
              const long long base = total / nclusters, extra = total % nclusters;
              const long long have = kprev < base * kblocks ? min(nclusters, total)
                                     : (kprev < (base + 1) * kblocks ? extra : 0);
              const unsigned need = 2u * static_cast<unsigned>(have);
              // Bounded spin: never a deadlock.  A wait that times out means
              // some pairs are not co-resident (other work on the GPU); this
              // producer then stops waiting for the rest of the launch.
              int spin = 0;
              for (; spin < 4096; ++spin) {
                unsigned v;
                asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p.sync + c - 1) : "memory");
                if (v >= need) break;
                __nanosleep(128);
              }
              if (spin == 4096) sync_wait = false;
            }
          }
          const unsigned long long w0 = tick();
          mbar_wait(&empty[s], ph ^ 1);
          if (p.prof) prof_acc += clock64() - w0;
          uint8_t* st = smem + s * Cfg::STAGE_BYTES;
          if constexpr (kSplitA) {
            // A streams from HBM with only STAGES boxes in flight per CTA
            // (the loop measured latency-bound: producer and MMA both
            // waiting, QSG_TC_PROF); prefetch the A boxes `prefetch`
            // k-blocks ahead into L2 so the stage loads hit L2.
            if (p.prefetch > 0) {
              const long long gp = gk + p.prefetch;
              const long long tp = gp / kblocks;
              if (tp < my_tiles) {
                long long mp_pair;
                int np_tile;
                pair_tile_coords(cluster + tp * nclusters, m_pairs, p.n_tiles, mp_pair, np_tile, p.group_m);
                const int prow = static_cast<int>(mp_pair * 256 + static_cast<long long>(rank) * BM);
                const int pk = static_cast<int>(gp % kblocks) * kBK;
                tma_prefetch_2d(&map_a, pk, prow);
                tma_prefetch_2d(&map_alo, pk, prow);
              }
            }
            // Both CTAs' bytes complete on the leader's full[s].
            uint32_t bar = smem_u32(&full[s]);
            if (rank == 0) mbar_expect_tx(&full[s], 2 * Cfg::STAGE_BYTES);
            else asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(bar) : "r"(bar));
            tma_load_2d_pair(&map_a, bar, st, kb * kBK, row0);
            tma_load_2d_pair(&map_alo, bar, st + Cfg::A_B / 2, kb * kBK, row0);
            tma_load_2d_pair(&map_bhi, bar, st + Cfg::A_B, kb * kBK, brow0);
            tma_load_2d_pair(&map_blo, bar, st + Cfg::A_B + Cfg::B_B, kb * kBK, brow0);
            if (++s == Cfg::STAGES) { s = 0; ph ^= 1; }
            continue;
          }
          const bool tail = p.half_tail && kb == kblocks - 1;
          mbar_expect_tx(&full[s], tail ? Cfg::STAGE_BYTES - Cfg::A_B / 2 : Cfg::STAGE_BYTES);
          tma_load_2d(&map_a, &full[s], st, kb * kBK, row0);
          if (!tail) tma_load_2d(&map_a, &full[s], st + Cfg::A_B / 2, kb * kBK + kBK / 2, row0);
          tma_load_2d(&map_bhi, &full[s], st + Cfg::A_B, kb * kBK, brow0);
          tma_load_2d(&map_blo, &full[s], st + Cfg::A_B + Cfg::B_B, kb * kBK, brow0);
          if (++s == Cfg::STAGES) { s = 0; ph ^= 1; }
        }
      }
    }
    if (p.prof && lane == 0) p.prof[8 * blockIdx.x + 0] = prof_acc;
  } else if (warp == 1) {
    if (rank == 0) {
      // The whole warp runs the issue loop (warp-uniform descriptors stay
      // in uniform registers); one elected lane issues each tcgen05 op.
      constexpr uint32_t idesc = f16_idesc_pair<kPairBN>();
      const uint32_t leader = elect_one();
      int s = 0, c = 0;
      uint32_t ph = 0;
      for (long long q = 0; q < total_chunks; ++q) {
        const int buf = static_cast<int>(q % Cfg::NBUF);
        const unsigned long long w0 = tick();
        mbar_wait_cluster(&acc_empty[buf], static_cast<uint32_t>(((q / Cfg::NBUF) & 1) ^ 1));
        if (p.prof) prof_acc += clock64() - w0;
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t d = tmem + static_cast<uint32_t>(buf * kPairBN);
        const int kb_end = min(kblocks, (c + 1) * p.chunk);
        for (int kb = c * p.chunk; kb < kb_end; ++kb) {
          const unsigned long long f0 = tick();
          if constexpr (kSplitA) mbar_wait(&full[s], ph);
          else mbar_wait_cluster(&conv[s], ph);
          if (p.prof && lane == 0) atomicAdd(p.prof + 8 * blockIdx.x + 2, clock64() - f0);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t st = smem_u32(smem + s * Cfg::STAGE_BYTES);
          // 64-K stages: SW128 planes (128-byte rows); 32-K stages: SW64 (64-byte rows, 512-byte atoms)
          const uint64_t b_hi = kBK == 64 ? kmajor_sw128_desc(st + Cfg::A_B) : kmajor_sw64_desc(st + Cfg::A_B, 512);
          const uint64_t b_lo = kBK == 64 ? kmajor_sw128_desc(st + Cfg::A_B + Cfg::B_B)
                                          : kmajor_sw64_desc(st + Cfg::A_B + Cfg::B_B, 512);
          const uint64_t a0 = kmajor_sw64_desc(st, 1024);
          const bool first = kb == c * p.chunk;
          const int nkk = (p.half_tail && kb == kblocks - 1) ? 2 : kBK / 16;  // zero-filled B half not needed
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk) {
            if (kk == nkk) break;
            uint64_t a_hi, a_lo;
            if constexpr (kSplitA) {  // +32 B per K=16 step
              a_hi = (kBK == 64 ? kmajor_sw128_desc(st) : kmajor_sw64_desc(st, 512)) + static_cast<uint64_t>(kk * 2);
              a_lo = (kBK == 64 ? kmajor_sw128_desc(st + Cfg::A_B / 2) : kmajor_sw64_desc(st + Cfg::A_B / 2, 512)) +
                     static_cast<uint64_t>(kk * 2);
            } else {
              a_hi = a0 + static_cast<uint64_t>(((kk >> 1) * (Cfg::A_B / 2) + (kk & 1) * 32) >> 4);
              a_lo = a_hi + (512 >> 4);
            }
            const uint64_t adv = static_cast<uint64_t>(kk * 32 >> 4);
            umma2_f16_if(leader, d, a_hi, b_hi + adv, idesc, (first && kk == 0) ? 0u : 1u);
            umma2_f16_if(leader, d, a_hi, b_lo + adv, idesc, 1u);
            if (p.passes >= 3) umma2_f16_if(leader, d, a_lo, b_hi + adv, idesc, 1u);
          }
          umma2_commit_both_if(leader, &empty[s]);
          if (++s == Cfg::STAGES) { s = 0; ph ^= 1; }
        }
        umma2_commit_both_if(leader, &acc_full[buf]);
        if (++c == nchunks) c = 0;
      }
      if (p.prof && lane == 0) p.prof[8 * blockIdx.x + 1] = prof_acc;
    } else if (lane == 0) {
      // Peer CTA: relay its workers' (CTA-scope, cheap) arrivals to the
      // leader's barriers.  The cluster-scope release this needs costs a
      // GPU-scope membar; issued here, by a thread with no outstanding
      // global stores, it stays off the worker warps' critical path.
      int s = 0;
      uint32_t ph = 0;
      for (long long q = 0; q <= total_chunks; ++q) {
        if (!kSplitA && q < total_chunks) {
          const int c = static_cast<int>(q % nchunks);
          const int kb_end = min(kblocks, (c + 1) * p.chunk);
          for (int kb = c * p.chunk; kb < kb_end; ++kb) {
            mbar_wait(&conv[s], ph);
            mbar_arrive_remote(&conv[s], 0);
            if (++s == Cfg::STAGES) { s = 0; ph ^= 1; }
          }
        }
        if (q >= 1) {
          const long long qq = q - 1;
          const int buf = static_cast<int>(qq % Cfg::NBUF);
          mbar_wait(&acc_empty[buf], static_cast<uint32_t>((qq / Cfg::NBUF) & 1));
          mbar_arrive_remote(&acc_empty[buf], 0);
        }
      }
    }
    __syncwarp();
  } else {
    const int quad = warp & 3;
    const int half = (warp - 2) >> 2;
    // kDirect 1 / 3 read the accumulator straight from TMEM in the epilogue
    // (3: the tile's two promotion chunks sit in consecutive ring buffers
    // and are summed there, in round-to-nearest fp32, per 16-column slab).
    constexpr bool kFromTmem = kDirect == 1 || kDirect == 3;
    float acc[kFromTmem ? 1 : HALF];
#pragma unroll
    for (int i = 0; i < (kFromTmem ? 1 : HALF); ++i) acc[i] = 0.f;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(quad * 32) << 16) + static_cast<uint32_t>(half * HALF);
    const int sa = tc_pending_shift(p.meta_a, p.norm_a), sb = tc_pending_shift(p.meta_b, p.norm_b);
    const int ea = p.a_presplit ? p.meta_a->split_exp : f16_exp(p.meta_a), eb = f16_exp(p.meta_b);
    const int shift = sa + sb;            // the reference's renormalisation (recorded in log_scale)
    const int unscale = shift + ea + eb;  // + the fp16 operand scaling
    const float scale_a = scalbnf(1.f, ea);
    // 2^-unscale as one or two exact power-of-two factors (cheaper than
    // scalbnf per element, same rounding: a single multiply by 2^u is exact
    // unless the result is subnormal, which both round identically).
    const int u1 = min(max(-unscale, -126), 127), u2 = -unscale - u1;
    const float f1 = __int_as_float((127 + u1) << 23);
    const float f2 = u2 == 0 ? 1.f : scalbnf(1.f, u2);
    // Split output: y = acc * 2^-t with |acc| <= 2k * max|A_s| * max|B_s| <
    // 2^(log2k + 1 + EA + EB) (A_s, B_s: the scaled operands the MMA saw,
    // EA / EB their exact max exponents), so t = log2k + 1 + EA + EB - 15
    // keeps |y| below 2^15 without knowing C's max.  Using the operands'
    // true maxima (not the 2^15 cap) keeps the headroom from compounding
    // along chains of split hand-offs.  data = y * 2^-split_exp with
    // split_exp = unscale - t.
    int t_split = 0;
    {
      const int xa = max_exp(p.meta_a), xb = max_exp(p.meta_b);
      if (xa > -1000 && xb > -1000) t_split = min(max(p.log2k + 1 + (xa + ea) + (xb + eb) - 15, -126), 126);
    }
    const float fy = __int_as_float((127 - t_split) << 23);
    uint8_t* const c_bytes = reinterpret_cast<uint8_t*>(p.c);
    const long long lo_plane = 4 * p.c_total;
    // Fused output permutation: the column part of a float4's offset is
    // f(c0 / 2) + f(2 * (lane & 3)) (disjoint bits of the complex column).
    long long lane_col_off = 0;
    // Fused permutation: per-warp table of the stored rows' offsets.
    uint32_t* const row_tab =
        reinterpret_cast<uint32_t*>(epi_stage + (kWorkers / 32) * Cfg::EPI_WARP_FLOATS) + (warp - 2) * 32;
    if (p.store_perm)
      for (int b = 0; b < 3 && b < p.ncol_bits; ++b)
        if (((2 * (lane & 3)) >> b) & 1) lane_col_off += 1ll << p.col_pos[b];
    auto col_bit = [&](int b) { return p.ncol_bits > b ? 1ll << p.col_pos[b] : 0ll; };
    // sum_b bit_b(x) << pos[b] over the warp's lanes (distinct bit positions:
    // the sum is an OR, reduced as two 32-bit halves).
    auto warp_bits = [&](long long x, int pos_lo, int pos_hi) {
      unsigned long long t = 0;
      if (pos_lo >= 0 && ((x >> lane) & 1)) t |= 1ull << pos_lo;
      if (pos_hi >= 0 && ((x >> (lane + 32)) & 1)) t |= 1ull << pos_hi;
      const unsigned lo = __reduce_or_sync(0xffffffffu, static_cast<unsigned>(t));
      const unsigned hi = __reduce_or_sync(0xffffffffu, static_cast<unsigned>(t >> 32));
      return static_cast<long long>((static_cast<unsigned long long>(hi) << 32) | lo);
    };
    float local = 0.f;
    unsigned long long prof_w[3] = {0, 0, 0};
    // Raw-A stage conversion, serviced cooperatively: the same warps convert
    // the stages of chunk q and write the epilogue of chunk q - 1.  Converting
    // all of chunk q first (each stage gated by the MMA freeing a smem slot)
    // left the tensor pipe idle during every epilogue (~51% busy on the
    // k = 256 class); now the epilogue polls between slabs and converts any
    // stage that has landed, so the MMA of chunk q runs under the epilogue
    // of chunk q - 1.  Cursor: next (chunk, k-block) to convert.
    int cv_s = 0;
    uint32_t cv_ph = 0;
    long long cv_q = 0;
    int cv_kb = 0;
    auto convert_stage = [&](int kb) {
      uint8_t* st = smem + cv_s * Cfg::STAGE_BYTES;
      // In place, warp-local: each 8-row group g of a box (1 KiB of raw
      // fp32) becomes its hi (512 B) and lo (512 B) SW64 atoms, so A_hi
      // / A_lo are 8-row atoms at a 1 KiB stride (SBO) and no warp
      // touches another warp's rows.  Lane = (row rl, 8-column group cg).
      const int rl = lane >> 2, cg = lane & 3;
      const int iters = (p.half_tail && kb == kblocks - 1 ? 1 : 2) * (BM / 8) / (kWorkers / 32);
#pragma unroll 1
      for (int it = 0; it < iters; ++it) {
        const int gi = it * (kWorkers / 32) + (warp - 2);  // 0..31 over both boxes
        uint8_t* grp = st + (gi >> 4) * (Cfg::A_B / 2) + (gi & 15) * 1024;
        const float4 x0 = *reinterpret_cast<const float4*>(grp + rl * 128 + (((2 * cg) ^ rl) << 4));
        const float4 x1 = *reinterpret_cast<const float4*>(grp + rl * 128 + (((2 * cg + 1) ^ rl) << 4));
        __syncwarp();
        uint4 h, l;
        split_f16x8(x0, x1, scale_a, h, l);
        const int off = rl * 64 + ((cg ^ ((rl >> 1) & 3)) << 4);
        *reinterpret_cast<uint4*>(grp + off) = h;
        *reinterpret_cast<uint4*>(grp + 512 + off) = l;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&conv[cv_s]);  // this warp's rows are converted
      if (++cv_s == Cfg::STAGES) { cv_s = 0; cv_ph ^= 1; }
    };
    // Convert stages of chunks <= q_lim: all of them (block) or only those
    // whose TMA has landed (poll).
    auto service = [&](long long q_lim, bool block) {
      if constexpr (!kSplitA) {
        while (cv_q <= q_lim && cv_q < total_chunks) {
          const int c = static_cast<int>(cv_q % nchunks);
          const int kb = c * p.chunk + cv_kb;
          if (block) mbar_wait(&full[cv_s], cv_ph);
          else if (!__shfl_sync(0xffffffffu, mbar_test(&full[cv_s], cv_ph) ? 1 : 0, 0)) return;  // warp-uniform
          convert_stage(kb);
          if (++cv_kb == min(kblocks, (c + 1) * p.chunk) - c * p.chunk) { cv_kb = 0; ++cv_q; }
        }
      }
    };
    for (long long q = 0; q <= total_chunks; ++q) {
      if (q == 0 || p.convert_ahead) service(q, true);
      if (q >= 1) {
        const long long qq = q - 1;
        const int buf = static_cast<int>(qq % Cfg::NBUF);
        const unsigned long long a0 = tick();
        if constexpr (kSplitA) {
          mbar_wait(&acc_full[buf], static_cast<uint32_t>((qq / Cfg::NBUF) & 1));
        } else {
          while (!__shfl_sync(0xffffffffu, mbar_test(&acc_full[buf], static_cast<uint32_t>((qq / Cfg::NBUF) & 1)) ? 1 : 0, 0))
            service(q, false);
        }
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const unsigned long long a1 = tick();
        if (p.prof) prof_w[0] += a1 - a0;
        if constexpr (!kDirect) {
#pragma unroll
          for (int j = 0; j < HALF / 16; ++j) {
            float v[16];
            tmem_ld16(lane_base + static_cast<uint32_t>(buf * kPairBN + 16 * j), v);
#pragma unroll
            for (int i = 0; i < 16; ++i) acc[16 * j + i] += v[i];
          }
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(&acc_empty[buf]);
        } else if constexpr (kDirect == 2) {
          // Early release: the whole accumulator slice goes to registers in
          // one burst of TMEM loads (one wait), and the buffer is handed
          // back to the MMA before any conversion or store.  With two 256-
          // column buffers the MMA otherwise waits for the slab-by-slab
          // epilogue of tile t before it may start tile t + 2.
#pragma unroll
          for (int j = 0; j < HALF / 16; ++j)
            tmem_ld16_nowait(lane_base + static_cast<uint32_t>(buf * kPairBN + 16 * j), &acc[16 * j]);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(&acc_empty[buf]);
        }
        const unsigned long long a2 = tick();
        if (p.prof) prof_w[1] += a2 - a1;
        const int prev = static_cast<int>((qq + Cfg::NBUF - 1) % Cfg::NBUF);  // kDirect 3: the tile's first chunk
        // 16 accumulator columns of this lane's row straight from TMEM.
        auto tmem16 = [&](int col, float* v) {
          tmem_ld16(lane_base + static_cast<uint32_t>(buf * kPairBN + col), v);
          if constexpr (kDirect == 3) {
            float w[16];
            tmem_ld16(lane_base + static_cast<uint32_t>(prev * kPairBN + col), w);
#pragma unroll
            for (int i = 0; i < 16; ++i) v[i] = w[i] + v[i];
          }
        };
        if (kDirect == 1 || kDirect == 2 || qq % nchunks == nchunks - 1) {
          long long m_pair;
          int n_tile;
          pair_tile_coords(cluster + (qq / nchunks) * nclusters, m_pairs, p.n_tiles, m_pair, n_tile, p.group_m);
          const long long row_base = m_pair * 256 + static_cast<long long>(rank) * BM + quad * 32;
          float* base = p.c + row_base * p.n2 + static_cast<long long>(n_tile) * kPairBN + half * HALF;
          float* stg = epi_stage + (warp - 2) * Cfg::EPI_WARP_FLOATS;
          long long my_row_off = 0, col_tile_off = 0;
          if (p.store_perm) {
            // row_base is a multiple of 32: its bits and the lane's are
            // disjoint.  Lane b reduces bit b (and b + 32); the positions are
            // re-read per tile (not kept in registers next to acc[]).
            const int rp0 = lane < p.nrow_bits ? p.row_pos[lane] : -1;
            const int rp1 = lane + 32 < p.nrow_bits ? p.row_pos[lane + 32] : -1;
            const int cpl = lane < p.ncol_bits ? p.col_pos[lane] : -1;
            my_row_off = warp_bits(row_base, rp0, rp1);
            for (int b = 0; b < 5 && b < p.nrow_bits; ++b)
              if ((lane >> b) & 1) my_row_off += 1ll << p.row_pos[b];
            const long long gcol = (static_cast<long long>(n_tile) * kPairBN + half * HALF) / 2;
            col_tile_off = warp_bits(gcol, cpl, -1);
          }
          // The rows' offsets, read back per store (no shuffles, no registers).
          if (p.store_perm) row_tab[lane] = static_cast<uint32_t>((my_row_off + col_tile_off) >> 3);
          bool stored = false;
          if constexpr (kLane) {
            static_assert((kDirect == 0 || kDirect == 1) && HALF >= 16, "lane stores: promoted or direct tiles");
            {
              // Split output, lane = row, no staging: every 8 complex of the
              // lane's row are one 32-byte run per plane (complex column
              // bits 0..2 are the output's bits 0..2 under the fused
              // permutation; natural order needs n % 8 == 0), written as one
              // STG.256 per plane straight from registers.  Its own
              // instantiation, so the staged paths' registers stay out.  The
              // max is kept on the split values y = acc * 2^-t and rescaled
              // once per tile (an exact power of two).
              const long long row_off =
                  p.store_perm ? my_row_off + col_tile_off
                               : (row_base + lane) * (p.n2 / 2) + (static_cast<long long>(n_tile) * kPairBN + half * HALF) / 2;
              float ymax = 0.f;
#pragma unroll
              for (int g = 0; g < HALF / 16; ++g) {
                if ((g & 1) == 0) service(q, false);
                float a16[16];
                if constexpr (kFromTmem) {
                  tmem16(16 * g, a16);
                } else {
#pragma unroll
                  for (int i = 0; i < 16; ++i) a16[i] = acc[16 * g + i];
                }
                uint32_t hh[8], ll[8];
#pragma unroll
                for (int t = 0; t < 8; ++t) {
                  const float y0 = a16[2 * t] * fy, y1 = a16[2 * t + 1] * fy;
                  ymax = fmaxf(ymax, y0 * y0 + y1 * y1);
                  const __half2 h = __floats2half2_rn(y0, y1);
                  const float2 g2 = __half22float2(h);
                  hh[t] = h2_bits(h);
                  ll[t] = h2_bits(__floats2half2_rn(y0 - g2.x, y1 - g2.y));
                }
                const long long o =
                    row_off + (p.store_perm ? ((g & 1) ? col_bit(3) : 0ll) + ((g & 2) ? col_bit(4) : 0ll) +
                                                  ((g & 4) ? col_bit(5) : 0ll)
                                            : 8ll * g);
                st_global_v8(c_bytes + 4 * o, hh, p.stream_store != 0);
                st_global_v8(c_bytes + lo_plane + 4 * o, ll, p.stream_store != 0);
              }
              local = fmaxf(local, scalbnf(ymax, 2 * (t_split - unscale)));
              stored = true;
            }
          }
          if constexpr (HALF >= 32 && kDirect) {
            if (p.c_split && !stored) {
              // Split output in 32-column slabs: lane = row stages 32 floats
              // (chunk c of row r at 16-byte slot c ^ (r & 7): conflict-free
              // both ways), then 4 lanes per row convert 4 complex each and
              // store 64-byte runs per plane (2x the 32-byte runs of 16-column
              // slabs; complex column bits 0..1 in-lane, 2..3 = lane & 3).
              // Short-K steps -15-20%.  Single-chunk (kDirect) tiles only: next
              // to the 128 promoted floats of the multi-chunk path ptxas spills
              // ~0.5 KB per thread, so those keep the 16-column slabs.
              const uint32_t stg_row = smem_u32(stg) + lane * 128;  // this lane's staged row
              const uint32_t stg_rd = smem_u32(stg) + (lane >> 2) * 128;
              const int sw = (lane >> 2) & 7;  // r & 7 of every row this lane reads
#pragma unroll
              for (int c0 = 0; c0 < HALF; c0 += 32) {
                service(q, false);
#pragma unroll
                for (int h16 = 0; h16 < 2; ++h16) {
                  float a16[16];
                  if constexpr (kFromTmem) {
                    tmem16(c0 + 16 * h16, a16);
                  } else {
#pragma unroll
                    for (int i = 0; i < 16; ++i) a16[i] = acc[c0 + 16 * h16 + i];
                  }
#pragma unroll
                  for (int i = 0; i < 4; ++i) {
                    float4 v =
                        make_float4(a16[4 * i] * f1, a16[4 * i + 1] * f1, a16[4 * i + 2] * f1, a16[4 * i + 3] * f1);
                    if (u2 != 0) { v.x *= f2; v.y *= f2; v.z *= f2; v.w *= f2; }
                    local = fmaxf(local, fmaxf(v.x * v.x + v.y * v.y, v.z * v.z + v.w * v.w));
                    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(stg_row + (((4 * h16 + i) ^ (lane & 7)) << 4)),
                                 "f"(a16[4 * i] * fy), "f"(a16[4 * i + 1] * fy), "f"(a16[4 * i + 2] * fy),
                                 "f"(a16[4 * i + 3] * fy)
                                 : "memory");
                  }
                }
                __syncwarp();
                const int g = lane & 3;
                const long long jg = (g & 1) * 4 + ((g >> 1) ? col_bit(3) : 0ll) + ((c0 >> 5) & 1 ? col_bit(4) : 0ll) +
                                     ((c0 >> 6) & 1 ? col_bit(5) : 0ll);
#pragma unroll
                for (int it = 0; it < 4; ++it) {
                  const int r = it * 8 + (lane >> 2);
                  float4 v0, v1;
                  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                               : "=f"(v0.x), "=f"(v0.y), "=f"(v0.z), "=f"(v0.w)
                               : "r"(stg_rd + it * 1024 + (((2 * g) ^ sw) << 4)));
                  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                               : "=f"(v1.x), "=f"(v1.y), "=f"(v1.z), "=f"(v1.w)
                               : "r"(stg_rd + it * 1024 + (((2 * g + 1) ^ sw) << 4)));
                  const long long o = p.store_perm
                                          ? (static_cast<long long>(row_tab[r]) << 3) + jg
                                          : ((base - p.c) + static_cast<long long>(r) * p.n2 + c0 + 8 * g) >> 1;
                  const float x[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
                  uint32_t hh[4], ll[4];
#pragma unroll
                  for (int j = 0; j < 4; ++j) {
                    const __half2 h = __floats2half2_rn(x[2 * j], x[2 * j + 1]);
                    const float2 gg = __half22float2(h);
                    hh[j] = h2_bits(h);
                    ll[j] = h2_bits(__floats2half2_rn(x[2 * j] - gg.x, x[2 * j + 1] - gg.y));
                  }
                  if (p.stream_store) {
                    __stcs(reinterpret_cast<uint4*>(c_bytes + 4 * o), make_uint4(hh[0], hh[1], hh[2], hh[3]));
                    __stcs(reinterpret_cast<uint4*>(c_bytes + lo_plane + 4 * o), make_uint4(ll[0], ll[1], ll[2], ll[3]));
                  } else {
                    *reinterpret_cast<uint4*>(c_bytes + 4 * o) = make_uint4(hh[0], hh[1], hh[2], hh[3]);
                    *reinterpret_cast<uint4*>(c_bytes + lo_plane + 4 * o) = make_uint4(ll[0], ll[1], ll[2], ll[3]);
                  }
                }
                __syncwarp();
              }
              stored = true;
            }
          }
          if (!stored) {
#pragma unroll
          for (int c0 = 0; c0 < HALF; c0 += 16) {
            if ((c0 & 31) == 0) service(q, false);
            float a16[16];
            if constexpr (kFromTmem) {
              tmem16(c0, a16);
            } else {
#pragma unroll
              for (int i = 0; i < 16; ++i) a16[i] = acc[c0 + i];
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              float4 v = make_float4(a16[4 * i] * f1, a16[4 * i + 1] * f1, a16[4 * i + 2] * f1, a16[4 * i + 3] * f1);
              if (u2 != 0) { v.x *= f2; v.y *= f2; v.z *= f2; v.w *= f2; }
              local = fmaxf(local, fmaxf(v.x * v.x + v.y * v.y, v.z * v.z + v.w * v.w));
              if ((HALF < 32 || !kDirect) && p.c_split)
                v = make_float4(a16[4 * i] * fy, a16[4 * i + 1] * fy, a16[4 * i + 2] * fy, a16[4 * i + 3] * fy);
              *reinterpret_cast<float4*>(stg + lane * Cfg::EPI_PITCH + 4 * i) = v;
            }
            __syncwarp();
            // column bits 3..5 of this 8-complex run (c0 < HALF <= 128: jhi < 64)
            const long long jc =
                ((c0 >> 4) & 1 ? col_bit(3) : 0ll) + ((c0 >> 5) & 1 ? col_bit(4) : 0ll) + ((c0 >> 6) & 1 ? col_bit(5) : 0ll);
            if ((HALF < 32 || !kDirect) && p.c_split) {
              // Split output, 4 complex per lane: one 16-byte hi and one
              // 16-byte lo store (half the store instructions of 2 complex).
#pragma unroll
              for (int it = 0; it < 2; ++it) {
                const int r = it * 16 + (lane >> 1), hf = lane & 1;
                const float4 v0 = *reinterpret_cast<const float4*>(stg + r * Cfg::EPI_PITCH + 8 * hf);
                const float4 v1 = *reinterpret_cast<const float4*>(stg + r * Cfg::EPI_PITCH + 8 * hf + 4);
                long long o;  // complex offset of v0.xy (col bits 0..2 are the output's bits 0..2)
                if (p.store_perm) {
                  o = (static_cast<long long>(row_tab[r]) << 3) + jc + 4 * hf;
                } else {
                  o = ((base - p.c) + static_cast<long long>(r) * p.n2 + c0 + 8 * hf) >> 1;
                }
                const float x[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
                uint32_t hh[4], ll[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  const __half2 h = __floats2half2_rn(x[2 * j], x[2 * j + 1]);
                  const float2 g = __half22float2(h);
                  hh[j] = h2_bits(h);
                  ll[j] = h2_bits(__floats2half2_rn(x[2 * j] - g.x, x[2 * j + 1] - g.y));
                }
                if (p.stream_store) {
                  __stcs(reinterpret_cast<uint4*>(c_bytes + 4 * o), make_uint4(hh[0], hh[1], hh[2], hh[3]));
                  __stcs(reinterpret_cast<uint4*>(c_bytes + lo_plane + 4 * o), make_uint4(ll[0], ll[1], ll[2], ll[3]));
                } else {
                  *reinterpret_cast<uint4*>(c_bytes + 4 * o) = make_uint4(hh[0], hh[1], hh[2], hh[3]);
                  *reinterpret_cast<uint4*>(c_bytes + lo_plane + 4 * o) = make_uint4(ll[0], ll[1], ll[2], ll[3]);
                }
              }
              __syncwarp();
              continue;
            }
#pragma unroll
            for (int it = 0; it < 4; ++it) {
              const int r = it * 8 + (lane >> 2), c4 = lane & 3;
              const float4 v = *reinterpret_cast<const float4*>(stg + r * Cfg::EPI_PITCH + 4 * c4);
              long long o;  // complex offset of v.xy in C
              if (p.store_perm) {
                o = (static_cast<long long>(row_tab[r]) << 3) + jc + lane_col_off;
              } else {
                o = ((base - p.c) + static_cast<long long>(r) * p.n2 + c0 + 4 * c4) >> 1;
              }
              if (p.stream_store) __stcs(reinterpret_cast<float4*>(p.c + 2 * o), v);
              else *reinterpret_cast<float4*>(p.c + 2 * o) = v;
            }
            __syncwarp();
          }
          }
          if constexpr (kFromTmem) {
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            if (lane == 0) {
              mbar_arrive(&acc_empty[buf]);
              if constexpr (kDirect == 3) mbar_arrive(&acc_empty[prev]);
            }
          } else if constexpr (kDirect == 0) {
#pragma unroll
            for (int i = 0; i < HALF; ++i) acc[i] = 0.f;
          }
          if (p.prof) prof_w[2] += clock64() - a2;
        }
      }
    }
    if (p.prof && warp == 2 && lane == 0) {
      p.prof[8 * blockIdx.x + 3] = prof_w[0];
      p.prof[8 * blockIdx.x + 4] = prof_w[1];
      p.prof[8 * blockIdx.x + 5] = prof_w[2];
    }
    if (p.meta_c) {
      for (int o = 16; o > 0; o >>= 1) local = fmaxf(local, __shfl_xor_sync(0xffffffffu, local, o));
      if (lane == 0 && local > 0.f) atomicMax(&p.meta_c->maxsq_bits, __float_as_uint(local));
      if (blockIdx.x == 0 && threadIdx.x == 64) {
        p.meta_c->log_scale = (p.meta_a ? p.meta_a->log_scale : 0.0) + (p.meta_b ? p.meta_b->log_scale : 0.0) + shift;
        if (p.c_split) p.meta_c->split_exp = unscale - t_split;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();
  if (p.prof && threadIdx.x == 0) p.prof[8 * blockIdx.x + 6] = clock64() - prof_t0;
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(Cfg::TMEM_COLS));
  }
}

// A (complex, [m][k] = fp32 [m][2k]) -> A hi / lo fp16 planes [m][2k], scaled by 2^ea.
__global__ void __launch_bounds__(256) tc_prep_a_f16_kernel(const float4* __restrict__ a, uint2* __restrict__ hi,
                                                            uint2* __restrict__ lo, long long n4,
                                                            const TMeta* __restrict__ meta_a) {
  const float s = scalbnf(1.f, f16_exp(meta_a));
  for (long long i = blockIdx.x * 256ll + threadIdx.x; i < n4; i += static_cast<long long>(gridDim.x) * 256) {
    const float4 x = a[i];
    const __half2 h0 = __floats2half2_rn(x.x * s, x.y * s), h1 = __floats2half2_rn(x.z * s, x.w * s);
    const float2 f0 = __half22float2(h0), f1 = __half22float2(h1);
    hi[i] = make_uint2(h2_bits(h0), h2_bits(h1));
    lo[i] = make_uint2(h2_bits(__floats2half2_rn(x.x * s - f0.x, x.y * s - f0.y)),
                       h2_bits(__floats2half2_rn(x.z * s - f1.x, x.w * s - f1.y)));
  }
}

// B (complex) -> B_r^T hi / lo fp16 planes [2n][2k] scaled by 2^eb.
__global__ void __launch_bounds__(256) tc_prep_b_f16_kernel(const float2* __restrict__ b, __half* __restrict__ hi,
                                                            __half* __restrict__ lo, long long n, long long k, int tb,
                                                            const TMeta* __restrict__ meta_b, long long pitch) {
  __shared__ float2 tile[32][33];
  const long long j0 = static_cast<long long>(blockIdx.x) * 32, p0 = static_cast<long long>(blockIdx.y) * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int r = ty; r < 32; r += 8) {
    if (!tb) {
      const long long p = p0 + r, j = j0 + tx;
      tile[r][tx] = (p < k && j < n) ? b[p * n + j] : make_float2(0.f, 0.f);
    } else {
      const long long j = j0 + r, p = p0 + tx;
      tile[tx][r] = (p < k && j < n) ? b[j * k + p] : make_float2(0.f, 0.f);
    }
  }
  __syncthreads();
  const float s = scalbnf(1.f, f16_exp(meta_b));
  for (int r = ty; r < 32; r += 8) {
    const long long j = j0 + r, p = p0 + tx;
    if (j >= n || p >= k) continue;
    const float2 v = tile[tx][r];
    const float re = v.x * s, im = v.y * s;
    const __half2 h0 = __floats2half2_rn(re, -im), h1 = __floats2half2_rn(im, re);
    const float2 f0 = __half22float2(h0), f1 = __half22float2(h1);
    const long long row0 = (2 * j) * pitch + 2 * p, row1 = (2 * j + 1) * pitch + 2 * p;
    *reinterpret_cast<__half2*>(hi + row0) = h0;
    *reinterpret_cast<__half2*>(hi + row1) = h1;
    *reinterpret_cast<__half2*>(lo + row0) = __floats2half2_rn(re - f0.x, -im - f0.y);
    *reinterpret_cast<__half2*>(lo + row1) = __floats2half2_rn(im - f1.x, re - f1.y);
  }
}

// B (complex, [k][n] or [n][k]) -> B_r^T hi/lo planes [2n][2k] fp32.
__global__ void __launch_bounds__(256) tc_prep_b_kernel(const float2* __restrict__ b, float* __restrict__ hi,
                                                        float* __restrict__ lo, long long n, long long k, int tb) {
  __shared__ float2 tile[32][33];  // [p_local][j_local]
  const long long j0 = static_cast<long long>(blockIdx.x) * 32, p0 = static_cast<long long>(blockIdx.y) * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  for (int r = ty; r < 32; r += 8) {
    if (!tb) {  // B[p][j], j contiguous
      const long long p = p0 + r, j = j0 + tx;
      tile[r][tx] = (p < k && j < n) ? b[p * n + j] : make_float2(0.f, 0.f);
    } else {    // B[j][p], p contiguous
      const long long j = j0 + r, p = p0 + tx;
      tile[tx][r] = (p < k && j < n) ? b[j * k + p] : make_float2(0.f, 0.f);
    }
  }
  __syncthreads();
  const long long k2 = 2 * k;
  for (int r = ty; r < 32; r += 8) {
    const long long j = j0 + r, p = p0 + tx;
    if (j >= n || p >= k) continue;
    const float2 v = tile[tx][r];
    const float re = v.x, im = v.y;
    const float h0 = tf32_rna(re), h1 = tf32_rna(-im), h2 = tf32_rna(im), h3 = h0;
    const long long row0 = (2 * j) * k2 + 2 * p, row1 = (2 * j + 1) * k2 + 2 * p;
    *reinterpret_cast<float2*>(hi + row0) = make_float2(h0, h1);
    *reinterpret_cast<float2*>(hi + row1) = make_float2(h2, h3);
    *reinterpret_cast<float2*>(lo + row0) = make_float2(re - h0, -im - h1);
    *reinterpret_cast<float2*>(lo + row1) = make_float2(im - h2, re - h3);
  }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<EncodeFn>(nullptr);
    return reinterpret_cast<EncodeFn>(p);
  }();
  if (!fn) throw std::runtime_error("CUDA error in cuTensorMapEncodeTiled lookup: entry point unavailable");
  return fn;
}

// TMA L2 promotion 256 B (measured best of none / 64 / 128 / 256 B on s026).
constexpr CUtensorMapL2promotion kL2Promo = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;

// 2-D fp32 K-major map: inner dim `cols` (contiguous), outer `rows`; box
// [box_rows x 32] with 128-byte swizzle.
CUtensorMap make_map(const void* base, long long cols, long long rows, int box_rows) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * 4};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(BK), static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box,
                                 estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, kL2Promo,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("CUDA error in cuTensorMapEncodeTiled: code " + std::to_string(r));
  return m;
}

// Row pitch (elements) of the fp16 B_r^T planes (padding the pitch was
// measured: no gain, more DRAM traffic).
long long b16_pitch(std::int64_t k) { return 2 * k; }

// fp16 map: inner dim `cols` (contiguous), box [box_rows x kb] with kb = 64
// (128 B rows, SW128) or 32 (64 B rows, SW64).
CUtensorMap make_map_f16(const void* base, long long cols, long long rows, long long pitch, int box_rows,
                         int kb = BK16) {
  CUtensorMap m;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(pitch) * 2};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(kb), static_cast<cuuint32_t>(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(base), dims, strides, box,
                                 estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                 kb == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B, kL2Promo,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("CUDA error in cuTensorMapEncodeTiled: code " + std::to_string(r));
  return m;
}

// QSG_TC_PROF=1 (diagnostics only; synchronises after every pair launch):
// per-CTA cycle counters of the pair kernel's roles, reported to stderr as
// fractions of the kernel's cycles (tc_prof_report).
unsigned long long*& tc_prof_storage() {
  static unsigned long long* buf = nullptr;
  return buf;
}

unsigned long long* tc_prof_buffer(cudaStream_t stream) {
  static const bool on = std::getenv("QSG_TC_PROF") && std::getenv("QSG_TC_PROF")[0] == '1';
  unsigned long long*& buf = tc_prof_storage();
  if (!on) return nullptr;
  if (!buf && cudaMalloc(&buf, 8 * sizeof(unsigned long long) * 512) != cudaSuccess) return nullptr;
  cudaMemsetAsync(buf, 0, 8 * sizeof(unsigned long long) * 512, stream);
  return buf;
}

void tc_prof_report(std::int64_t m, std::int64_t n, std::int64_t k, cudaStream_t stream) {
  unsigned long long* buf = tc_prof_storage();
  if (!buf) return;
  std::vector<unsigned long long> h(8 * 512);
  cudaStreamSynchronize(stream);
  cudaMemcpy(h.data(), buf, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  double sum[7] = {0, 0, 0, 0, 0, 0, 0};
  int ctas = 0, leaders = 0;
  for (int c = 0; c < 512; ++c) {
    if (h[8 * c + 6] == 0) continue;
    ++ctas;
    const double tot = static_cast<double>(h[8 * c + 6]);
    for (int f = 0; f < 6; ++f) sum[f] += h[8 * c + f] / tot;
    if (h[8 * c + 2] != 0) ++leaders;
    sum[6] += tot;
  }
  if (ctas == 0) return;
  std::fprintf(stderr,
               "qsg-prof m=%lld n=%lld k=%lld ctas=%d cycles=%.3g | producer wait-free-stage %.1f%% | MMA wait-TMEM "
               "%.1f%% wait-stage %.1f%% | workers wait-acc %.1f%% promote %.1f%% epilogue %.1f%%\n",
               static_cast<long long>(m), static_cast<long long>(n), static_cast<long long>(k), ctas, sum[6] / ctas,
               100 * sum[0] / ctas, 100 * sum[1] / std::max(leaders, 1), 100 * sum[2] / std::max(leaders, 1),
               100 * sum[3] / ctas, 100 * sum[4] / ctas, 100 * sum[5] / ctas);
}

int env_int(const char* name, int dflt) {
  const char* env = std::getenv(name);
  const int v = env ? std::atoi(env) : dflt;
  return v >= 1 ? v : dflt;
}

int chunk_blocks() {
  const char* env = std::getenv("QSG_TC_CHUNK");
  const int v = env ? std::atoi(env) : kChunkDefault;
  return v >= 1 ? v : kChunkDefault;
}

// Persistent grid: one CTA pair per SM pair (74 on a 148-SM B200).
long long pair_slots() {
  static long long n = [] {
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return static_cast<long long>(std::max(1, sms / 2));
  }();
  return n;
}

// Co-resident CTA pairs of a pair kernel (GPCs with an odd number of free
// SMs cannot host a pair on their last SM): the persistent grid must not
// exceed it, or the surplus clusters run as a serial tail wave.
template <typename Kern>
long long resident_pairs(Kern kernel, int smem) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(2 * pair_slots()));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = static_cast<size_t>(smem);
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, reinterpret_cast<const void*>(kernel), &cfg) != cudaSuccess || n <= 0) {
    cudaGetLastError();
    n = static_cast<int>(pair_slots());
  }
  if (std::getenv("QSG_TC_DEBUG")) std::fprintf(stderr, "qsg: %d co-resident CTA pairs (smem %d)\n", n, smem);
  return std::min<long long>(n, pair_slots());
}

// The CTA-pair kernel covers 256 x 256 (real) tiles; QSG_TC_2SM=0 disables it.
int pair_bn(std::int64_t n) {
  static const int cap = env_int("QSG_TC_PAIR_BN_MAX", 256);  // A/B knob
  for (int bn : {256, 128, 64, 32})
    if (bn <= cap && (2 * n) % bn == 0) return bn;
  return 0;
}

// QSG_TC_DIRECT2=1: short-K tiles promoted in two chunks run as 128-column
// tiles whose two chunk accumulators are summed in the epilogue straight
// from TMEM (kDirect 3: 4 ring buffers of 128 columns) instead of through
// 128 promotion registers per thread.  Measured 3-4% slower than the
// register path on configs 2/3/4 (the 128-column tiles cost more than the
// registers), so off by default.
bool two_chunk_direct(std::int64_t k) {
  const char* env = std::getenv("QSG_TC_DIRECT2");
  if (!(env && env[0] == '1')) return false;
  const std::int64_t kblocks = (2 * k + BK16 - 1) / BK16;
  return kblocks <= 8 && kblocks >= 2 && std::min<std::int64_t>(env_int("QSG_TC_SHORTK_CHUNKS", kShortKChunks), kblocks) == 2;
}

// Column tile of the fp16 pair kernel for a GEMM shape.
int f16_bn(std::int64_t n, std::int64_t k) {
  const int bn = pair_bn(n);
  return (bn == 256 && two_chunk_direct(k)) ? 128 : bn;
}

bool use_pair(std::int64_t m, std::int64_t n) {
  const char* env = std::getenv("QSG_TC_2SM");
  if (env && env[0] == '0') return false;
  return m % 256 == 0 && pair_bn(n) > 0;
}

template <int BN>
cudaError_t launch_pair(const GemmArgs& g, const float* bhi, const float* blo, cudaStream_t stream) {
  const CUtensorMap ma = make_map(g.a, 2 * g.k, g.m, BM);
  const CUtensorMap mbh = make_map(bhi, 2 * g.k, 2 * g.n, BN / 2);
  const CUtensorMap mbl = make_map(blo, 2 * g.k, 2 * g.n, BN / 2);
  TcParams p{};
  p.c = static_cast<float*>(g.c);
  p.m = g.m;
  p.n2 = 2 * g.n;
  p.kblocks = static_cast<int>((2 * g.k) / BK);
  p.meta_a = g.meta_a;
  p.meta_b = g.meta_b;
  p.meta_c = g.meta_c;
  p.norm_a = g.norm_a;
  p.norm_b = g.norm_b;
  p.chunk = chunk_blocks();
  p.store_perm = g.store_perm ? 1 : 0;
  p.nrow_bits = g.nrow_bits;
  p.ncol_bits = g.ncol_bits;
  std::memcpy(p.row_pos, g.row_pos, sizeof p.row_pos);
  std::memcpy(p.col_pos, g.col_pos, sizeof p.col_pos);
  const long long pairs = (g.m / 256) * ((2 * g.n) / BN);
  if (pairs >= (1ll << 31)) return cudaErrorInvalidValue;  // pair_tile_coords divides in 32 bits
  p.n_tiles = static_cast<int>((2 * g.n) / BN);
  static const long long slots = [] {
    cudaFuncSetAttribute(cgemm_tc2_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, Tc2Cfg<BN>::SMEM);
    return resident_pairs(cgemm_tc2_kernel<BN>, Tc2Cfg<BN>::SMEM);
  }();
  const long long clusters = std::min<long long>(pairs, slots);
  cgemm_tc2_kernel<BN><<<static_cast<unsigned>(2 * clusters), kThreads, Tc2Cfg<BN>::SMEM, stream>>>(ma, mbh, mbl, p);
  return cudaGetLastError();
}

// Operand precision of the CTA-pair path: 3xFP16 with power-of-two operand
// scaling (default) or 3xTF32 (QSG_TC_PREC=tf32).
bool use_f16(std::int64_t m, std::int64_t n, std::int64_t k) {
  const char* env = std::getenv("QSG_TC_PREC");
  if (env && std::strcmp(env, "tf32") == 0) return false;
  return use_pair(m, n) && (2 * k) % (BK16 / 2) == 0;
}

// K-sync checkpoint spacing in k-blocks (QSG_TC_SYNC; 0 disables).
int sync_every() {
  const char* env = std::getenv("QSG_TC_SYNC");
  return env ? std::max(0, std::atoi(env)) : 16;
}

// Counters for every checkpoint of the longest per-pair run (at most all
// tiles on one pair); 0 when K-sync is off.
std::int64_t sync_bytes(std::int64_t m, std::int64_t n, std::int64_t k) {
  const int every = sync_every();
  const std::int64_t kblocks = (2 * k + 31) / 32;  // 32-K stages (QSG_TC_STAGEK=32) count twice the 64-K blocks
  if (every <= 0 || !use_pair(m, n)) return 0;
  const std::int64_t tiles = (m / 256) * ((2 * n) / f16_bn(n, k));
  return ((((tiles * kblocks) / every + 2) * 4 + 255) / 256) * 256;  // checkpoints of the longest run (1 pair)
}

// Pre-split A: a streaming pass converts A to fp16 hi / lo planes so the
// GEMM's stages are pure TMA -> MMA (tensor pipe ~98% busy instead of ~68%
// with the in-kernel conversion on the critical path).  The pass moves
// 16 B per complex element of A; the GEMM spends ~8n flop on each, so it
// pays from n ~ 1024 complex columns up (measured: s026 / s038 of config 2
// and the 2^15 cubes of config 5 gain 20-30%, the n = 256 steps lose).
// QSG_TC_SPLITA=0/1 forces it off/on (where the shape allows).
bool split_a(std::int64_t m, std::int64_t n, std::int64_t k) {
  if (!use_f16(m, n, k) || (2 * k) % BK16 != 0) return false;
  const char* env = std::getenv("QSG_TC_SPLITA");
  if (env) return env[0] == '1';
  return n >= 1024;
}

template <int BN>
cudaError_t launch_f16_pair(const GemmArgs& g, const TMeta* meta_a, const TMeta* meta_b, const __half* bhi,
                            const __half* blo, unsigned int* sync, const __half* ahi, const __half* alo,
                            cudaStream_t stream) {
  const bool split = ahi != nullptr;
  // 64-K stages (3 in flight).  32-K stages (6 in flight, SW64 planes; the
  // kernel's kBK = 32 instantiation) measured 2-6% slower on the long-K
  // steps: the per-stage barrier / commit overhead outweighs the deeper TMA
  // lookahead.  QSG_TC_STAGEK=32 selects them for short-K (k <= 256)
  // pre-split tiles, whose A streams from HBM (more bytes in flight).
  static const bool stage32 = env_int("QSG_TC_STAGEK", 64) == 32;
  // k <= 16 (one 32-K block): 32-K stages always -- a 64-K box would stage
  // half zero-fill and twice the L2 reads (the m = 2^27 bond-closing steps).
  const int kb = (split && ((stage32 && 2 * g.k <= 512) || 2 * g.k <= 32)) ? 32 : BK16;
  const CUtensorMap ma = split ? make_map_f16(ahi, 2 * g.k, g.m, 2 * g.k, BM, kb) : make_map(g.a, 2 * g.k, g.m, BM);
  const CUtensorMap mal = split ? make_map_f16(alo, 2 * g.k, g.m, 2 * g.k, BM, kb) : ma;
  const CUtensorMap mbh = make_map_f16(bhi, 2 * g.k, 2 * g.n, b16_pitch(g.k), BN / 2, kb);
  const CUtensorMap mbl = make_map_f16(blo, 2 * g.k, 2 * g.n, b16_pitch(g.k), BN / 2, kb);
  TcParams p{};
  p.c = static_cast<float*>(g.c);
  p.m = g.m;
  p.n2 = 2 * g.n;
  p.kblocks = static_cast<int>((2 * g.k + kb - 1) / kb);
  p.half_tail = (2 * g.k) % kb != 0 ? 1 : 0;
  p.group_m = env_int("QSG_TC_GROUPM", kGroupM);
  p.sync = sync;
  p.sync_every = sync_every();
  p.a_presplit = g.a_presplit ? 1 : 0;
  p.c_split = g.c_split ? 1 : 0;
  int l2k = 0;
  while ((std::int64_t{1} << l2k) < g.k) ++l2k;
  p.log2k = l2k;
  p.c_total = g.m * g.n;
  p.stream_store = std::getenv("QSG_TC_STCS") && std::getenv("QSG_TC_STCS")[0] == '0' ? 0 : 1;  // measured ~2% on config 2
  {
    // Lane-per-row split stores (QSG_TC_LANESTORE=0: the staged slab paths):
    // 32-byte aligned planes and 8-complex runs per row.
    const char* ls = std::getenv("QSG_TC_LANESTORE");
    const bool on = !(ls && ls[0] == '0');
    p.lane_store = on && g.c_split && reinterpret_cast<std::uintptr_t>(g.c) % 32 == 0 && p.c_total % 8 == 0 &&
                           (g.store_perm || g.n % 8 == 0)
                       ? 1
                       : 0;
  }
  p.passes = env_int("QSG_TC_PASSES", 3) == 2 ? 2 : 3;  // 2: inaccurate, measures MMA-count vs power only
  p.prof = tc_prof_buffer(stream);
  p.prefetch = env_int("QSG_TC_PREFETCH", 0) > 0 ? env_int("QSG_TC_PREFETCH", 0) : 0;
  p.convert_ahead = std::getenv("QSG_TC_SERVICE") && std::getenv("QSG_TC_SERVICE")[0] == '0' ? 1 : 0;
  p.meta_a = meta_a;
  p.meta_b = meta_b;
  p.meta_c = g.meta_c;
  p.norm_a = g.norm_a && g.meta_a != nullptr;
  p.norm_b = g.norm_b && g.meta_b != nullptr;
  // Promotion interval: 128 real K (2 k-blocks; relative error ~1e-6,
  // linear in the interval, tests/tc_accuracy).  Short-K tiles (k <= 256,
  // at most 512 real K) run as ONE chunk: no promotion, the epilogue stores
  // straight from TMEM (kDirect).  Every promotion is a TMEM hand-off
  // between the MMA and the worker warps that also write the tile epilogue;
  // measured on config 2: 4 chunks per k=256 tile -> 2 chunks 25-35% faster,
  // 2 -> 1 another 21% (batch -4%), amplitudes vs the FP32-SIMT engine
  // rel-L2 9.3e-6 -> 1.5e-5, batch fidelity 1 - 2e-11 (north star: 1 - 1e-6).
  const char* chunk_env = std::getenv("QSG_TC_CHUNK");
  const int per128 = 128 / kb;  // k-blocks per 128 real K
  if (chunk_env) p.chunk = std::max(1, chunk_blocks() * per128 / 4);
  else if (p.kblocks <= 4 * per128) {
    // Short K (<= 512 real K): a k = 256 tile in QSG_TC_SHORTK_CHUNKS
    // promotion chunks (1 = one unpromoted TMEM chunk, stored straight from
    // TMEM); shorter tiles keep the same chunk LENGTH (256 real K by
    // default), so k <= 128 is one chunk, stored directly (config 4's
    // k = 128 class 12.3 -> 7.x ms) at the accuracy the k = 256 chunks have.
    const int parts = std::min(env_int("QSG_TC_SHORTK_CHUNKS", kShortKChunks), 4 * per128);
    p.chunk = std::min(p.kblocks, (4 * per128 + parts - 1) / parts);
  } else {
    p.chunk = per128;
  }
  p.store_perm = g.store_perm ? 1 : 0;
  p.nrow_bits = g.nrow_bits;
  p.ncol_bits = g.ncol_bits;
  std::memcpy(p.row_pos, g.row_pos, sizeof p.row_pos);
  std::memcpy(p.col_pos, g.col_pos, sizeof p.col_pos);
  const long long pairs = (g.m / 256) * ((2 * g.n) / BN);
  if (pairs >= (1ll << 31)) return cudaErrorInvalidValue;  // pair_tile_coords divides in 32 bits
  p.n_tiles = static_cast<int>((2 * g.n) / BN);
  // One column tile: no pair shares an A slab with another (B is one small
  // tile), so K-sync only adds a grid-wide wait every `sync_every` tiles
  // (config 4's m = 2^27, n = k = 16 steps: -5% without it).
  if (p.n_tiles == 1) p.sync = nullptr;
  static const long long slots = [] {
    cudaFuncSetAttribute(cgemm_f16_pair_kernel<BN, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         Tc5Cfg<BN>::SMEM);
    cudaFuncSetAttribute(cgemm_f16_pair_kernel<BN, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         Tc5Cfg<BN>::SMEM);
    return resident_pairs(cgemm_f16_pair_kernel<BN, false>, Tc5Cfg<BN>::SMEM);
  }();
  static const bool attrs_direct3 = [] {
    if constexpr (BN <= 128) {
      cudaFuncSetAttribute(cgemm_f16_pair_kernel<BN, false, BK16, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           Tc5Cfg<BN>::SMEM);
      cudaFuncSetAttribute(cgemm_f16_pair_kernel<BN, true, BK16, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           Tc5Cfg<BN>::SMEM);
    }
    return true;
  }();
  (void)attrs_direct3;
  static const bool attrs_direct = [] {
    cudaFuncSetAttribute(cgemm_f16_pair_kernel<BN, false, BK16, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         Tc5Cfg<BN>::SMEM);
    cudaFuncSetAttribute(cgemm_f16_pair_kernel<BN, true, BK16, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         Tc5Cfg<BN>::SMEM);
    cudaFuncSetAttribute(cgemm_f16_pair_kernel<BN, false, BK16, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         Tc5Cfg<BN>::SMEM);
    cudaFuncSetAttribute(cgemm_f16_pair_kernel<BN, true, BK16, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         Tc5Cfg<BN>::SMEM);
    return true;
  }();
  (void)attrs_direct;
  const long long clusters = std::min<long long>(pairs, slots);
  const unsigned grid = static_cast<unsigned>(2 * clusters);
  const bool direct = p.kblocks <= p.chunk && !(std::getenv("QSG_TC_DIRECT") && std::getenv("QSG_TC_DIRECT")[0] == '0');
  // Early TMEM release for single-chunk tiles (QSG_TC_EARLY=0: slab-by-slab reads).
  static const bool early = std::getenv("QSG_TC_EARLY") && std::getenv("QSG_TC_EARLY")[0] == '1';
  if (kb == 32) {
    static const bool attrs32 = [] {
      cudaFuncSetAttribute(cgemm_f16_pair_kernel<BN, true, 32, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           Tc5Cfg<BN, 32>::SMEM);
      cudaFuncSetAttribute(cgemm_f16_pair_kernel<BN, true, 32, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           Tc5Cfg<BN, 32>::SMEM);
      return true;
    }();
    (void)attrs32;
    if (p.lane_store) {
      static const bool attrs32l = [] {
        cudaFuncSetAttribute(cgemm_f16_pair_kernel<BN, true, 32, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             Tc5Cfg<BN, 32>::SMEM);
        cudaFuncSetAttribute(cgemm_f16_pair_kernel<BN, true, 32, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             Tc5Cfg<BN, 32>::SMEM);
        return true;
      }();
      (void)attrs32l;
      if (direct)
        cgemm_f16_pair_kernel<BN, true, 32, 1, true><<<grid, kThreads, Tc5Cfg<BN, 32>::SMEM, stream>>>(ma, mal, mbh, mbl, p);
      else
        cgemm_f16_pair_kernel<BN, true, 32, 0, true><<<grid, kThreads, Tc5Cfg<BN, 32>::SMEM, stream>>>(ma, mal, mbh, mbl, p);
      return cudaGetLastError();
    }
    if (direct)
      cgemm_f16_pair_kernel<BN, true, 32, 1><<<grid, kThreads, Tc5Cfg<BN, 32>::SMEM, stream>>>(ma, mal, mbh, mbl, p);
    else
      cgemm_f16_pair_kernel<BN, true, 32, 0><<<grid, kThreads, Tc5Cfg<BN, 32>::SMEM, stream>>>(ma, mal, mbh, mbl, p);
    return cudaGetLastError();
  }
  const bool direct3 = !direct && BN <= 128 && p.kblocks <= 8 && (p.kblocks + p.chunk - 1) / p.chunk == 2 &&
                       two_chunk_direct(g.k);
  if constexpr (BN <= 128) {
    if (direct3) {
      if (split)
        cgemm_f16_pair_kernel<BN, true, BK16, 3><<<grid, kThreads, Tc5Cfg<BN>::SMEM, stream>>>(ma, mal, mbh, mbl, p);
      else
        cgemm_f16_pair_kernel<BN, false, BK16, 3><<<grid, kThreads, Tc5Cfg<BN>::SMEM, stream>>>(ma, mal, mbh, mbl, p);
      return cudaGetLastError();
    }
  }
  if (p.lane_store && !(direct && early)) {
    static const bool attrs_lane = [] {
      cudaFuncSetAttribute(cgemm_f16_pair_kernel<BN, true, BK16, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           Tc5Cfg<BN>::SMEM);
      cudaFuncSetAttribute(cgemm_f16_pair_kernel<BN, false, BK16, 0, true>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, Tc5Cfg<BN>::SMEM);
      cudaFuncSetAttribute(cgemm_f16_pair_kernel<BN, true, BK16, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           Tc5Cfg<BN>::SMEM);
      cudaFuncSetAttribute(cgemm_f16_pair_kernel<BN, false, BK16, 1, true>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, Tc5Cfg<BN>::SMEM);
      return true;
    }();
    (void)attrs_lane;
    if (direct && split)
      cgemm_f16_pair_kernel<BN, true, BK16, 1, true><<<grid, kThreads, Tc5Cfg<BN>::SMEM, stream>>>(ma, mal, mbh, mbl, p);
    else if (direct)
      cgemm_f16_pair_kernel<BN, false, BK16, 1, true><<<grid, kThreads, Tc5Cfg<BN>::SMEM, stream>>>(ma, mal, mbh, mbl, p);
    else if (split)
      cgemm_f16_pair_kernel<BN, true, BK16, 0, true><<<grid, kThreads, Tc5Cfg<BN>::SMEM, stream>>>(ma, mal, mbh, mbl, p);
    else
      cgemm_f16_pair_kernel<BN, false, BK16, 0, true><<<grid, kThreads, Tc5Cfg<BN>::SMEM, stream>>>(ma, mal, mbh, mbl, p);
    return cudaGetLastError();
  }
  if (direct && split && early)
    cgemm_f16_pair_kernel<BN, true, BK16, 2><<<grid, kThreads, Tc5Cfg<BN>::SMEM, stream>>>(ma, mal, mbh, mbl, p);
  else if (direct && early)
    cgemm_f16_pair_kernel<BN, false, BK16, 2><<<grid, kThreads, Tc5Cfg<BN>::SMEM, stream>>>(ma, mal, mbh, mbl, p);
  else if (direct && split)
    cgemm_f16_pair_kernel<BN, true, BK16, 1><<<grid, kThreads, Tc5Cfg<BN>::SMEM, stream>>>(ma, mal, mbh, mbl, p);
  else if (direct)
    cgemm_f16_pair_kernel<BN, false, BK16, 1><<<grid, kThreads, Tc5Cfg<BN>::SMEM, stream>>>(ma, mal, mbh, mbl, p);
  else if (split)
    cgemm_f16_pair_kernel<BN, true><<<grid, kThreads, Tc5Cfg<BN>::SMEM, stream>>>(ma, mal, mbh, mbl, p);
  else
    cgemm_f16_pair_kernel<BN, false><<<grid, kThreads, Tc5Cfg<BN>::SMEM, stream>>>(ma, mal, mbh, mbl, p);
  return cudaGetLastError();
}

int tc_bn(std::int64_t n) {
  const char* env = std::getenv("QSG_TC_BN");
  const int want = env ? std::atoi(env) : 256;
  if (want == 256 && (2 * n) % 256 == 0) return 256;
  return 128;
}

template <int BN>
void setup_attr() {
  static std::once_flag once;
  std::call_once(once, [] {
    cudaFuncSetAttribute(cgemm_tc_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, TcCfg<BN>::SMEM);
  });
}


// ---------------------------------------------------------------------------
// 3M (Gauss / Karatsuba) complex products on the same CTA-pair kernel.
//   P1 = Ar Br,  P2 = Ai Bi,  P3 = (Ar + Ai)(Br + Bi)
//   Re C = P1 - P2,  Im C = P3 - P1 - P2
// three REAL GEMMs of the complex shape (3 m n k MACs) instead of the 2x2
// embedding's one real GEMM of 4 m n k MACs: 25% fewer tensor-core passes,
// which under the board's power cap is the lever left (measured: dropping a
// third of the MMAs ran config 2 / 5 1.22-1.26x faster).  Each real product
// is the pair kernel on a "complex" shape (m, n/2, k/2): A = the [m][k] real
// plane pair, B^T = the [n][k] real plane pair, C = [m][n] fp32.  Operand
// planes are built by one streaming pass each (A: 20 B per complex element,
// B: small), the products go to workspace, and a combine pass forms C,
// applies the operands' pending renormalisation and updates TMeta.  Used on
// compute-heavy steps only (n, k >= kMin3M): the operand passes cost ~300/n
// and the combine ~480/k of the GEMM's time, and the step loses the fused
// store / split hand-offs (the combine writes complex64 in natural order).
// Measured: config 5's 2^15 cubes 1007 -> 839 ms, config 2 506 -> 403 ms per
// batch; at n = k = 1024 (config 5's 2^20 x 2^10 x 2^10 steps) it lost 35%.
constexpr std::int64_t kMin3M = 4096;

// |S| = |Re + Im| <= sqrt(2) max|z|: one exponent below the 2x2 path's.
__device__ __forceinline__ int f16_exp_3m(const TMeta* m) { return f16_exp(m) - 1; }

__device__ __forceinline__ void split16(float x, __half& hi, __half& lo) {
  hi = __float2half_rn(x);
  lo = __float2half_rn(x - __half2float(hi));
}

// A (complex [m][k]: raw fp32, or split fp16 hi | lo planes of the 2x2 path
// with value (hi + lo) 2^-split_exp) -> Ar, Ai, S = Ar + Ai, each as fp16
// hi | lo planes [m][k] scaled by 2^(f16_exp(meta) - 1).
__device__ __forceinline__ uint32_t pack_h2(__half lo, __half hi) {
  return static_cast<uint32_t>(__half_as_ushort(lo)) | (static_cast<uint32_t>(__half_as_ushort(hi)) << 16);
}

__global__ void __launch_bounds__(256) tc3m_prep_a_kernel(const void* __restrict__ a, int presplit,
                                                          long long count, const TMeta* __restrict__ meta,
                                                          __half* __restrict__ planes, TMeta* __restrict__ scratch) {
  const int ea = f16_exp_3m(meta);
  const float s = scalbnf(1.f, ea - (presplit ? meta->split_exp : 0));
  if (blockIdx.x == 0 && threadIdx.x == 0) scratch->split_exp = ea;
  __half* const arh = planes;
  __half* const arl = arh + count;
  __half* const aih = arl + count;
  __half* const ail = aih + count;
  __half* const ssh = ail + count;
  __half* const ssl = ssh + count;
  const long long stride = static_cast<long long>(gridDim.x) * 256;
  // 8 complex per thread and pass: 2 x 32-byte reads, 6 x 16-byte plane
  // writes (count % 8 == 0 keeps every plane 16-byte aligned); the element
  // arithmetic is the scalar tail's.
  const bool aligned = ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(planes)) & 15) == 0;
  const long long n8 = count % 8 == 0 && aligned ? count / 8 : 0;
  for (long long v = blockIdx.x * 256ll + threadIdx.x; v < n8; v += stride) {
    float re[8], im[8];
    if (presplit) {
      const uint4* hp = reinterpret_cast<const uint4*>(a) + 2 * v;
      const uint4* lp = reinterpret_cast<const uint4*>(reinterpret_cast<const __half2*>(a) + count) + 2 * v;
      const uint4 hw[2] = {__ldcs(hp), __ldcs(hp + 1)}, lw[2] = {__ldcs(lp), __ldcs(lp + 1)};
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const uint32_t hs[4] = {hw[q].x, hw[q].y, hw[q].z, hw[q].w}, ls[4] = {lw[q].x, lw[q].y, lw[q].z, lw[q].w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const __half2 h = *reinterpret_cast<const __half2*>(&hs[t]), l = *reinterpret_cast<const __half2*>(&ls[t]);
          re[4 * q + t] = __low2float(h) + __low2float(l);
          im[4 * q + t] = __high2float(h) + __high2float(l);
        }
      }
    } else {
      const float4* fp = reinterpret_cast<const float4*>(a) + 4 * v;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float4 f = __ldcs(fp + q);
        re[2 * q] = f.x;
        im[2 * q] = f.y;
        re[2 * q + 1] = f.z;
        im[2 * q + 1] = f.w;
      }
    }
    uint32_t w[6][4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      __half h[6][2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const float r = re[2 * t + u] * s, m = im[2 * t + u] * s;
        split16(r, h[0][u], h[1][u]);
        split16(m, h[2][u], h[3][u]);
        split16(r + m, h[4][u], h[5][u]);
      }
#pragma unroll
      for (int pl = 0; pl < 6; ++pl) w[pl][t] = pack_h2(h[pl][0], h[pl][1]);
    }
    __half* const dst[6] = {arh, arl, aih, ail, ssh, ssl};
#pragma unroll
    for (int pl = 0; pl < 6; ++pl)
      __stcs(reinterpret_cast<uint4*>(dst[pl]) + v, make_uint4(w[pl][0], w[pl][1], w[pl][2], w[pl][3]));
  }
  for (long long i = 8 * n8 + blockIdx.x * 256ll + threadIdx.x; i < count; i += stride) {
    float re, im;
    if (presplit) {
      const __half2 h = reinterpret_cast<const __half2*>(a)[i];
      const __half2 l = reinterpret_cast<const __half2*>(a)[count + i];
      re = __low2float(h) + __low2float(l);
      im = __high2float(h) + __high2float(l);
    } else {
      const float2 v = reinterpret_cast<const float2*>(a)[i];
      re = v.x;
      im = v.y;
    }
    re *= s;
    im *= s;
    split16(re, arh[i], arl[i]);
    split16(im, aih[i], ail[i]);
    split16(re + im, ssh[i], ssl[i]);
  }
}

// B (complex [k][n], or [n][k] when tb) -> B^T real planes [n][k]: Br, Bi,
// T = Br + Bi, each fp16 hi | lo scaled by 2^(f16_exp(meta) - 1).  Tiles of
// 128 k x 32 n through shared memory (stored [n][k]); every lane then writes
// 4 consecutive k (8 bytes) per plane, a warp one 256-byte run of one n row.
__global__ void __launch_bounds__(256) tc3m_prep_b_kernel(const float2* __restrict__ b, long long n, long long k,
                                                          int tb, const TMeta* __restrict__ meta,
                                                          __half* __restrict__ planes) {
  constexpr int TK = 128, TN = 32, PITCH = TK + 1;
  __shared__ float2 tile[TN][PITCH];
  const long long j0 = static_cast<long long>(blockIdx.x) * TN, p0 = static_cast<long long>(blockIdx.y) * TK;
  const int lane = threadIdx.x & 31, wy = threadIdx.x >> 5;
  if (!tb) {
    for (int r = wy; r < TK; r += 8) {  // row p of B [k][n]: lanes over n
      const long long p = p0 + r, j = j0 + lane;
      tile[lane][r] = (p < k && j < n) ? b[p * n + j] : make_float2(0.f, 0.f);
    }
  } else {
    for (int r = wy; r < TN; r += 8) {  // row j of B^T [n][k]: lanes over k
      const long long j = j0 + r;
#pragma unroll
      for (int c = 0; c < TK / 32; ++c) {
        const long long p = p0 + 32 * c + lane;
        tile[r][32 * c + lane] = (p < k && j < n) ? b[j * k + p] : make_float2(0.f, 0.f);
      }
    }
  }
  __syncthreads();
  const float s = scalbnf(1.f, f16_exp_3m(meta));
  const long long nk = n * k;
  const bool vec = k % 4 == 0 && (reinterpret_cast<uintptr_t>(planes) & 7) == 0;
  for (int r = wy; r < TN; r += 8) {
    const long long j = j0 + r, p = p0 + 4 * lane;
    if (j >= n || p >= k) continue;
    if (vec) {  // p .. p + 3 all < k (k % 4 == 0, p % 4 == 0)
      uint32_t w[6][2];
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        __half h[6][2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const float2 v = tile[r][4 * lane + 2 * t + u];
          split16(v.x * s, h[0][u], h[1][u]);
          split16(v.y * s, h[2][u], h[3][u]);
          split16((v.x + v.y) * s, h[4][u], h[5][u]);
        }
#pragma unroll
        for (int pl = 0; pl < 6; ++pl) w[pl][t] = pack_h2(h[pl][0], h[pl][1]);
      }
      const long long o = j * k + p;
#pragma unroll
      for (int pl = 0; pl < 6; ++pl)
        *reinterpret_cast<uint2*>(planes + pl * nk + o) = make_uint2(w[pl][0], w[pl][1]);
    } else {
      for (int u = 0; u < 4 && p + u < k; ++u) {
        const float2 v = tile[r][4 * lane + u];
        const long long o = j * k + p + u;
        split16(v.x * s, planes[o], planes[nk + o]);
        split16(v.y * s, planes[2 * nk + o], planes[3 * nk + o]);
        split16((v.x + v.y) * s, planes[4 * nk + o], planes[5 * nk + o]);
      }
    }
  }
}

// C = (P1 - P2) + i (P3 - P1 - P2), times the operands' pending power-of-two
// renormalisation; max |c|^2 -> meta_c, log_scale as the pair epilogue sets it.
__global__ void __launch_bounds__(256) tc3m_combine_kernel(const float4* __restrict__ p1, const float4* __restrict__ p2,
                                                           const float4* __restrict__ p3, float4* __restrict__ c,
                                                           long long n4, const TMeta* meta_a, const TMeta* meta_b,
                                                           int norm_a, int norm_b, TMeta* meta_c) {
  const int shift = tc_pending_shift(meta_a, norm_a) + tc_pending_shift(meta_b, norm_b);
  const float f = scalbnf(1.f, -shift);
  float local = 0.f;
  for (long long i = blockIdx.x * 256ll + threadIdx.x; i < n4; i += static_cast<long long>(gridDim.x) * 256) {
    const float4 a = p1[i], b = p2[i], d = p3[i];
    const float4 lo = make_float4((a.x - b.x) * f, (d.x - a.x - b.x) * f, (a.y - b.y) * f, (d.y - a.y - b.y) * f);
    const float4 hi = make_float4((a.z - b.z) * f, (d.z - a.z - b.z) * f, (a.w - b.w) * f, (d.w - a.w - b.w) * f);
    c[2 * i] = lo;
    c[2 * i + 1] = hi;
    local = fmaxf(local, fmaxf(fmaxf(lo.x * lo.x + lo.y * lo.y, lo.z * lo.z + lo.w * lo.w),
                               fmaxf(hi.x * hi.x + hi.y * hi.y, hi.z * hi.z + hi.w * hi.w)));
  }
  if (meta_c) {
    for (int o = 16; o > 0; o >>= 1) local = fmaxf(local, __shfl_xor_sync(0xffffffffu, local, o));
    if ((threadIdx.x & 31) == 0 && local > 0.f) atomicMax(&meta_c->maxsq_bits, __float_as_uint(local));
    if (blockIdx.x == 0 && threadIdx.x == 0)
      meta_c->log_scale = (meta_a ? meta_a->log_scale : 0.0) + (meta_b ? meta_b->log_scale : 0.0) + shift;
  }
}

// B scratch meta: max |z| doubled (max |z|^2 x 4), so f16_exp(meta_b3) is
// the exponent the 3M B planes were scaled with.
__global__ void tc3m_scale_meta_kernel(TMeta* m) {
  const unsigned bits = m->maxsq_bits;
  if (bits != 0 && bits < 0x7f800000u) m->maxsq_bits = __float_as_uint(__uint_as_float(bits) * 4.f);
}

bool use_3m(std::int64_t m, std::int64_t n, std::int64_t k) {
  const char* env = std::getenv("QSG_TC_3M");  // 0: the 2x2 embedding everywhere
  const bool on = !(env && env[0] == '0');
  return on && n >= kMin3M && k >= kMin3M && n % 2 == 0 && k % 2 == 0 && use_f16(m, n / 2, k / 2) &&
         (k % BK16) == 0;
}

// Workspace: [metas | sync | A planes 12 m k | B planes 12 n k | P1 P2 P3 12 m n] bytes.
std::int64_t ws3m_bytes(std::int64_t m, std::int64_t n, std::int64_t k) {
  return kF16Scratch + sync_bytes(m, n / 2, k / 2) + 12 * m * k + 12 * n * k + 12 * m * n;
}

cudaError_t cgemm_tc_3m(const GemmArgs& g, const TMeta* ma, const TMeta* mb, cudaStream_t stream, int* launches) {
  char* ws = static_cast<char*>(g.workspace);
  TMeta* metas = reinterpret_cast<TMeta*>(ws);  // [2] scan scratch (caller), [3] A, [4] B, [5] C scratch
  TMeta* meta_a3 = metas + 3;
  TMeta* meta_b3 = metas + 4;
  TMeta* meta_c3 = metas + 5;
  const std::int64_t sb = sync_bytes(g.m, g.n / 2, g.k / 2);
  unsigned int* sync = sb > 0 ? reinterpret_cast<unsigned int*>(ws + kF16Scratch) : nullptr;
  __half* ap = reinterpret_cast<__half*>(ws + kF16Scratch + sb);
  __half* bp = ap + 6 * g.m * g.k;
  float* pp = reinterpret_cast<float*>(bp + 6 * g.n * g.k);
  const long long mk = g.m * g.k, nk = g.n * g.k, mn = g.m * g.n;
  // B's scratch meta: max |z|^2 x 4 so that f16_exp gives the planes' exponent (f16_exp - 1).
  cudaError_t e = cudaMemcpyAsync(meta_b3, mb, sizeof(TMeta), cudaMemcpyDeviceToDevice, stream);
  if (e != cudaSuccess) return e;
  {
    const long long items = mk % 8 == 0 ? mk / 8 : mk;
    const int blocks = static_cast<int>(std::min<long long>((items + 255) / 256, 148 * 16));
    tc3m_prep_a_kernel<<<blocks, 256, 0, stream>>>(g.a, g.a_presplit ? 1 : 0, mk, ma, ap, meta_a3);
    dim3 grid(static_cast<unsigned>((g.n + 31) / 32), static_cast<unsigned>((g.k + 127) / 128));
    tc3m_prep_b_kernel<<<grid, 256, 0, stream>>>(static_cast<const float2*>(g.b), g.n, g.k, g.trans_b ? 1 : 0, mb, bp);
    tc3m_scale_meta_kernel<<<1, 1, 0, stream>>>(meta_b3);
    if (launches) *launches += 3;
  }
  GemmArgs r{};
  r.m = g.m;
  r.n = g.n / 2;  // real [m][n] output = "complex" [m][n/2]
  r.k = g.k / 2;  // real K = k
  r.a_presplit = true;
  r.meta_a = meta_a3;
  r.meta_b = meta_b3;
  r.meta_c = meta_c3;
  r.norm_a = r.norm_b = false;
  for (int t = 0; t < 3; ++t) {
    r.a = ap + 2 * t * mk;
    r.c = pp + t * mn;
    const __half* bhi = bp + 2 * t * nk;
    const __half* blo = bhi + nk;
    if (sync) {
      e = cudaMemsetAsync(sync, 0, static_cast<size_t>(sb), stream);
      if (e != cudaSuccess) return e;
    }
    const __half* ahi = static_cast<const __half*>(r.a);
    const __half* alo = ahi + mk;
    switch (f16_bn(r.n, r.k)) {
      case 256: e = launch_f16_pair<256>(r, meta_a3, meta_b3, bhi, blo, sync, ahi, alo, stream); break;
      case 128: e = launch_f16_pair<128>(r, meta_a3, meta_b3, bhi, blo, sync, ahi, alo, stream); break;
      case 64: e = launch_f16_pair<64>(r, meta_a3, meta_b3, bhi, blo, sync, ahi, alo, stream); break;
      default: e = launch_f16_pair<32>(r, meta_a3, meta_b3, bhi, blo, sync, ahi, alo, stream); break;
    }
    if (e != cudaSuccess) return e;
    if (launches) ++*launches;
  }
  const long long n4 = mn / 4;
  const int blocks = static_cast<int>(std::min<long long>((n4 + 255) / 256, 148 * 16));
  tc3m_combine_kernel<<<blocks, 256, 0, stream>>>(reinterpret_cast<const float4*>(pp),
                                                  reinterpret_cast<const float4*>(pp + mn),
                                                  reinterpret_cast<const float4*>(pp + 2 * mn),
                                                  static_cast<float4*>(g.c), n4, g.meta_a, g.meta_b,
                                                  g.norm_a && g.meta_a ? 1 : 0, g.norm_b && g.meta_b ? 1 : 0, g.meta_c);
  if (launches) ++*launches;
  return cudaGetLastError();
}
}  // namespace

bool tc_enabled() {
  const char* env = std::getenv("QSG_TENSOR_CORES");
  return !(env && env[0] == '0');
}

bool cgemm_tc_supported(std::int64_t m, std::int64_t n, std::int64_t k, bool trans_a, bool /*trans_b*/) {
  if (trans_a || m <= 0 || n <= 0 || k <= 0 || (2 * k) % BK != 0) return false;
  return (m % BM == 0 && (2 * n) % 128 == 0) || use_pair(m, n);
}

bool cgemm_tc_eligible(std::int64_t m, std::int64_t n, std::int64_t k, bool trans_a, bool trans_b) {
  if (!tc_enabled() || !cgemm_tc_supported(m, n, k, trans_a, trans_b)) return false;
  // Worth it for real work (>= ~1 GFLOP).  The persistent CTA-pair kernel
  // streams even single-k-block tiles well; the 1-CTA kernel needs K >= 64.
  const char* env = std::getenv("QSG_TC_MIN_FLOPS");  // tests force small shapes onto the TC path
  const double min_flops = env ? std::atof(env) : 1e9;
  if (8.0 * static_cast<double>(m) * n * k < min_flops) return false;
  return use_pair(m, n) ? k >= 16 : k >= 64;
}

bool cgemm_tc_store_perm_supported(std::int64_t m, std::int64_t n, std::int64_t k, bool trans_a, bool trans_b) {
  return cgemm_tc_supported(m, n, k, trans_a, trans_b) && use_pair(m, n) && !use_3m(m, n, k);
}

bool cgemm_tc_split_ok(std::int64_t m, std::int64_t n, std::int64_t k, bool trans_a, bool trans_b) {
  // Any fp16 pair shape (a half k-block tail reads zero-filled plane columns it never multiplies).
  return cgemm_tc_supported(m, n, k, trans_a, trans_b) && use_pair(m, n) && !use_3m(m, n, k);
}

std::int64_t cgemm_tc_workspace_bytes(std::int64_t m, std::int64_t n, std::int64_t k, bool, bool, bool a_presplit) {
  if (use_3m(m, n, k)) return ws3m_bytes(m, n, k);
  if (a_presplit || use_f16(m, n, k))  // operand maxima + K-sync counters + fp16 B_r^T hi + lo (+ pre-split A)
    return kF16Scratch + sync_bytes(m, n, k) + 2 * (2 * n) * b16_pitch(k) * 2 +
           (!a_presplit && split_a(m, n, k) ? 8 * m * k : 0);
  return 2 * (2 * n) * (2 * k) * 4;                                     // fp32 B_r^T hi + lo
}

double cgemm_tc_rate(std::int64_t m, std::int64_t n, std::int64_t k) {
  if (use_3m(m, n, k)) return 5.5e14;   // 3 real products instead of the 4-MAC embedding
  if (split_a(m, n, k)) return 4.5e14;  // measured 450-630 TF/s (config 2 s026 / config 5 cubes)
  if (use_f16(m, n, k)) return 3.5e14;  // in-kernel A conversion: ~68% tensor-pipe occupancy
  return 1.5e14;                        // 3xTF32
}

double cgemm_tc_prep_bytes(std::int64_t m, std::int64_t n, std::int64_t k) {
  const double nb = static_cast<double>(n) * static_cast<double>(k);  // complex elements of B
  if (use_3m(m, n, k))  // A planes, B planes, three fp32 products written + read, C written
    return 20.0 * static_cast<double>(m) * static_cast<double>(k) + 32.0 * nb +
           32.0 * static_cast<double>(m) * static_cast<double>(n);
  if (!use_f16(m, n, k)) return 40.0 * nb;                            // read 8, write 32 (fp32 hi + lo)
  return 24.0 * nb + (split_a(m, n, k) ? 16.0 * static_cast<double>(m) * static_cast<double>(k) : 0.0);
}

cudaError_t cgemm_tc(const GemmArgs& g, cudaStream_t stream, int* launches) {
  if (!cgemm_tc_supported(g.m, g.n, g.k, g.trans_a, g.trans_b))
    throw std::invalid_argument("cgemm_tc: shape not supported by the tensor-core path");
  if (g.workspace == nullptr || g.workspace_bytes < cgemm_tc_workspace_bytes(g.m, g.n, g.k, g.trans_a, g.trans_b, g.a_presplit))
    throw std::invalid_argument("cgemm_tc: workspace too small");
  if (g.store_perm && !use_pair(g.m, g.n))
    throw std::invalid_argument("cgemm_tc: fused output permutation needs the CTA-pair path");
  if (g.store_perm && !use_pair(g.m, g.n))
    throw std::invalid_argument("cgemm_tc: fused output permutation needs the CTA-pair path");
  if ((g.a_presplit || g.c_split) && !cgemm_tc_split_ok(g.m, g.n, g.k, g.trans_a, g.trans_b))
    throw std::invalid_argument("cgemm_tc: split operand storage needs the fp16 CTA-pair path");
  if (g.a_presplit && g.meta_a == nullptr) throw std::invalid_argument("cgemm_tc: pre-split A needs its meta");
  if (g.a_presplit || g.c_split || use_f16(g.m, g.n, g.k)) {
    // Operand maxima for the fp16 scaling: the producers' device metas when
    // present, else a max |z|^2 scan into workspace scratch.
    TMeta* scratch = static_cast<TMeta*>(g.workspace);
    const TMeta* ma = g.meta_a;
    const TMeta* mb = g.meta_b;
    if (!ma || !mb) {
      cudaError_t e = cudaMemsetAsync(scratch, 0, 2 * sizeof(TMeta), stream);
      if (e != cudaSuccess) return e;
    }
    if (!ma) {
      cudaError_t e = max_abs_sq(g.a, g.m * g.k, scratch, stream, launches);
      if (e != cudaSuccess) return e;
      ma = scratch;
    }
    if (!mb) {
      cudaError_t e = max_abs_sq(g.b, g.n * g.k, scratch + 1, stream, launches);
      if (e != cudaSuccess) return e;
      mb = scratch + 1;
    }
    if (use_3m(g.m, g.n, g.k)) {
      if (g.store_perm || g.c_split) throw std::invalid_argument("cgemm_tc: the 3M path writes natural-order complex64");
      return cgemm_tc_3m(g, ma, mb, stream, launches);
    }
    const std::int64_t sb = sync_bytes(g.m, g.n, g.k);
    unsigned int* sync = sb > 0 ? reinterpret_cast<unsigned int*>(static_cast<char*>(g.workspace) + kF16Scratch) : nullptr;
    if (sync) {
      cudaError_t e = cudaMemsetAsync(sync, 0, static_cast<size_t>(sb), stream);
      if (e != cudaSuccess) return e;
    }
    __half* bhi = reinterpret_cast<__half*>(static_cast<char*>(g.workspace) + kF16Scratch + sb);
    __half* blo = bhi + (2 * g.n) * b16_pitch(g.k);
    dim3 grid(static_cast<unsigned>((g.n + 31) / 32), static_cast<unsigned>((g.k + 31) / 32));
    tc_prep_b_f16_kernel<<<grid, 256, 0, stream>>>(static_cast<const float2*>(g.b), bhi, blo, g.n, g.k,
                                                    g.trans_b ? 1 : 0, mb, b16_pitch(g.k));
    if (launches) ++*launches;
    __half* ahi = nullptr;
    __half* alo = nullptr;
    if (g.a_presplit) {
      ahi = static_cast<__half*>(const_cast<void*>(g.a));
      alo = ahi + 2 * g.m * g.k;
    } else if (split_a(g.m, g.n, g.k)) {
      ahi = blo + (2 * g.n) * b16_pitch(g.k);
      alo = ahi + g.m * 2 * g.k;
      const long long n4 = g.m * 2 * g.k / 4;
      const int blocks = static_cast<int>(std::min<long long>((n4 + 255) / 256, 148 * 16));
      tc_prep_a_f16_kernel<<<blocks, 256, 0, stream>>>(static_cast<const float4*>(g.a), reinterpret_cast<uint2*>(ahi),
                                                       reinterpret_cast<uint2*>(alo), n4, ma);
      if (launches) ++*launches;
    }
    cudaError_t e = cudaSuccess;
    switch (f16_bn(g.n, g.k)) {
      case 256: e = launch_f16_pair<256>(g, ma, mb, bhi, blo, sync, ahi, alo, stream); break;
      case 128: e = launch_f16_pair<128>(g, ma, mb, bhi, blo, sync, ahi, alo, stream); break;
      case 64: e = launch_f16_pair<64>(g, ma, mb, bhi, blo, sync, ahi, alo, stream); break;
      default: e = launch_f16_pair<32>(g, ma, mb, bhi, blo, sync, ahi, alo, stream); break;
    }
    if (launches) ++*launches;
    tc_prof_report(g.m, g.n, g.k, stream);
    return e;
  }
  float* bhi = static_cast<float*>(g.workspace);
  float* blo = bhi + (2 * g.n) * (2 * g.k);
  {
    dim3 grid(static_cast<unsigned>((g.n + 31) / 32), static_cast<unsigned>((g.k + 31) / 32));
    tc_prep_b_kernel<<<grid, 256, 0, stream>>>(static_cast<const float2*>(g.b), bhi, blo, g.n, g.k, g.trans_b ? 1 : 0);
    if (launches) ++*launches;
  }
  if (g.store_perm && !use_pair(g.m, g.n))
    throw std::invalid_argument("cgemm_tc: fused output permutation needs the CTA-pair path");
  if (use_pair(g.m, g.n)) {
    cudaError_t e = cudaSuccess;
    switch (pair_bn(g.n)) {
      case 256: e = launch_pair<256>(g, bhi, blo, stream); break;
      case 128: e = launch_pair<128>(g, bhi, blo, stream); break;
      case 64: e = launch_pair<64>(g, bhi, blo, stream); break;
      default: e = launch_pair<32>(g, bhi, blo, stream); break;
    }
    if (launches) ++*launches;
    return e;
  }
  const int bn = tc_bn(g.n);
  const CUtensorMap ma = make_map(g.a, 2 * g.k, g.m, BM);
  const CUtensorMap mbh = make_map(bhi, 2 * g.k, 2 * g.n, bn);
  const CUtensorMap mbl = make_map(blo, 2 * g.k, 2 * g.n, bn);
  TcParams p{};
  p.c = static_cast<float*>(g.c);
  p.m = g.m;
  p.n2 = 2 * g.n;
  p.kblocks = static_cast<int>((2 * g.k) / BK);
  p.meta_a = g.meta_a;
  p.meta_b = g.meta_b;
  p.meta_c = g.meta_c;
  p.norm_a = g.norm_a;
  p.norm_b = g.norm_b;
  p.chunk = chunk_blocks();
  const long long mt = g.m / BM, nt = (2 * g.n) / bn;
  if (mt * nt > 2147483647LL || g.m > 2147483647LL) throw std::length_error("cgemm_tc: too many tiles");
  p.n_tiles = static_cast<int>(nt);
  dim3 grid(static_cast<unsigned>(mt * nt));
  if (bn == 256) {
    setup_attr<256>();
    cgemm_tc_kernel<256><<<grid, kThreads, TcCfg<256>::SMEM, stream>>>(ma, mbh, mbl, p);
  } else {
    setup_attr<128>();
    cgemm_tc_kernel<128><<<grid, kThreads, TcCfg<128>::SMEM, stream>>>(ma, mbh, mbl, p);
  }
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace qsg::dev
