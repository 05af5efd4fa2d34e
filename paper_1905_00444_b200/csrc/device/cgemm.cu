// K2 (general path): complex64 GEMM on the FP32 pipes, the contraction
// core of contract_ttgt (include/qsim/contraction.hpp:208-214: row-major
// C = A * B, FP32 accumulate).  Each complex multiply-add is 4 FFMA, i.e.
// exactly the 8 flops of the Eq.(1) model.
//
// This is the shape-general kernel: any m, n, k (including the tiny and
// skinny steps of every plan), operands in N or T layout so the executor
// can skip permutes, and split-K for small outputs with long reductions.
// The large, aligned steps go to the tcgen05 kernel (cgemm_tc.cu) when it
// is enabled.
//
// Fused epilogue (normalize_inplace, tensor.hpp:209-224, called after every
// step at src/engine.cpp:233): the operands' pending power-of-two shifts
// are applied to the accumulator (exact), max|c|^2 is reduced per block and
// atomically merged into the output's TMeta, and block (0,0,0) writes the
// output log_scale.  No extra pass over the output is needed.
#include <algorithm>
#include <cstdint>
#include <stdexcept>

#include "kernels.hpp"

namespace qsg::dev {

__device__ __forceinline__ int pending_shift(const TMeta* m, bool norm) {
  if (!norm || m == nullptr) return 0;
  const unsigned bits = m->maxsq_bits;
  if (bits == 0) return 0;
  const double mx = sqrt(static_cast<double>(__uint_as_float(bits)));
  int e = 0;
  const double fr = frexp(mx, &e);
  return fr == 0.5 ? e - 1 : e;
}

namespace {

constexpr int BM = 64, BN = 128, BK = 8, NT = 256;

struct KParams {
  const float2* a;
  const float2* b;
  float2* c;
  float2* partial;  // split-K partials [splits][m][n] or null
  long long m, n, k, kchunk;
  long long m_tiles;  // tiles are linearised over grid.x, m fastest (no 65535 grid.y limit)
  const TMeta* meta_a;
  const TMeta* meta_b;
  TMeta* meta_c;
  int norm_a, norm_b;
};

__device__ __forceinline__ void cfma(float2& acc, const float2 a, const float2 b) {
  acc.x = fmaf(a.x, b.x, acc.x);
  acc.x = fmaf(-a.y, b.y, acc.x);
  acc.y = fmaf(a.x, b.y, acc.y);
  acc.y = fmaf(a.y, b.x, acc.y);
}

__device__ __forceinline__ void block_max_to_meta(float local, TMeta* meta) {
  __shared__ float red[NT / 32];
  for (int o = 16; o > 0; o >>= 1) local = fmaxf(local, __shfl_xor_sync(0xffffffffu, local, o));
  const int warp = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) red[warp] = local;
  __syncthreads();
  if (threadIdx.x == 0) {
    float mx = red[0];
    for (int w = 1; w < NT / 32; ++w) mx = fmaxf(mx, red[w]);
    if (mx > 0.f) atomicMax(&meta->maxsq_bits, __float_as_uint(mx));
  }
}

// Output column of accumulator j (0..7) of thread column tx (0..15):
// pairs 2 tx + 32 (j / 2) + (j % 2), so each B / C access is a 16-byte pair.
__device__ __forceinline__ int simt_col(int tx, int j) { return 2 * tx + 32 * (j >> 1) + (j & 1); }

template <bool TA, bool TB>
__global__ void __launch_bounds__(NT, 2) cgemm_simt_kernel(const KParams p) {
  __shared__ __align__(16) float2 As[2][BK][BM + 2];
  __shared__ __align__(16) float2 Bs[2][BK][BN + 2];
  const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
  const long long m0 = (static_cast<long long>(blockIdx.x) % p.m_tiles) * BM;
  const long long n0 = (static_cast<long long>(blockIdx.x) / p.m_tiles) * BN;
  const long long kbeg = static_cast<long long>(blockIdx.z) * p.kchunk;
  const long long kend = min(p.k, kbeg + p.kchunk);
  const long long M = p.m, N = p.n, K = p.k;

  float2 ra[2], rb[4];
  auto load = [&](long long k0) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int idx = tid + i * NT;
      long long row, col;
      if (!TA) { row = idx / BK; col = idx % BK; } else { col = idx / BM; row = idx % BM; }
      const long long gm = m0 + row, gk = k0 + col;
      ra[i] = (gm < M && gk < kend) ? (TA ? p.a[gk * M + gm] : p.a[gm * K + gk]) : make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int idx = tid + i * NT;
      long long kr, nc;
      if (!TB) { kr = idx / BN; nc = idx % BN; } else { nc = idx / BK; kr = idx % BK; }
      const long long gk = k0 + kr, gn = n0 + nc;
      rb[i] = (gn < N && gk < kend) ? (TB ? p.b[gn * K + gk] : p.b[gk * N + gn]) : make_float2(0.f, 0.f);
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int idx = tid + i * NT;
      if (!TA) As[buf][idx % BK][idx / BK] = ra[i]; else As[buf][idx / BM][idx % BM] = ra[i];
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int idx = tid + i * NT;
      if (!TB) Bs[buf][idx / BN][idx % BN] = rb[i]; else Bs[buf][idx % BK][idx / BK] = rb[i];
    }
  };

  float2 acc[4][8];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = make_float2(0.f, 0.f);

  int buf = 0;
  if (kbeg < kend) {
    load(kbeg);
    store(0);
  }
  __syncthreads();
  for (long long k0 = kbeg; k0 < kend; k0 += BK) {
    const bool more = k0 + BK < kend;
    if (more) load(k0 + BK);
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      const float4 a01 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 4]);
      const float4 a23 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 4 + 2]);
      const float2 av[4] = {make_float2(a01.x, a01.y), make_float2(a01.z, a01.w), make_float2(a23.x, a23.y),
                            make_float2(a23.z, a23.w)};
      // Thread tx owns column pairs 2 tx + 32 jj + {0, 1}: one 16-byte shared
      // load per pair (4 LDS.128 instead of 8 LDS.64 per k).
      float2 bv[8];
#pragma unroll
      for (int jj = 0; jj < 4; ++jj) {
        const float4 q = *reinterpret_cast<const float4*>(&Bs[buf][kk][2 * tx + 32 * jj]);
        bv[2 * jj] = make_float2(q.x, q.y);
        bv[2 * jj + 1] = make_float2(q.z, q.w);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) cfma(acc[i][j], av[i], bv[j]);
    }
    if (more) store(buf ^ 1);
    __syncthreads();
    buf ^= 1;
  }

  if (p.partial) {
    float2* out = p.partial + static_cast<long long>(blockIdx.z) * M * N;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const long long gm = m0 + ty * 4 + i;
      if (gm >= M) continue;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const long long gn = n0 + simt_col(tx, j);
        if (gn < N) out[gm * N + gn] = acc[i][j];
      }
    }
    return;
  }

  const int sa = pending_shift(p.meta_a, p.norm_a), sb = pending_shift(p.meta_b, p.norm_b);
  const int shift = sa + sb;
  float local = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const long long gm = m0 + ty * 4 + i;
#pragma unroll
    for (int j = 0; j < 8; j += 2) {
      const long long gn = n0 + simt_col(tx, j);
      if (gm >= M) continue;
      const float2 v0 = make_float2(scalbnf(acc[i][j].x, -shift), scalbnf(acc[i][j].y, -shift));
      const float2 v1 = make_float2(scalbnf(acc[i][j + 1].x, -shift), scalbnf(acc[i][j + 1].y, -shift));
      if (gn + 1 < N && (N & 1) == 0) {  // the pair is adjacent and 16-byte aligned
        *reinterpret_cast<float4*>(p.c + gm * N + gn) = make_float4(v0.x, v0.y, v1.x, v1.y);
        local = fmaxf(local, fmaxf(v0.x * v0.x + v0.y * v0.y, v1.x * v1.x + v1.y * v1.y));
      } else {
        if (gn < N) {
          p.c[gm * N + gn] = v0;
          local = fmaxf(local, v0.x * v0.x + v0.y * v0.y);
        }
        if (gn + 1 < N) {
          p.c[gm * N + gn + 1] = v1;
          local = fmaxf(local, v1.x * v1.x + v1.y * v1.y);
        }
      }
    }
  }
  if (p.meta_c) {
    block_max_to_meta(local, p.meta_c);
    if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && threadIdx.x == 0)
      p.meta_c->log_scale = (p.meta_a ? p.meta_a->log_scale : 0.0) + (p.meta_b ? p.meta_b->log_scale : 0.0) + shift;
  }
}

__global__ void __launch_bounds__(NT) splitk_reduce_kernel(const KParams p, int splits) {
  const long long mn = p.m * p.n;
  const int sa = pending_shift(p.meta_a, p.norm_a), sb = pending_shift(p.meta_b, p.norm_b);
  const int shift = sa + sb;
  float local = 0.f;
  for (long long i = blockIdx.x * static_cast<long long>(NT) + threadIdx.x; i < mn;
       i += static_cast<long long>(gridDim.x) * NT) {
    float2 s = p.partial[i];
    for (int z = 1; z < splits; ++z) {
      const float2 t = p.partial[z * mn + i];
      s.x += t.x;
      s.y += t.y;
    }
    const float2 v = make_float2(scalbnf(s.x, -shift), scalbnf(s.y, -shift));
    p.c[i] = v;
    local = fmaxf(local, v.x * v.x + v.y * v.y);
  }
  if (p.meta_c) {
    block_max_to_meta(local, p.meta_c);
    if (blockIdx.x == 0 && threadIdx.x == 0)
      p.meta_c->log_scale = (p.meta_a ? p.meta_a->log_scale : 0.0) + (p.meta_b ? p.meta_b->log_scale : 0.0) + shift;
  }
}

// Narrow-N variant (n <= 16): the 64 x 128 tile above wastes 7/8 of its
// FFMAs and stores on n = 16 (the bond-closing steps of the column sweeps,
// e.g. m = 2^20 x n = 16 x k = 16 with A in T layout).  Here a thread owns
// one output row and all n columns: A is staged per 32-k chunk through
// shared memory with coalesced loads (T layout: along m; N layout: along k),
// B's chunk (<= 32 x 16) is broadcast from shared memory, and each thread
// stores its contiguous row.  HBM-bound: 8 (m k + m n) bytes per launch.
constexpr int NR = 128, NKC = 32;

template <bool TA, bool TB, int NNW>
__global__ void __launch_bounds__(NR) cgemm_narrow_kernel(const KParams p) {
  __shared__ __align__(16) float2 As[NKC][NR + 1];
  __shared__ float2 Bs[NKC][NNW];
  const int tid = threadIdx.x;
  const long long m0 = static_cast<long long>(blockIdx.x) * NR;
  const long long M = p.m, N = p.n, K = p.k;
  float2 acc[NNW];
#pragma unroll
  for (int j = 0; j < NNW; ++j) acc[j] = make_float2(0.f, 0.f);
  for (long long k0 = 0; k0 < K; k0 += NKC) {
    const int kc = static_cast<int>(min(static_cast<long long>(NKC), K - k0));
#pragma unroll 4
    for (int i = 0; i < NKC; ++i) {
      const int idx = tid + i * NR;
      int r, kk;
      if (TA) { kk = idx / NR; r = idx % NR; } else { r = idx / NKC; kk = idx % NKC; }
      const long long gm = m0 + r;
      As[kk][r] = (gm < M && kk < kc) ? (TA ? p.a[(k0 + kk) * M + gm] : p.a[gm * K + k0 + kk]) : make_float2(0.f, 0.f);
    }
    for (int idx = tid; idx < NKC * NNW; idx += NR) {
      const int kk = idx / NNW, j = idx % NNW;
      Bs[kk][j] = (kk < kc && j < N) ? (TB ? p.b[j * K + k0 + kk] : p.b[(k0 + kk) * N + j]) : make_float2(0.f, 0.f);
    }
    __syncthreads();
    for (int kk = 0; kk < kc; ++kk) {
      const float2 a = As[kk][tid];
#pragma unroll
      for (int j = 0; j < NNW; ++j) cfma(acc[j], a, Bs[kk][j]);
    }
    __syncthreads();
  }
  const int sa = pending_shift(p.meta_a, p.norm_a), sb = pending_shift(p.meta_b, p.norm_b);
  const int shift = sa + sb;
  float local = 0.f;
  const long long gm = m0 + tid;
  if (N == NNW && m0 + NR <= M) {
    // Full block: its 128 rows x NNW columns are one contiguous run of C.
    // Stage them through the (now idle) A buffer -- 16-byte chunk c of row
    // r at slot c ^ (r mod NNW/2), conflict-free both ways -- and store the
    // run with consecutive threads on consecutive 16-byte pieces.
    constexpr int CH = NNW / 2;  // float4 chunks per row
    float4* stage = reinterpret_cast<float4*>(&As[0][0]);
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const float4 v = make_float4(scalbnf(acc[2 * c].x, -shift), scalbnf(acc[2 * c].y, -shift),
                                   scalbnf(acc[2 * c + 1].x, -shift), scalbnf(acc[2 * c + 1].y, -shift));
      local = fmaxf(local, fmaxf(v.x * v.x + v.y * v.y, v.z * v.z + v.w * v.w));
      stage[tid * CH + (c ^ (tid & (CH - 1)))] = v;
    }
    __syncthreads();
    float4* out = reinterpret_cast<float4*>(p.c + m0 * N);
#pragma unroll 4
    for (int l = tid; l < NR * CH; l += NR) {
      const int r = l / CH, c = l % CH;
      out[l] = stage[r * CH + (c ^ (r & (CH - 1)))];
    }
  } else if (gm < M) {
#pragma unroll
    for (int j = 0; j < NNW; ++j) {
      const float2 v = make_float2(scalbnf(acc[j].x, -shift), scalbnf(acc[j].y, -shift));
      acc[j] = v;
      local = fmaxf(local, v.x * v.x + v.y * v.y);
    }
    if (N == NNW) {
      float4* row = reinterpret_cast<float4*>(p.c + gm * N);
#pragma unroll
      for (int j = 0; j < NNW; j += 2) row[j / 2] = make_float4(acc[j].x, acc[j].y, acc[j + 1].x, acc[j + 1].y);
    } else {
#pragma unroll
      for (int j = 0; j < NNW; ++j)
        if (j < N) p.c[gm * N + j] = acc[j];
    }
  }
  if (p.meta_c) {
    for (int o = 16; o > 0; o >>= 1) local = fmaxf(local, __shfl_xor_sync(0xffffffffu, local, o));
    if ((tid & 31) == 0 && local > 0.f) atomicMax(&p.meta_c->maxsq_bits, __float_as_uint(local));
    if (blockIdx.x == 0 && tid == 0)
      p.meta_c->log_scale = (p.meta_a ? p.meta_a->log_scale : 0.0) + (p.meta_b ? p.meta_b->log_scale : 0.0) + shift;
  }
}

bool use_narrow(std::int64_t m, std::int64_t n) { return n <= 32 && m >= 1024; }

template <int NNW>
void launch_narrow(const GemmArgs& g, const KParams& p, cudaStream_t stream) {
  const dim3 grid(static_cast<unsigned>((g.m + NR - 1) / NR));
  if (g.trans_a) {
    if (g.trans_b) cgemm_narrow_kernel<true, true, NNW><<<grid, NR, 0, stream>>>(p);
    else cgemm_narrow_kernel<true, false, NNW><<<grid, NR, 0, stream>>>(p);
  } else {
    if (g.trans_b) cgemm_narrow_kernel<false, true, NNW><<<grid, NR, 0, stream>>>(p);
    else cgemm_narrow_kernel<false, false, NNW><<<grid, NR, 0, stream>>>(p);
  }
}

int sm_count() {
  static int n = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

int choose_splits(std::int64_t m, std::int64_t n, std::int64_t k) {
  const std::int64_t tiles = ((m + BM - 1) / BM) * ((n + BN - 1) / BN);
  const std::int64_t want = 2 * static_cast<std::int64_t>(sm_count());
  std::int64_t s = 1;
  if (tiles < want && k >= 32) {
    // Few tiles: split K over idle SMs.  Each K step of this kernel is a
    // dependent global-load round trip (~2.5 us at one or two CTAs), so the
    // small side contractions of the Bristlecone plans (m = 16, n = 256,
    // k = 256: 2 tiles, 80 us) are latency-bound; chunks of >= 16 K there
    // (>= 256 K on long K, as before).
    const std::int64_t min_chunk = k >= 512 ? 256 : 2 * BK;
    s = std::min<std::int64_t>((want + tiles - 1) / tiles, k / min_chunk);
    // Cap the occupancy partial buffer at 1 GiB.
    while (s > 1 && s * m * n * 8 > (std::int64_t{1} << 30)) --s;
  }
  // Accuracy: one FFMA chain per output element over the whole of a long K
  // grows its rounding error with K (config 2's k = 32768 / 65536 steps put
  // the FP32 engine's smallest amplitude at 1.5e-4 relative); K/4096-way
  // split-K with the ordered fp32 reduction bounds every chain at 4096
  // terms.  Partial buffers up to 16 GiB (s026: 8 x 2 GiB).
  if (k >= 8192) {
    std::int64_t sa = std::min<std::int64_t>(16, k / 4096);
    while (sa > 1 && sa * m * n * 8 > (std::int64_t{16} << 30)) --sa;
    s = std::max(s, sa);
  }
  return static_cast<int>(std::max<std::int64_t>(s, 1));
}

}  // namespace

bool cgemm_narrow(std::int64_t m, std::int64_t n) { return use_narrow(m, n); }

std::int64_t cgemm_workspace_bytes(std::int64_t m, std::int64_t n, std::int64_t k) {
  if (use_narrow(m, n)) return 0;
  const int s = choose_splits(m, n, k);
  return s > 1 ? static_cast<std::int64_t>(s) * m * n * 8 : 0;
}

cudaError_t cgemm(const GemmArgs& g, cudaStream_t stream, int* launches) {
  if (g.m < 0 || g.n < 0 || g.k < 0) throw std::invalid_argument("cgemm: negative extent");
  if (g.m == 0 || g.n == 0) return cudaSuccess;
  KParams p{};
  p.a = static_cast<const float2*>(g.a);
  p.b = static_cast<const float2*>(g.b);
  p.c = static_cast<float2*>(g.c);
  p.m = g.m;
  p.n = g.n;
  p.k = g.k;
  p.meta_a = g.meta_a;
  p.meta_b = g.meta_b;
  p.meta_c = g.meta_c;
  p.norm_a = g.norm_a;
  p.norm_b = g.norm_b;
  if (use_narrow(g.m, g.n) && g.k > 0) {
    const std::int64_t blocks = (g.m + NR - 1) / NR;
    if (blocks > 0x7fffffff) throw std::length_error("cgemm: m too large for the grid");
    if (g.n <= 16) launch_narrow<16>(g, p, stream);
    else launch_narrow<32>(g, p, stream);
    if (launches) ++*launches;
    return cudaGetLastError();
  }
  int splits = choose_splits(g.m, g.n, g.k);
  if (splits > 1 && (g.workspace == nullptr || g.workspace_bytes < cgemm_workspace_bytes(g.m, g.n, g.k))) splits = 1;
  std::int64_t kchunk = g.k;
  if (splits > 1) {
    kchunk = ((g.k + splits - 1) / splits + BK - 1) / BK * BK;
    splits = static_cast<int>((g.k + kchunk - 1) / kchunk);
    p.partial = static_cast<float2*>(g.workspace);
  }
  p.kchunk = std::max<std::int64_t>(kchunk, 1);
  const std::int64_t gx = (g.m + BM - 1) / BM, gy = (g.n + BN - 1) / BN;
  if (gx * gy > 0x7fffffff) throw std::length_error("cgemm: m x n too large for the grid");
  p.m_tiles = gx;
  dim3 grid(static_cast<unsigned>(gx * gy), 1, static_cast<unsigned>(splits));
  if (g.trans_a) {
    if (g.trans_b) cgemm_simt_kernel<true, true><<<grid, NT, 0, stream>>>(p);
    else cgemm_simt_kernel<true, false><<<grid, NT, 0, stream>>>(p);
  } else {
    if (g.trans_b) cgemm_simt_kernel<false, true><<<grid, NT, 0, stream>>>(p);
    else cgemm_simt_kernel<false, false><<<grid, NT, 0, stream>>>(p);
  }
  if (launches) ++*launches;
  if (splits > 1) {
    const std::int64_t mn = g.m * g.n;
    const std::int64_t blocks = std::min<std::int64_t>((mn + NT - 1) / NT, sm_count() * 8);
    splitk_reduce_kernel<<<static_cast<unsigned>(blocks), NT, 0, stream>>>(p, splits);
    if (launches) ++*launches;
  }
  return cudaGetLastError();
}

}  // namespace qsg::dev
