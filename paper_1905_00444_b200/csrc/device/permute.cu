// K1: complex64 tensor permutation (replaces qsim::transpose,
// include/qsim/tensor.hpp:135-197, and the slice copies of apply_cut /
// slice_axis, tensor.hpp:236-264 -- a cut is an offset + dropped stride).
//
// Domain tensors have only extent-2 axes, so a permutation is a permutation
// of address bits: output bit j of the element index reads input bit
// inpos[j].  The kernel moves 2^t-element tiles (t <= 10, 8 KiB) through
// shared memory:
//   tile bits T = {output bits 0..4} U {the 5 output bits with the lowest
//   input positions}, topped up to 10 bits.  Loads enumerate T in input
//   order (a warp reads 32 consecutive input elements = 256 B), stores
//   enumerate T in output order (a warp writes 256 B contiguous), so both
//   HBM streams are fully coalesced and every byte moves exactly once
//   (16 B/element of algorithmic traffic).
// The remaining bits index tiles; a block walks tiles grid-stride.  Tile
// offset tables live in shared memory (dynamic indices would serialise the
// constant cache).  Pure data movement: the result is bit-identical to
// qsim::transpose.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "kernels.hpp"

namespace qsg::dev {
namespace {

constexpr int kMaxBits = 48;
constexpr int kTileBits = 10;
constexpr int kThreads = 256;

struct BitPermParams {
  long long in_base;
  long long ntiles;
  int tbits;   // bits in a tile
  int nrest;   // bits indexing tiles
  // Tile tables: load index e = (hi5 << 5) | lo5.
  long long in_lo[32], in_hi[32];    // input offsets
  long long out_lo[32], out_hi[32];  // output offsets (store index f)
  unsigned short f_lo[32], f_hi[32]; // store index of load index e
  unsigned char rest_in[kMaxBits], rest_out[kMaxBits];
};

__device__ __forceinline__ int swz(int f) { return f ^ ((f >> 5) & 31); }

// E = float2 (one complex64) or float4 (two adjacent complex64 that stay
// adjacent: output bit 0 reads input bit 0 -- 16-byte loads and stores).
template <typename E>
__global__ void __launch_bounds__(kThreads) permute_bits_kernel(const E* __restrict__ in, E* __restrict__ out,
                                                                const BitPermParams p) {
  __shared__ E tile[1 << kTileBits];
  __shared__ long long s_in_lo[32], s_in_hi[32], s_out_lo[32], s_out_hi[32];
  __shared__ unsigned short s_f_lo[32], s_f_hi[32];
  __shared__ unsigned char s_rin[kMaxBits], s_rout[kMaxBits];
  const int tid = threadIdx.x;
  if (tid < 32) {
    s_in_lo[tid] = p.in_lo[tid];
    s_in_hi[tid] = p.in_hi[tid];
    s_out_lo[tid] = p.out_lo[tid];
    s_out_hi[tid] = p.out_hi[tid];
    s_f_lo[tid] = p.f_lo[tid];
    s_f_hi[tid] = p.f_hi[tid];
  }
  if (tid < kMaxBits) {
    s_rin[tid] = p.rest_in[tid];
    s_rout[tid] = p.rest_out[tid];
  }
  __syncthreads();
  const int tsize = 1 << p.tbits;
  const int lane = tid & 31;
  // Tile base offsets: lane k contributes tile bit k (and k + 32).
  auto bases = [&](long long t, long long& base_in, long long& base_out) {
    unsigned long long bin = 0, bout = 0;
    for (int k = lane; k < p.nrest; k += 32)
      if ((t >> k) & 1) {
        bin |= 1ull << s_rin[k];
        bout |= 1ull << s_rout[k];
      }
    const unsigned bin_lo = __reduce_or_sync(0xffffffffu, static_cast<unsigned>(bin));
    const unsigned bin_hi = __reduce_or_sync(0xffffffffu, static_cast<unsigned>(bin >> 32));
    const unsigned bout_lo = __reduce_or_sync(0xffffffffu, static_cast<unsigned>(bout));
    const unsigned bout_hi = __reduce_or_sync(0xffffffffu, static_cast<unsigned>(bout >> 32));
    base_in = p.in_base + static_cast<long long>((static_cast<unsigned long long>(bin_hi) << 32) | bin_lo);
    base_out = static_cast<long long>((static_cast<unsigned long long>(bout_hi) << 32) | bout_lo);
  };
  constexpr int kPer = (1 << kTileBits) / kThreads;
  E v[kPer];
  auto load = [&](long long base_in) {
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const int e = tid + j * kThreads;
      if (e < tsize) v[j] = __ldcs(in + base_in + s_in_lo[e & 31] + s_in_hi[e >> 5]);
    }
  };
  // Software pipeline: the next tile's loads are in flight while the current
  // tile drains from shared memory to HBM.
  long long t = blockIdx.x;
  if (t >= p.ntiles) return;
  long long base_in, base_out;
  bases(t, base_in, base_out);
  load(base_in);
  while (true) {
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const int e = tid + j * kThreads;
      if (e < tsize) tile[swz(s_f_lo[e & 31] | s_f_hi[e >> 5])] = v[j];
    }
    __syncthreads();
    const long long cur_out = base_out;
    const long long tn = t + gridDim.x;
    if (tn < p.ntiles) {
      bases(tn, base_in, base_out);
      load(base_in);
    }
#pragma unroll
    for (int j = 0; j < kPer; ++j) {
      const int f = tid + j * kThreads;
      if (f < tsize) __stcs(out + cur_out + s_out_lo[f & 31] + s_out_hi[f >> 5], tile[swz(f)]);
    }
    if (tn >= p.ntiles) break;
    t = tn;
    __syncthreads();
  }
}

constexpr int kMaxRank = 64;
struct GatherParams {
  long long base;
  long long count;
  int rank;
  long long extent[kMaxRank];
  long long istride[kMaxRank];
};

// Mixed-radix gather for non-power-of-two extents (test shapes only).
__global__ void __launch_bounds__(kThreads) permute_gather_kernel(const float2* __restrict__ in,
                                                                  float2* __restrict__ out,
                                                                  const GatherParams p) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < p.count;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    long long rem = i, off = p.base;
    for (int a = p.rank - 1; a >= 0; --a) {
      const long long e = p.extent[a];
      off += (rem % e) * p.istride[a];
      rem /= e;
    }
    out[i] = in[off];
  }
}

bool is_pow2(long long x) { return x > 0 && (x & (x - 1)) == 0; }
int ilog2(long long x) {
  int r = 0;
  while ((1ll << r) < x) ++r;
  return r;
}

int sm_count() {
  static int n = [] {
    int dev = 0, v = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v;
  }();
  return n;
}

template <typename E>
void launch_bits(const std::vector<int>& inpos, long long base, const E* src, E* dst, cudaStream_t stream,
                 int* launches) {
  const int r = static_cast<int>(inpos.size());
  if (r > kMaxBits) throw std::length_error("permute: tensor rank exceeds 48 address bits");
  std::vector<char> in_tile(static_cast<std::size_t>(r), 0);
  std::vector<int> tile;
  auto add = [&](int j) {
    if (!in_tile[static_cast<std::size_t>(j)]) {
      in_tile[static_cast<std::size_t>(j)] = 1;
      tile.push_back(j);
    }
  };
  std::vector<int> by_in(static_cast<std::size_t>(r));
  for (int j = 0; j < r; ++j) by_in[static_cast<std::size_t>(j)] = j;
  std::stable_sort(by_in.begin(), by_in.end(), [&](int x, int y) { return inpos[x] < inpos[y]; });
  const int target = std::min(kTileBits, r);
  for (int j = 0; j < std::min(5, r); ++j) add(j);
  for (int j = 0; j < std::min(5, r) && static_cast<int>(tile.size()) < target; ++j) add(by_in[static_cast<std::size_t>(j)]);
  for (int step = 5; static_cast<int>(tile.size()) < target; ++step) {
    if (step < r) add(step);
    if (static_cast<int>(tile.size()) < target && step < r) add(by_in[static_cast<std::size_t>(step)]);
  }
  const int t = static_cast<int>(tile.size());
  std::vector<int> load_order = tile, store_order = tile;
  std::sort(load_order.begin(), load_order.end(), [&](int x, int y) { return inpos[x] < inpos[y]; });
  std::sort(store_order.begin(), store_order.end());
  std::vector<int> store_rank(static_cast<std::size_t>(r), -1);
  for (int k = 0; k < t; ++k) store_rank[static_cast<std::size_t>(store_order[static_cast<std::size_t>(k)])] = k;

  BitPermParams p;
  std::memset(&p, 0, sizeof p);
  p.in_base = base;
  p.tbits = t;
  for (int e = 0; e < 32; ++e) {
    long long ilo = 0, ihi = 0, olo = 0, ohi = 0;
    unsigned flo = 0, fhi = 0;
    for (int k = 0; k < 5; ++k) {
      if (!((e >> k) & 1)) continue;
      if (k < t) {
        const int j = load_order[static_cast<std::size_t>(k)];
        ilo += 1ll << inpos[static_cast<std::size_t>(j)];
        flo |= 1u << store_rank[static_cast<std::size_t>(j)];
        olo += 1ll << store_order[static_cast<std::size_t>(k)];
      }
      if (k + 5 < t) {
        const int j = load_order[static_cast<std::size_t>(k + 5)];
        ihi += 1ll << inpos[static_cast<std::size_t>(j)];
        fhi |= 1u << store_rank[static_cast<std::size_t>(j)];
        ohi += 1ll << store_order[static_cast<std::size_t>(k + 5)];
      }
    }
    p.in_lo[e] = ilo;
    p.in_hi[e] = ihi;
    p.out_lo[e] = olo;
    p.out_hi[e] = ohi;
    p.f_lo[e] = static_cast<unsigned short>(flo);
    p.f_hi[e] = static_cast<unsigned short>(fhi);
  }
  int nrest = 0;
  for (int j = 0; j < r; ++j)
    if (!in_tile[static_cast<std::size_t>(j)]) {
      p.rest_in[nrest] = static_cast<unsigned char>(inpos[static_cast<std::size_t>(j)]);
      p.rest_out[nrest] = static_cast<unsigned char>(j);
      ++nrest;
    }
  p.nrest = nrest;
  p.ntiles = 1ll << nrest;
  const long long grid = std::min<long long>(p.ntiles, static_cast<long long>(sm_count()) * 8);
  permute_bits_kernel<E><<<static_cast<unsigned>(grid), kThreads, 0, stream>>>(src, dst, p);
  if (launches) ++*launches;
}

}  // namespace

cudaError_t permute(const void* in, std::int64_t base, void* out, int rank, const std::int64_t* extent,
                    const std::int64_t* istride, cudaStream_t stream, int* launches) {
  long long count = 1;
  bool bits = true;
  for (int a = 0; a < rank; ++a) {
    if (extent[a] < 1) throw std::invalid_argument("permute: extent < 1");
    count *= extent[a];
    if (!is_pow2(extent[a]) || (extent[a] > 1 && !is_pow2(istride[a]))) bits = false;
  }
  if (count == 0) return cudaSuccess;
  const auto* src = static_cast<const float2*>(in);
  auto* dst = static_cast<float2*>(out);

  if (bits) {
    // Output bit j (LSB = fastest output element) -> input bit inpos[j].
    std::vector<int> inpos;
    for (int a = rank - 1; a >= 0; --a) {
      const int w = ilog2(extent[a]);
      const int s = extent[a] > 1 ? ilog2(istride[a]) : 0;
      for (int b = 0; b < w; ++b) inpos.push_back(s + b);
    }
    if (static_cast<int>(inpos.size()) > kMaxBits) throw std::length_error("permute: tensor rank exceeds 48 address bits");
    // Element pairs that stay adjacent move as 16-byte units.
    const bool pairs = inpos.size() >= 2 && inpos[0] == 0 && base % 2 == 0 &&
                       reinterpret_cast<std::uintptr_t>(in) % 16 == 0 && reinterpret_cast<std::uintptr_t>(out) % 16 == 0;
    if (pairs) {
      std::vector<int> half(inpos.begin() + 1, inpos.end());
      for (auto& x : half) --x;
      launch_bits<float4>(half, base / 2, static_cast<const float4*>(in), static_cast<float4*>(out), stream, launches);
    } else {
      launch_bits<float2>(inpos, base, src, dst, stream, launches);
    }
    return cudaGetLastError();
  }

  if (rank > kMaxRank) throw std::length_error("permute: rank exceeds 64");
  GatherParams g;
  std::memset(&g, 0, sizeof g);
  g.base = base;
  g.count = count;
  g.rank = rank;
  for (int a = 0; a < rank; ++a) {
    g.extent[a] = extent[a];
    g.istride[a] = istride[a];
  }
  const long long grid = std::min<long long>((count + kThreads - 1) / kThreads, static_cast<long long>(sm_count()) * 16);
  permute_gather_kernel<<<static_cast<unsigned>(grid), kThreads, 0, stream>>>(src, dst, g);
  if (launches) ++*launches;
  return cudaGetLastError();
}

}  // namespace qsg::dev
