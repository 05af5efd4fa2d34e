// K3: per-slice accumulation of the final tensor into the amplitude batch
// (src/sampler.cpp:28-34 `acc[i] += cdouble(fin[i]) * exp2(log_scale)`;
// closed plans: scalar_value, include/qsim/tensor.hpp:325-329, summed at
// src/engine.cpp:352-356).  FP64, slice order = launch order on the stream,
// so the sum order is the reference's ascending slice order.  The per-slice
// contribution is also written out for the ordered cross-GPU reduction.
//
// Plus the standalone normalize_inplace pieces (tensor.hpp:209-224): a
// max|z|^2 reduction and an exact power-of-two rescale.
#include <cmath>
#include <cstring>

#include "kernels.hpp"

namespace qsg::dev {
namespace {

constexpr int NT = 256;

__global__ void __launch_bounds__(NT) accumulate_kernel(const float2* __restrict__ fin, const TMeta* meta,
                                                        double log_scale, long long count,
                                                        double2* __restrict__ acc,
                                                        double2* __restrict__ per_slice) {
  const double scale = exp2(meta ? meta->log_scale : log_scale);
  for (long long i = blockIdx.x * static_cast<long long>(NT) + threadIdx.x; i < count;
       i += static_cast<long long>(gridDim.x) * NT) {
    const float2 v = fin[i];
    const double2 c = make_double2(static_cast<double>(v.x) * scale, static_cast<double>(v.y) * scale);
    double2 a = acc[i];
    a.x += c.x;
    a.y += c.y;
    acc[i] = a;
    if (per_slice) per_slice[i] = c;
  }
}

__global__ void __launch_bounds__(NT) max_abs_sq_kernel(const float2* __restrict__ d, long long count, TMeta* meta) {
  float local = 0.f;
  for (long long i = blockIdx.x * static_cast<long long>(NT) + threadIdx.x; i < count;
       i += static_cast<long long>(gridDim.x) * NT) {
    const float2 v = d[i];
    local = fmaxf(local, v.x * v.x + v.y * v.y);
  }
  for (int o = 16; o > 0; o >>= 1) local = fmaxf(local, __shfl_xor_sync(0xffffffffu, local, o));
  __shared__ float red[NT / 32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = local;
  __syncthreads();
  if (threadIdx.x == 0) {
    float mx = red[0];
    for (int w = 1; w < NT / 32; ++w) mx = fmaxf(mx, red[w]);
    if (mx > 0.f) atomicMax(&meta->maxsq_bits, __float_as_uint(mx));
  }
}

__global__ void __launch_bounds__(NT) scale_pow2_kernel(float2* d, long long count, int shift) {
  for (long long i = blockIdx.x * static_cast<long long>(NT) + threadIdx.x; i < count;
       i += static_cast<long long>(gridDim.x) * NT) {
    float2 v = d[i];
    v.x = scalbnf(v.x, -shift);
    v.y = scalbnf(v.y, -shift);
    d[i] = v;
  }
}

unsigned grid_for(long long count) {
  long long g = (count + NT - 1) / NT;
  if (g > 148 * 16) g = 148 * 16;
  if (g < 1) g = 1;
  return static_cast<unsigned>(g);
}

}  // namespace

cudaError_t accumulate(const void* fin, const TMeta* meta, std::int64_t count, void* acc, void* per_slice,
                       cudaStream_t stream, int* launches) {
  if (count <= 0) return cudaSuccess;
  accumulate_kernel<<<grid_for(count), NT, 0, stream>>>(static_cast<const float2*>(fin), meta, 0.0, count,
                                                        static_cast<double2*>(acc), static_cast<double2*>(per_slice));
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t accumulate(const void* fin, double log_scale, std::int64_t count, void* acc, void* per_slice,
                       cudaStream_t stream, int* launches) {
  if (count <= 0) return cudaSuccess;
  accumulate_kernel<<<grid_for(count), NT, 0, stream>>>(static_cast<const float2*>(fin), nullptr, log_scale, count,
                                                        static_cast<double2*>(acc), static_cast<double2*>(per_slice));
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t max_abs_sq(const void* data, std::int64_t count, TMeta* meta, cudaStream_t stream, int* launches) {
  if (count <= 0) return cudaSuccess;
  max_abs_sq_kernel<<<grid_for(count), NT, 0, stream>>>(static_cast<const float2*>(data), count, meta);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t scale_pow2(void* data, std::int64_t count, int shift, cudaStream_t stream, int* launches) {
  if (count <= 0 || shift == 0) return cudaSuccess;
  scale_pow2_kernel<<<grid_for(count), NT, 0, stream>>>(static_cast<float2*>(data), count, shift);
  if (launches) ++*launches;
  return cudaGetLastError();
}

int host_shift_from_maxsq(unsigned int bits) {
  if (bits == 0) return 0;
  float f;
  std::memcpy(&f, &bits, sizeof f);
  const double mx = std::sqrt(static_cast<double>(f));
  int e = 0;
  const double fr = std::frexp(mx, &e);
  return fr == 0.5 ? e - 1 : e;
}

}  // namespace qsg::dev
