// Microbenchmark: tcgen05.ld throughput per SM (bytes/clk) for 4 / 8 / 16
// warps, x16 / x32 / x64 column loads (32x32b shape).  One CTA per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int NCOL>
__device__ __forceinline__ void ld(uint32_t taddr, uint32_t* v);
template <>
__device__ __forceinline__ void ld<16>(uint32_t t, uint32_t* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                 "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
               : "r"(t));
}
template <>
__device__ __forceinline__ void ld<32>(uint32_t t, uint32_t* v) {
  ld<16>(t, v);
  ld<16>(t + 16, v + 16);
}

template <int NCOL>
__global__ void bench(int iters, unsigned long long* out, uint32_t* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  const int quad = warp & 3, sub = warp >> 2;
  const uint32_t base = tmem + ((uint32_t)(quad * 32) << 16);
  uint32_t acc = 0;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    for (int c = 0; c < 256; c += NCOL) {
      uint32_t v[NCOL];
      ld<NCOL>(base + (uint32_t)((sub * 256 + c) & 511), v);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int i = 0; i < NCOL; ++i) acc += v[i];
    }
  }
  __syncthreads();
  const unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int NCOL>
void run(int warps) {
  const int iters = 2000, blocks = 148;
  unsigned long long* d;
  uint32_t* sink;
  cudaMalloc(&d, blocks * 8);
  cudaMalloc(&sink, blocks * warps * 32 * 4);
  bench<NCOL><<<blocks, warps * 32>>>(10, d, sink);
  bench<NCOL><<<blocks, warps * 32>>>(iters, d, sink);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  double cyc = 0;
  for (int i = 0; i < blocks; ++i) cyc += h[i];
  cyc /= blocks;
  const double bytes = (double)iters * 256 * 4 * 32 * warps;  // per CTA: 256 columns x 32 lanes x 4 B per warp-iter
  std::printf("warps %2d  x%-2d : %.1f B/clk per SM (%s)\n", warps, NCOL, bytes / cyc, cudaGetErrorString(e));
  cudaFree(d);
  cudaFree(sink);
}

int main() {
  for (int w : {4, 8, 16}) {
    run<16>(w);
    run<32>(w);
  }
  return 0;
}
