// Debug harness: C1 = A0 * B0 (written split), C2 = C1 * B1 (A pre-split),
// against the same chain in fp32 storage.  Build:
//   nvcc -std=c++20 -gencode arch=compute_100a,code=sm_100a -I paper_1905_00444_b200/csrc/device \
//        scripts/debug/split_chain.cu -o gpurun_out/split_chain -L paper_1905_00444_b200 -lqsg -Xlinker -rpath,$PWD/paper_1905_00444_b200
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include <cuda_runtime.h>
#include "kernels.hpp"
#include "kernels_tc.hpp"
using namespace qsg::dev;

int run(long long m, long long k0, long long n0, long long n1, int tb1, int perm) {
  printf("== m %lld k0 %lld n0 %lld n1 %lld tb1 %d perm %d\n", m, k0, n0, n1, tb1, perm);
  std::vector<float> hA(m * k0 * 2), hB0(k0 * n0 * 2), hB1(n0 * n1 * 2);
  srand(1);
  for (auto& x : hA) x = rand() / (float)RAND_MAX - 0.5f;
  for (auto& x : hB0) x = rand() / (float)RAND_MAX - 0.5f;
  for (auto& x : hB1) x = rand() / (float)RAND_MAX - 0.5f;
  float *A, *B0, *B1, *C1, *C2;
  TMeta* meta;
  cudaMalloc(&A, hA.size() * 4); cudaMalloc(&B0, hB0.size() * 4); cudaMalloc(&B1, hB1.size() * 4);
  cudaMalloc(&C1, m * n0 * 8); cudaMalloc(&C2, m * n1 * 8); cudaMalloc(&meta, 4 * sizeof(TMeta));
  cudaMemcpy(A, hA.data(), hA.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(B0, hB0.data(), hB0.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(B1, hB1.data(), hB1.size() * 4, cudaMemcpyHostToDevice);
  std::vector<float> out[2];
  for (int split = 0; split < 2; ++split) {
    cudaMemset(meta, 0, 4 * sizeof(TMeta));
    cudaMemset(C1, 0, m * n0 * 8);
    void* ws;
    const long long wsb = 1ll << 30;
    cudaMalloc(&ws, wsb);
    GemmArgs g{};
    g.a = A; g.b = B0; g.c = C1; g.m = m; g.n = n0; g.k = k0;
    g.meta_c = meta + 0; g.workspace = ws; g.workspace_bytes = wsb; g.c_split = split;
    if (perm) {  // identity layout expressed as a fused output permutation
      int nb = 0, mb = 0;
      while ((1ll << nb) < n0) ++nb;
      while ((1ll << mb) < m) ++mb;
      g.store_perm = true; g.nrow_bits = mb; g.ncol_bits = nb;
      for (int b = 0; b < nb; ++b) g.col_pos[b] = (unsigned char)b;
      for (int b = 0; b < mb; ++b) g.row_pos[b] = (unsigned char)(nb + b);
    }
    printf("gemm1 %s\n", cudaGetErrorString(cgemm_tc(g, 0)));
    GemmArgs h{};
    h.a = C1; h.b = B1; h.c = C2; h.m = m; h.n = n1; h.k = n0; h.trans_b = tb1;
    h.meta_a = meta + 0; h.norm_a = true; h.meta_c = meta + 1; h.workspace = ws; h.workspace_bytes = wsb;
    h.a_presplit = split;
    printf("gemm2 %s\n", cudaGetErrorString(cgemm_tc(h, 0)));
    cudaDeviceSynchronize();
    printf("sync %s\n", cudaGetErrorString(cudaGetLastError()));
    TMeta hm[2];
    cudaMemcpy(hm, meta, sizeof hm, cudaMemcpyDeviceToHost);
    printf("split=%d meta0 ls=%g maxsq=%g split_exp=%d meta1 ls=%g maxsq=%g\n", split, hm[0].log_scale,
           *(float*)&hm[0].maxsq_bits, hm[0].split_exp, hm[1].log_scale, *(float*)&hm[1].maxsq_bits);
    out[split].resize(m * n1 * 2);
    cudaMemcpy(out[split].data(), C2, m * n1 * 8, cudaMemcpyDeviceToHost);
    if (split) {
      std::vector<unsigned short> raw(8);
      cudaMemcpy(raw.data(), C1, 16, cudaMemcpyDeviceToHost);
      printf("C1 hi head: %04x %04x %04x %04x\n", raw[0], raw[1], raw[2], raw[3]);
    }
    cudaFree(ws);
  }
  double num = 0, den = 0;
  for (size_t i = 0; i < out[0].size(); ++i) {
    num += (out[0][i] - out[1][i]) * (double)(out[0][i] - out[1][i]);
    den += out[0][i] * (double)out[0][i];
  }
  printf("C2[0] %g %g vs %g %g ; rel L2 diff %g\n", out[0][0], out[0][1], out[1][0], out[1][1], sqrt(num / den));
  cudaFree(A); cudaFree(B0); cudaFree(B1); cudaFree(C1); cudaFree(C2); cudaFree(meta);
  return 0;
}

int main() {
  setvbuf(stdout, nullptr, _IONBF, 0);
  run(4096, 256, 256, 128, 0, 0);
  run(4096, 256, 256, 128, 1, 0);
  run(4096, 256, 256, 128, 0, 1);
  run(65536, 256, 256, 256, 0, 1);
  run(8192, 64, 1024, 1024, 1, 1);
  run(1 << 20, 32, 128, 256, 0, 1);
  return 0;
}
