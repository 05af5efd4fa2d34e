// Host-callable launchers for the sm_100a kernels of the contraction path.
//   K1  permute      qsim::transpose            include/qsim/tensor.hpp:135-197
//   K2  cgemm        the GEMM in contract_ttgt  include/qsim/contraction.hpp:208-214
//       + normalize  normalize_inplace fused    include/qsim/tensor.hpp:209-224
//   K3  accumulate   batch_amplitudes sum       src/sampler.cpp:28-34
// Complex64 data are float2 (re, im) interleaved, row-major, last axis
// fastest.  Every launcher is stream-ordered and never synchronises.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace qsg::dev {

// Per-tensor normalisation state, device resident.  The represented value
// of a tensor is data * 2^log_scale.  maxsq_bits is the float bit pattern of
// max |z|^2 over the data (atomicMax on non-negative floats as uint); a
// consumer applies the reference's power-of-two renormalisation shift
// (normalize_inplace) derived from it on the fly, which is exact.
struct TMeta {
  double log_scale;
  unsigned int maxsq_bits;
  // When the tensor is stored pre-split (fp16 hi plane | lo plane, see
  // GemmArgs::c_split): data = (hi + lo) * 2^-split_exp.
  int split_exp;
};

// ---- K1: permute -----------------------------------------------------------
// out[i_0..i_{r-1}] = in[base + sum_j i_j * istride[j]], output dense in
// the given axis order.  Covers transposes and cut views (fixed axes
// folded into base).  Uses the tiled bit-permutation kernel when every
// extent and stride is a power of two (all tensors of this domain), a
// mixed-radix gather otherwise.
cudaError_t permute(const void* in, std::int64_t base, void* out, int rank, const std::int64_t* extent,
                    const std::int64_t* istride, cudaStream_t stream, int* launches = nullptr);

// ---- K2: complex GEMM ------------------------------------------------------
// C[m][n] = sum_p A[m][p] * B[p][n] * 2^-(sa + sb), FP32 accumulate.
// trans_a: A stored [k][m]; trans_b: B stored [n][k].  sa/sb are the
// pending renormalisation shifts of the operands (from meta_a/meta_b when
// norm_a/norm_b; 0 otherwise).  meta_c receives log_scale and max|c|^2
// (maxsq must be 0 on entry).  workspace (may be null) enables split-K for
// small m*n with long k; workspace_bytes() gives the size needed.
struct GemmArgs {
  const void* a;
  const void* b;
  void* c;
  std::int64_t m, n, k;
  bool trans_a, trans_b;
  const TMeta* meta_a;
  const TMeta* meta_b;
  bool norm_a, norm_b;
  TMeta* meta_c;
  void* workspace;
  std::int64_t workspace_bytes;
  // Optional fused output permutation (tcgen05 CTA-pair path only): C is
  // stored at complex offset sum_b bit_b(row) << row_pos[b] +
  // sum_b bit_b(col) << col_pos[b] instead of row * n + col, i.e. directly in
  // the layout the consuming step wants.  row/col bit b = LSB-first bits of
  // the row (m) / complex column (n) index.  Requires col_pos[0..2] = 0,1,2.
  bool store_perm = false;
  int nrow_bits = 0, ncol_bits = 0;
  unsigned char row_pos[48] = {};
  unsigned char col_pos[24] = {};
  // Pre-split operand storage (tcgen05 fp16 CTA-pair path only).  A tensor
  // of N complex elements stored split occupies the same 8N bytes: an fp16
  // hi plane (re, im interleaved) in the first 4N bytes and the lo plane in
  // the last 4N, element o at byte 4o of each, value (hi + lo) *
  // 2^-meta.split_exp.  c_split: the epilogue writes C this way (exponent
  // from the operand bounds, so no second pass); a_presplit: A is read
  // this way (no conversion pass or in-kernel conversion).
  bool c_split = false;
  bool a_presplit = false;
};
std::int64_t cgemm_workspace_bytes(std::int64_t m, std::int64_t n, std::int64_t k);
// True when cgemm runs the narrow-N kernel (n <= 32, m >= 1024): one thread
// per output row, HBM-bound (8 (m k + m n + k n) bytes).
bool cgemm_narrow(std::int64_t m, std::int64_t n);
cudaError_t cgemm(const GemmArgs& g, cudaStream_t stream, int* launches = nullptr);

// ---- K3: accumulate --------------------------------------------------------
// contrib[i] = double(fin[i]) * 2^log_scale(meta); acc[i] += contrib[i];
// per_slice (nullable) receives contrib.
cudaError_t accumulate(const void* fin, const TMeta* meta, std::int64_t count, void* acc_double2,
                       void* per_slice_double2, cudaStream_t stream, int* launches = nullptr);
// Same with a host-side log_scale (C ABI qsg_accumulate_dev: no device meta).
cudaError_t accumulate(const void* fin, double log_scale, std::int64_t count, void* acc_double2,
                       void* per_slice_double2, cudaStream_t stream, int* launches = nullptr);

// ---- normalisation helpers (standalone normalize_inplace) --------------------
// max |z|^2 into meta->maxsq_bits (atomicMax; zero it first).
cudaError_t max_abs_sq(const void* data, std::int64_t count, TMeta* meta, cudaStream_t stream,
                       int* launches = nullptr);
// data *= 2^-shift (exact power-of-two scaling).
cudaError_t scale_pow2(void* data, std::int64_t count, int shift, cudaStream_t stream, int* launches = nullptr);

// Reference shift rule (tensor.hpp:215-217): frexp(max|z|) -> frac in
// [0.5,1); shift = exp - (frac == 0.5).  0 for an all-zero tensor.
int host_shift_from_maxsq(unsigned int maxsq_bits);

}  // namespace qsg::dev
