// K2 tensor-core path: complex64 GEMM as a real GEMM on tcgen05.  Default:
// the CTA-pair kind::f16 kernel with a 3xFP16 split (power-of-two operand
// scaling, promoted FP32 accumulation) for FP32-level accuracy; 3xTF32
// (kind::tf32) for shapes the pair kernel does not take or QSG_TC_PREC=tf32.
// See cgemm_tc.cu.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "kernels.hpp"

namespace qsg::dev {

// True when the shape/layout is handled by the tcgen05 kernel.
// Layout constraints of the kernel (m % 128, n % 64, k % 16, A row-major).
bool cgemm_tc_supported(std::int64_t m, std::int64_t n, std::int64_t k, bool trans_a, bool trans_b);
// Supported and worth it (the engine uses this).
bool cgemm_tc_eligible(std::int64_t m, std::int64_t n, std::int64_t k, bool trans_a, bool trans_b);
// The fused output permutation is available (CTA-pair kernel path).
bool cgemm_tc_store_perm_supported(std::int64_t m, std::int64_t n, std::int64_t k, bool trans_a, bool trans_b);
std::int64_t cgemm_tc_workspace_bytes(std::int64_t m, std::int64_t n, std::int64_t k, bool trans_a, bool trans_b,
                                      bool a_presplit = false);
// The fp16 CTA-pair kernel handles the shape, so C may be written split /
// A read pre-split (GemmArgs::c_split / a_presplit).
bool cgemm_tc_split_ok(std::int64_t m, std::int64_t n, std::int64_t k, bool trans_a, bool trans_b);
cudaError_t cgemm_tc(const GemmArgs& g, cudaStream_t stream, int* launches = nullptr);
// Planning model of the tensor-core path for a shape: sustained Eq.(1)
// flop/s and the HBM bytes of its operand preparation passes (B expansion,
// A pre-split), for the engine's layout / role cost model.
double cgemm_tc_rate(std::int64_t m, std::int64_t n, std::int64_t k);
double cgemm_tc_prep_bytes(std::int64_t m, std::int64_t n, std::int64_t k);
// Process-wide switch (QSG_TENSOR_CORES=0 disables); the engine also has
// a per-instance option.
bool tc_enabled();

}  // namespace qsg::dev
