// K2 tensor-core path (tcgen05 kind::tf32, 3xTF32 split) -- under
// construction; until validated on hardware every shape routes to the
// general FP32 kernel (cgemm.cu).
#include <cstdlib>
#include <stdexcept>

#include "kernels_tc.hpp"

namespace qsg::dev {

bool tc_enabled() {
  const char* env = std::getenv("QSG_TENSOR_CORES");
  return !(env && env[0] == '0');
}

bool cgemm_tc_eligible(std::int64_t, std::int64_t, std::int64_t, bool, bool) { return false; }

std::int64_t cgemm_tc_workspace_bytes(std::int64_t, std::int64_t, std::int64_t, bool, bool) { return 0; }

cudaError_t cgemm_tc(const GemmArgs&, cudaStream_t, int*) {
  throw std::runtime_error("cgemm_tc: tensor-core path not available");
}

}  // namespace qsg::dev
