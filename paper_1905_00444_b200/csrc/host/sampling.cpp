// x1 draws for amplitude batches: the reference's per-task RNG stream
// mt19937_64(mix_seed(seed, task)) and its bit-per-closed-qubit draw
// (src/sampler.cpp:155-157 seeding, :70-82 drawing).  Bit-exact.
#include <algorithm>
#include <random>

#include "qsg_host.hpp"

namespace qsg {

std::vector<int> draw_x1(int n, const std::vector<int>& open_qubits, std::uint64_t seed, std::uint64_t index) {
  std::mt19937_64 rng(mix_seed(seed, index));
  std::vector<int> x1(static_cast<std::size_t>(n), -1);
  std::uint64_t word = 0;
  int left = 0;
  for (int q = 0; q < n; ++q) {
    if (std::find(open_qubits.begin(), open_qubits.end(), q) != open_qubits.end()) continue;
    if (left == 0) {
      word = rng();
      left = 64;
    }
    x1[static_cast<std::size_t>(q)] = static_cast<int>(word & 1);
    word >>= 1;
    --left;
  }
  return x1;
}

}  // namespace qsg
