// Sampling and XEB on top of the device engine (reference
// include/qsim/sampler.hpp:17-88).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "engine.hpp"

namespace qsg {

struct SamplingConfig {
  std::size_t num_samples = 0;
  std::vector<int> x2_region;       // empty = the plan's open qubits
  bool amplitude_fraction_mode = false;  // FidelityMode::amplitude_fraction
  Fraction fraction{1, 1};
  double rejection_cap = 6.0;       // kappa
  std::uint64_t seed = 0;
};

struct SampleStats {
  std::uint64_t x1_draws = 0, redraws = 0, cap_hits = 0, candidates = 0;
  std::size_t exact_count = 0, uniform_count = 0;
};

struct XebReport {
  int n = 0;
  std::size_t size = 0;
  double mean_log_prob = 0.0, cross_entropy = 0.0, fidelity_estimate = 0.0;
  double hog_fraction = -1.0;
  bool hog_available = false;
  std::size_t zero_excluded = 0;
};

struct SampleOutput {
  std::vector<std::string> bitstrings;
  std::vector<double> probabilities;  // -1 where unknown (uniform share)
  SampleStats stats;
  XebReport self_xeb;
};

// sample() / sample_amplitude_fraction() (src/sampler.cpp:122-185).
SampleOutput sample(Engine& e, const SamplingConfig& cfg);

// xeb_score (src/sampler.cpp:187-215); hog_median may be null.
XebReport xeb_score(int n, const std::vector<double>& probs, const double* hog_median);

}  // namespace qsg
