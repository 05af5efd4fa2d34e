// Frugal rejection sampling with x1/x2 recycling on top of device amplitude
// batches, plus XEB/HOG scoring (SURVEY 8f "next" row 2: the consumer that
// turns amplitudes/s into samples/s).
//   sample / emit_one          proj/src/sampler.cpp:54-178
//   amplitude-fraction mode    proj/src/sampler.cpp:131-150, :180-185
//   xeb_score                  proj/src/sampler.cpp:187-215
// The RNG streams (mt19937_64(mix_seed(seed, i)) per sample, x1 bits from
// successive 64-bit words, candidate j = rng() % batch, 53-bit uniforms)
// follow the reference draw for draw, so a sample differs from the
// reference's only where an FP32 amplitude difference flips an accept test.
#include "sampler.hpp"

#include <algorithm>
#include <cmath>
#include <random>
#include <stdexcept>

namespace qsg {

namespace {

double uniform53(std::mt19937_64& rng) { return static_cast<double>(rng() >> 11) * 0x1p-53; }

}  // namespace

XebReport xeb_score(int n, const std::vector<double>& probs, const double* hog_median) {
  XebReport r;
  r.n = n;
  double sum_log = 0.0, sum_p = 0.0;
  std::size_t above = 0, used = 0;
  for (double p : probs) {
    if (p <= 0.0) {
      ++r.zero_excluded;
      continue;
    }
    ++used;
    sum_log += std::log(p);
    sum_p += p;
    if (hog_median && p > *hog_median) ++above;
  }
  r.size = used;
  if (used == 0) return r;
  r.mean_log_prob = sum_log / static_cast<double>(used);
  r.cross_entropy = -r.mean_log_prob;
  r.fidelity_estimate = std::exp2(static_cast<double>(n)) * (sum_p / static_cast<double>(used)) - 1.0;
  if (hog_median) {
    r.hog_available = true;
    r.hog_fraction = static_cast<double>(above) / static_cast<double>(used);
  }
  return r;
}

SampleOutput sample(Engine& e, const SamplingConfig& cfg) {
  const Circuit& c = e.circuit();
  const ContractionPlan& plan = e.plan();
  const int n = c.num_qubits();
  if (plan.open_qubits.empty()) throw std::invalid_argument("sample: plan must leave the x2 region open");
  if (!cfg.x2_region.empty()) {
    auto want = cfg.x2_region;
    std::sort(want.begin(), want.end());
    if (want != plan.open_qubits) throw std::invalid_argument("sample: x2 region does not match the plan's open qubits");
  }
  if (cfg.rejection_cap <= 0) throw std::invalid_argument("sample: rejection cap must be > 0");

  const bool amplitude_mode = cfg.amplitude_fraction_mode;
  std::size_t exact_count = cfg.num_samples;
  std::vector<std::int64_t> slice_ids;
  if (amplitude_mode) {
    const double f = static_cast<double>(cfg.fraction.num) / static_cast<double>(cfg.fraction.den);
    exact_count = static_cast<std::size_t>(std::llround(f * static_cast<double>(cfg.num_samples)));
    slice_ids = select_slices(Fraction{plan.num_slices, plan.num_slices}, plan.num_slices, cfg.seed);
  } else {
    slice_ids = select_slices(cfg.fraction, plan.num_slices, cfg.seed);
  }

  const auto& open = plan.open_qubits;
  const std::size_t batch = std::size_t{1} << open.size();
  const double scale = std::exp2(static_cast<double>(n)) / cfg.rejection_cap;

  SampleOutput out;
  out.bitstrings.assign(cfg.num_samples, {});
  out.probabilities.assign(cfg.num_samples, -1.0);
  out.stats.exact_count = exact_count;
  out.stats.uniform_count = cfg.num_samples - exact_count;

  std::vector<cdouble> amps;
  for (std::size_t i = 0; i < cfg.num_samples; ++i) {
    std::mt19937_64 rng(mix_seed(cfg.seed, i));
    if (amplitude_mode && i >= exact_count) {
      std::string bits(static_cast<std::size_t>(n), '0');
      for (auto& ch : bits) ch = static_cast<char>('0' + (rng() & 1));
      out.bitstrings[i] = std::move(bits);
      continue;
    }
    for (;;) {  // emit_one
      std::vector<int> x1(static_cast<std::size_t>(n), -1);
      std::uint64_t word = 0;
      int left = 0;
      for (int q = 0; q < n; ++q) {
        if (std::find(open.begin(), open.end(), q) != open.end()) continue;
        if (left == 0) {
          word = rng();
          left = 64;
        }
        x1[static_cast<std::size_t>(q)] = static_cast<int>(word & 1);
        word >>= 1;
        --left;
      }
      ++out.stats.x1_draws;
      e.prepare(x1);
      e.run(slice_ids, /*reset=*/true, /*per_slice=*/false);
      e.results(&amps, nullptr);
      bool accepted = false;
      for (std::size_t trial = 0; trial < batch && !accepted; ++trial) {
        const std::size_t j = rng() % batch;
        ++out.stats.candidates;
        const double p = std::norm(amps[j]);
        const double accept = p * scale;
        if (accept >= 1.0) {
          ++out.stats.cap_hits;
          accepted = true;
        } else {
          accepted = uniform53(rng) < accept;
        }
        if (accepted) {
          out.bitstrings[i] = merge_bits(x1, open, j);
          out.probabilities[i] = p;
        }
      }
      if (accepted) break;
      ++out.stats.redraws;
    }
  }
  std::vector<double> known;
  for (double p : out.probabilities)
    if (p >= 0) known.push_back(p);
  if (!known.empty()) out.self_xeb = xeb_score(n, known, nullptr);
  return out;
}

}  // namespace qsg
