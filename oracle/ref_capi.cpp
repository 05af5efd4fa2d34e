// extern "C" driver over the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp, compiled by oracle/Makefile into
// oracle/_ref/libqsim_ref.so).  TEST INFRASTRUCTURE ONLY: tests/, the
// golden-fixture generator and bench.py's CPU-baseline leg load it to get
// the reference's own answers and timings.  Nothing in the product path
// (paper_1905_00444_b200/) links or loads this library.
//
// Every entry point returns 0 on success and -1 on a C++ exception, whose
// message is available from ref_last_error().  Variable-length outputs use
// the (buf, cap) -> required-length convention.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <map>
#include <random>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "qsim/circuit.hpp"
#include "qsim/contraction.hpp"
#include "qsim/engine.hpp"
#include "qsim/network.hpp"
#include "qsim/oracle.hpp"
#include "qsim/plan.hpp"
#include "qsim/sampler.hpp"
#include "qsim/tensor.hpp"
#include "qsim/tensor_io.hpp"

#include <nlohmann/json.hpp>

extern "C" void scipy_openblas_set_num_threads64_(int);

using namespace qsim;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

std::int64_t put_string(const std::string& s, char* buf, std::int64_t cap) {
  if (buf && cap > 0) {
    const std::int64_t n = std::min<std::int64_t>(cap - 1, static_cast<std::int64_t>(s.size()));
    std::memcpy(buf, s.data(), static_cast<std::size_t>(n));
    buf[n] = '\0';
  }
  return static_cast<std::int64_t>(s.size());
}

std::vector<int> to_vec(const int* p, int n) { return std::vector<int>(p, p + n); }

// plan_kind: 0 = plan JSON text in `plan_text`, 1 = reference_plan_7x7,
// 2 = greedy plan_contraction(budget).
ContractionPlan make_plan(const Circuit& c, const std::vector<int>& open, int plan_kind,
                          const char* plan_text, std::int64_t budget) {
  NetworkShape shape = fold_shape(c, open);
  if (plan_kind == 0) return plan_from_json(plan_text, shape);
  if (plan_kind == 1) return reference_plan_7x7(shape);
  PlanOptions opts;
  opts.memory_budget = budget;
  return plan_contraction(shape, opts);
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_set_blas_threads(int n) { scipy_openblas_set_num_threads64_(n); }

std::uint64_t ref_mix_seed(std::uint64_t seed, std::uint64_t stream) { return mix_seed(seed, stream); }

int ref_generate_rqc(int rows, int cols, int m, std::uint64_t seed, char* buf, std::int64_t cap,
                     std::int64_t* len) {
  return guarded([&] { *len = put_string(serialize_circuit(generate_rqc(rows, cols, m, seed)), buf, cap); });
}

// Round-trips circuit text through parse + serialize (canonical form).
int ref_canonical_circuit(const char* text, char* buf, std::int64_t cap, std::int64_t* len) {
  return guarded([&] { *len = put_string(serialize_circuit(parse_circuit(std::string(text))), buf, cap); });
}

// Full double-precision state vector (2^n complex, interleaved re/im).
int ref_evolve(const char* text, double* out, std::int64_t cap_complex) {
  return guarded([&] {
    StateVector sv = evolve(parse_circuit(std::string(text)));
    const auto& a = sv.amplitudes();
    if (static_cast<std::int64_t>(a.size()) > cap_complex) throw std::length_error("ref_evolve: buffer too small");
    for (std::size_t i = 0; i < a.size(); ++i) {
      out[2 * i] = a[i].real();
      out[2 * i + 1] = a[i].imag();
    }
  });
}

// Plan JSON (plan_to_json of the annotated plan).
int ref_plan_json(const char* text, const int* open, int nopen, int plan_kind, const char* plan_text,
                  std::int64_t budget, char* buf, std::int64_t cap, std::int64_t* len) {
  return guarded([&] {
    Circuit c = parse_circuit(std::string(text));
    ContractionPlan plan = make_plan(c, to_vec(open, nopen), plan_kind, plan_text, budget);
    *len = put_string(plan_to_json(plan), buf, cap);
  });
}

// Folded network (after the optional cut) as concatenated QTNS dumps, node
// order q = 0..n-1.  out_bits: one entry per qubit, -1 = open.
int ref_fold_qtns(const char* text, const int* out_bits, int n, const char* plan_text,
                  std::int64_t slice_id, char* buf, std::int64_t cap, std::int64_t* len) {
  return guarded([&] {
    Circuit c = parse_circuit(std::string(text));
    GridNetwork net = fold_worldlines(c, to_vec(out_bits, n));
    if (plan_text && plan_text[0]) {
      ContractionPlan plan = plan_from_json(plan_text, net.shape());
      net = apply_cut(net, plan.cut, slice_id);
    }
    std::ostringstream os;
    for (const auto& t : net.nodes) write_tensor(os, t);
    const std::string s = os.str();
    *len = static_cast<std::int64_t>(s.size());
    if (buf && cap >= *len) std::memcpy(buf, s.data(), s.size());
  });
}

int ref_select_slices(std::int64_t num, std::int64_t den, std::int64_t num_slices, std::uint64_t seed,
                      std::int64_t* out) {
  return guarded([&] {
    auto ids = select_slices(Fraction{num, den}, num_slices, seed);
    std::copy(ids.begin(), ids.end(), out);
  });
}

// amplitude_batch (src/sampler.cpp:111-120): x1 bits per qubit (-1 = open),
// out = 2^|open| complex doubles (interleaved) in batch-index order, plus
// the merged bitstrings (n chars each, concatenated) if bits_out != null.
int ref_amplitude_batch(const char* text, const char* plan_text, int plan_kind, const int* x1, int n,
                        const std::int64_t* slice_ids, std::int64_t nslices, double* out,
                        char* bits_out) {
  return guarded([&] {
    Circuit c = parse_circuit(std::string(text));
    std::vector<int> open;
    for (int q = 0; q < n; ++q)
      if (x1[q] < 0) open.push_back(q);
    ContractionPlan plan = make_plan(c, open, plan_kind, plan_text, 0);
    std::vector<std::int64_t> ids(slice_ids, slice_ids + nslices);
    ExecOptions exec;
    auto res = amplitude_batch(c, plan, to_vec(x1, n), ids, exec);
    for (std::size_t i = 0; i < res.size(); ++i) {
      out[2 * i] = res[i].second.real();
      out[2 * i + 1] = res[i].second.imag();
      if (bits_out) std::memcpy(bits_out + i * static_cast<std::size_t>(n), res[i].first.data(), static_cast<std::size_t>(n));
    }
  });
}

// run_amplitudes (src/engine.cpp:300-378) on a closed plan.  bitstrings are
// nb concatenated n-char strings.  out: nb complex doubles; slice ids
// executed are written to ids_out (k entries) when non-null.
int ref_run_amplitudes(const char* text, const char* plan_text, int plan_kind, const char* bitstrings,
                       int nb, int n, std::int64_t frac_num, std::int64_t frac_den, int workers,
                       std::uint64_t seed, double* out, std::int64_t* ids_out, std::uint64_t* flops_out) {
  return guarded([&] {
    Circuit c = parse_circuit(std::string(text));
    ContractionPlan plan = make_plan(c, {}, plan_kind, plan_text, 0);
    std::vector<std::string> bits;
    for (int b = 0; b < nb; ++b) bits.emplace_back(bitstrings + static_cast<std::size_t>(b) * n, static_cast<std::size_t>(n));
    Fraction f{frac_num, frac_den};
    if (frac_den <= 0) f = Fraction{plan.num_slices, plan.num_slices};
    auto res = run_amplitudes(c, plan, bits, f, workers, seed);
    for (int b = 0; b < nb; ++b) {
      out[2 * b] = res.amplitudes[static_cast<std::size_t>(b)].amplitude.real();
      out[2 * b + 1] = res.amplitudes[static_cast<std::size_t>(b)].amplitude.imag();
    }
    if (ids_out) std::copy(res.slice_ids.begin(), res.slice_ids.end(), ids_out);
    if (flops_out) *flops_out = res.metrics.total_flops;
  });
}

// qsim::transpose on a tensor with labels "a0".."a{r-1}"; perm[i] = input
// axis placed at output position i.  complex64 interleaved in/out.
int ref_transpose(int rank, const std::int64_t* dims, const float* in, const int* perm, float* out) {
  return guarded([&] {
    std::vector<Label> labels;
    std::vector<std::int64_t> d(dims, dims + rank);
    for (int i = 0; i < rank; ++i) labels.push_back("a" + std::to_string(i));
    const std::int64_t vol = Tensorf::volume_from_dims(d);
    std::vector<cfloat> data(static_cast<std::size_t>(vol));
    std::memcpy(data.data(), in, static_cast<std::size_t>(vol) * sizeof(cfloat));
    Tensorf t(labels, d, std::move(data));
    std::vector<Label> order;
    for (int i = 0; i < rank; ++i) order.push_back(labels[static_cast<std::size_t>(perm[i])]);
    Tensorf u = transpose(t, order);
    std::memcpy(out, u.data().data(), static_cast<std::size_t>(vol) * sizeof(cfloat));
  });
}

// qsim::contract_ttgt then normalize_inplace, as execute_slice does
// (src/engine.cpp:211-233).  Labels are small integers; the output is in
// the label order given by out_labels (the plan's sorted order), log_scale
// returned separately.
int ref_contract_step(int lrank, const int* llab, const std::int64_t* ldims, const float* ldata, double lscale,
                      int rrank, const int* rlab, const std::int64_t* rdims, const float* rdata, double rscale,
                      int orank, const int* olab, float* out, double* oscale, std::uint64_t* flops,
                      int normalize) {
  return guarded([&] {
    auto mk = [](int rank, const int* lab, const std::int64_t* dims, const float* data, double ls) {
      std::vector<Label> labels;
      for (int i = 0; i < rank; ++i) labels.push_back("L" + std::to_string(1000 + lab[i]));
      std::vector<std::int64_t> d(dims, dims + rank);
      const std::int64_t vol = Tensorf::volume_from_dims(d);
      std::vector<cfloat> v(static_cast<std::size_t>(vol));
      std::memcpy(v.data(), data, static_cast<std::size_t>(vol) * sizeof(cfloat));
      return Tensorf(labels, d, std::move(v), ls);
    };
    Tensorf a = mk(lrank, llab, ldims, ldata, lscale);
    Tensorf b = mk(rrank, rlab, rdims, rdata, rscale);
    ContractionSpec spec = infer_spec(a.labels(), b.labels());
    for (int i = 0; i < orank; ++i) spec.output_labels.push_back("L" + std::to_string(1000 + olab[i]));
    FlopCounter fc;
    Tensorf c = contract_ttgt(a, b, spec, &fc);
    if (normalize) normalize_inplace(c);
    std::memcpy(out, c.data().data(), static_cast<std::size_t>(c.volume()) * sizeof(cfloat));
    *oscale = c.log_scale();
    *flops = fc.total();
  });
}

// CPU baseline: runs the reference's per-step kernels (contract_ttgt +
// normalize_inplace, the body of execute_slice, src/engine.cpp:204-240) over
// the first `nsteps` plan steps of one slice, for `ntasks` independent
// (x1, slice) tasks spread over `threads` std::threads (the reference's
// schedule()).  Reports wall seconds and Eq.(1) flops executed.
int ref_execute_prefix(const char* text, const char* plan_text, int plan_kind, const int* open, int nopen,
                       int nsteps, int ntasks, int threads, std::uint64_t seed, double* seconds,
                       std::uint64_t* flops) {
  return guarded([&] {
    Circuit c = parse_circuit(std::string(text));
    const int n = c.num_qubits();
    std::vector<int> openv = to_vec(open, nopen);
    ContractionPlan plan = make_plan(c, openv, plan_kind, plan_text, 0);
    const int steps = std::min<int>(nsteps, static_cast<int>(plan.steps.size()));
    std::vector<GridNetwork> nets;
    std::vector<std::int64_t> sids;
    for (int t = 0; t < ntasks; ++t) {
      std::mt19937_64 rng(mix_seed(seed, static_cast<std::uint64_t>(t)));
      std::vector<int> x1(static_cast<std::size_t>(n), 0);
      for (int q = 0; q < n; ++q) x1[static_cast<std::size_t>(q)] = static_cast<int>(rng() & 1);
      for (int q : openv) x1[static_cast<std::size_t>(q)] = -1;
      GridNetwork folded = fold_worldlines(c, x1);
      const std::int64_t sid = static_cast<std::int64_t>(rng() % static_cast<std::uint64_t>(plan.num_slices));
      nets.push_back(apply_cut(folded, plan.cut, sid));
      sids.push_back(sid);
    }
    FlopCounter counter;
    auto t0 = std::chrono::steady_clock::now();
    schedule(static_cast<std::size_t>(ntasks), threads, [&](std::size_t task) {
      std::map<std::string, Tensorf> live;
      const auto& net = nets[task];
      for (std::size_t q = 0; q < net.nodes.size(); ++q) live[node_name(static_cast<int>(q))] = net.nodes[q];
      for (int si = 0; si < steps; ++si) {
        const auto& step = plan.steps[static_cast<std::size_t>(si)];
        auto li = live.find(step.lhs);
        auto ri = live.find(step.rhs);
        ContractionSpec spec = infer_spec(li->second.labels(), ri->second.labels());
        spec.output_labels = step.out_labels;
        Tensorf out = contract_ttgt(li->second, ri->second, spec, &counter);
        normalize_inplace(out);
        live.erase(li);
        live.erase(step.rhs);
        live[step.out] = std::move(out);
      }
    });
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *flops = counter.total();
  });
}

// sample() (src/sampler.cpp:122-178) on a plan with open qubits; bitstrings
// (M * n chars) and probabilities out.
int ref_sample(const char* text, const char* plan_text, std::int64_t num_samples, std::int64_t frac_num,
               std::int64_t frac_den, int amplitude_mode, double cap, std::uint64_t seed, char* bits_out,
               double* probs_out) {
  return guarded([&] {
    Circuit c = parse_circuit(std::string(text));
    // The plan JSON carries its open qubits.
    auto j = nlohmann::json::parse(plan_text);
    std::vector<int> open = j.at("open_qubits").get<std::vector<int>>();
    ContractionPlan plan = plan_from_json(plan_text, fold_shape(c, open));
    SamplingConfig cfg;
    cfg.num_samples = static_cast<std::size_t>(num_samples);
    cfg.fraction = frac_den > 0 ? Fraction{frac_num, frac_den} : Fraction{plan.num_slices, plan.num_slices};
    cfg.mode = amplitude_mode ? FidelityMode::amplitude_fraction : FidelityMode::path_fraction;
    cfg.rejection_cap = cap;
    cfg.seed = seed;
    auto out = sample(c, plan, cfg);
    const int n = c.num_qubits();
    for (std::size_t i = 0; i < out.bitstrings.size(); ++i) {
      std::memcpy(bits_out + i * static_cast<std::size_t>(n), out.bitstrings[i].data(), static_cast<std::size_t>(n));
      probs_out[i] = out.probabilities[i];
    }
  });
}

}  // extern "C"
