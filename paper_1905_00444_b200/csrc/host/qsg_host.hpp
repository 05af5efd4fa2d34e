// Host-side model of the qFlex-style amplitude path: circuits (GRCS text),
// the worldline fold into a 2-D grid network, contraction plans with cut
// slicing, and slice selection.  Mirrors the reference's public surface in
// namespace qsim (names, argument meaning, exception types and message
// prefixes) so the reference's drivers and tests read the same against it:
//
//   circuit   <- include/qsim/circuit.hpp, src/circuit.cpp
//   network   <- include/qsim/network.hpp, src/network.cpp
//   plan      <- include/qsim/plan.hpp,    src/plan.cpp
//   seeds     <- include/qsim/types.hpp:25-46, src/engine.cpp:26-50,285-298
//
// Everything here is host bookkeeping; the numeric work of the hot path
// (permute, contraction GEMM, accumulation) runs on the GPU (engine.hpp).
#pragma once

#include <complex>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace qsg {

using cfloat = std::complex<float>;
using cdouble = std::complex<double>;
using Label = std::string;

// ---- seeds / hashes (include/qsim/types.hpp:25-46) -------------------------
std::uint64_t mix_seed(std::uint64_t seed, std::uint64_t stream);
std::uint64_t fnv1a(const void* data, std::size_t len, std::uint64_t h = 0xcbf29ce484222325ull);

// ---- circuit (include/qsim/circuit.hpp) ------------------------------------
enum class GateKind { H, T, XHalf, YHalf, CZ };

struct Mat2 {
  cdouble a[4];  // row-major u00 u01 u10 u11
  const cdouble& operator()(int r, int c) const { return a[2 * r + c]; }
};

const char* gate_name(GateKind k);
Mat2 gate_matrix(GateKind k);

struct Gate {
  GateKind kind;
  int cycle;
  int q0;
  int q1 = -1;
  bool two_qubit() const { return q1 >= 0; }
  friend bool operator==(const Gate&, const Gate&) = default;
};

struct Circuit {
  int rows = 0, cols = 0;
  std::vector<Gate> gates;
  int num_qubits() const { return rows * cols; }
  int cycles() const;
  int depth_m() const { return cycles() - 2; }
  int row_of(int q) const { return q / cols; }
  int col_of(int q) const { return q % cols; }
  bool adjacent(int a, int b) const;
  void canonicalize();
  friend bool operator==(const Circuit&, const Circuit&) = default;
};

struct CircuitError : std::runtime_error {
  CircuitError(const std::string& msg, int line = 0);
  int line;
};

Circuit parse_circuit(const std::string& text, int rows_hint = 0, int cols_hint = 0);
std::string serialize_circuit(const Circuit& c);
Circuit generate_rqc(int rows, int cols, int m, std::uint64_t seed, bool t_only_first = true);
Circuit generate_rqc_masked(int rows, int cols, const std::string& mask, int m, std::uint64_t seed,
                            bool t_only_first = true);
std::string bristlecone_mask(int active);  // 11x12 diamond: 72, 70 or 60 active cells
int cz_layout_of_cycle(int c);
std::vector<std::pair<int, int>> cz_layout_edges(int layout, int rows, int cols);
void validate_circuit(const Circuit& c);

// ---- tensors on the host (node tensors, test I/O) ---------------------------
struct HostTensor {
  std::vector<Label> labels;
  std::vector<std::int64_t> dims;
  std::vector<cfloat> data;  // row-major, last label fastest
  double log_scale = 0.0;
  std::int64_t volume() const { return static_cast<std::int64_t>(data.size()); }
  int rank() const { return static_cast<int>(labels.size()); }
  int axis(const Label& l) const;
  bool has_label(const Label& l) const;
};

// ---- network (include/qsim/network.hpp) -------------------------------------
struct BondRef {
  Label label;
  int q0, q1;
  int cycle;
};

struct TensorShape {
  std::vector<Label> labels;
  std::vector<std::int64_t> dims;
  std::int64_t volume() const;
  std::int64_t bytes() const { return volume() * 8; }
  std::int64_t dim(const Label& l) const;
  bool has_label(const Label& l) const;
};

struct NetworkShape {
  int rows = 0, cols = 0;
  std::vector<TensorShape> nodes;
  std::vector<BondRef> bonds;
  std::vector<int> open_qubits;
};

struct GridNetwork {
  int rows = 0, cols = 0;
  std::vector<HostTensor> nodes;
  std::vector<BondRef> bonds;
  std::vector<int> open_qubits;
  NetworkShape shape() const;
};

Label bond_label(int cycle, int q0, int q1);
Label open_label(int q);
std::string node_name(int q);

GridNetwork fold_worldlines(const Circuit& c, const std::vector<int>& out_bits,
                            const std::vector<int>& in_bits);
GridNetwork fold_worldlines(const Circuit& c, const std::vector<int>& out_bits);
NetworkShape fold_shape(const Circuit& c, const std::vector<int>& open_qubits = {});

// ---- plan (include/qsim/plan.hpp) -------------------------------------------
struct Cut {
  std::vector<Label> labels;
  std::int64_t group = 1;
};

struct PlanStep {
  std::string out, lhs, rhs;
  std::vector<Label> out_labels;
  std::int64_t out_volume = 0;
  std::uint64_t flops = 0;
  double intensity = 0.0;
  std::int64_t working_set = 0;
};

struct ContractionPlan {
  Cut cut;
  std::int64_t num_slices = 1;
  std::vector<int> open_qubits;
  std::vector<PlanStep> steps;
  std::string final_tensor;
  std::uint64_t flops_per_slice = 0;
  std::int64_t peak_memory = 0;
  int max_rank = 0;
};

struct PlanOptions {
  std::int64_t memory_budget = 0;
  int max_cut_labels = 24;
};

std::uint64_t flop_count(std::uint64_t v0, std::uint64_t v1, std::uint64_t v2);
double log2_volume(const TensorShape& t);  // sum of log2 extents (overflow-free size test)
std::int64_t step_working_set(std::int64_t lhs_bytes, std::int64_t rhs_bytes, std::int64_t out_bytes);

NetworkShape sliced_shape(const NetworkShape& s, const Cut& cut);
std::int64_t cut_slice_count(const NetworkShape& s, const Cut& cut);
// Index of the first grouped (whole-kept) cut label; labels before it are
// fixed per slice (src/plan.cpp:25-42).
std::size_t cut_fixed_count(const NetworkShape& s, const Cut& cut);
// Mixed-radix digits of a slice id over the fixed cut labels, first label
// most significant (src/plan.cpp:96-101).
std::vector<std::int64_t> cut_digits(const NetworkShape& s, const Cut& cut, std::int64_t slice_id);
GridNetwork apply_cut(const GridNetwork& net, const Cut& cut, std::int64_t slice_id);

void annotate_plan(const NetworkShape& shape, ContractionPlan& plan);
ContractionPlan plan_contraction(const NetworkShape& shape, const PlanOptions& opts = {});
// Contraction-tree rewrite (not in the reference; opt-in): T = A x B read
// once by U = T x C becomes W = B x C, U = A x W (or with A and B swapped)
// when that cuts the pair's Eq.(1) flops by >= 25% without a larger
// intermediate, repeated to a fixed point.  Collapses chains that expand a
// tensor by a small node and contract the expansion with the next small
// node (X.(Y.Z) for (X.Y).Z).  Same amplitudes up to rounding, same cut and
// slices; outputs renamed positionally.
ContractionPlan reassociate_plan(const NetworkShape& shape, const ContractionPlan& plan, int* rewrites = nullptr);
std::string plan_to_json(const ContractionPlan& plan);
ContractionPlan plan_from_json(const std::string& text, const NetworkShape& shape);
std::vector<int> plan_json_open_qubits(const std::string& text);
ContractionPlan reference_plan_7x7(const NetworkShape& shape);
std::vector<int> reference_open_qubits_7x7();

// ---- slice selection (src/engine.cpp:26-50, 285-298) ------------------------
struct Fraction {
  std::int64_t num = 1, den = 1;
};
Fraction parse_fraction(const std::string& text);
std::vector<std::int64_t> select_slices(Fraction f, std::int64_t num_slices, std::uint64_t seed);

// Random x1 for task `index` (src/sampler.cpp:70-82, 155-157): closed
// qubits get bits from mt19937_64(mix_seed(seed, index)); open ones -1.
std::vector<int> draw_x1(int n, const std::vector<int>& open_qubits, std::uint64_t seed, std::uint64_t index);

// Batch index -> bitstring (src/sampler.cpp:38-52).
std::string merge_bits(const std::vector<int>& x1_bits, const std::vector<int>& open_sorted,
                       std::size_t batch_index);

}  // namespace qsg
