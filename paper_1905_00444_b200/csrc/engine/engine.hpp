// Device executor for the sliced contraction (replaces execute_slice,
// proj/src/engine.cpp:182-245, and the slice loops of batch_amplitudes,
// src/sampler.cpp:17-36, and run_amplitudes, src/engine.cpp:300-378).
//
// A plan is compiled ONCE into a static device program:
//   * node tensors live in one region of a single HBM arena: the worldline
//     fold with every output wire open, uploaded ONCE per circuit; an x1
//     batch projects closed outputs by a half offset on axis 0 and a cut is
//     a per-slice base offset plus dropped strides, so neither fold nor
//     apply_cut moves data per batch or slice;
//   * each plan step becomes [K1 permute of an operand when its layout is
//     unusable] + one K2 CGEMM writing C = [lfree, rfree].  The executor
//     picks the contracted-label order and N/T operand layouts that avoid
//     permutes, and never permutes outputs back to sorted order (only the
//     final tensor is put in sorted open-label order, the one layout the
//     reference exposes, src/sampler.cpp:38-40);
//   * intermediates, permute scratch and split-K workspaces get static
//     arena offsets from a liveness-based first-fit packing, so a slice
//     does no allocation and every slice reuses the same layout;
//   * renormalisation state (TMeta) is device resident; nothing
//     synchronises with the host inside a slice.
// Slices run back to back on one stream; K3 accumulates them in order.
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../device/kernels.hpp"
#include "../host/qsg_host.hpp"

namespace qsg {

struct EngineOptions {
  int device = 0;
  bool profile = false;     // CUDA events around every kernel op
  bool tensor_cores = true; // allow the tcgen05 GEMM for eligible steps
  bool compile_only = false; // build the program listing without touching a device
  // Out-of-core execution (ExecOptions, include/qsim/engine.hpp:22-27): a
  // contraction whose working set (in + out + max) exceeds memory_budget
  // bytes runs as pieces (src/plan.cpp:355-472) through a device-side
  // pipeline of depth pipeline_depth (src/engine.cpp:52-180); its operands
  // and result live in pinned host memory.  0 = everything in HBM.
  // < 0: automatic -- in HBM if the program fits device_memory (0: the
  // device's free memory), else the largest power-of-two budget that fits.
  std::int64_t memory_budget = 0;
  int pipeline_depth = 2;
  std::int64_t device_memory = 0;
  // Replay a run identical to the previous one (same slices, x1 views and
  // flags) as a CUDA graph captured on its second occurrence: the
  // launch-bound small configurations (config 1: ~140 kernels in 0.5 ms)
  // stop paying one host launch per kernel.  Off while profiling and for
  // out-of-core programs; QSG_GRAPH=0 disables.
  bool graphs = true;
};

struct OpProfile {
  int kind;          // 0 permute, 1 gemm, 2 accumulate/final
  int step;          // plan step index (-1 for the final op)
  std::int64_t m, n, k;      // gemm shape (permute: elements in m)
  std::uint64_t flops;       // Eq.(1) flops of the step (gemm ops)
  std::int64_t bytes;        // algorithmic bytes moved (permute: 16 B/elem)
  double ms_total;           // summed over executions
  std::int64_t executions;
  int tc;                    // 1 if the tcgen05 kernel ran
};

class Engine {
 public:
  Engine(const Circuit& c, const ContractionPlan& plan, const EngineOptions& opt);
  ~Engine();
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;

  const Circuit& circuit() const { return circuit_; }
  const ContractionPlan& plan() const { return plan_; }
  std::int64_t batch_size() const { return batch_; }
  std::int64_t arena_bytes() const { return arena_bytes_; }
  std::int64_t memory_budget() const { return opt_.memory_budget; }  // the resolved budget (0 = all in HBM)
  std::int64_t host_arena_bytes() const { return host_arena_bytes_; }
  std::int64_t node_bytes() const { return node_bytes_; }
  cudaStream_t stream() const { return stream_; }
  int device() const { return opt_.device; }

  // Selects the x1 batch (one entry per qubit, -1 exactly on the plan's open
  // qubits).  The open fold is resident (uploaded once by the constructor),
  // so this only sets per-node view offsets: no fold, no H2D.  Returns the
  // H2D byte count (0).
  std::int64_t prepare(const std::vector<int>& x1_bits);

  // Node region (the open fold, node_bytes() of complex64) in host order.
  // fold_nodes: the open fold of another instance of the same circuit
  // layout (same grid, depth and CZ pattern, e.g. another gate draw) into
  // host memory; throws if its fold shape differs.  load_nodes: async H2D
  // of such a region on the engine stream (pinned host memory overlaps);
  // later runs use the new circuit instance.  export_nodes: D2H copy.
  void fold_nodes(const Circuit& c, void* host, std::int64_t bytes) const;
  void load_nodes(const void* host, std::int64_t bytes);
  void export_nodes(void* host, std::int64_t bytes);

  // Runs the slices in the given order on the engine stream (async).
  // reset: zero the batch accumulator first.  per_slice: keep every
  // slice's contribution (slot i for slice_ids[i]).
  void run(const std::vector<std::int64_t>& slice_ids, bool reset, bool per_slice);

  // Copies results to the host (synchronises the stream).
  void results(std::vector<cdouble>* amps, std::vector<cdouble>* per_slice);
  // The batch in the engine's pinned staging buffer (synchronises; valid
  // until the next results call): no allocation on the hot path.
  const cdouble* results_pinned();
  // Asynchronous result staging (two slots): D2H of the batch accumulator
  // into a pinned slot + event, enqueued after the current run; the host
  // collects it later, so it can prepare the next batch meanwhile.
  void stage_results(int slot);
  const cdouble* staged_results(int slot);  // waits for that slot's copy
  void synchronize();

  std::int64_t launches() const { return launches_; }
  // Rows of per-slice contributions the last run() kept (0 without per_slice).
  std::int64_t per_slice_rows() const { return per_slice_used_; }
  std::vector<OpProfile> profile();  // synchronises
  void reset_profile();
  void set_profile(bool on);
  std::string describe() const;      // human-readable program listing

 private:
  struct Buffer {
    std::int64_t bytes = 0;
    int first = 0, last = 0;
    std::int64_t offset = 0;
    bool host = false;  // pinned host arena (out-of-core tensors)
  };
  struct Operand {
    int buf = -1;
    std::int64_t off = 0;   // elements, static part
    int node = -1;          // node whose per-slice cut offset applies
  };
  struct Op {
    int kind = 0;  // 0 permute, 1 gemm, 2 final accumulate
    int step = -1;
    Operand src;   // permute source / accumulate source
    std::vector<std::int64_t> ext, istr;
    int dst = -1;  // permute destination buffer
    Operand a, b;  // gemm
    int c = -1;
    std::int64_t m = 0, n = 0, k = 0;
    bool ta = false, tb = false;
    int meta_a = -1, meta_b = -1, meta_c = -1;
    int ws = -1;
    std::int64_t ws_bytes = 0;
    bool tc = false;
    std::int64_t count = 0;  // accumulate / permute elements
    std::uint64_t flops = 0;
    bool store_perm = false;  // fused output permutation (see dev::GemmArgs)
    int nrow_bits = 0, ncol_bits = 0;
    std::array<unsigned char, 48> row_pos{};
    std::array<unsigned char, 24> col_pos{};
    bool c_split = false;     // C written as fp16 hi | lo planes (dev::GemmArgs::c_split)
    bool a_presplit = false;  // A read as fp16 hi | lo planes
    // Out-of-core GEMM: m / n row-column blocks (m0, mp, n0, np) streamed
    // through the device pipeline; C in host memory.
    bool ooc = false;
    std::vector<std::array<std::int64_t, 4>> pieces;
    // Out-of-core operand gathers: instead of a K1 permute into a host copy,
    // each piece's block is gathered (K1) straight from the source view
    // (extents / strides in GEMM order; A: split rows = first ga_split
    // dims, B: split columns = dims from gb_split on).
    bool a_gather = false, b_gather = false;
    std::vector<std::int64_t> ga_ext, ga_str, gb_ext, gb_str;
    std::size_t ga_split = 0, gb_split = 0;
  };

  void compile();
  void split_handoffs();
  void pack_buffers();
  void* ptr(const Operand& o, const std::vector<std::int64_t>& node_off) const;
  char* base_of(int buf) const;
  static std::vector<std::array<std::int64_t, 4>> decompose_pieces(std::int64_t m, std::int64_t n, std::int64_t k,
                                                                   std::int64_t budget);
  void launch_op(std::size_t i, const std::vector<std::int64_t>& node_off, void* per_slice_slot);
  void launch_ooc_gemm(const Op& op, const std::vector<std::int64_t>& node_off, int* launches);
  void gather_block(const char* src, std::vector<std::int64_t> ext, const std::vector<std::int64_t>& str,
                    std::size_t lo, std::size_t hi, std::int64_t r0, std::int64_t rp, char* dst, int* launches);

  void pack_nodes(const GridNetwork& f, void* host) const;

  Circuit circuit_;
  ContractionPlan plan_;
  NetworkShape shape_;       // fold layout (open label at axis 0)
  EngineOptions opt_;
  cudaStream_t stream_ = nullptr;
  std::int64_t batch_ = 1;

  // Node layout (full, uncut) inside the node region.
  std::vector<std::int64_t> node_elem_off_, node_vol_;
  std::vector<std::vector<std::int64_t>> node_full_strides_;
  std::vector<std::vector<int>> node_cut_axes_;  // per node: fixed cut index -> axis
  std::vector<std::int64_t> node_wire_stride_;   // stride of axis 0 (the output wire)
  std::vector<char> closed_;                     // 1 = output projected by x1
  std::vector<std::int64_t> node_x1_off_;        // per-node view offset of the current x1
  std::int64_t node_bytes_ = 0;

  std::vector<Buffer> bufs_;
  std::vector<Op> ops_;
  std::int64_t arena_bytes_ = 0;
  char* arena_ = nullptr;
  // Out-of-core: pinned host arena (mapped) for oversized steps' tensors,
  // device scratch slots for their pieces, the copy stream and its events.
  std::int64_t host_arena_bytes_ = 0;
  char* host_arena_ = nullptr;
  std::int64_t ooc_slot_bytes_ = 0;
  char* ooc_scratch_ = nullptr;
  cudaStream_t copy_stream_ = nullptr;   // out-of-core loads (H2D)
  cudaStream_t store_stream_ = nullptr;  // out-of-core stores (D2H)
  std::vector<cudaEvent_t> ooc_ev_;
  dev::TMeta* metas_ = nullptr;
  int nmeta_ = 0;
  double2* acc_ = nullptr;
  double2* acc_host_ = nullptr;  // pinned staging of the batch for results()
  struct Stage {
    double2* host = nullptr;
    cudaEvent_t ev = nullptr;
  };
  Stage stage_[2];
  double2* per_slice_ = nullptr;
  std::int64_t per_slice_cap_ = 0;
  std::int64_t per_slice_used_ = 0;
  std::int64_t per_slice_base_ = 0;  // first row the current run writes
  std::int64_t launches_ = 0;
  // CUDA graph of the last repeated run (see EngineOptions::graphs).
  void enqueue_run(const std::vector<std::int64_t>& slice_ids, bool reset, bool per_slice);
  std::vector<std::int64_t> run_key(const std::vector<std::int64_t>& slice_ids, bool reset, bool per_slice) const;
  std::vector<std::int64_t> last_key_, graph_key_;
  cudaGraphExec_t graph_exec_ = nullptr;
  std::int64_t graph_launches_ = 0;
  bool graphs_ok_ = true;

  std::vector<cudaEvent_t> ev_;
  std::vector<double> op_ms_;
  std::vector<std::int64_t> op_execs_;
  bool events_pending_ = false;
};

// Reference-named drivers on top of the engine.
// amplitude_batch (src/sampler.cpp:111-120): (bitstring, amplitude) pairs.
std::vector<std::pair<std::string, cdouble>> amplitude_batch(Engine& e, const std::vector<int>& x1_bits,
                                                             const std::vector<std::int64_t>& slice_ids);

// run_amplitudes failure attributed to a slice, as the reference's JobError
// (include/qsim/engine.hpp:81-84, src/engine.cpp:38-39): message +
// " (slice N)", N = the slice of the lowest failing task (src/engine.cpp:247-283).
struct JobError : std::runtime_error {
  JobError(const std::string& msg, std::int64_t slice)
      : std::runtime_error(msg + " (slice " + std::to_string(slice) + ")"), slice_id(slice) {}
  std::int64_t slice_id;
};

struct AmplitudeOutput {
  std::vector<std::pair<std::string, cdouble>> amplitudes;
  std::vector<std::int64_t> slice_ids;
  std::uint64_t total_flops = 0;
};
// run_amplitudes (src/engine.cpp:300-378) for closed plans.
AmplitudeOutput run_amplitudes(Engine& e, const std::vector<std::string>& bitstrings, Fraction f, std::uint64_t seed);

// Many x1 draws in one contraction (GPU batching of amplitude_batch): the
// plan with the x1 qubits that vary across draws opened as well -- same
// order and cut, every draw's 2^|open| amplitudes are entries of the wider
// batch.  widen_plan annotates it; amplitude_batches runs an engine built
// on it once and gathers each draw's (bitstring, amplitude) list in the
// reference's order (src/sampler.cpp:111-120).
ContractionPlan widen_plan(const Circuit& c, const ContractionPlan& plan, const std::vector<int>& extra_open);
std::vector<std::vector<std::pair<std::string, cdouble>>> amplitude_batches(
    Engine& wide, const std::vector<int>& base_open, const std::vector<std::vector<int>>& x1_list,
    const std::vector<std::int64_t>& slice_ids, bool with_bitstrings = true);
// Same, flat buffers: x1_list nx1 x n ints; writes nx1 x 2^|base| (re, im)
// and, if bits_out, the bitstrings (n chars each) in the same order.
// Pipelined form of amplitude_batches_into: submit enqueues the contraction
// and the D2H of its batch into staging slot `slot` (0/1) and returns;
// collect waits for that slot and gathers the per-draw amplitudes.  The
// draw list passed to collect must be the one given to submit.
void amplitude_batches_submit(Engine& wide, const std::vector<int>& base_open, const int* x1_list, std::size_t nx1,
                              const std::vector<std::int64_t>& slice_ids, int slot);
void amplitude_batches_collect(Engine& wide, const std::vector<int>& base_open, const int* x1_list, std::size_t nx1,
                               int slot, double* amps_out, char* bits_out);
void amplitude_batches_into(Engine& wide, const std::vector<int>& base_open, const int* x1_list, std::size_t nx1,
                            const std::vector<std::int64_t>& slice_ids, double* amps_out, char* bits_out);

}  // namespace qsg
