/*
 * qsg.h -- C ABI of the B200-native sliced tensor-network amplitude path.
 *
 * The reference (qsim, /root/reference/proj) is a header-only C++ API with
 * no FFI; these entry points are the plain-C boundary a maintainer binds
 * from any host language (ctypes / cgo / JNI stubs in INTEGRATION.md).  Each
 * function names the reference interface it replaces (file:line relative to
 * the reference's proj/ directory).
 *
 * Conventions
 *   - Every function returns a qsg_status; on failure qsg_last_error()
 *     returns a thread-local message whose prefix matches the reference's
 *     exception message, and qsg_last_error_line() the 1-based circuit line
 *     for QSG_ERR_CIRCUIT (CircuitError::line, include/qsim/circuit.hpp:72).
 *   - complex64 data are interleaved float pairs (re, im), row-major, last
 *     axis fastest (qsim::Tensor, include/qsim/tensor.hpp:17-20).  complex128
 *     results are interleaved double pairs.
 *   - Variable-length text outputs use (buf, cap, *len): *len receives the
 *     full length; the text is copied (NUL-terminated) when cap > *len.
 *   - "host" pointers are CPU memory; "dev" pointers are CUDA device memory.
 *   - There is no CPU fallback: functions that compute need a CUDA device
 *     and return QSG_ERR_CUDA without one.
 */
#ifndef QSG_H_
#define QSG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum qsg_status {
  QSG_OK = 0,
  QSG_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument                 */
  QSG_ERR_LENGTH = 2,           /* std::length_error (volume overflow)   */
  QSG_ERR_OUT_OF_RANGE = 3,     /* std::out_of_range (slice id, index)   */
  QSG_ERR_RUNTIME = 4,          /* std::runtime_error                    */
  QSG_ERR_CUDA = 5,             /* CUDA runtime failure / no device      */
  QSG_ERR_OOM = 6,              /* device memory exhausted               */
  QSG_ERR_CIRCUIT = 7           /* qsim::CircuitError (parse/validation) */
} qsg_status;

const char* qsg_last_error(void);
int qsg_last_error_line(void);
/* Slice of a failed job (qsg_run_amplitudes): the lowest failing task's
 * slice id, also appended to the message as " (slice N)" -- the reference's
 * JobError (include/qsim/engine.hpp:81-84, src/engine.cpp:38-39, 247-283).
 * -1 when the last error was not attributed to a slice. */
int64_t qsg_last_error_slice(void);
const char* qsg_version(void);
int qsg_device_count(int* count);

/* ---------------------------------------------------------------------------
 * Host-side model (bit-exact with the reference)
 * ------------------------------------------------------------------------- */

/* splitmix64 stream derivation; qsim::mix_seed, include/qsim/types.hpp:25-30 */
uint64_t qsg_mix_seed(uint64_t seed, uint64_t stream);

/* Eq.(1) flops 8*sqrt(v0*v1*v2); qsim::flop_count, include/qsim/contraction.hpp:46-56 */
int qsg_flop_count(uint64_t v0, uint64_t v1, uint64_t v2, uint64_t* flops);

/* serialize_circuit(generate_rqc(...)); src/circuit.cpp:243-294, :206-220 */
int qsg_generate_rqc(int rows, int cols, int m, uint64_t seed, int t_only_first, char* buf, int64_t cap,
                     int64_t* len);

/* generate_rqc on a masked grid (no reference counterpart; its generator is
 * rectangle-only, src/circuit.cpp:227-241): mask = rows*cols '0'/'1' chars;
 * CZ layouts keep only active-active edges, inactive cells get only the
 * cycle-0 and final H.  qsg_bristlecone_mask: the 11x12 diamond with 72,
 * 70 or 60 active cells (SURVEY 8d construction). */
int qsg_generate_rqc_masked(int rows, int cols, const char* mask, int m, uint64_t seed, int t_only_first, char* buf,
                            int64_t cap, int64_t* len);
int qsg_bristlecone_mask(int active, char* buf, int64_t cap, int64_t* len);

/* serialize_circuit(parse_circuit(text)); src/circuit.cpp:128-220 */
int qsg_canonical_circuit(const char* text, char* buf, int64_t cap, int64_t* len);

/* rows, cols, qubits, cycles of parse_circuit(text) */
int qsg_circuit_info(const char* text, int* rows, int* cols, int* qubits, int* cycles);

/* Annotated plan JSON (plan_to_json).  kind: 0 = plan JSON in plan_text
 * (plan_from_json, src/plan.cpp:508-532), 1 = reference_plan_7x7
 * (src/plan.cpp:556-633), 2 = greedy plan_contraction(budget)
 * (src/plan.cpp:299-353).  open = open output qubits (fold_shape). */
int qsg_plan_json(const char* circuit_text, const int* open, int nopen, int kind, const char* plan_text,
                  int64_t budget, char* buf, int64_t cap, int64_t* len);

/* fold_worldlines (+ apply_cut when plan_text is non-empty) as concatenated
 * QTNS tensor dumps (include/qsim/tensor_io.hpp:12-41), node order 0..n-1.
 * out_bits: n entries, -1 = open.  src/network.cpp:106-149, src/plan.cpp:89-115 */
int qsg_fold_qtns(const char* circuit_text, const int* out_bits, int n, const char* plan_text, int64_t slice_id,
                  char* buf, int64_t cap, int64_t* len);

/* select_slices; src/engine.cpp:285-298.  out: num entries */
int qsg_select_slices(int64_t num, int64_t den, int64_t num_slices, uint64_t seed, int64_t* out);

/* x1 for sampling task `index`: mt19937_64(mix_seed(seed, index)), one bit
 * per closed qubit, -1 on open qubits (src/sampler.cpp:70-82, 155-157). */
int qsg_draw_x1(int n, const int* open, int nopen, uint64_t seed, uint64_t index, int* x1_out);

/* ---------------------------------------------------------------------------
 * Kernels on device memory (stream-ordered, asynchronous)
 * ------------------------------------------------------------------------- */

/* K1: out[i_0..i_{r-1}] = in[base + sum_j i_j * istride[j]], out dense.
 * Replaces qsim::transpose (include/qsim/tensor.hpp:135) and the copies of
 * slice_axis/apply_cut (tensor.hpp:236, src/plan.cpp:89). */
int qsg_permute_dev(const void* in_dev, int64_t base, void* out_dev, int rank, const int64_t* extent,
                    const int64_t* istride, void* stream);

/* K2: C[m][n] = A x B, complex64, FP32 accumulate; trans_a: A is [k][m];
 * trans_b: B is [n][k].  The GEMM of qsim::contract_ttgt
 * (include/qsim/contraction.hpp:208-214). */
int qsg_cgemm_dev(const void* a_dev, const void* b_dev, void* c_dev, int64_t m, int64_t n, int64_t k, int trans_a,
                  int trans_b, void* stream);

/* K2 on the tcgen05 tensor cores at FP32-level accuracy: CTA-pair 3xFP16
 * with power-of-two operand scaling when m % 256 == 0 (the production
 * path), 3xTF32 otherwise (QSG_TC_PREC=tf32 forces it).  Requires
 * m % 128 == 0, 2n % 32 == 0, k % 16 == 0, A row-major.
 * qsg_cgemm_tc_workspace_bytes returns the device scratch the call needs
 * (operand maxima, K-sync counters, B / A fp16 planes), or -1 for an
 * ineligible shape.  qsg_cgemm_tc_dev is stream-ordered and asynchronous:
 * no allocation, no synchronisation; the caller owns `workspace_dev`
 * (>= the returned size, reusable once the call has completed on `stream`).
 * QSG_ERR_INVALID_ARGUMENT for an ineligible shape or a short workspace. */
int64_t qsg_cgemm_tc_workspace_bytes(int64_t m, int64_t n, int64_t k, int trans_b);
int qsg_cgemm_tc_dev(const void* a_dev, const void* b_dev, void* c_dev, int64_t m, int64_t n, int64_t k, int trans_b,
                     void* workspace_dev, int64_t workspace_bytes, void* stream);

/* K3: acc[i] += double(fin[i]) * 2^log_scale for i < count (complex128
 * acc), and per_slice[i] = that contribution when per_slice_dev is not NULL.
 * The per-slice accumulation of batch_amplitudes (src/sampler.cpp:28-34).
 * Stream-ordered and asynchronous (log_scale is passed by value). */
int qsg_accumulate_dev(const void* fin_dev, double log_scale, int64_t count, void* acc_dev, void* per_slice_dev,
                       void* stream);

/* ---------------------------------------------------------------------------
 * Tensor operations on host buffers, computed on the GPU (synchronous)
 * ------------------------------------------------------------------------- */

/* qsim::transpose (include/qsim/tensor.hpp:135-197); perm[i] = input axis
 * placed at output position i.  Bit-identical to the reference. */
int qsg_transpose(int rank, const int64_t* dims, const float* in_host, const int* perm, float* out_host);

/* qsim::contract_ttgt (include/qsim/contraction.hpp:186-226) followed, when
 * normalize != 0, by normalize_inplace (tensor.hpp:209) as execute_slice
 * does (src/engine.cpp:227-233).  Labels are integers; contracted = shared
 * labels; the output is written in out_labels order. */
int qsg_contract(int lrank, const int* llab, const int64_t* ldims, const float* ldata, double lscale, int rrank,
                 const int* rlab, const int64_t* rdims, const float* rdata, double rscale, int orank,
                 const int* olab, float* out, double* oscale, uint64_t* flops, int normalize);

/* normalize_inplace (include/qsim/tensor.hpp:209-224) on a host buffer.
 * *log_scale is updated; *nonzero = 0 for an all-zero tensor (untouched). */
int qsg_normalize(float* data_host, int64_t count, double* log_scale, int* nonzero);

/* ---------------------------------------------------------------------------
 * Engine: the sliced contraction path (execute_slice / amplitude_batch /
 * run_amplitudes) on one GPU
 * ------------------------------------------------------------------------- */

typedef struct qsg_engine qsg_engine;

enum { QSG_ENGINE_PROFILE = 1, QSG_ENGINE_NO_TENSOR_CORES = 2 };

/* Parses the circuit, loads + annotates the plan (kind as qsg_plan_json;
 * the open qubits come from the plan JSON, or reference_open_qubits_7x7 for
 * kind 1, or `open` for kind 2), and compiles the device program. */
int qsg_engine_create(const char* circuit_text, int kind, const char* plan_text, const int* open, int nopen,
                      int device, int flags, qsg_engine** out);
/* As qsg_engine_create, with the reference's ExecOptions (include/qsim/
 * engine.hpp:22-27): a contraction whose working set exceeds memory_budget
 * bytes (0 = no limit) is decomposed into pieces (src/plan.cpp:355-472) and
 * run through a pipeline of pipeline_depth pieces in flight
 * (src/engine.cpp:52-180); its tensors live in pinned host memory and only
 * the pieces occupy the device.  Error "indivisible contraction still over
 * budget" (runtime error) as the reference.  memory_budget -1: automatic --
 * everything in HBM if the program fits the device's free memory, else the
 * largest power-of-two budget whose out-of-core program fits. */
int qsg_engine_create_ex(const char* circuit_text, int kind, const char* plan_text, const int* open, int nopen,
                         int device, int flags, int64_t memory_budget, int pipeline_depth, qsg_engine** out);
int qsg_engine_destroy(qsg_engine* e);

/* Compiles the device program for (circuit, plan) WITHOUT a device and
 * returns its listing (ops, shapes, GEMM path, arena bytes) -- for planning
 * and CPU-side checks.  Arguments as qsg_engine_create. */
int qsg_program_listing(const char* circuit_text, int kind, const char* plan_text, const int* open, int nopen,
                        int flags, char* buf, int64_t cap, int64_t* len);
/* As qsg_program_listing with a memory budget (out-of-core placement);
 * memory_budget -1 = automatic for a device of device_memory bytes. */
int qsg_program_listing_ex(const char* circuit_text, int kind, const char* plan_text, const int* open, int nopen,
                           int flags, int64_t memory_budget, int64_t device_memory, char* buf, int64_t cap,
                           int64_t* len);

typedef struct qsg_engine_info {
  int64_t num_qubits, num_slices, batch_size, num_steps, max_rank;
  int64_t peak_memory;        /* reference annotate_plan prediction */
  int64_t arena_bytes;        /* this engine's static device arena   */
  int64_t node_bytes;         /* H2D bytes per prepare               */
  uint64_t flops_per_slice;   /* Eq.(1), exact                      */
  int64_t num_ops;
} qsg_engine_info;
int qsg_engine_get_info(qsg_engine* e, qsg_engine_info* info);
int qsg_engine_plan_json(qsg_engine* e, char* buf, int64_t cap, int64_t* len);
int qsg_engine_describe(qsg_engine* e, char* buf, int64_t cap, int64_t* len);
int qsg_engine_open_qubits(qsg_engine* e, int* out /* num_open entries */);

/* Fold for x1 (n entries, -1 exactly on the open qubits) and upload. */
int qsg_engine_prepare(qsg_engine* e, const int* x1_bits, int n, int64_t* h2d_bytes);
/* Node region (the open fold: info.node_bytes of complex64, engine order).
 * A new instance of the same circuit layout (same grid, depth and CZ
 * pattern; e.g. another single-qubit gate draw) reuses the engine's plan,
 * arena and kernels: fold it on the host (qsg_engine_fold_nodes; fails if the
 * fold shape differs), then qsg_engine_load_nodes (async H2D on the engine
 * stream; pass pinned memory to overlap, keep it alive until the next
 * synchronize).  This is the reference's per-circuit tensor construction,
 * fold_worldlines at src/network.cpp:106-155, with the upload split out.
 * qsg_engine_export_nodes copies the resident region back (synchronises). */
int qsg_engine_fold_nodes(qsg_engine* e, const char* circuit_text, void* host_nodes, int64_t bytes);
int qsg_engine_load_nodes(qsg_engine* e, const void* host_nodes, int64_t bytes);
int qsg_engine_export_nodes(qsg_engine* e, void* host_nodes, int64_t bytes);
/* Run slices (async, engine stream).  reset: zero the batch accumulator;
 * per_slice: keep each slice's contribution (appended after the previous
 * run's rows when reset = 0 and that run kept rows, so a batch split over
 * several runs keeps one row per slice in run order). */
int qsg_engine_run(qsg_engine* e, const int64_t* slice_ids, int64_t k, int reset, int per_slice);
/* Batch amplitudes (batch_size complex128) and, if non-null, per-slice
 * contributions (k x batch_size complex128); synchronises. */
int qsg_engine_results(qsg_engine* e, double* amps_host, double* per_slice_host);
int qsg_engine_stream(qsg_engine* e, void** stream);
int qsg_engine_synchronize(qsg_engine* e);
int qsg_engine_launches(qsg_engine* e, int64_t* launches);
/* Rows (slices) of per-slice contributions kept by the engine's last run
 * (0 when that run -- including the internal runs of qsg_amplitude_batch,
 * qsg_run_amplitudes, qsg_sample -- did not keep them); per_slice_host of
 * qsg_engine_results receives rows x batch_size complex128 values. */
int qsg_engine_per_slice_rows(qsg_engine* e, int64_t* rows);

typedef struct qsg_op_profile {
  int32_t kind;  /* 0 permute, 1 gemm, 2 accumulate */
  int32_t step;
  int64_t m, n, k;
  uint64_t flops;
  int64_t bytes;
  double ms_total;
  int64_t executions;
  int32_t tensor_cores;
  int32_t pad;
} qsg_op_profile;
int qsg_engine_profile(qsg_engine* e, qsg_op_profile* out, int cap, int* count);
/* Turns per-op CUDA-event timing on/off (off by default unless created with
 * QSG_ENGINE_PROFILE; timing syncs the stream once per slice). */
int qsg_engine_set_profile(qsg_engine* e, int on);
int qsg_engine_reset_profile(qsg_engine* e);

/* amplitude_batch (src/sampler.cpp:111-120) in one call on host buffers:
 * amps: batch_size complex128; bitstrings (nullable): batch_size * n chars. */
int qsg_amplitude_batch(qsg_engine* e, const int* x1_bits, int n, const int64_t* slice_ids, int64_t k,
                        double* amps_host, char* bitstrings_host);

/* GPU batching of many x1 draws (no reference counterpart; it serves
 * amplitude_batch, src/sampler.cpp:111-120, for a list of draws).
 * qsg_widen_plan: the plan (kind as qsg_plan_json) with extra qubits opened
 * -- same order and cut -- as JSON; build the engine from it (kind 0).
 * qsg_amplitude_batches: one contraction on that engine for nx1 draws (each
 * n entries, -1 exactly on the nbase base open qubits; they may differ only
 * on qubits the widened plan opened).  Writes nx1 x 2^nbase amplitudes
 * (re, im) and bitstrings, each draw in the reference's batch order. */
int qsg_widen_plan(const char* circuit_text, int kind, const char* plan_text, const int* open, int nopen,
                   const int* extra_open, int nextra, char* buf, int64_t cap, int64_t* len);
/* Contraction-tree rewrite (no reference counterpart; opt-in planner pass
 * over plans loaded like qsg_plan_json, src/plan.cpp:508-552): a step output
 * T = A x B read once by U = T x C becomes W = B x C, U = A x W (or A, B
 * swapped) when that cuts the pair's Eq.(1) flops by >= 25% without a larger
 * intermediate, to a fixed point.  Same cut, slices and amplitudes (up to
 * rounding); JSON out, *rewrites = number of rewrites. */
int qsg_reassociate_plan(const char* circuit_text, int kind, const char* plan_text, const int* open, int nopen,
                         char* buf, int64_t cap, int64_t* len, int* rewrites);
int qsg_amplitude_batches(qsg_engine* e, const int* base_open, int nbase, const int* x1_list, int nx1, int n,
                          const int64_t* slice_ids, int64_t k, double* amps_host, char* bitstrings_host);
/* Pipelined qsg_amplitude_batches: _submit validates the draws, enqueues the
 * contraction and the D2H of its batch into pinned staging slot `slot`
 * (0 or 1) on the engine stream and returns at once; _collect waits for
 * that slot and writes the per-draw amplitudes (and bitstrings, if non-NULL)
 * exactly as qsg_amplitude_batches does.  Pass collect the same draw list.
 * With two slots the host gathers batch i while the GPU runs batch i + 1. */
int qsg_amplitude_batches_submit(qsg_engine* e, const int* base_open, int nbase, const int* x1_list, int nx1, int n,
                                 const int64_t* slice_ids, int64_t k, int slot);
int qsg_amplitude_batches_collect(qsg_engine* e, const int* base_open, int nbase, const int* x1_list, int nx1, int n,
                                  int slot, double* amps_host, char* bitstrings_host);

/* run_amplitudes (src/engine.cpp:300-378) for closed plans: nb bitstrings
 * of n chars, fraction num/den (den <= 0: all slices), seed.  out: nb
 * complex128; ids_out (nullable): the k slice ids; flops: Eq.(1) total. */
int qsg_run_amplitudes(qsg_engine* e, const char* bitstrings, int nb, int n, int64_t frac_num, int64_t frac_den,
                       uint64_t seed, double* out, int64_t* ids_out, uint64_t* flops);

/* ---------------------------------------------------------------------------
 * Sampling and XEB on device amplitude batches (SURVEY 8f "next")
 * ------------------------------------------------------------------------- */

typedef struct qsg_sample_stats {
  uint64_t x1_draws, redraws, cap_hits, candidates;
  int64_t exact_count, uniform_count;
} qsg_sample_stats;

typedef struct qsg_xeb_report {
  int32_t n, hog_available;
  int64_t size, zero_excluded;
  double mean_log_prob, cross_entropy, fidelity_estimate, hog_fraction;
} qsg_xeb_report;

/* sample() (src/sampler.cpp:122-178; amplitude_fraction_mode = 1 is
 * sample_amplitude_fraction, :180-185): frugal rejection sampling with x1/x2
 * recycling over the engine's open qubits.  Fraction frac_num/frac_den
 * (den <= 0: all slices), rejection cap kappa, seed.  Outputs: M bitstrings
 * of n chars (concatenated), M probabilities (-1 = uniform share), stats,
 * and the self-XEB of the emitted probabilities. */
int qsg_sample(qsg_engine* e, int64_t num_samples, int64_t frac_num, int64_t frac_den, int amplitude_fraction_mode,
               double rejection_cap, uint64_t seed, char* bitstrings_out, double* probs_out, qsg_sample_stats* stats,
               qsg_xeb_report* self_xeb);

/* xeb_score (src/sampler.cpp:187-215): cross entropy -<log p>, fidelity
 * 2^n <p> - 1 over p > 0 (zeros excluded and counted), HOG fraction above
 * `hog_median` when has_median != 0. */
int qsg_xeb_score(int n, const double* probs, int64_t count, int has_median, double hog_median, qsg_xeb_report* out);

#ifdef __cplusplus
}
#endif

#endif /* QSG_H_ */
