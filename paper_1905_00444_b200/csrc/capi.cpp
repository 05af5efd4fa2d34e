// extern "C" boundary (include/qsg.h).  Translates C++ exceptions into
// qsg_status codes + a thread-local message (the reference's exception
// types and message prefixes, see include/qsg.h), and implements the
// host-buffer conveniences on top of the device kernels and the engine.
#include "../../include/qsg.h"

#include <algorithm>
#include <cstring>
#include <memory>
#include <new>
#include <sstream>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "device/kernels.hpp"
#include "device/kernels_tc.hpp"
#include "engine/engine.hpp"
#include "engine/sampler.hpp"
#include "host/qsg_host.hpp"

struct qsg_engine {
  std::unique_ptr<qsg::Engine> impl;
};

namespace {

thread_local std::string g_err;
thread_local int g_err_line = 0;
thread_local std::int64_t g_err_slice = -1;

template <class F>
int guarded(F&& f) {
  g_err_slice = -1;
  try {
    f();
    return QSG_OK;
  } catch (const qsg::JobError& e) {
    g_err = e.what();
    g_err_slice = e.slice_id;
    return QSG_ERR_RUNTIME;
  } catch (const qsg::CircuitError& e) {
    g_err = e.what();
    g_err_line = e.line;
    return QSG_ERR_CIRCUIT;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return QSG_ERR_INVALID_ARGUMENT;
  } catch (const std::length_error& e) {
    g_err = e.what();
    return QSG_ERR_LENGTH;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return QSG_ERR_OUT_OF_RANGE;
  } catch (const std::bad_alloc& e) {
    g_err = std::string("host allocation failed: ") + e.what();
    return QSG_ERR_OOM;
  } catch (const std::runtime_error& e) {
    g_err = e.what();
    if (g_err.rfind("CUDA error", 0) == 0) {
      return g_err.find("out of memory") != std::string::npos ? QSG_ERR_OOM : QSG_ERR_CUDA;
    }
    return QSG_ERR_RUNTIME;
  } catch (const std::exception& e) {
    g_err = e.what();
    return QSG_ERR_RUNTIME;
  }
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

void put_text(const std::string& s, char* buf, std::int64_t cap, std::int64_t* len) {
  if (len) *len = static_cast<std::int64_t>(s.size());
  if (buf && cap > static_cast<std::int64_t>(s.size())) {
    std::memcpy(buf, s.data(), s.size());
    buf[s.size()] = '\0';
  }
}

// RAII device buffer.
struct DevBuf {
  void* p = nullptr;
  explicit DevBuf(std::size_t bytes) { cuda_check(cudaMalloc(&p, std::max<std::size_t>(bytes, 16)), "cudaMalloc"); }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

std::vector<std::int64_t> strides_of(const std::vector<std::int64_t>& dims) {
  std::vector<std::int64_t> s(dims.size());
  std::int64_t acc = 1;
  for (std::size_t i = dims.size(); i-- > 0;) {
    s[i] = acc;
    acc *= dims[i];
  }
  return s;
}

std::int64_t volume_of(const std::vector<std::int64_t>& dims) {
  std::int64_t v = 1;
  for (auto d : dims) {
    if (d < 1) throw std::invalid_argument("tensor: dims must be >= 1");
    v *= d;
  }
  return v;
}

void require_device() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n < 1)
    throw std::runtime_error("CUDA error in device query: no CUDA device (this library has no CPU fallback)");
}

qsg::ContractionPlan make_plan(const qsg::Circuit& c, int kind, const char* plan_text, const std::vector<int>& open,
                               std::int64_t budget) {
  if (kind == 0) {
    const std::string text = plan_text ? plan_text : "";
    return qsg::plan_from_json(text, qsg::fold_shape(c, qsg::plan_json_open_qubits(text)));
  }
  if (kind == 1) return qsg::reference_plan_7x7(qsg::fold_shape(c, qsg::reference_open_qubits_7x7()));
  if (kind == 2) {
    qsg::PlanOptions o;
    o.memory_budget = budget;
    return qsg::plan_contraction(qsg::fold_shape(c, open), o);
  }
  throw std::invalid_argument("plan kind must be 0 (json), 1 (reference 7x7) or 2 (greedy)");
}

void write_qtns(std::ostringstream& os, const qsg::HostTensor& t) {
  auto put = [&](const void* p, std::size_t n) { os.write(static_cast<const char*>(p), static_cast<std::streamsize>(n)); };
  os.write("QTNS", 4);
  const std::uint32_t ver = 1, rank = static_cast<std::uint32_t>(t.rank());
  put(&ver, 4);
  put(&rank, 4);
  for (int i = 0; i < t.rank(); ++i) {
    const auto& l = t.labels[static_cast<std::size_t>(i)];
    const auto len = static_cast<std::uint16_t>(l.size());
    put(&len, 2);
    put(l.data(), len);
    const auto d = static_cast<std::uint64_t>(t.dims[static_cast<std::size_t>(i)]);
    put(&d, 8);
  }
  put(&t.log_scale, 8);
  put(t.data.data(), t.data.size() * sizeof(qsg::cfloat));
}

}  // namespace

extern "C" {

const char* qsg_last_error(void) { return g_err.c_str(); }
int qsg_last_error_line(void) { return g_err_line; }
int64_t qsg_last_error_slice(void) { return g_err_slice; }
const char* qsg_version(void) { return "qsg 0.1 (sm_100a)"; }

int qsg_device_count(int* count) {
  return guarded([&] {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) n = 0;
    *count = n;
  });
}

uint64_t qsg_mix_seed(uint64_t seed, uint64_t stream) { return qsg::mix_seed(seed, stream); }

int qsg_flop_count(uint64_t v0, uint64_t v1, uint64_t v2, uint64_t* flops) {
  return guarded([&] { *flops = qsg::flop_count(v0, v1, v2); });
}

int qsg_generate_rqc(int rows, int cols, int m, uint64_t seed, int t_only_first, char* buf, int64_t cap, int64_t* len) {
  return guarded([&] {
    put_text(qsg::serialize_circuit(qsg::generate_rqc(rows, cols, m, seed, t_only_first != 0)), buf, cap, len);
  });
}

int qsg_generate_rqc_masked(int rows, int cols, const char* mask, int m, uint64_t seed, int t_only_first, char* buf,
                            int64_t cap, int64_t* len) {
  return guarded([&] {
    put_text(qsg::serialize_circuit(qsg::generate_rqc_masked(rows, cols, mask ? mask : "", m, seed, t_only_first != 0)),
             buf, cap, len);
  });
}

int qsg_bristlecone_mask(int active, char* buf, int64_t cap, int64_t* len) {
  return guarded([&] { put_text(qsg::bristlecone_mask(active), buf, cap, len); });
}

int qsg_canonical_circuit(const char* text, char* buf, int64_t cap, int64_t* len) {
  return guarded([&] { put_text(qsg::serialize_circuit(qsg::parse_circuit(text)), buf, cap, len); });
}

int qsg_circuit_info(const char* text, int* rows, int* cols, int* qubits, int* cycles) {
  return guarded([&] {
    const qsg::Circuit c = qsg::parse_circuit(text);
    *rows = c.rows;
    *cols = c.cols;
    *qubits = c.num_qubits();
    *cycles = c.cycles();
  });
}

int qsg_plan_json(const char* circuit_text, const int* open, int nopen, int kind, const char* plan_text, int64_t budget,
                  char* buf, int64_t cap, int64_t* len) {
  return guarded([&] {
    const qsg::Circuit c = qsg::parse_circuit(circuit_text);
    const std::vector<int> o(open, open + nopen);
    put_text(qsg::plan_to_json(make_plan(c, kind, plan_text, o, budget)), buf, cap, len);
  });
}

int qsg_fold_qtns(const char* circuit_text, const int* out_bits, int n, const char* plan_text, int64_t slice_id,
                  char* buf, int64_t cap, int64_t* len) {
  return guarded([&] {
    const qsg::Circuit c = qsg::parse_circuit(circuit_text);
    qsg::GridNetwork net = qsg::fold_worldlines(c, std::vector<int>(out_bits, out_bits + n));
    if (plan_text && plan_text[0]) {
      const qsg::ContractionPlan plan = qsg::plan_from_json(plan_text, net.shape());
      net = qsg::apply_cut(net, plan.cut, slice_id);
    }
    std::ostringstream os;
    for (const auto& t : net.nodes) write_qtns(os, t);
    const std::string s = os.str();
    *len = static_cast<std::int64_t>(s.size());
    if (buf && cap >= *len) std::memcpy(buf, s.data(), s.size());
  });
}

int qsg_select_slices(int64_t num, int64_t den, int64_t num_slices, uint64_t seed, int64_t* out) {
  return guarded([&] {
    const auto ids = qsg::select_slices(qsg::Fraction{num, den}, num_slices, seed);
    std::copy(ids.begin(), ids.end(), out);
  });
}

int qsg_draw_x1(int n, const int* open, int nopen, uint64_t seed, uint64_t index, int* x1_out) {
  return guarded([&] {
    const auto x1 = qsg::draw_x1(n, std::vector<int>(open, open + nopen), seed, index);
    std::copy(x1.begin(), x1.end(), x1_out);
  });
}

int qsg_permute_dev(const void* in_dev, int64_t base, void* out_dev, int rank, const int64_t* extent,
                    const int64_t* istride, void* stream) {
  return guarded([&] {
    cuda_check(qsg::dev::permute(in_dev, base, out_dev, rank, extent, istride, static_cast<cudaStream_t>(stream)),
               "permute");
  });
}

int qsg_cgemm_dev(const void* a_dev, const void* b_dev, void* c_dev, int64_t m, int64_t n, int64_t k, int trans_a,
                  int trans_b, void* stream) {
  return guarded([&] {
    qsg::dev::GemmArgs g{};
    g.a = a_dev;
    g.b = b_dev;
    g.c = c_dev;
    g.m = m;
    g.n = n;
    g.k = k;
    g.trans_a = trans_a != 0;
    g.trans_b = trans_b != 0;
    cuda_check(qsg::dev::cgemm(g, static_cast<cudaStream_t>(stream)), "cgemm");
  });
}

int64_t qsg_cgemm_tc_workspace_bytes(int64_t m, int64_t n, int64_t k, int trans_b) {
  if (m <= 0 || n <= 0 || k <= 0 || !qsg::dev::cgemm_tc_supported(m, n, k, false, trans_b != 0)) return -1;
  return qsg::dev::cgemm_tc_workspace_bytes(m, n, k, false, trans_b != 0);
}

int qsg_cgemm_tc_dev(const void* a_dev, const void* b_dev, void* c_dev, int64_t m, int64_t n, int64_t k, int trans_b,
                     void* workspace_dev, int64_t workspace_bytes, void* stream) {
  return guarded([&] {
    if (!qsg::dev::cgemm_tc_supported(m, n, k, false, trans_b != 0))
      throw std::invalid_argument("cgemm_tc: shape not eligible for the tensor-core path");
    const std::int64_t ws = qsg::dev::cgemm_tc_workspace_bytes(m, n, k, false, trans_b != 0);
    if (workspace_dev == nullptr || workspace_bytes < ws)
      throw std::invalid_argument("cgemm_tc: workspace smaller than qsg_cgemm_tc_workspace_bytes()");
    qsg::dev::GemmArgs g{};
    g.a = a_dev;
    g.b = b_dev;
    g.c = c_dev;
    g.m = m;
    g.n = n;
    g.k = k;
    g.trans_b = trans_b != 0;
    g.workspace = workspace_dev;
    g.workspace_bytes = workspace_bytes;
    cuda_check(qsg::dev::cgemm_tc(g, static_cast<cudaStream_t>(stream)), "cgemm_tc");
  });
}

int qsg_accumulate_dev(const void* fin_dev, double log_scale, int64_t count, void* acc_dev, void* per_slice_dev,
                       void* stream) {
  return guarded([&] {
    if (count < 0) throw std::invalid_argument("accumulate: negative count");
    cuda_check(qsg::dev::accumulate(fin_dev, log_scale, count, acc_dev, per_slice_dev, static_cast<cudaStream_t>(stream)),
               "accumulate");
  });
}

int qsg_transpose(int rank, const int64_t* dims, const float* in_host, const int* perm, float* out_host) {
  return guarded([&] {
    std::vector<std::int64_t> d(dims, dims + rank);
    std::vector<char> seen(static_cast<std::size_t>(rank), 0);
    for (int i = 0; i < rank; ++i) {
      if (perm[i] < 0 || perm[i] >= rank) throw std::invalid_argument("tensor: no label (axis out of range)");
      if (seen[static_cast<std::size_t>(perm[i])]) throw std::invalid_argument("transpose: order is not a permutation");
      seen[static_cast<std::size_t>(perm[i])] = 1;
    }
    const std::int64_t vol = volume_of(d);
    require_device();
    const auto st = strides_of(d);
    std::vector<std::int64_t> ext(static_cast<std::size_t>(rank)), istr(static_cast<std::size_t>(rank));
    for (int i = 0; i < rank; ++i) {
      ext[static_cast<std::size_t>(i)] = d[static_cast<std::size_t>(perm[i])];
      istr[static_cast<std::size_t>(i)] = st[static_cast<std::size_t>(perm[i])];
    }
    DevBuf a(static_cast<std::size_t>(vol) * 8), b(static_cast<std::size_t>(vol) * 8);
    cuda_check(cudaMemcpy(a.p, in_host, static_cast<std::size_t>(vol) * 8, cudaMemcpyHostToDevice), "H2D");
    cuda_check(qsg::dev::permute(a.p, 0, b.p, rank, ext.data(), istr.data(), nullptr), "permute");
    cuda_check(cudaMemcpy(out_host, b.p, static_cast<std::size_t>(vol) * 8, cudaMemcpyDeviceToHost), "D2H");
  });
}

int qsg_contract(int lrank, const int* llab, const int64_t* ldims, const float* ldata, double lscale, int rrank,
                 const int* rlab, const int64_t* rdims, const float* rdata, double rscale, int orank, const int* olab,
                 float* out, double* oscale, uint64_t* flops, int normalize) {
  return guarded([&] {
    std::vector<int> L(llab, llab + lrank), R(rlab, rlab + rrank);
    std::vector<std::int64_t> Ld(ldims, ldims + lrank), Rd(rdims, rdims + rrank);
    auto find = [](const std::vector<int>& v, int x) { return static_cast<int>(std::find(v.begin(), v.end(), x) - v.begin()); };
    for (const auto* v : {&L, &R}) {
      auto s = *v;
      std::sort(s.begin(), s.end());
      if (std::adjacent_find(s.begin(), s.end()) != s.end()) throw std::invalid_argument("tensor: duplicate label");
    }
    // contraction.hpp:65-93 (analyze) with the infer_spec contracted set.
    std::vector<int> con, lfree, rfree;
    std::int64_t m = 1, n = 1, k = 1;
    for (int i = 0; i < lrank; ++i) {
      const int j = find(R, L[static_cast<std::size_t>(i)]);
      if (j < rrank) {
        if (Ld[static_cast<std::size_t>(i)] != Rd[static_cast<std::size_t>(j)])
          throw std::invalid_argument("contract: extent mismatch on " + std::to_string(L[static_cast<std::size_t>(i)]));
        con.push_back(L[static_cast<std::size_t>(i)]);
        k *= Ld[static_cast<std::size_t>(i)];
      } else {
        lfree.push_back(L[static_cast<std::size_t>(i)]);
        m *= Ld[static_cast<std::size_t>(i)];
      }
    }
    for (int i = 0; i < rrank; ++i)
      if (find(L, R[static_cast<std::size_t>(i)]) >= lrank) {
        rfree.push_back(R[static_cast<std::size_t>(i)]);
        n *= Rd[static_cast<std::size_t>(i)];
      }
    constexpr std::int64_t kMax = std::int64_t{1} << 33;
    if (m * k > kMax || k * n > kMax || m * n > kMax) throw std::length_error("contract_ttgt: volume overflow");
    std::vector<int> natural = lfree;
    natural.insert(natural.end(), rfree.begin(), rfree.end());
    std::vector<int> want = orank > 0 ? std::vector<int>(olab, olab + orank) : natural;
    {
      auto a = want, b = natural;
      std::sort(a.begin(), a.end());
      std::sort(b.begin(), b.end());
      if (a != b) throw std::invalid_argument("transpose: order is not a permutation");
    }
    require_device();
    const std::int64_t vl = volume_of(Ld), vr = volume_of(Rd);
    const auto ls = strides_of(Ld), rs = strides_of(Rd);
    DevBuf dl(static_cast<std::size_t>(vl) * 8), dr(static_cast<std::size_t>(vr) * 8);
    DevBuf pl(static_cast<std::size_t>(vl) * 8), pr(static_cast<std::size_t>(vr) * 8);
    DevBuf dc(static_cast<std::size_t>(m * n) * 8), po(static_cast<std::size_t>(m * n) * 8);
    DevBuf meta(sizeof(qsg::dev::TMeta));
    cuda_check(cudaMemcpy(dl.p, ldata, static_cast<std::size_t>(vl) * 8, cudaMemcpyHostToDevice), "H2D");
    cuda_check(cudaMemcpy(dr.p, rdata, static_cast<std::size_t>(vr) * 8, cudaMemcpyHostToDevice), "H2D");
    cuda_check(cudaMemset(meta.p, 0, sizeof(qsg::dev::TMeta)), "memset");
    // L -> [lfree, con], R -> [con, rfree]  (contraction.hpp:193-203)
    std::vector<std::int64_t> ext, istr;
    for (int l : lfree) { ext.push_back(Ld[static_cast<std::size_t>(find(L, l))]); istr.push_back(ls[static_cast<std::size_t>(find(L, l))]); }
    for (int l : con) { ext.push_back(Ld[static_cast<std::size_t>(find(L, l))]); istr.push_back(ls[static_cast<std::size_t>(find(L, l))]); }
    cuda_check(qsg::dev::permute(dl.p, 0, pl.p, static_cast<int>(ext.size()), ext.data(), istr.data(), nullptr), "permute");
    ext.clear();
    istr.clear();
    for (int l : con) { ext.push_back(Rd[static_cast<std::size_t>(find(R, l))]); istr.push_back(rs[static_cast<std::size_t>(find(R, l))]); }
    for (int l : rfree) { ext.push_back(Rd[static_cast<std::size_t>(find(R, l))]); istr.push_back(rs[static_cast<std::size_t>(find(R, l))]); }
    cuda_check(qsg::dev::permute(dr.p, 0, pr.p, static_cast<int>(ext.size()), ext.data(), istr.data(), nullptr), "permute");
    qsg::dev::GemmArgs g{};
    g.a = pl.p;
    g.b = pr.p;
    g.c = dc.p;
    g.m = m;
    g.n = n;
    g.k = k;
    g.meta_c = meta.as<qsg::dev::TMeta>();
    const std::int64_t ws_bytes = qsg::dev::cgemm_workspace_bytes(m, n, k);
    std::unique_ptr<DevBuf> ws;
    if (ws_bytes > 0) {
      ws = std::make_unique<DevBuf>(static_cast<std::size_t>(ws_bytes));
      g.workspace = ws->p;
      g.workspace_bytes = ws_bytes;
    }
    cuda_check(qsg::dev::cgemm(g, nullptr), "cgemm");
    // Output permute to the requested order.
    void* result = dc.p;
    if (want != natural) {
      std::vector<std::int64_t> cd;
      for (int l : natural) cd.push_back(find(L, l) < lrank ? Ld[static_cast<std::size_t>(find(L, l))] : Rd[static_cast<std::size_t>(find(R, l))]);
      const auto cs = strides_of(cd);
      ext.clear();
      istr.clear();
      for (int l : want) {
        const auto j = static_cast<std::size_t>(find(natural, l));
        ext.push_back(cd[j]);
        istr.push_back(cs[j]);
      }
      cuda_check(qsg::dev::permute(dc.p, 0, po.p, static_cast<int>(ext.size()), ext.data(), istr.data(), nullptr), "permute");
      result = po.p;
    }
    double scale = lscale + rscale;
    if (normalize) {
      qsg::dev::TMeta h{};
      cuda_check(cudaMemcpy(&h, meta.p, sizeof h, cudaMemcpyDeviceToHost), "D2H");
      const int shift = qsg::dev::host_shift_from_maxsq(h.maxsq_bits);
      cuda_check(qsg::dev::scale_pow2(result, m * n, shift, nullptr), "scale");
      scale += shift;
    }
    cuda_check(cudaMemcpy(out, result, static_cast<std::size_t>(m * n) * 8, cudaMemcpyDeviceToHost), "D2H");
    *oscale = scale;
    *flops = qsg::flop_count(static_cast<std::uint64_t>(vl), static_cast<std::uint64_t>(vr), static_cast<std::uint64_t>(m * n));
  });
}

int qsg_normalize(float* data_host, int64_t count, double* log_scale, int* nonzero) {
  return guarded([&] {
    require_device();
    DevBuf d(static_cast<std::size_t>(count) * 8), meta(sizeof(qsg::dev::TMeta));
    cuda_check(cudaMemcpy(d.p, data_host, static_cast<std::size_t>(count) * 8, cudaMemcpyHostToDevice), "H2D");
    cuda_check(cudaMemset(meta.p, 0, sizeof(qsg::dev::TMeta)), "memset");
    cuda_check(qsg::dev::max_abs_sq(d.p, count, meta.as<qsg::dev::TMeta>(), nullptr), "max");
    qsg::dev::TMeta h{};
    cuda_check(cudaMemcpy(&h, meta.p, sizeof h, cudaMemcpyDeviceToHost), "D2H");
    *nonzero = h.maxsq_bits != 0;
    if (!*nonzero) return;
    const int shift = qsg::dev::host_shift_from_maxsq(h.maxsq_bits);
    if (shift == 0) return;
    cuda_check(qsg::dev::scale_pow2(d.p, count, shift, nullptr), "scale");
    cuda_check(cudaMemcpy(data_host, d.p, static_cast<std::size_t>(count) * 8, cudaMemcpyDeviceToHost), "D2H");
    *log_scale += shift;
  });
}

int qsg_engine_create(const char* circuit_text, int kind, const char* plan_text, const int* open, int nopen, int device,
                      int flags, qsg_engine** out) {
  return guarded([&] {
    require_device();
    const qsg::Circuit c = qsg::parse_circuit(circuit_text);
    const qsg::ContractionPlan plan = make_plan(c, kind, plan_text, std::vector<int>(open, open + nopen), 0);
    qsg::EngineOptions o;
    o.device = device;
    o.profile = (flags & QSG_ENGINE_PROFILE) != 0;
    o.tensor_cores = (flags & QSG_ENGINE_NO_TENSOR_CORES) == 0;
    auto e = std::make_unique<qsg_engine>();
    e->impl = std::make_unique<qsg::Engine>(c, plan, o);
    *out = e.release();
  });
}

int qsg_engine_create_ex(const char* circuit_text, int kind, const char* plan_text, const int* open, int nopen,
                         int device, int flags, int64_t memory_budget, int pipeline_depth, qsg_engine** out) {
  return guarded([&] {
    require_device();
    if (memory_budget < -1 || pipeline_depth < 1)
      throw std::invalid_argument("engine: memory_budget >= -1 (-1: automatic), pipeline_depth >= 1");
    const qsg::Circuit c = qsg::parse_circuit(circuit_text);
    const qsg::ContractionPlan plan = make_plan(c, kind, plan_text, std::vector<int>(open, open + nopen), 0);
    qsg::EngineOptions o;
    o.device = device;
    o.profile = (flags & QSG_ENGINE_PROFILE) != 0;
    o.tensor_cores = (flags & QSG_ENGINE_NO_TENSOR_CORES) == 0;
    o.memory_budget = memory_budget;
    o.pipeline_depth = pipeline_depth;
    auto e = std::make_unique<qsg_engine>();
    e->impl = std::make_unique<qsg::Engine>(c, plan, o);
    *out = e.release();
  });
}

int qsg_program_listing_ex(const char* circuit_text, int kind, const char* plan_text, const int* open, int nopen,
                           int flags, int64_t memory_budget, int64_t device_memory, char* buf, int64_t cap,
                           int64_t* len) {
  return guarded([&] {
    const qsg::Circuit c = qsg::parse_circuit(circuit_text);
    const qsg::ContractionPlan plan = make_plan(c, kind, plan_text, std::vector<int>(open, open + nopen), 0);
    qsg::EngineOptions o;
    o.compile_only = true;
    o.tensor_cores = (flags & QSG_ENGINE_NO_TENSOR_CORES) == 0;
    o.memory_budget = memory_budget;
    o.device_memory = device_memory;
    qsg::Engine e(c, plan, o);
    put_text(e.describe(), buf, cap, len);
  });
}

int qsg_program_listing(const char* circuit_text, int kind, const char* plan_text, const int* open, int nopen,
                        int flags, char* buf, int64_t cap, int64_t* len) {
  return guarded([&] {
    const qsg::Circuit c = qsg::parse_circuit(circuit_text);
    const qsg::ContractionPlan plan = make_plan(c, kind, plan_text, std::vector<int>(open, open + nopen), 0);
    qsg::EngineOptions o;
    o.compile_only = true;
    o.tensor_cores = (flags & QSG_ENGINE_NO_TENSOR_CORES) == 0;
    qsg::Engine e(c, plan, o);
    put_text(e.describe(), buf, cap, len);
  });
}

int qsg_engine_destroy(qsg_engine* e) {
  return guarded([&] { delete e; });
}

int qsg_engine_get_info(qsg_engine* e, qsg_engine_info* info) {
  return guarded([&] {
    const auto& p = e->impl->plan();
    info->num_qubits = e->impl->circuit().num_qubits();
    info->num_slices = p.num_slices;
    info->batch_size = e->impl->batch_size();
    info->num_steps = static_cast<std::int64_t>(p.steps.size());
    info->max_rank = p.max_rank;
    info->peak_memory = p.peak_memory;
    info->arena_bytes = e->impl->arena_bytes();
    info->node_bytes = e->impl->node_bytes();
    info->flops_per_slice = p.flops_per_slice;
    info->num_ops = static_cast<std::int64_t>(e->impl->profile().size());
  });
}

int qsg_engine_plan_json(qsg_engine* e, char* buf, int64_t cap, int64_t* len) {
  return guarded([&] { put_text(qsg::plan_to_json(e->impl->plan()), buf, cap, len); });
}

int qsg_engine_describe(qsg_engine* e, char* buf, int64_t cap, int64_t* len) {
  return guarded([&] { put_text(e->impl->describe(), buf, cap, len); });
}

int qsg_engine_open_qubits(qsg_engine* e, int* out) {
  return guarded([&] {
    const auto& o = e->impl->plan().open_qubits;
    std::copy(o.begin(), o.end(), out);
  });
}

int qsg_engine_prepare(qsg_engine* e, const int* x1_bits, int n, int64_t* h2d_bytes) {
  return guarded([&] {
    const std::int64_t b = e->impl->prepare(std::vector<int>(x1_bits, x1_bits + n));
    if (h2d_bytes) *h2d_bytes = b;
  });
}

int qsg_engine_fold_nodes(qsg_engine* e, const char* circuit_text, void* host_nodes, int64_t bytes) {
  return guarded([&] { e->impl->fold_nodes(qsg::parse_circuit(circuit_text), host_nodes, bytes); });
}

int qsg_engine_load_nodes(qsg_engine* e, const void* host_nodes, int64_t bytes) {
  return guarded([&] { e->impl->load_nodes(host_nodes, bytes); });
}

int qsg_engine_export_nodes(qsg_engine* e, void* host_nodes, int64_t bytes) {
  return guarded([&] { e->impl->export_nodes(host_nodes, bytes); });
}

int qsg_engine_run(qsg_engine* e, const int64_t* slice_ids, int64_t k, int reset, int per_slice) {
  return guarded([&] { e->impl->run(std::vector<std::int64_t>(slice_ids, slice_ids + k), reset != 0, per_slice != 0); });
}

int qsg_engine_results(qsg_engine* e, double* amps_host, double* per_slice_host) {
  return guarded([&] {
    std::vector<qsg::cdouble> amps, ps;
    e->impl->results(amps_host ? &amps : nullptr, per_slice_host ? &ps : nullptr);
    if (amps_host) std::memcpy(amps_host, amps.data(), amps.size() * sizeof(qsg::cdouble));
    if (per_slice_host) std::memcpy(per_slice_host, ps.data(), ps.size() * sizeof(qsg::cdouble));
  });
}

int qsg_engine_stream(qsg_engine* e, void** stream) {
  return guarded([&] { *stream = static_cast<void*>(e->impl->stream()); });
}

int qsg_engine_synchronize(qsg_engine* e) {
  return guarded([&] { e->impl->synchronize(); });
}

int qsg_engine_per_slice_rows(qsg_engine* e, int64_t* rows) {
  return guarded([&] { *rows = e->impl->per_slice_rows(); });
}

int qsg_engine_launches(qsg_engine* e, int64_t* launches) {
  return guarded([&] { *launches = e->impl->launches(); });
}

int qsg_engine_profile(qsg_engine* e, qsg_op_profile* out, int cap, int* count) {
  return guarded([&] {
    const auto prof = e->impl->profile();
    *count = static_cast<int>(prof.size());
    for (int i = 0; i < cap && i < *count; ++i) {
      const auto& p = prof[static_cast<std::size_t>(i)];
      out[i] = qsg_op_profile{p.kind, p.step, p.m, p.n, p.k, p.flops, p.bytes, p.ms_total, p.executions, p.tc, 0};
    }
  });
}

int qsg_engine_set_profile(qsg_engine* e, int on) {
  return guarded([&] { e->impl->set_profile(on != 0); });
}

int qsg_engine_reset_profile(qsg_engine* e) {
  return guarded([&] { e->impl->reset_profile(); });
}

int qsg_amplitude_batch(qsg_engine* e, const int* x1_bits, int n, const int64_t* slice_ids, int64_t k, double* amps_host,
                        char* bitstrings_host) {
  return guarded([&] {
    const auto res = qsg::amplitude_batch(*e->impl, std::vector<int>(x1_bits, x1_bits + n),
                                          std::vector<std::int64_t>(slice_ids, slice_ids + k));
    for (std::size_t i = 0; i < res.size(); ++i) {
      amps_host[2 * i] = res[i].second.real();
      amps_host[2 * i + 1] = res[i].second.imag();
      if (bitstrings_host) std::memcpy(bitstrings_host + i * static_cast<std::size_t>(n), res[i].first.data(), static_cast<std::size_t>(n));
    }
  });
}

int qsg_widen_plan(const char* circuit_text, int kind, const char* plan_text, const int* open, int nopen,
                   const int* extra_open, int nextra, char* buf, int64_t cap, int64_t* len) {
  return guarded([&] {
    const qsg::Circuit c = qsg::parse_circuit(circuit_text);
    const qsg::ContractionPlan plan = make_plan(c, kind, plan_text, std::vector<int>(open, open + nopen), 0);
    put_text(qsg::plan_to_json(qsg::widen_plan(c, plan, std::vector<int>(extra_open, extra_open + nextra))), buf, cap,
             len);
  });
}

int qsg_reassociate_plan(const char* circuit_text, int kind, const char* plan_text, const int* open, int nopen,
                         char* buf, int64_t cap, int64_t* len, int* rewrites) {
  return guarded([&] {
    const qsg::Circuit c = qsg::parse_circuit(circuit_text);
    const qsg::ContractionPlan plan = make_plan(c, kind, plan_text, std::vector<int>(open, open + nopen), 0);
    int r = 0;
    put_text(qsg::plan_to_json(qsg::reassociate_plan(qsg::fold_shape(c, plan.open_qubits), plan, &r)), buf, cap, len);
    if (rewrites) *rewrites = r;
  });
}

int qsg_amplitude_batches(qsg_engine* e, const int* base_open, int nbase, const int* x1_list, int nx1, int n,
                          const int64_t* slice_ids, int64_t k, double* amps_host, char* bitstrings_host) {
  return guarded([&] {
    if (n != e->impl->circuit().num_qubits()) throw std::invalid_argument("fold: bitstring length != qubit count");
    if (nx1 < 0) throw std::invalid_argument("amplitude_batches: negative draw count");
    qsg::amplitude_batches_into(*e->impl, std::vector<int>(base_open, base_open + nbase), x1_list,
                                static_cast<std::size_t>(nx1), std::vector<std::int64_t>(slice_ids, slice_ids + k),
                                amps_host, bitstrings_host);
  });
}

int qsg_amplitude_batches_submit(qsg_engine* e, const int* base_open, int nbase, const int* x1_list, int nx1, int n,
                                 const int64_t* slice_ids, int64_t k, int slot) {
  return guarded([&] {
    if (nx1 < 0) throw std::invalid_argument("amplitude_batches: negative draw count");
    if (n != e->impl->circuit().num_qubits()) throw std::invalid_argument("fold: bitstring length != qubit count");
    qsg::amplitude_batches_submit(*e->impl, std::vector<int>(base_open, base_open + nbase), x1_list,
                                  static_cast<std::size_t>(nx1), std::vector<std::int64_t>(slice_ids, slice_ids + k),
                                  slot);
  });
}

int qsg_amplitude_batches_collect(qsg_engine* e, const int* base_open, int nbase, const int* x1_list, int nx1, int n,
                                  int slot, double* amps_out, char* bits_out) {
  return guarded([&] {
    if (nx1 < 0) throw std::invalid_argument("amplitude_batches: negative draw count");
    if (n != e->impl->circuit().num_qubits()) throw std::invalid_argument("fold: bitstring length != qubit count");
    qsg::amplitude_batches_collect(*e->impl, std::vector<int>(base_open, base_open + nbase), x1_list,
                                   static_cast<std::size_t>(nx1), slot, amps_out, bits_out);
  });
}

int qsg_run_amplitudes(qsg_engine* e, const char* bitstrings, int nb, int n, int64_t frac_num, int64_t frac_den,
                       uint64_t seed, double* out, int64_t* ids_out, uint64_t* flops) {
  return guarded([&] {
    std::vector<std::string> bits;
    for (int b = 0; b < nb; ++b) bits.emplace_back(bitstrings + static_cast<std::size_t>(b) * n, static_cast<std::size_t>(n));
    qsg::Fraction f{frac_num, frac_den};
    if (frac_den <= 0) f = qsg::Fraction{e->impl->plan().num_slices, e->impl->plan().num_slices};
    const auto res = qsg::run_amplitudes(*e->impl, bits, f, seed);
    for (int b = 0; b < nb; ++b) {
      out[2 * b] = res.amplitudes[static_cast<std::size_t>(b)].second.real();
      out[2 * b + 1] = res.amplitudes[static_cast<std::size_t>(b)].second.imag();
    }
    if (ids_out) std::copy(res.slice_ids.begin(), res.slice_ids.end(), ids_out);
    if (flops) *flops = res.total_flops;
  });
}

namespace {
qsg_xeb_report to_c(const qsg::XebReport& r) {
  qsg_xeb_report o{};
  o.n = r.n;
  o.hog_available = r.hog_available ? 1 : 0;
  o.size = static_cast<int64_t>(r.size);
  o.zero_excluded = static_cast<int64_t>(r.zero_excluded);
  o.mean_log_prob = r.mean_log_prob;
  o.cross_entropy = r.cross_entropy;
  o.fidelity_estimate = r.fidelity_estimate;
  o.hog_fraction = r.hog_fraction;
  return o;
}
}  // namespace

int qsg_sample(qsg_engine* e, int64_t num_samples, int64_t frac_num, int64_t frac_den, int amplitude_fraction_mode,
               double rejection_cap, uint64_t seed, char* bitstrings_out, double* probs_out, qsg_sample_stats* stats,
               qsg_xeb_report* self_xeb) {
  return guarded([&] {
    qsg::SamplingConfig cfg;
    cfg.num_samples = static_cast<std::size_t>(num_samples);
    const auto K = e->impl->plan().num_slices;
    cfg.fraction = frac_den > 0 ? qsg::Fraction{frac_num, frac_den} : qsg::Fraction{K, K};
    if (cfg.fraction.den < 1 || cfg.fraction.num < 1 || cfg.fraction.num > cfg.fraction.den)
      throw std::invalid_argument("fraction out of range");
    cfg.amplitude_fraction_mode = amplitude_fraction_mode != 0;
    cfg.rejection_cap = rejection_cap;
    cfg.seed = seed;
    const auto out = qsg::sample(*e->impl, cfg);
    const int n = e->impl->circuit().num_qubits();
    for (std::size_t i = 0; i < out.bitstrings.size(); ++i) {
      if (bitstrings_out) std::memcpy(bitstrings_out + i * static_cast<std::size_t>(n), out.bitstrings[i].data(), static_cast<std::size_t>(n));
      if (probs_out) probs_out[i] = out.probabilities[i];
    }
    if (stats) {
      stats->x1_draws = out.stats.x1_draws;
      stats->redraws = out.stats.redraws;
      stats->cap_hits = out.stats.cap_hits;
      stats->candidates = out.stats.candidates;
      stats->exact_count = static_cast<int64_t>(out.stats.exact_count);
      stats->uniform_count = static_cast<int64_t>(out.stats.uniform_count);
    }
    if (self_xeb) *self_xeb = to_c(out.self_xeb);
  });
}

int qsg_xeb_score(int n, const double* probs, int64_t count, int has_median, double hog_median, qsg_xeb_report* out) {
  return guarded([&] {
    const std::vector<double> p(probs, probs + count);
    *out = to_c(qsg::xeb_score(n, p, has_median ? &hog_median : nullptr));
  });
}

}  // extern "C"
