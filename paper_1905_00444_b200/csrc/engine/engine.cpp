// Device executor: plan -> static device program -> per-slice replay.
// See engine.hpp for the design; reference behaviour cited inline.
#include "engine.hpp"

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <map>
#include <set>
#include <numeric>
#include <sstream>
#include <stdexcept>

#include "../device/kernels_tc.hpp"

namespace qsg {

namespace {

void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

constexpr std::int64_t kAlign = 256;

std::int64_t align_up(std::int64_t x) { return (x + kAlign - 1) / kAlign * kAlign; }

std::vector<std::int64_t> row_major_strides(const std::vector<std::int64_t>& dims) {
  std::vector<std::int64_t> s(dims.size());
  std::int64_t acc = 1;
  for (std::size_t i = dims.size(); i-- > 0;) {
    s[i] = acc;
    acc *= dims[i];
  }
  return s;
}

// A tensor as the program sees it at compile time.
struct View {
  int buf = -1;
  std::int64_t off = 0;
  int node = -1;
  std::vector<Label> labels;
  std::vector<std::int64_t> dims;
  std::vector<std::int64_t> strides;
  int meta = -1;  // -1: node tensor (never renormalised)
  std::int64_t volume() const {
    std::int64_t v = 1;
    for (auto d : dims) v *= d;
    return v;
  }
  bool dense() const { return strides == row_major_strides(dims); }
  std::int64_t dim_of(const Label& l) const {
    for (std::size_t i = 0; i < labels.size(); ++i)
      if (labels[i] == l) return dims[i];
    throw std::invalid_argument("execute: no label " + l);
  }
  std::int64_t stride_of(const Label& l) const {
    for (std::size_t i = 0; i < labels.size(); ++i)
      if (labels[i] == l) return strides[i];
    throw std::invalid_argument("execute: no label " + l);
  }
  bool has(const Label& l) const { return std::find(labels.begin(), labels.end(), l) != labels.end(); }
};

bool seq_equal(const std::vector<Label>& a, std::size_t a0, const std::vector<Label>& b) {
  if (a0 + b.size() > a.size()) return false;
  for (std::size_t i = 0; i < b.size(); ++i)
    if (a[a0 + i] != b[i]) return false;
  return true;
}

}  // namespace

Engine::Engine(const Circuit& c, const ContractionPlan& plan, const EngineOptions& opt)
    : circuit_(c), plan_(plan), opt_(opt) {
  if (!opt_.compile_only) {
    check(cudaSetDevice(opt_.device), "cudaSetDevice");
    check(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "cudaStreamCreate");
  }
  // Device-side fold: the worldline fold with EVERY output wire left open is
  // independent of x1; projecting a closed output onto bit b is taking half
  // b of axis 0 (src/network.cpp:138-147), i.e. a view offset.  So the open
  // fold is uploaded once per engine and an x1 batch only moves node views.
  const int nq = c.num_qubits();
  for (int q : plan_.open_qubits)
    if (q < 0 || q >= nq) throw std::invalid_argument("engine: plan open qubits do not match the circuit fold");
  GridNetwork open_fold = fold_worldlines(c, std::vector<int>(static_cast<std::size_t>(nq), -1));
  shape_ = open_fold.shape();
  closed_.assign(static_cast<std::size_t>(nq), 1);
  for (int q : plan_.open_qubits) closed_[static_cast<std::size_t>(q)] = 0;
  node_x1_off_.assign(static_cast<std::size_t>(nq), 0);
  batch_ = std::int64_t{1} << plan_.open_qubits.size();
  auto build = [&] {
    ooc_slot_bytes_ = 0;
    compile();
    split_handoffs();
    pack_buffers();
  };
  if (opt_.memory_budget >= 0) {
    build();
  } else {
    // Automatic: the in-HBM program if it fits the device, else the largest
    // power-of-two contraction budget whose out-of-core program fits.
    std::int64_t avail = opt_.device_memory;
    if (avail <= 0 && !opt_.compile_only) {
      std::size_t free_b = 0, total_b = 0;
      check(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
      avail = static_cast<std::int64_t>(free_b);
    }
    if (avail <= 0) avail = std::int64_t{180} << 30;
    avail = avail / 100 * 92;  // headroom for the CUDA context, metas, accumulators
    auto device_need = [&] {
      return arena_bytes_ + ooc_slot_bytes_ * std::max(1, opt_.pipeline_depth);
    };
    opt_.memory_budget = 0;
    build();
    for (std::int64_t b = std::int64_t{1} << 42; device_need() > avail; b >>= 1) {
      if (b < (std::int64_t{1} << 20)) throw std::runtime_error("engine: no contraction budget fits the device memory");
      opt_.memory_budget = b;
      build();
    }
  }
  op_ms_.assign(ops_.size(), 0.0);
  op_execs_.assign(ops_.size(), 0);
  if (opt_.compile_only) return;  // program listing only (no device)
  check(cudaMalloc(&arena_, static_cast<std::size_t>(std::max<std::int64_t>(arena_bytes_, kAlign))), "arena cudaMalloc");
  if (host_arena_bytes_ > 0) {
    check(cudaHostAlloc(reinterpret_cast<void**>(&host_arena_), static_cast<std::size_t>(host_arena_bytes_),
                        cudaHostAllocMapped | cudaHostAllocPortable),
          "host arena cudaHostAlloc");
    const int depth = std::max(1, opt_.pipeline_depth);
    check(cudaMalloc(&ooc_scratch_, static_cast<std::size_t>(ooc_slot_bytes_) * static_cast<std::size_t>(depth)),
          "out-of-core scratch cudaMalloc");
    check(cudaStreamCreateWithFlags(&copy_stream_, cudaStreamNonBlocking), "cudaStreamCreate");
    check(cudaStreamCreateWithFlags(&store_stream_, cudaStreamNonBlocking), "cudaStreamCreate");
    ooc_ev_.resize(3 * static_cast<std::size_t>(depth) + 2);
    for (auto& e : ooc_ev_) check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
  }
  check(cudaMalloc(&metas_, sizeof(dev::TMeta) * static_cast<std::size_t>(std::max(nmeta_, 1))), "meta cudaMalloc");
  check(cudaMemset(metas_, 0, sizeof(dev::TMeta) * static_cast<std::size_t>(std::max(nmeta_, 1))), "meta memset");
  check(cudaMalloc(&acc_, sizeof(double2) * static_cast<std::size_t>(batch_)), "acc cudaMalloc");
  check(cudaMemset(acc_, 0, sizeof(double2) * static_cast<std::size_t>(batch_)), "acc memset");
  {  // one-time upload of the open fold (x1-independent node tensors)
    std::vector<cfloat> host(static_cast<std::size_t>(node_bytes_ / 8), cfloat{});
    pack_nodes(open_fold, host.data());
    check(cudaMemcpy(arena_ + bufs_[0].offset, host.data(), static_cast<std::size_t>(node_bytes_), cudaMemcpyHostToDevice),
          "node upload");
  }
  op_ms_.assign(ops_.size(), 0.0);
  op_execs_.assign(ops_.size(), 0);
  set_profile(opt_.profile);
}

void Engine::set_profile(bool on) {
  opt_.profile = on;
  if (on && ev_.empty()) {
    check(cudaSetDevice(opt_.device), "cudaSetDevice");
    ev_.resize(2 * ops_.size());
    for (auto& e : ev_) check(cudaEventCreate(&e), "cudaEventCreate");
  }
}

Engine::~Engine() {
  if (opt_.compile_only) return;
  cudaSetDevice(opt_.device);
  if (stream_) cudaStreamSynchronize(stream_);
  for (auto e : ev_) cudaEventDestroy(e);
  if (arena_) cudaFree(arena_);
  if (host_arena_) cudaFreeHost(host_arena_);
  if (ooc_scratch_) cudaFree(ooc_scratch_);
  for (auto e : ooc_ev_) cudaEventDestroy(e);
  if (copy_stream_) cudaStreamDestroy(copy_stream_);
  if (store_stream_) cudaStreamDestroy(store_stream_);
  if (metas_) cudaFree(metas_);
  if (acc_) cudaFree(acc_);
  if (acc_host_) cudaFreeHost(acc_host_);
  for (auto& st : stage_) {
    if (st.host) cudaFreeHost(st.host);
    if (st.ev) cudaEventDestroy(st.ev);
  }
  if (per_slice_) cudaFree(per_slice_);
  if (graph_exec_) cudaGraphExecDestroy(graph_exec_);
  if (stream_) cudaStreamDestroy(stream_);
}

void Engine::compile() {
  // ---- node region ---------------------------------------------------------
  const std::size_t n = shape_.nodes.size();
  node_elem_off_.assign(n, 0);
  node_vol_.assign(n, 0);
  node_full_strides_.assign(n, {});
  node_cut_axes_.assign(n, {});
  node_wire_stride_.assign(n, 0);
  std::int64_t elems = 0;
  for (std::size_t q = 0; q < n; ++q) {
    node_elem_off_[q] = elems;
    node_vol_[q] = shape_.nodes[q].volume();
    node_full_strides_[q] = row_major_strides(shape_.nodes[q].dims);
    elems += align_up(node_vol_[q] * 8) / 8;
  }
  node_bytes_ = elems * 8;
  bufs_.clear();
  ops_.clear();
  bufs_.push_back(Buffer{node_bytes_, 0, 1 << 30, 0});  // buffer 0: node region, always live

  const std::size_t fixed = cut_fixed_count(shape_, plan_.cut);
  std::map<std::string, View> live;
  for (std::size_t q = 0; q < n; ++q) {
    const auto& node = shape_.nodes[q];
    View v;
    v.buf = 0;
    v.off = node_elem_off_[q];
    v.node = static_cast<int>(q);
    std::vector<int> cut_axes(fixed, -1);
    // Axis 0 is the output wire; a closed output is a per-x1 half offset.
    node_wire_stride_[q] = node_full_strides_[q][0];
    for (std::size_t a = closed_[q] ? 1 : 0; a < node.labels.size(); ++a) {
      auto it = std::find(plan_.cut.labels.begin(), plan_.cut.labels.begin() + static_cast<std::ptrdiff_t>(fixed),
                          node.labels[a]);
      if (it != plan_.cut.labels.begin() + static_cast<std::ptrdiff_t>(fixed)) {
        cut_axes[static_cast<std::size_t>(it - plan_.cut.labels.begin())] = static_cast<int>(a);
        continue;
      }
      v.labels.push_back(node.labels[a]);
      v.dims.push_back(node.dims[a]);
      v.strides.push_back(node_full_strides_[q][a]);
    }
    node_cut_axes_[q] = cut_axes;
    live[node_name(static_cast<int>(q))] = std::move(v);
  }

  auto new_buf = [&](std::int64_t bytes) {
    Buffer b;
    b.bytes = align_up(std::max<std::int64_t>(bytes, 8));
    b.first = b.last = static_cast<int>(ops_.size());
    bufs_.push_back(b);
    return static_cast<int>(bufs_.size()) - 1;
  };
  auto touch = [&](int buf) {
    if (buf > 0) bufs_[static_cast<std::size_t>(buf)].last = static_cast<int>(ops_.size());
  };
  auto as_operand = [](const View& v) { return Operand{v.buf, v.off, v.node}; };
  // Emits K1 making `v` dense in `order`; returns the new view.
  auto permute_to = [&](const View& v, const std::vector<Label>& order, int step, bool host = false) {
    Op op;
    op.kind = 0;
    op.step = step;
    op.src = as_operand(v);
    View out;
    out.meta = v.meta;
    for (const auto& l : order) {
      op.ext.push_back(v.dim_of(l));
      op.istr.push_back(v.stride_of(l));
      out.labels.push_back(l);
      out.dims.push_back(v.dim_of(l));
    }
    out.strides = row_major_strides(out.dims);
    op.count = out.volume();
    touch(v.buf);
    op.dst = new_buf(op.count * 8);
    bufs_[static_cast<std::size_t>(op.dst)].host = host;
    out.buf = op.dst;
    out.off = 0;
    ops_.push_back(op);
    return out;
  };

  nmeta_ = static_cast<int>(plan_.steps.size());
  for (std::size_t si = 0; si < plan_.steps.size(); ++si) {
    const auto& step = plan_.steps[si];
    auto li = live.find(step.lhs), ri = live.find(step.rhs);
    if (li == live.end() || ri == live.end())
      throw std::invalid_argument("execute: missing operand " + step.lhs + " or " + step.rhs);
    View L = li->second, R = ri->second;
    live.erase(li);
    live.erase(step.rhs);

    std::int64_t k = 1;
    std::vector<Label> con_l;
    for (const auto& l : L.labels)
      if (R.has(l)) {
        if (L.dim_of(l) != R.dim_of(l)) throw std::invalid_argument("contract: extent mismatch on " + l);
        con_l.push_back(l);
        k *= L.dim_of(l);
      }
    std::vector<Label> con_r;
    for (const auto& l : R.labels)
      if (L.has(l)) con_r.push_back(l);
    const std::int64_t ml = L.volume() / k, nr = R.volume() / k;
    constexpr std::int64_t kMaxVolume = std::int64_t{1} << 33;  // contraction.hpp:95, :189-191
    if (ml * k > kMaxVolume || k * nr > kMaxVolume || ml * nr > kMaxVolume)
      throw std::length_error("contract_ttgt: volume overflow");

    // Operand roles and layouts, by a time model.  C = [A free, B free];
    // either L or R takes the A role (streamed, rows of C), the contracted
    // order comes from either operand, and an operand is used in place when
    // dense with the contracted labels as a suffix/prefix (A: N or T, B: N
    // or T) -- otherwise K1 permutes it to the N layout.  The tcgen05 GEMM
    // needs A in N layout and expands B (40 B per element), so forcing a
    // permute of A can pay for itself on large steps.
    struct Choice {
      bool swap = false, use_a = false, ta = false, use_b = false, tb = false, tc = false;
      std::vector<Label> con;
      double cost = 0.0;
    };
    const double flops = static_cast<double>(step.flops);
    constexpr double kHbm = 5.0e12, kSimtRate = 4.0e13;
    constexpr std::int64_t kMaxTcWorkspace = std::int64_t{48} << 30;  // B_r^T planes (+ pre-split A planes)
    auto evaluate = [&](bool swap, const std::vector<Label>& con, bool force_permute_a) {
      const View& X = swap ? R : L;
      const View& Y = swap ? L : R;
      Choice ch;
      ch.swap = swap;
      ch.con = con;
      const std::size_t nc = con.size();
      if (X.dense() && !force_permute_a) {
        if (seq_equal(X.labels, X.labels.size() - nc, con)) { ch.use_a = true; ch.ta = false; }
        else if (seq_equal(X.labels, 0, con)) { ch.use_a = true; ch.ta = true; }
      }
      if (Y.dense()) {
        if (seq_equal(Y.labels, 0, con)) { ch.use_b = true; ch.tb = false; }
        else if (seq_equal(Y.labels, Y.labels.size() - nc, con)) { ch.use_b = true; ch.tb = true; }
      }
      const std::int64_t mm = X.volume() / k, nn2 = Y.volume() / k;
      const bool ta = ch.use_a && ch.ta, tb = ch.use_b && ch.tb;
      ch.tc = opt_.tensor_cores && dev::cgemm_tc_eligible(mm, nn2, k, ta, tb) &&
              dev::cgemm_tc_workspace_bytes(mm, nn2, k, ta, tb) <= kMaxTcWorkspace;
      const double bytes = (ch.use_a ? 0.0 : 16.0 * X.volume()) + (ch.use_b ? 0.0 : 16.0 * Y.volume()) +
                           (ch.tc ? dev::cgemm_tc_prep_bytes(mm, nn2, k) : 0.0);
      double gemm_s;
      if (ch.tc) {
        gemm_s = flops / dev::cgemm_tc_rate(mm, nn2, k);
      } else if (dev::cgemm_narrow(mm, nn2)) {  // HBM-bound narrow-N kernel
        gemm_s = 8.0 * static_cast<double>(mm * k + mm * nn2 + k * nn2) / kHbm;
      } else {  // 64 x 128 tiles: padded rows / columns are computed too
        const double pad = static_cast<double>((mm + 63) / 64 * 64) / static_cast<double>(mm) *
                           static_cast<double>((nn2 + 127) / 128 * 128) / static_cast<double>(nn2);
        gemm_s = flops * pad / kSimtRate;
      }
      ch.cost = bytes / kHbm + gemm_s;
      return ch;
    };
    Choice best = evaluate(false, con_l, false);
    for (bool swap : {false, true})
      for (const auto* con : {&con_l, &con_r})
        for (bool force : {false, true}) {
          Choice c = evaluate(swap, *con, force);
          if (c.cost < best.cost) best = c;
        }

    // Lookahead: the labels the consuming step will contract this output
    // against (its other operand's label set).
    // Lookahead: the labels the consuming step will contract this output
    // against (its other operand's label set), and the same one step further
    // (the consumer's consumer, for the output's row-bit order below).
    auto consumer_of = [&](const std::string& name, std::size_t from, std::set<Label>& con) -> std::size_t {
      for (std::size_t sj = from; sj < plan_.steps.size(); ++sj) {
        const auto& nx = plan_.steps[sj];
        if (nx.lhs != name && nx.rhs != name) continue;
        const std::string& other = nx.lhs == name ? nx.rhs : nx.lhs;
        auto lv = live.find(other);
        if (lv != live.end()) {
          con.insert(lv->second.labels.begin(), lv->second.labels.end());
        } else {
          for (std::size_t sk = 0; sk < sj; ++sk)
            if (plan_.steps[sk].out == other)
              con.insert(plan_.steps[sk].out_labels.begin(), plan_.steps[sk].out_labels.end());
        }
        return sj;
      }
      return plan_.steps.size();
    };
    std::set<Label> next_con;
    const std::size_t next_step = consumer_of(step.out, si + 1, next_con);
    const bool has_next = next_step < plan_.steps.size();
    // Contraction distance of this output's labels along its chain of
    // consumers (1 = the next step, 2 = the one after, ...; labels never
    // contracted within kLook steps: kLook + 1).
    constexpr int kLook = 8;
    std::map<Label, int> use_dist;
    {
      std::string name = step.out;
      std::size_t from = si + 1;
      for (int d = 1; d <= kLook; ++d) {
        std::set<Label> con;
        const std::size_t sj = consumer_of(name, from, con);
        if (sj >= plan_.steps.size()) break;
        for (const auto& l : con)
          if (!use_dist.count(l)) use_dist[l] = d;
        name = plan_.steps[sj].out;
        from = sj + 1;
      }
    }
    auto dist_of = [&](const Label& l) {
      auto it = use_dist.find(l);
      return it == use_dist.end() ? kLook + 1 : it->second;
    };
    // Free labels the next step contracts go last (they become the
    // trailing bits of the output, so it is usable there without a permute).
    auto next_last = [&](std::vector<Label> v) {
      std::stable_partition(v.begin(), v.end(), [&](const Label& l) { return next_con.count(l) == 0; });
      return v;
    };

    const View& X = best.swap ? R : L;
    const View& Y = best.swap ? L : R;
    std::vector<Label> xfree, yfree;
    for (const auto& l : X.labels)
      if (!Y.has(l)) xfree.push_back(l);
    for (const auto& l : Y.labels)
      if (!X.has(l)) yfree.push_back(l);
    xfree = next_last(xfree);
    yfree = next_last(yfree);
    // Out-of-core (ExecOptions::memory_budget semantics, src/engine.cpp:216-222):
    // the step's working set exceeds the budget, or an operand already lives
    // in host memory.  Its permuted operands and its result go to the
    // pinned host arena; the GEMM runs as device pieces.
    const std::int64_t xm = X.volume() / k, yn = Y.volume() / k;
    const bool ooc = opt_.memory_budget > 0 &&
                     (step_working_set(8 * xm * k, 8 * k * yn, 8 * xm * yn) > opt_.memory_budget ||
                      bufs_[static_cast<std::size_t>(X.buf)].host || bufs_[static_cast<std::size_t>(Y.buf)].host);
    View A = X, B = Y;
    // An out-of-core step gathers its operands' blocks per piece instead
    // (no permuted host copy): the view is just reordered.
    auto reorder = [](const View& v, const std::vector<Label>& order) {
      View r = v;
      r.labels = order;
      r.dims.clear();
      r.strides.clear();
      for (const auto& l : order) {
        r.dims.push_back(v.dim_of(l));
        r.strides.push_back(v.stride_of(l));
      }
      return r;
    };
    bool a_gather = false, b_gather = false;
    if (!best.use_a) {
      std::vector<Label> order = xfree;
      order.insert(order.end(), best.con.begin(), best.con.end());
      if (ooc) {
        A = reorder(X, order);
        a_gather = true;
      } else {
        A = permute_to(X, order, static_cast<int>(si), ooc);
      }
      best.ta = false;
    }
    if (!best.use_b) {
      std::vector<Label> order = best.con;
      order.insert(order.end(), yfree.begin(), yfree.end());
      if (ooc) {
        B = reorder(Y, order);
        b_gather = true;
      } else {
        B = permute_to(Y, order, static_cast<int>(si), ooc);
      }
      best.tb = false;
    }
    // Free-label orders as laid out in the operands.
    std::vector<Label> a_free, b_free;
    for (const auto& l : A.labels)
      if (!Y.has(l)) a_free.push_back(l);
    for (const auto& l : B.labels)
      if (!X.has(l)) b_free.push_back(l);

    Op g;
    g.kind = 1;
    g.step = static_cast<int>(si);
    g.a = as_operand(A);
    g.b = as_operand(B);
    g.m = X.volume() / k;
    g.n = Y.volume() / k;
    g.k = k;
    g.ta = best.ta;
    g.tb = best.tb;
    g.meta_a = A.meta;
    g.meta_b = B.meta;
    g.meta_c = static_cast<int>(si);
    g.flops = step.flops;
    g.tc = opt_.tensor_cores && dev::cgemm_tc_eligible(g.m, g.n, k, g.ta, g.tb) &&
           dev::cgemm_tc_workspace_bytes(g.m, g.n, k, g.ta, g.tb) <= kMaxTcWorkspace;
    g.ws_bytes = g.tc ? dev::cgemm_tc_workspace_bytes(g.m, g.n, k, g.ta, g.tb) : dev::cgemm_workspace_bytes(g.m, g.n, k);
    touch(A.buf);
    touch(B.buf);
    g.c = new_buf(g.m * g.n * 8);
    g.ooc = ooc;
    g.a_gather = a_gather;
    g.b_gather = b_gather;
    if (a_gather) {
      g.ga_ext = A.dims;
      g.ga_str = A.strides;
      g.ga_split = xfree.size();
    }
    if (b_gather) {
      g.gb_ext = B.dims;
      g.gb_str = B.strides;
      g.gb_split = best.con.size();
    }
    if (ooc) {
      bufs_[static_cast<std::size_t>(g.c)].host = true;
      g.tc = opt_.tensor_cores;  // decided per piece
      g.ws_bytes = 0;
      g.pieces = decompose_pieces(g.m, g.n, k, opt_.memory_budget);
      for (const auto& pc : g.pieces) {
        const std::int64_t ws = opt_.tensor_cores && dev::cgemm_tc_eligible(pc[1], pc[3], k, g.ta, g.tb)
                                    ? dev::cgemm_tc_workspace_bytes(pc[1], pc[3], k, g.ta, g.tb)
                                    : dev::cgemm_workspace_bytes(pc[1], pc[3], k);
        ooc_slot_bytes_ = std::max(ooc_slot_bytes_, align_up(pc[1] * k * 8) + align_up(k * pc[3] * 8) +
                                                        align_up(pc[1] * pc[3] * 8) + align_up(std::max<std::int64_t>(ws, 8)));
      }
    } else if (g.ws_bytes > 0) {
      g.ws = new_buf(g.ws_bytes);
    }

    // Output layout.  Natural GEMM order is [a_free, b_free]; when the
    // tcgen05 pair kernel runs, the epilogue can scatter C straight into
    // [free_next..., a_free ∩ con_next, b_free ∩ con_next] -- the layout the
    // consuming step uses in place -- provided the three lowest column bits
    // stay the three lowest output bits (64-byte store runs).
    std::vector<Label> out_order = a_free;
    out_order.insert(out_order.end(), b_free.begin(), b_free.end());
    if (has_next && !ooc && g.tc && dev::cgemm_tc_store_perm_supported(g.m, g.n, k, g.ta, g.tb) && a_free.size() <= 48 &&
        b_free.size() <= 24 && b_free.size() >= 3) {
      std::vector<Label> fr, cn;
      for (const auto& l : a_free) (next_con.count(l) ? cn : fr).push_back(l);
      std::vector<Label> cn_b;
      for (const auto& l : b_free) (next_con.count(l) ? cn_b : fr).push_back(l);
      // Lookahead layout (QSG_LAYOUT2=0 disables): the remaining free labels
      // ordered by how soon a later step contracts them, soonest lowest.
      // The next step's A then has the labels its own consumer contracts as
      // its lowest ROW bits, which its fused store puts right above its
      // column run: consecutive rows land in adjacent runs, and along a
      // sweep whole tiles become contiguous blocks (Bristlecone-70's k = 256
      // class 122 -> 106 ms per slice with the two-step version).
      static const bool layout2 = !(std::getenv("QSG_LAYOUT2") && std::getenv("QSG_LAYOUT2")[0] == '0');
      if (layout2)
        std::stable_sort(fr.begin(), fr.end(), [&](const Label& a, const Label& b) { return dist_of(a) > dist_of(b); });
      std::vector<Label> cand = fr;
      cand.insert(cand.end(), cn.begin(), cn.end());
      cand.insert(cand.end(), cn_b.begin(), cn_b.end());
      bool ok = cand != out_order;
      for (const auto& l : cand) ok = ok && (A.has(l) ? A.dim_of(l) : B.dim_of(l)) == 2;
      for (std::size_t t = 1; t <= 3 && ok; ++t) ok = cand[cand.size() - t] == b_free[b_free.size() - t];
      if (ok) {
        auto pos = [&](const Label& l) {
          return static_cast<unsigned char>(cand.size() - 1 - (std::find(cand.begin(), cand.end(), l) - cand.begin()));
        };
        g.store_perm = true;
        g.nrow_bits = static_cast<int>(a_free.size());
        g.ncol_bits = static_cast<int>(b_free.size());
        for (std::size_t b = 0; b < a_free.size(); ++b) g.row_pos[b] = pos(a_free[a_free.size() - 1 - b]);
        for (std::size_t b = 0; b < b_free.size(); ++b) g.col_pos[b] = pos(b_free[b_free.size() - 1 - b]);
        out_order = cand;
      }
    }
    ops_.push_back(g);

    View C;
    C.buf = g.c;
    C.off = 0;
    C.meta = static_cast<int>(si);
    C.labels = out_order;
    for (const auto& l : C.labels) C.dims.push_back(A.has(l) ? A.dim_of(l) : B.dim_of(l));
    C.strides = row_major_strides(C.dims);
    live[step.out] = std::move(C);
  }

  if (live.size() != 1) throw std::invalid_argument("execute: plan left multiple tensors");
  View F = live.begin()->second;
  std::vector<Label> want;
  for (int q : plan_.open_qubits) want.push_back(open_label(q));
  std::sort(want.begin(), want.end());
  {
    std::vector<Label> have = F.labels;
    std::sort(have.begin(), have.end());
    if (have != want) throw std::invalid_argument("execute: final tensor does not match the open qubits");
  }
  if (F.labels != want || !F.dense()) F = permute_to(F, want, -1);
  Op acc;
  acc.kind = 2;
  acc.src = as_operand(F);
  acc.meta_c = F.meta;
  acc.count = F.volume();
  touch(F.buf);
  ops_.push_back(acc);
  if (F.meta < 0) {
    // Single-node network: no step produced a meta; use a zeroed slot.
    ops_.back().meta_c = nmeta_;
    ++nmeta_;
  }
}

// GEMM -> GEMM hand-offs in split storage: when a tensor-core GEMM's output
// is read by exactly one op, and that op is a tensor-core GEMM using it in
// place as its A operand (N layout, whole tensor), the producer's epilogue
// writes fp16 hi | lo planes and the consumer streams them with no
// conversion (dev::GemmArgs::c_split / a_presplit).  QSG_TC_CSPLIT=0 turns
// this off.
void Engine::split_handoffs() {
  const char* env = std::getenv("QSG_TC_CSPLIT");
  if (!opt_.tensor_cores || (env && env[0] == '0')) return;
  const char* only = std::getenv("QSG_TC_CSPLIT_ONLY");  // debugging: restrict to one producer step
  for (std::size_t i = 0; i < ops_.size(); ++i) {
    Op& pr = ops_[i];
    if (pr.kind != 1 || !pr.tc || pr.ooc || !dev::cgemm_tc_split_ok(pr.m, pr.n, pr.k, pr.ta, pr.tb)) continue;
    if (only && (std::string(",") + only + ",").find("," + std::to_string(pr.step) + ",") == std::string::npos) continue;
    int reader = -1, readers = 0;
    for (std::size_t j = i + 1; j < ops_.size(); ++j) {
      const Op& q = ops_[j];
      const bool reads = (q.kind != 1 && q.src.buf == pr.c) || (q.kind == 1 && (q.a.buf == pr.c || q.b.buf == pr.c));
      if (reads) {
        ++readers;
        reader = static_cast<int>(j);
      }
    }
    if (readers != 1) continue;
    Op& co = ops_[static_cast<std::size_t>(reader)];
    if (co.kind != 1 || !co.tc || co.ooc || co.a.buf != pr.c || co.b.buf == pr.c || co.a.off != 0 || co.a.node >= 0 || co.ta ||
        co.m * co.k != pr.m * pr.n || co.meta_a != pr.meta_c || !dev::cgemm_tc_split_ok(co.m, co.n, co.k, co.ta, co.tb))
      continue;
    pr.c_split = true;
    co.a_presplit = true;
    co.ws_bytes = dev::cgemm_tc_workspace_bytes(co.m, co.n, co.k, co.ta, co.tb, true);
    if (co.ws >= 0) bufs_[static_cast<std::size_t>(co.ws)].bytes = align_up(std::max<std::int64_t>(co.ws_bytes, 8));
  }
}

// m / n blocks of an oversized contraction (src/plan.cpp:355-472 halves the
// widest axis of the largest of m, n, k until the piece fits).  Pieces here
// split only m and n: every output element keeps its whole K loop, so the
// result is the in-core one (no partial-sum accumulation or renormalisation
// of partial sums), and halving powers of two keeps pieces tensor-core shaped.
std::vector<std::array<std::int64_t, 4>> Engine::decompose_pieces(std::int64_t m, std::int64_t n, std::int64_t k,
                                                                   std::int64_t budget) {
  std::vector<std::array<std::int64_t, 4>> out;
  std::vector<std::array<std::int64_t, 4>> stack{{0, m, 0, n}};
  while (!stack.empty()) {
    const auto p = stack.back();
    stack.pop_back();
    if (step_working_set(8 * p[1] * k, 8 * k * p[3], 8 * p[1] * p[3]) <= budget) {
      out.push_back(p);
      continue;
    }
    const bool split_m = p[1] >= p[3] ? p[1] > 1 : p[3] <= 1;
    if ((split_m && p[1] < 2) || (!split_m && p[3] < 2))
      throw std::runtime_error("indivisible contraction still over budget");
    const std::int64_t len = split_m ? p[1] : p[3], half = len / 2;
    auto lo = p, hi = p;
    (split_m ? lo[1] : lo[3]) = half;
    (split_m ? hi[0] : hi[2]) += half;
    (split_m ? hi[1] : hi[3]) = len - half;
    stack.push_back(hi);  // the low half pops first (stable order)
    stack.push_back(lo);
  }
  return out;
}

// K1 gather of one piece block on the copy stream: dims [lo, hi) of the
// (ext, str) view carry the split index; the block [r0, r0 + rp) fixes their
// leading digits (rp divides their product, r0 % rp == 0), the other dims
// stay whole.  Output dense in the view's order.
void Engine::gather_block(const char* src, std::vector<std::int64_t> ext, const std::vector<std::int64_t>& str,
                          std::size_t lo, std::size_t hi, std::int64_t r0, std::int64_t rp, char* dst, int* launches) {
  std::int64_t base = 0, place = 1;
  for (std::size_t i = hi; i-- > lo;) {
    const std::int64_t e = ext[i], digit = (r0 / place) % e;
    if (place * e > rp) {
      base += digit * str[i];
      ext[i] = place < rp ? rp / place : 1;  // straddling dim keeps a sub-range, higher ones a single digit
    }
    place *= e;
  }
  std::vector<std::int64_t> e2, s2;
  for (std::size_t i = 0; i < ext.size(); ++i)
    if (ext[i] > 1) {
      e2.push_back(ext[i]);
      s2.push_back(str[i]);
    }
  if (e2.empty()) {
    e2.push_back(1);
    s2.push_back(1);
  }
  check(dev::permute(src, base, dst, static_cast<int>(e2.size()), e2.data(), s2.data(), copy_stream_, launches),
        "ooc gather");
}

// Five-stage pipeline of one out-of-core GEMM (src/engine.cpp:52-180):
// acquire a scratch slot, load the A row block and B column block
// (host->device copies on the copy stream; 2-D copies for strided blocks),
// execute on the engine stream, store the C block (device->host), release.
// pipeline_depth slots are in flight, so loads and stores of neighbouring
// pieces overlap the GEMM of the current one.
void Engine::launch_ooc_gemm(const Op& op, const std::vector<std::int64_t>& node_off, int* launches) {
  const int depth = std::max(1, opt_.pipeline_depth);
  const char* A = static_cast<const char*>(ptr(op.a, node_off));
  const char* B = static_cast<const char*>(ptr(op.b, node_off));
  char* C = base_of(op.c);
  const std::int64_t k = op.k;
  // Loads (H2D) on copy_stream_, stores (D2H) on store_stream_: both link
  // directions stay busy; per-slot events order the reuse of a slot.
  const std::size_t nd = static_cast<std::size_t>(depth);
  cudaEvent_t start = ooc_ev_[3 * nd], done = ooc_ev_[3 * nd + 1];
  check(cudaEventRecord(start, stream_), "event");
  check(cudaStreamWaitEvent(copy_stream_, start, 0), "wait");
  check(cudaStreamWaitEvent(store_stream_, start, 0), "wait");
  for (std::size_t i = 0; i < op.pieces.size(); ++i) {
    const auto& pc = op.pieces[i];
    const std::int64_t m0 = pc[0], mp = pc[1], n0 = pc[2], np = pc[3];
    const std::size_t slot = i % static_cast<std::size_t>(depth);
    char* sA = ooc_scratch_ + static_cast<std::int64_t>(slot) * ooc_slot_bytes_;
    char* sB = sA + align_up(mp * k * 8);
    char* sC = sB + align_up(k * np * 8);
    char* sW = sC + align_up(mp * np * 8);
    cudaEvent_t loaded = ooc_ev_[3 * slot], computed = ooc_ev_[3 * slot + 1], stored = ooc_ev_[3 * slot + 2];
    // load: after the slot's previous GEMM has read its A / B blocks
    if (i >= nd) check(cudaStreamWaitEvent(copy_stream_, computed, 0), "wait");
    if (op.a_gather) {
      gather_block(A, op.ga_ext, op.ga_str, 0, op.ga_split, m0, mp, sA, launches);
    } else if (!op.ta)
      check(cudaMemcpyAsync(sA, A + m0 * k * 8, static_cast<std::size_t>(mp * k * 8), cudaMemcpyDefault, copy_stream_),
            "ooc load A");
    else
      check(cudaMemcpy2DAsync(sA, static_cast<std::size_t>(mp * 8), A + m0 * 8, static_cast<std::size_t>(op.m * 8),
                              static_cast<std::size_t>(mp * 8), static_cast<std::size_t>(k), cudaMemcpyDefault,
                              copy_stream_),
            "ooc load A");
    if (op.b_gather)
      gather_block(B, op.gb_ext, op.gb_str, op.gb_split, op.gb_ext.size(), n0, np, sB, launches);
    else if (op.tb)
      check(cudaMemcpyAsync(sB, B + n0 * k * 8, static_cast<std::size_t>(np * k * 8), cudaMemcpyDefault, copy_stream_),
            "ooc load B");
    else
      check(cudaMemcpy2DAsync(sB, static_cast<std::size_t>(np * 8), B + n0 * 8, static_cast<std::size_t>(op.n * 8),
                              static_cast<std::size_t>(np * 8), static_cast<std::size_t>(k), cudaMemcpyDefault,
                              copy_stream_),
            "ooc load B");
    check(cudaEventRecord(loaded, copy_stream_), "event");
    // execute (engine stream): after the load, and after the slot's previous C block was stored
    check(cudaStreamWaitEvent(stream_, loaded, 0), "wait");
    if (i >= nd) check(cudaStreamWaitEvent(stream_, stored, 0), "wait");
    dev::GemmArgs g{};
    g.a = sA;
    g.b = sB;
    g.c = sC;
    g.m = mp;
    g.n = np;
    g.k = k;
    g.trans_a = op.ta;
    g.trans_b = op.tb;
    g.meta_a = op.meta_a >= 0 ? metas_ + op.meta_a : nullptr;
    g.meta_b = op.meta_b >= 0 ? metas_ + op.meta_b : nullptr;
    g.norm_a = op.meta_a >= 0;
    g.norm_b = op.meta_b >= 0;
    g.meta_c = metas_ + op.meta_c;
    g.workspace = sW;
    const bool tc = op.tc && dev::cgemm_tc_eligible(mp, np, k, op.ta, op.tb);
    g.workspace_bytes = tc ? dev::cgemm_tc_workspace_bytes(mp, np, k, op.ta, op.tb) : dev::cgemm_workspace_bytes(mp, np, k);
    if (tc) check(dev::cgemm_tc(g, stream_, launches), "cgemm_tc");
    else check(dev::cgemm(g, stream_, launches), "cgemm");
    check(cudaEventRecord(computed, stream_), "event");
    // store (store stream)
    check(cudaStreamWaitEvent(store_stream_, computed, 0), "wait");
    check(cudaMemcpy2DAsync(C + (m0 * op.n + n0) * 8, static_cast<std::size_t>(op.n * 8), sC,
                            static_cast<std::size_t>(np * 8), static_cast<std::size_t>(np * 8),
                            static_cast<std::size_t>(mp), cudaMemcpyDefault, store_stream_),
          "ooc store C");
    check(cudaEventRecord(stored, store_stream_), "event");
  }
  check(cudaEventRecord(done, store_stream_), "event");
  check(cudaStreamWaitEvent(stream_, done, 0), "wait");
}

void Engine::pack_buffers() {
  // First-fit over lifetimes, largest buffers first within equal starts.
  std::vector<int> order(bufs_.size());
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) {
    if (bufs_[static_cast<std::size_t>(x)].first != bufs_[static_cast<std::size_t>(y)].first)
      return bufs_[static_cast<std::size_t>(x)].first < bufs_[static_cast<std::size_t>(y)].first;
    return bufs_[static_cast<std::size_t>(x)].bytes > bufs_[static_cast<std::size_t>(y)].bytes;
  });
  std::vector<int> placed;
  arena_bytes_ = 0;
  host_arena_bytes_ = 0;
  for (int id : order) {
    Buffer& b = bufs_[static_cast<std::size_t>(id)];
    std::vector<std::pair<std::int64_t, std::int64_t>> busy;
    for (int p : placed) {
      const Buffer& o = bufs_[static_cast<std::size_t>(p)];
      if (o.host == b.host && o.first <= b.last && b.first <= o.last) busy.emplace_back(o.offset, o.offset + o.bytes);
    }
    std::sort(busy.begin(), busy.end());
    std::int64_t off = 0;
    for (const auto& [lo, hi] : busy) {
      if (off + b.bytes <= lo) break;
      off = std::max(off, hi);
    }
    b.offset = off;
    (b.host ? host_arena_bytes_ : arena_bytes_) = std::max(b.host ? host_arena_bytes_ : arena_bytes_, off + b.bytes);
    placed.push_back(id);
  }
}

char* Engine::base_of(int buf) const {
  const Buffer& b = bufs_[static_cast<std::size_t>(buf)];
  return (b.host ? host_arena_ : arena_) + b.offset;
}

void* Engine::ptr(const Operand& o, const std::vector<std::int64_t>& node_off) const {
  std::int64_t e = o.off;
  if (o.node >= 0) e += node_off[static_cast<std::size_t>(o.node)];
  return base_of(o.buf) + e * 8;
}

std::int64_t Engine::prepare(const std::vector<int>& x1_bits) {
  if (static_cast<int>(x1_bits.size()) != circuit_.num_qubits())
    throw std::invalid_argument("fold: bitstring length != qubit count");
  std::vector<int> open;
  for (std::size_t q = 0; q < x1_bits.size(); ++q) {
    if (x1_bits[q] < 0) open.push_back(static_cast<int>(q));
    else if (x1_bits[q] > 1) throw std::invalid_argument("fold: output bits must be 0, 1 or -1 (open)");
  }
  if (open != plan_.open_qubits) throw std::invalid_argument("x1 open qubits do not match the plan's open qubits");
  for (std::size_t q = 0; q < x1_bits.size(); ++q)
    node_x1_off_[q] = closed_[q] ? x1_bits[q] * node_wire_stride_[q] : 0;
  return 0;  // node tensors are resident; x1 only selects views
}

namespace {
bool same_layout(const NetworkShape& a, const NetworkShape& b) {
  if (a.rows != b.rows || a.cols != b.cols || a.nodes.size() != b.nodes.size() || a.bonds.size() != b.bonds.size() ||
      a.open_qubits != b.open_qubits)
    return false;
  for (std::size_t i = 0; i < a.nodes.size(); ++i)
    if (a.nodes[i].labels != b.nodes[i].labels || a.nodes[i].dims != b.nodes[i].dims) return false;
  for (std::size_t i = 0; i < a.bonds.size(); ++i)
    if (a.bonds[i].label != b.bonds[i].label || a.bonds[i].q0 != b.bonds[i].q0 || a.bonds[i].q1 != b.bonds[i].q1)
      return false;
  return true;
}
}  // namespace

void Engine::fold_nodes(const Circuit& c, void* host, std::int64_t bytes) const {
  if (bytes != node_bytes_) throw std::invalid_argument("fold_nodes: buffer size != node_bytes");
  if (c.num_qubits() != circuit_.num_qubits()) throw std::invalid_argument("fold_nodes: qubit count differs");
  GridNetwork f = fold_worldlines(c, std::vector<int>(static_cast<std::size_t>(c.num_qubits()), -1));
  if (!same_layout(f.shape(), shape_)) throw std::invalid_argument("fold_nodes: circuit fold shape differs from the engine's");
  pack_nodes(f, host);
}

void Engine::pack_nodes(const GridNetwork& f, void* host) const {
  cfloat* out = static_cast<cfloat*>(host);
  std::fill(out, out + node_bytes_ / 8, cfloat{});
  for (std::size_t q = 0; q < f.nodes.size(); ++q)
    std::copy(f.nodes[q].data.begin(), f.nodes[q].data.end(), out + node_elem_off_[q]);
}

void Engine::load_nodes(const void* host, std::int64_t bytes) {
  if (bytes != node_bytes_) throw std::invalid_argument("load_nodes: size != node_bytes");
  check(cudaSetDevice(opt_.device), "cudaSetDevice");
  check(cudaMemcpyAsync(arena_ + bufs_[0].offset, host, static_cast<std::size_t>(bytes), cudaMemcpyHostToDevice, stream_),
        "node load");
}

void Engine::export_nodes(void* host, std::int64_t bytes) {
  if (bytes != node_bytes_) throw std::invalid_argument("export_nodes: size != node_bytes");
  check(cudaSetDevice(opt_.device), "cudaSetDevice");
  check(cudaMemcpyAsync(host, arena_ + bufs_[0].offset, static_cast<std::size_t>(bytes), cudaMemcpyDeviceToHost, stream_),
        "node export");
  check(cudaStreamSynchronize(stream_), "sync");
}

void Engine::launch_op(std::size_t i, const std::vector<std::int64_t>& node_off, void* per_slice_slot) {
  const Op& op = ops_[i];
  int launches = 0;
  if (opt_.profile) check(cudaEventRecord(ev_[2 * i], stream_), "event");
  if (op.kind == 0) {
    const std::int64_t base = op.src.off + (op.src.node >= 0 ? node_off[static_cast<std::size_t>(op.src.node)] : 0);
    check(dev::permute(base_of(op.src.buf), base, base_of(op.dst), static_cast<int>(op.ext.size()),
                       op.ext.data(), op.istr.data(), stream_, &launches),
          "permute");
  } else if (op.kind == 1 && op.ooc) {
    launch_ooc_gemm(op, node_off, &launches);
  } else if (op.kind == 1) {
    dev::GemmArgs g{};
    g.a = ptr(op.a, node_off);
    g.b = ptr(op.b, node_off);
    g.c = base_of(op.c);
    g.m = op.m;
    g.n = op.n;
    g.k = op.k;
    g.trans_a = op.ta;
    g.trans_b = op.tb;
    g.meta_a = op.meta_a >= 0 ? metas_ + op.meta_a : nullptr;
    g.meta_b = op.meta_b >= 0 ? metas_ + op.meta_b : nullptr;
    g.norm_a = op.meta_a >= 0;
    g.norm_b = op.meta_b >= 0;
    g.meta_c = metas_ + op.meta_c;
    g.workspace = op.ws >= 0 ? base_of(op.ws) : nullptr;
    g.workspace_bytes = op.ws_bytes;
    g.store_perm = op.store_perm;
    g.c_split = op.c_split;
    g.a_presplit = op.a_presplit;
    g.nrow_bits = op.nrow_bits;
    g.ncol_bits = op.ncol_bits;
    std::copy(op.row_pos.begin(), op.row_pos.end(), g.row_pos);
    std::copy(op.col_pos.begin(), op.col_pos.end(), g.col_pos);
    if (op.tc) check(dev::cgemm_tc(g, stream_, &launches), "cgemm_tc");
    else check(dev::cgemm(g, stream_, &launches), "cgemm");
  } else {
    check(dev::accumulate(ptr(op.src, node_off), metas_ + op.meta_c, op.count, acc_, per_slice_slot, stream_, &launches),
          "accumulate");
  }
  if (opt_.profile) check(cudaEventRecord(ev_[2 * i + 1], stream_), "event");
  launches_ += launches;
}

std::vector<std::int64_t> Engine::run_key(const std::vector<std::int64_t>& slice_ids, bool reset, bool per_slice) const {
  std::vector<std::int64_t> key(slice_ids);
  key.push_back(-1);
  key.insert(key.end(), node_x1_off_.begin(), node_x1_off_.end());
  key.push_back(reset ? 1 : 0);
  key.push_back(per_slice ? 1 : 0);
  key.push_back(reinterpret_cast<std::int64_t>(per_slice_));
  key.push_back(per_slice_base_);
  return key;
}

void Engine::run(const std::vector<std::int64_t>& slice_ids, bool reset, bool per_slice) {
  check(cudaSetDevice(opt_.device), "cudaSetDevice");
  // Validate every id before anything is queued or captured: a bad id must
  // neither leave the accumulator half-updated nor poison graph capture.
  for (const auto id : slice_ids) (void)cut_digits(shape_, plan_.cut, id);
  if (per_slice) {
    // Rows append after the previous run's when the accumulator is kept
    // (reset = false): K runs of one slice each leave K rows, in run order.
    const std::int64_t base = (!reset && per_slice_used_ > 0) ? per_slice_used_ : 0;
    const std::int64_t need = (base + static_cast<std::int64_t>(slice_ids.size())) * batch_;
    if (need > per_slice_cap_) {
      const std::int64_t cap = std::max(need, 2 * per_slice_cap_);
      double2* grown = nullptr;
      check(cudaMalloc(&grown, sizeof(double2) * static_cast<std::size_t>(cap)), "per-slice cudaMalloc");
      if (base > 0)
        check(cudaMemcpyAsync(grown, per_slice_, sizeof(double2) * static_cast<std::size_t>(base * batch_),
                              cudaMemcpyDeviceToDevice, stream_),
              "per-slice copy");
      check(cudaStreamSynchronize(stream_), "sync");
      if (per_slice_) cudaFree(per_slice_);
      per_slice_ = grown;
      per_slice_cap_ = cap;
    }
    per_slice_base_ = base;
    per_slice_used_ = base + static_cast<std::int64_t>(slice_ids.size());
  } else {
    per_slice_base_ = 0;
    per_slice_used_ = 0;
  }
  if (events_pending_) profile();  // fold finished timings before reusing events
  static const bool env_off = std::getenv("QSG_GRAPH") && std::getenv("QSG_GRAPH")[0] == '0';
  const bool graphable = opt_.graphs && graphs_ok_ && !env_off && !opt_.profile && host_arena_bytes_ == 0;
  if (!graphable) {
    enqueue_run(slice_ids, reset, per_slice);
    return;
  }
  auto key = run_key(slice_ids, reset, per_slice);
  if (graph_exec_ && key == graph_key_) {
    check(cudaGraphLaunch(graph_exec_, stream_), "graph launch");
    launches_ += graph_launches_;
    return;
  }
  if (key != last_key_) {  // first occurrence: eager (also the first-use setup of every kernel)
    last_key_ = std::move(key);
    enqueue_run(slice_ids, reset, per_slice);
    return;
  }
  // Second identical run in a row: capture it once, replay from now on.
  if (graph_exec_) {
    cudaGraphExecDestroy(graph_exec_);
    graph_exec_ = nullptr;
  }
  const std::int64_t before = launches_;
  cudaGraph_t graph = nullptr;
  check(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal), "graph capture");
  try {
    enqueue_run(slice_ids, reset, per_slice);
  } catch (...) {
    cudaStreamEndCapture(stream_, &graph);
    if (graph) cudaGraphDestroy(graph);
    graphs_ok_ = false;
    launches_ = before;
    cudaGetLastError();
    enqueue_run(slice_ids, reset, per_slice);
    return;
  }
  const cudaError_t ce = cudaStreamEndCapture(stream_, &graph);
  cudaError_t ie = ce;
  if (ce == cudaSuccess) ie = cudaGraphInstantiate(&graph_exec_, graph, 0);
  if (graph) cudaGraphDestroy(graph);
  if (ie != cudaSuccess) {  // capture unsupported here: stay eager
    graph_exec_ = nullptr;
    graphs_ok_ = false;
    launches_ = before;
    cudaGetLastError();
    enqueue_run(slice_ids, reset, per_slice);
    return;
  }
  graph_launches_ = launches_ - before;
  graph_key_ = last_key_;
  check(cudaGraphLaunch(graph_exec_, stream_), "graph launch");
}

void Engine::enqueue_run(const std::vector<std::int64_t>& slice_ids, bool reset, bool per_slice) {
  if (reset) check(cudaMemsetAsync(acc_, 0, sizeof(double2) * static_cast<std::size_t>(batch_), stream_), "acc reset");
  // QSG_FAIL_SLICES=a,b,...: fault injection for the failure-attribution
  // tests (a run that reaches one of these slices throws).
  static const std::vector<std::int64_t> fail = [] {
    std::vector<std::int64_t> v;
    if (const char* env = std::getenv("QSG_FAIL_SLICES")) {
      std::string t(env);
      std::size_t pos = 0;
      while (pos < t.size()) {
        const std::size_t c = t.find(',', pos);
        v.push_back(std::stoll(t.substr(pos, c == std::string::npos ? std::string::npos : c - pos)));
        if (c == std::string::npos) break;
        pos = c + 1;
      }
    }
    return v;
  }();
  for (std::size_t s = 0; s < slice_ids.size(); ++s) {
    if (!fail.empty() && std::find(fail.begin(), fail.end(), slice_ids[s]) != fail.end())
      throw std::runtime_error("injected failure");
    const auto digits = cut_digits(shape_, plan_.cut, slice_ids[s]);
    std::vector<std::int64_t> node_off(node_x1_off_);
    for (std::size_t q = 0; q < node_vol_.size(); ++q)
      for (std::size_t ci = 0; ci < node_cut_axes_[q].size(); ++ci) {
        const int ax = node_cut_axes_[q][ci];
        if (ax >= 0) node_off[q] += digits[ci] * node_full_strides_[q][static_cast<std::size_t>(ax)];
      }
    check(cudaMemsetAsync(metas_, 0, sizeof(dev::TMeta) * static_cast<std::size_t>(nmeta_), stream_), "meta reset");
    void* slot =
        per_slice ? static_cast<void*>(per_slice_ + (per_slice_base_ + static_cast<std::int64_t>(s)) * batch_) : nullptr;
    for (std::size_t i = 0; i < ops_.size(); ++i) {
      launch_op(i, node_off, slot);
    }
    if (opt_.profile) {
      // Events are reused per slice: harvest this slice's timings.
      check(cudaStreamSynchronize(stream_), "profile sync");
      for (std::size_t i = 0; i < ops_.size(); ++i) {
        float ms = 0.f;
        check(cudaEventElapsedTime(&ms, ev_[2 * i], ev_[2 * i + 1]), "elapsed");
        op_ms_[i] += ms;
        op_execs_[i] += 1;
      }
    }
  }
}

void Engine::results(std::vector<cdouble>* amps, std::vector<cdouble>* per_slice) {
  check(cudaSetDevice(opt_.device), "cudaSetDevice");
  const std::size_t acc_bytes = sizeof(double2) * static_cast<std::size_t>(batch_);
  if (amps) {
    amps->resize(static_cast<std::size_t>(batch_));
    // Large batches (widened x1 plans: 2^16 amplitudes) go through a pinned
    // staging buffer: a pageable D2H runs at a fraction of the link rate.
    if (acc_bytes >= (64u << 10) && !acc_host_) check(cudaMallocHost(&acc_host_, acc_bytes), "pinned staging");
    check(cudaMemcpyAsync(acc_host_ ? static_cast<void*>(acc_host_) : static_cast<void*>(amps->data()), acc_, acc_bytes,
                          cudaMemcpyDeviceToHost, stream_),
          "result copy");
  }
  if (per_slice) {
    per_slice->resize(static_cast<std::size_t>(per_slice_used_ * batch_));
    if (per_slice_used_ > 0)
      check(cudaMemcpyAsync(per_slice->data(), per_slice_, sizeof(double2) * per_slice->size(), cudaMemcpyDeviceToHost,
                            stream_),
            "per-slice copy");
  }
  check(cudaStreamSynchronize(stream_), "result sync");
  if (amps && acc_host_) std::memcpy(amps->data(), acc_host_, acc_bytes);
}

const cdouble* Engine::results_pinned() {
  check(cudaSetDevice(opt_.device), "cudaSetDevice");
  const std::size_t acc_bytes = sizeof(double2) * static_cast<std::size_t>(batch_);
  if (!acc_host_) check(cudaMallocHost(&acc_host_, acc_bytes), "pinned staging");
  check(cudaMemcpyAsync(acc_host_, acc_, acc_bytes, cudaMemcpyDeviceToHost, stream_), "result copy");
  check(cudaStreamSynchronize(stream_), "result sync");
  return reinterpret_cast<const cdouble*>(acc_host_);
}

void Engine::stage_results(int slot) {
  if (slot < 0 || slot > 1) throw std::out_of_range("stage_results: slot must be 0 or 1");
  check(cudaSetDevice(opt_.device), "cudaSetDevice");
  const std::size_t acc_bytes = sizeof(double2) * static_cast<std::size_t>(batch_);
  auto& st = stage_[static_cast<std::size_t>(slot)];
  if (!st.host) check(cudaMallocHost(&st.host, acc_bytes), "pinned staging");
  if (!st.ev) check(cudaEventCreateWithFlags(&st.ev, cudaEventDisableTiming), "event");
  check(cudaMemcpyAsync(st.host, acc_, acc_bytes, cudaMemcpyDeviceToHost, stream_), "result copy");
  check(cudaEventRecord(st.ev, stream_), "event record");
}

const cdouble* Engine::staged_results(int slot) {
  if (slot < 0 || slot > 1 || !stage_[static_cast<std::size_t>(slot)].ev)
    throw std::invalid_argument("staged_results: nothing staged in this slot");
  auto& st = stage_[static_cast<std::size_t>(slot)];
  check(cudaEventSynchronize(st.ev), "staged result sync");
  return reinterpret_cast<const cdouble*>(st.host);
}

void Engine::synchronize() {
  check(cudaSetDevice(opt_.device), "cudaSetDevice");
  check(cudaStreamSynchronize(stream_), "sync");
}

std::vector<OpProfile> Engine::profile() {
  synchronize();
  events_pending_ = false;
  std::vector<OpProfile> out;
  for (std::size_t i = 0; i < ops_.size(); ++i) {
    const Op& op = ops_[i];
    OpProfile p{};
    p.kind = op.kind;
    p.step = op.step;
    p.m = op.kind == 1 ? op.m : op.count;
    p.n = op.kind == 1 ? op.n : 0;
    p.k = op.kind == 1 ? op.k : 0;
    p.flops = op.kind == 1 ? op.flops : 0;
    p.bytes = op.kind == 0 ? 16 * op.count : op.kind == 1 ? 8 * (op.m * op.k + op.k * op.n + op.m * op.n) : 24 * op.count;
    p.ms_total = op_ms_[i];
    p.executions = op_execs_[i];
    p.tc = op.tc ? 1 : 0;
    out.push_back(p);
  }
  return out;
}

void Engine::reset_profile() {
  std::fill(op_ms_.begin(), op_ms_.end(), 0.0);
  std::fill(op_execs_.begin(), op_execs_.end(), 0);
}

std::string Engine::describe() const {
  // "[r0 r1 ... | c0 c1 ...]": output bit positions of the GEMM row / column bits.
  auto perm_text = [](const Op& op) {
    std::string t = " [";
    for (int b = 0; b < op.nrow_bits; ++b) t += std::to_string(op.row_pos[b]) + " ";
    t += "|";
    for (int b = 0; b < op.ncol_bits; ++b) t += " " + std::to_string(op.col_pos[b]);
    return t + "]";
  };
  std::ostringstream os;
  os << "arena " << arena_bytes_ << " B, nodes " << node_bytes_ << " B, ops " << ops_.size();
  if (host_arena_bytes_ > 0)
    os << ", host arena " << host_arena_bytes_ << " B, pipeline scratch " << ooc_slot_bytes_ << " B x "
       << std::max(1, opt_.pipeline_depth);
  os << "\n";
  for (const auto& op : ops_) {
    if (op.kind == 0) os << "  permute step " << op.step << " elems " << op.count << " rank " << op.ext.size() << "\n";
    else if (op.kind == 1)
      os << "  gemm    step " << op.step << " m " << op.m << " n " << op.n << " k " << op.k << " flops " << op.flops
         << (op.ta ? " TA" : "") << (op.tb ? " TB" : "") << (op.tc ? " tc" : " simt") << " ws " << op.ws_bytes
         << (op.store_perm ? " fused-store" : "") << (op.store_perm ? perm_text(op) : std::string())
         << (op.c_split ? " split-out" : "")
         << (op.a_presplit ? " split-in" : "")
         << (op.ooc ? " ooc pieces " + std::to_string(op.pieces.size()) : std::string()) << "\n";
    else os << "  accumulate " << op.count << "\n";
  }
  return os.str();
}

std::vector<std::pair<std::string, cdouble>> amplitude_batch(Engine& e, const std::vector<int>& x1_bits,
                                                             const std::vector<std::int64_t>& slice_ids) {
  e.prepare(x1_bits);
  e.run(slice_ids, /*reset=*/true, /*per_slice=*/false);
  std::vector<cdouble> amps;
  e.results(&amps, nullptr);
  std::vector<std::pair<std::string, cdouble>> out;
  out.reserve(amps.size());
  for (std::size_t j = 0; j < amps.size(); ++j) out.emplace_back(merge_bits(x1_bits, e.plan().open_qubits, j), amps[j]);
  return out;
}

ContractionPlan widen_plan(const Circuit& c, const ContractionPlan& plan, const std::vector<int>& extra_open) {
  std::set<int> open(plan.open_qubits.begin(), plan.open_qubits.end());
  for (int q : extra_open) {
    if (q < 0 || q >= c.num_qubits()) throw std::invalid_argument("widen_plan: qubit out of range");
    open.insert(q);
  }
  ContractionPlan p = plan;
  p.open_qubits.assign(open.begin(), open.end());
  annotate_plan(fold_shape(c, p.open_qubits), p);  // same order and cut, wider open wires
  return p;
}

namespace {
// Validates a draw list against the widened plan; returns the widened x1.
std::vector<int> widened_x1(const Engine& wide, const std::vector<int>& base_open, const int* x1_list,
                            std::size_t nx1) {
  const int n = wide.circuit().num_qubits();
  const auto& wopen = wide.plan().open_qubits;
  std::vector<char> is_open(static_cast<std::size_t>(n), 0), is_base(static_cast<std::size_t>(n), 0);
  for (int q : wopen) is_open[static_cast<std::size_t>(q)] = 1;
  if (!std::is_sorted(base_open.begin(), base_open.end()))
    throw std::invalid_argument("amplitude_batches: base open qubits must be sorted (the plan's order)");
  for (int q : base_open) {
    if (q < 0 || q >= n || !is_open[static_cast<std::size_t>(q)])
      throw std::invalid_argument("amplitude_batches: base open qubits must be open in the widened plan");
    is_base[static_cast<std::size_t>(q)] = 1;
  }
  auto draw = [&](std::size_t t) { return x1_list + t * static_cast<std::size_t>(n); };
  // One contraction: the widened plan's closed qubits must agree across the list.
  std::vector<int> x1w(static_cast<std::size_t>(n), -1);
  if (nx1 == 0) return x1w;
  for (int q = 0; q < n; ++q)
    if (!is_open[static_cast<std::size_t>(q)]) x1w[static_cast<std::size_t>(q)] = draw(0)[q];
  for (std::size_t t = 0; t < nx1; ++t) {
    const int* x1 = draw(t);
    for (int q = 0; q < n; ++q) {
      const int b = x1[q];
      if ((b < 0) != static_cast<bool>(is_base[static_cast<std::size_t>(q)]))
        throw std::invalid_argument("x1 open qubits do not match the plan's open qubits");
      if (b > 1) throw std::invalid_argument("fold: output bits must be 0, 1 or -1 (open)");
      if (!is_open[static_cast<std::size_t>(q)] && b != x1w[static_cast<std::size_t>(q)])
        throw std::invalid_argument("amplitude_batches: x1 draws differ on a qubit the widened plan keeps closed");
    }
  }
  return x1w;
}
}  // namespace

void amplitude_batches_submit(Engine& wide, const std::vector<int>& base_open, const int* x1_list, std::size_t nx1,
                              const std::vector<std::int64_t>& slice_ids, int slot) {
  const std::vector<int> x1w = widened_x1(wide, base_open, x1_list, nx1);
  if (nx1 == 0) return;
  wide.prepare(x1w);
  wide.run(slice_ids, /*reset=*/true, /*per_slice=*/false);
  wide.stage_results(slot);
}

void amplitude_batches_collect(Engine& wide, const std::vector<int>& base_open, const int* x1_list, std::size_t nx1,
                               int slot, double* amps_out, char* bits_out) {
  if (nx1 == 0) return;
  const int n = wide.circuit().num_qubits();
  const auto& wopen = wide.plan().open_qubits;
  auto draw = [&](std::size_t t) { return x1_list + t * static_cast<std::size_t>(n); };
  const cdouble* amps = wide.staged_results(slot);
  // Batch index of a full bitstring: bit (|open|-1-r) <-> r-th smallest open qubit (src/sampler.cpp:41-52).
  // wide index = fixed part (this draw's bits on the extra open qubits) + the
  // base batch index's bits scattered to the base qubits' positions.
  const std::size_t nw = wopen.size(), nb = base_open.size(), per = std::size_t{1} << nb;
  std::vector<std::size_t> base_pos(nb), extra_bit;
  std::vector<int> extra_q;
  for (std::size_t r = 0; r < nw; ++r) {
    const int q = wopen[r];
    const std::size_t bit = std::size_t{1} << (nw - 1 - r);
    const auto it = std::find(base_open.begin(), base_open.end(), q);
    if (it == base_open.end()) {
      extra_q.push_back(q);
      extra_bit.push_back(bit);
    } else {
      base_pos[static_cast<std::size_t>(it - base_open.begin())] = bit;  // base r-th smallest <-> batch bit nb-1-r
    }
  }
  std::vector<std::size_t> scatter(per);  // wide-index part of each base batch index
  for (std::size_t j = 0; j < per; ++j) {
    std::size_t idx = 0;
    for (std::size_t r = 0; r < nb; ++r)
      if ((j >> (nb - 1 - r)) & 1) idx |= base_pos[r];
    scatter[j] = idx;
  }
  for (std::size_t t = 0; t < nx1; ++t) {
    std::size_t fixed = 0;
    for (std::size_t e = 0; e < extra_q.size(); ++e)
      if (draw(t)[extra_q[e]] == 1) fixed |= extra_bit[e];
    double* out = amps_out + 2 * t * per;
    for (std::size_t j = 0; j < per; ++j) {
      const cdouble a = amps[fixed | scatter[j]];
      out[2 * j] = a.real();
      out[2 * j + 1] = a.imag();
    }
    if (bits_out) {
      const std::vector<int> x1(draw(t), draw(t) + n);
      for (std::size_t j = 0; j < per; ++j) {
        const std::string b = merge_bits(x1, base_open, j);
        std::memcpy(bits_out + (t * per + j) * static_cast<std::size_t>(n), b.data(), static_cast<std::size_t>(n));
      }
    }
  }
}

void amplitude_batches_into(Engine& wide, const std::vector<int>& base_open, const int* x1_list, std::size_t nx1,
                            const std::vector<std::int64_t>& slice_ids, double* amps_out, char* bits_out) {
  amplitude_batches_submit(wide, base_open, x1_list, nx1, slice_ids, 0);
  amplitude_batches_collect(wide, base_open, x1_list, nx1, 0, amps_out, bits_out);
}

std::vector<std::vector<std::pair<std::string, cdouble>>> amplitude_batches(
    Engine& wide, const std::vector<int>& base_open, const std::vector<std::vector<int>>& x1_list,
    const std::vector<std::int64_t>& slice_ids, bool with_bitstrings) {
  const int n = wide.circuit().num_qubits();
  std::vector<int> flat;
  flat.reserve(x1_list.size() * static_cast<std::size_t>(n));
  for (const auto& x1 : x1_list) {
    if (static_cast<int>(x1.size()) != n) throw std::invalid_argument("fold: bitstring length != qubit count");
    flat.insert(flat.end(), x1.begin(), x1.end());
  }
  const std::size_t per = std::size_t{1} << base_open.size();
  std::vector<double> amps(2 * per * x1_list.size());
  std::vector<char> bits(with_bitstrings ? per * x1_list.size() * static_cast<std::size_t>(n) : 0);
  amplitude_batches_into(wide, base_open, flat.data(), x1_list.size(), slice_ids, amps.data(),
                         with_bitstrings ? bits.data() : nullptr);
  std::vector<std::vector<std::pair<std::string, cdouble>>> out(x1_list.size());
  for (std::size_t t = 0; t < x1_list.size(); ++t) {
    out[t].reserve(per);
    for (std::size_t j = 0; j < per; ++j) {
      const std::size_t o = t * per + j;
      out[t].emplace_back(with_bitstrings ? std::string(bits.data() + o * static_cast<std::size_t>(n), static_cast<std::size_t>(n))
                                          : std::string(),
                          cdouble(amps[2 * o], amps[2 * o + 1]));
    }
  }
  return out;
}

AmplitudeOutput run_amplitudes(Engine& e, const std::vector<std::string>& bitstrings, Fraction f, std::uint64_t seed) {
  const int n = e.circuit().num_qubits();
  if (!e.plan().open_qubits.empty()) throw std::invalid_argument("run_amplitudes: plan must close every output");
  for (const auto& b : bitstrings)
    if (static_cast<int>(b.size()) != n) throw std::invalid_argument("bitstring length != qubit count: " + b);
  AmplitudeOutput out;
  out.slice_ids = select_slices(f, e.plan().num_slices, seed);
  for (const auto& b : bitstrings) {
    std::vector<int> bits(static_cast<std::size_t>(n));
    for (int q = 0; q < n; ++q) {
      if (b[static_cast<std::size_t>(q)] != '0' && b[static_cast<std::size_t>(q)] != '1')
        throw std::invalid_argument("bitstring: bad character");
      bits[static_cast<std::size_t>(q)] = b[static_cast<std::size_t>(q)] - '0';
    }
    e.prepare(bits);
    std::vector<cdouble> amps;
    try {
      e.run(out.slice_ids, true, false);
      e.results(&amps, nullptr);
    } catch (const std::exception& ex) {
      // The batch runs asynchronously; attribute the failure the way the
      // reference's schedule() does (lowest failing task): re-run the
      // slices one at a time, synchronously, and report the first that fails.
      const std::string first = ex.what();
      for (const auto id : out.slice_ids) {
        try {
          e.run({id}, true, false);
          e.synchronize();
        } catch (const std::exception& ex2) {
          throw JobError(ex2.what(), id);
        }
      }
      throw JobError(first, out.slice_ids.empty() ? -1 : out.slice_ids.front());
    }
    out.amplitudes.emplace_back(b, amps[0]);
    out.total_flops += e.plan().flops_per_slice * out.slice_ids.size();
  }
  return out;
}

}  // namespace qsg
