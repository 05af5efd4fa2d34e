// Contraction plans: cut slicing, step annotation, the greedy planner, plan
// JSON I/O, the hand-crafted 7x7 region schedule, and slice selection.
//   cut grouping / slice ids   proj/src/plan.cpp:25-115
//   annotate_plan              proj/src/plan.cpp:122-210
//   greedy planner + cuts      proj/src/plan.cpp:212-353
//   plan JSON                  proj/src/plan.cpp:481-552
//   reference_plan_7x7         proj/src/plan.cpp:554-633
//   flop model Eq.(1)          include/qsim/contraction.hpp:43-56
//   fraction / select_slices   proj/src/engine.cpp:26-37, 285-298
#include <algorithm>
#include <limits>
#include <cmath>
#include <cstdio>
#include <map>
#include <set>
#include <tuple>

#include "json.hpp"
#include "qsg_host.hpp"

namespace qsg {

std::uint64_t flop_count(std::uint64_t v0, std::uint64_t v1, std::uint64_t v2) {
  const unsigned __int128 prod = static_cast<unsigned __int128>(v0) * v1 * v2;
  auto root = static_cast<std::uint64_t>(std::sqrt(static_cast<double>(prod)));
  while (root > 0 && static_cast<unsigned __int128>(root) * root > prod) --root;
  while (static_cast<unsigned __int128>(root + 1) * (root + 1) <= prod) ++root;
  if (static_cast<unsigned __int128>(root) * root != prod)
    throw std::invalid_argument("flop_count: volume product is not a perfect square");
  return 8 * root;
}

double log2_volume(const TensorShape& t) {
  double v = 0.0;
  for (auto d : t.dims) v += std::log2(static_cast<double>(d));
  return v;
}

std::int64_t step_working_set(std::int64_t l, std::int64_t r, std::int64_t o) {
  return l + r + o + std::max({l, r, o});
}

namespace {

std::string step_name(int i) {
  char buf[24];
  std::snprintf(buf, sizeof buf, "s%03d", i);
  return buf;
}

std::int64_t label_extent(const NetworkShape& s, const Label& l) {
  for (const auto& node : s.nodes)
    if (node.has_label(l)) return node.dim(l);
  throw std::invalid_argument("cut label " + l + " not in network");
}

}  // namespace

std::size_t cut_fixed_count(const NetworkShape& s, const Cut& cut) {
  if (cut.group <= 1) return cut.labels.size();
  std::int64_t acc = 1;
  std::size_t i = cut.labels.size();
  while (i > 0 && acc < cut.group) acc *= label_extent(s, cut.labels[--i]);
  if (acc != cut.group) throw std::invalid_argument("cut group does not divide the trailing multi-index");
  return i;
}

std::int64_t cut_slice_count(const NetworkShape& s, const Cut& cut) {
  const std::size_t fixed = cut_fixed_count(s, cut);
  std::int64_t count = 1;
  for (std::size_t i = 0; i < cut.labels.size(); ++i) {
    const std::int64_t d = label_extent(s, cut.labels[i]);
    if (i < fixed) count *= d;
  }
  return count;
}

std::vector<std::int64_t> cut_digits(const NetworkShape& s, const Cut& cut, std::int64_t slice_id) {
  const std::size_t fixed = cut_fixed_count(s, cut);
  std::vector<std::int64_t> radix(fixed);
  std::int64_t total = 1;
  for (std::size_t i = 0; i < cut.labels.size(); ++i) {
    const std::int64_t d = label_extent(s, cut.labels[i]);
    if (i < fixed) {
      radix[i] = d;
      total *= d;
    }
  }
  if (slice_id < 0 || slice_id >= total) throw std::out_of_range("apply_cut: slice_id out of range");
  std::vector<std::int64_t> digit(fixed, 0);
  for (std::size_t i = fixed; i-- > 0;) {
    digit[i] = slice_id % radix[i];
    slice_id /= radix[i];
  }
  return digit;
}

NetworkShape sliced_shape(const NetworkShape& s, const Cut& cut) {
  const std::size_t fixed = cut_fixed_count(s, cut);
  const std::set<Label> gone(cut.labels.begin(), cut.labels.begin() + static_cast<std::ptrdiff_t>(fixed));
  NetworkShape out = s;
  for (auto& node : out.nodes) {
    TensorShape kept;
    for (std::size_t i = 0; i < node.labels.size(); ++i)
      if (!gone.count(node.labels[i])) {
        kept.labels.push_back(node.labels[i]);
        kept.dims.push_back(node.dims[i]);
      }
    node = std::move(kept);
  }
  std::erase_if(out.bonds, [&](const BondRef& b) { return gone.count(b.label) > 0; });
  return out;
}

GridNetwork apply_cut(const GridNetwork& net, const Cut& cut, std::int64_t slice_id) {
  const NetworkShape shape = net.shape();
  const auto digit = cut_digits(shape, cut, slice_id);
  GridNetwork out = net;
  for (std::size_t i = 0; i < digit.size(); ++i) {
    const Label& l = cut.labels[i];
    for (auto& node : out.nodes) {
      if (!node.has_label(l)) continue;
      // Fix axis `ax` to digit[i] and drop it.
      const int ax = node.axis(l);
      std::int64_t outer = 1, inner = 1;
      for (int a = 0; a < ax; ++a) outer *= node.dims[static_cast<std::size_t>(a)];
      for (std::size_t a = static_cast<std::size_t>(ax) + 1; a < node.dims.size(); ++a) inner *= node.dims[a];
      const std::int64_t d = node.dims[static_cast<std::size_t>(ax)];
      std::vector<cfloat> kept;
      kept.reserve(static_cast<std::size_t>(outer * inner));
      for (std::int64_t o = 0; o < outer; ++o) {
        const cfloat* base = node.data.data() + (o * d + digit[i]) * inner;
        kept.insert(kept.end(), base, base + inner);
      }
      node.data.swap(kept);
      node.labels.erase(node.labels.begin() + ax);
      node.dims.erase(node.dims.begin() + ax);
    }
  }
  const std::set<Label> gone(cut.labels.begin(), cut.labels.begin() + static_cast<std::ptrdiff_t>(digit.size()));
  std::erase_if(out.bonds, [&](const BondRef& b) { return gone.count(b.label) > 0; });
  return out;
}

namespace {

// Labels of a pairwise product in (lhs-only, rhs-only) order.
TensorShape merge_free(const TensorShape& a, const TensorShape& b) {
  TensorShape out;
  for (std::size_t i = 0; i < a.labels.size(); ++i)
    if (!b.has_label(a.labels[i])) {
      out.labels.push_back(a.labels[i]);
      out.dims.push_back(a.dims[i]);
    }
  for (std::size_t i = 0; i < b.labels.size(); ++i)
    if (!a.has_label(b.labels[i])) {
      out.labels.push_back(b.labels[i]);
      out.dims.push_back(b.dims[i]);
    }
  return out;
}

TensorShape sorted_shape(const TensorShape& t) {
  std::vector<std::size_t> idx(t.labels.size());
  for (std::size_t i = 0; i < idx.size(); ++i) idx[i] = i;
  std::sort(idx.begin(), idx.end(), [&](std::size_t x, std::size_t y) { return t.labels[x] < t.labels[y]; });
  TensorShape s;
  for (auto i : idx) {
    s.labels.push_back(t.labels[i]);
    s.dims.push_back(t.dims[i]);
  }
  return s;
}

}  // namespace

void annotate_plan(const NetworkShape& shape, ContractionPlan& plan) {
  const NetworkShape sliced = sliced_shape(shape, plan.cut);
  plan.num_slices = cut_slice_count(shape, plan.cut);
  plan.open_qubits = shape.open_qubits;

  std::map<std::string, TensorShape> live;
  for (std::size_t q = 0; q < sliced.nodes.size(); ++q) live[node_name(static_cast<int>(q))] = sliced.nodes[q];

  plan.flops_per_slice = 0;
  plan.peak_memory = 0;
  plan.max_rank = 0;
  std::int64_t live_bytes = 0;
  for (const auto& [name, t] : live) {
    plan.max_rank = std::max(plan.max_rank, static_cast<int>(t.labels.size()));
    live_bytes += t.bytes();
  }

  for (auto& step : plan.steps) {
    auto li = live.find(step.lhs);
    auto ri = live.find(step.rhs);
    if (li == live.end() || ri == live.end())
      throw std::invalid_argument("plan: step operand missing or already consumed: " + step.lhs + " x " + step.rhs);
    if (live.count(step.out)) throw std::invalid_argument("plan: duplicate tensor " + step.out);
    const TensorShape& a = li->second;
    const TensorShape& b = ri->second;
    TensorShape out = sorted_shape(merge_free(a, b));
    // Overflow guard: the reference silently wraps int64
    // volumes / uint64 flops here for large greedy plans.  Reject instead.
    const double lo = log2_volume(out), la = log2_volume(a), lb = log2_volume(b);
    if (lo >= 59.0)
      throw std::length_error("plan: step " + step.out + " has rank " + std::to_string(out.labels.size()) +
                              ": volume 2^" + std::to_string(static_cast<int>(lo)) + " overflows int64 bytes");
    if (3.0 + 0.5 * (la + lb + lo) >= 63.0)
      throw std::length_error("plan: step " + step.out + " flops overflow uint64");

    step.out_labels = out.labels;
    step.out_volume = out.volume();
    step.flops = flop_count(static_cast<std::uint64_t>(a.volume()), static_cast<std::uint64_t>(b.volume()),
                            static_cast<std::uint64_t>(out.volume()));
    step.intensity = static_cast<double>(step.flops) /
                     static_cast<double>(8 * (a.volume() + b.volume() + out.volume()));
    step.working_set = step_working_set(a.bytes(), b.bytes(), out.bytes());
    const std::int64_t scratch = std::max({a.bytes(), b.bytes(), out.bytes()});
    plan.peak_memory = std::max(plan.peak_memory, live_bytes + out.bytes() + scratch);
    plan.flops_per_slice += step.flops;
    plan.max_rank = std::max(plan.max_rank, static_cast<int>(out.labels.size()));

    live_bytes += out.bytes() - a.bytes() - b.bytes();
    live.erase(step.lhs);
    live.erase(step.rhs);
    live[step.out] = std::move(out);
  }

  if (live.size() != 1)
    throw std::invalid_argument("plan: steps leave " + std::to_string(live.size()) + " tensors, expected 1");
  plan.final_tensor = live.begin()->first;
  std::vector<Label> want;
  for (int q : shape.open_qubits) want.push_back(open_label(q));
  std::sort(want.begin(), want.end());
  if (live.begin()->second.labels != want)
    throw std::invalid_argument("plan: final tensor does not match the open qubits");
  if (plan.peak_memory == 0) plan.peak_memory = live_bytes;
}

ContractionPlan reassociate_plan(const NetworkShape& shape, const ContractionPlan& in, int* rewrites) {
  ContractionPlan p = in;
  annotate_plan(shape, p);
  const NetworkShape sliced = sliced_shape(shape, p.cut);
  auto flops_of = [](const TensorShape& a, const TensorShape& b, const TensorShape& o) {
    return std::exp2(3.0 + 0.5 * (log2_volume(a) + log2_volume(b) + log2_volume(o)));
  };
  int count = 0, fresh = 0;
  for (bool changed = true; changed;) {
    changed = false;
    std::map<std::string, TensorShape> shp;
    for (std::size_t q = 0; q < sliced.nodes.size(); ++q) shp[node_name(static_cast<int>(q))] = sliced.nodes[q];
    for (const auto& st : p.steps) shp[st.out] = sorted_shape(merge_free(shp.at(st.lhs), shp.at(st.rhs)));
    for (std::size_t i = 0; i < p.steps.size() && !changed; ++i) {
      const PlanStep& si = p.steps[i];
      std::size_t j = i + 1;
      while (j < p.steps.size() && p.steps[j].lhs != si.out && p.steps[j].rhs != si.out) ++j;
      if (j == p.steps.size()) continue;  // the final tensor
      const std::string c = p.steps[j].lhs == si.out ? p.steps[j].rhs : p.steps[j].lhs;
      const TensorShape& T = shp.at(si.out);
      const TensorShape& U = shp.at(p.steps[j].out);
      const double old_cost = flops_of(shp.at(si.lhs), shp.at(si.rhs), T) + flops_of(T, shp.at(c), U);
      double best = old_cost;
      std::string keep, join;
      for (int side = 0; side < 2; ++side) {
        const std::string& x = side == 0 ? si.lhs : si.rhs;  // stays, meets W last
        const std::string& y = side == 0 ? si.rhs : si.lhs;  // joins c first
        const TensorShape W = sorted_shape(merge_free(shp.at(y), shp.at(c)));
        if (log2_volume(W) > std::max(log2_volume(T), log2_volume(U))) continue;  // no larger intermediates
        const double cost = flops_of(shp.at(y), shp.at(c), W) + flops_of(shp.at(x), W, U);
        if (cost < best) {
          best = cost;
          keep = x;
          join = y;
        }
      }
      if (keep.empty() || best > 0.75 * old_cost) continue;
      PlanStep w, u;
      w.out = "r" + std::to_string(fresh++);
      w.lhs = join;
      w.rhs = c;
      u.out = p.steps[j].out;
      u.lhs = keep;
      u.rhs = w.out;
      p.steps[j] = u;
      p.steps.insert(p.steps.begin() + static_cast<std::ptrdiff_t>(j), w);
      p.steps.erase(p.steps.begin() + static_cast<std::ptrdiff_t>(i));
      ++count;
      changed = true;
    }
  }
  // Positional names, as plan_from_json assigns them.
  std::map<std::string, std::string> rename;
  for (std::size_t i = 0; i < p.steps.size(); ++i) rename[p.steps[i].out] = step_name(static_cast<int>(i));
  auto ren = [&](const std::string& n) {
    auto it = rename.find(n);
    return it == rename.end() ? n : it->second;
  };
  for (auto& st : p.steps) {
    st.lhs = ren(st.lhs);
    st.rhs = ren(st.rhs);
    st.out = ren(st.out);
  }
  annotate_plan(shape, p);
  if (rewrites) *rewrites = count;
  return p;
}

namespace {

// Greedy pairing by (result volume, Eq.1 flops, lexicographic names);
// deterministic in the shape (proj/src/plan.cpp:214-281).
std::vector<PlanStep> greedy_steps(const NetworkShape& shape) {
  std::vector<std::pair<std::string, TensorShape>> pool;
  for (std::size_t q = 0; q < shape.nodes.size(); ++q) pool.emplace_back(node_name(static_cast<int>(q)), shape.nodes[q]);
  std::vector<PlanStep> steps;
  int next = 0;
  // Candidate cost: exact (volume, flops) while they fit (the reference's
  // keys, so small plans are identical); past 2^60 elements the reference
  // wraps int64 / uint128 -- here such candidates sort after every exact
  // one, by log2 volume then log2 flops (overflow fix).
  struct Cost {
    bool big = false;
    double lvol = 0.0, lfl = 0.0;
    std::int64_t vol = 0;
    std::uint64_t fl = 0;
  };
  auto less = [](const Cost& x, const Cost& y) -> int {  // -1: x cheaper, 1: y cheaper, 0: tie
    if (x.big != y.big) return x.big ? 1 : -1;
    if (!x.big) return std::tie(x.vol, x.fl) < std::tie(y.vol, y.fl) ? -1 : (std::tie(y.vol, y.fl) < std::tie(x.vol, x.fl) ? 1 : 0);
    return std::tie(x.lvol, x.lfl) < std::tie(y.lvol, y.lfl) ? -1 : (std::tie(y.lvol, y.lfl) < std::tie(x.lvol, x.lfl) ? 1 : 0);
  };
  while (pool.size() > 1) {
    bool have = false;
    Cost best;
    std::pair<std::string, std::string> best_key;
    std::size_t bi = 0, bj = 0;
    for (std::size_t i = 0; i < pool.size(); ++i)
      for (std::size_t j = i + 1; j < pool.size(); ++j) {
        const TensorShape m = merge_free(pool[i].second, pool[j].second);
        Cost c;
        c.lvol = log2_volume(m);
        const double la = log2_volume(pool[i].second), lb = log2_volume(pool[j].second);
        c.lfl = 3.0 + 0.5 * (la + lb + c.lvol);
        c.big = c.lvol >= 60.0 || la >= 60.0 || lb >= 60.0 || c.lfl >= 63.0;
        if (!c.big) {
          c.vol = m.volume();
          c.fl = flop_count(static_cast<std::uint64_t>(pool[i].second.volume()),
                            static_cast<std::uint64_t>(pool[j].second.volume()), static_cast<std::uint64_t>(c.vol));
        }
        auto names = std::minmax(pool[i].first, pool[j].first);
        std::pair<std::string, std::string> key{names.first, names.second};
        const int cmp = have ? less(c, best) : -1;
        if (cmp < 0 || (cmp == 0 && key < best_key)) {
          have = true;
          best = c;
          best_key = key;
          bi = i;
          bj = j;
        }
      }
    PlanStep st;
    st.lhs = best_key.first;
    st.rhs = best_key.second;
    st.out = step_name(next++);
    TensorShape merged = merge_free(pool[bi].second, pool[bj].second);
    if (bj > bi) std::swap(bi, bj);
    pool.erase(pool.begin() + static_cast<std::ptrdiff_t>(bi));
    pool.erase(pool.begin() + static_cast<std::ptrdiff_t>(bj));
    pool.emplace_back(st.out, std::move(merged));
    steps.push_back(std::move(st));
  }
  return steps;
}

ContractionPlan greedy_plan(const NetworkShape& shape, const Cut& cut) {
  ContractionPlan p;
  p.cut = cut;
  p.steps = greedy_steps(sliced_shape(shape, cut));
  annotate_plan(shape, p);
  return p;
}

// For the budgeted cut search: a greedy plan whose sizes overflow (the
// reference would wrap) counts as infinitely large instead of aborting the
// search, so cuts can still bring it under the budget.
ContractionPlan greedy_plan_or_huge(const NetworkShape& shape, const Cut& cut) {
  try {
    return greedy_plan(shape, cut);
  } catch (const std::length_error&) {
    ContractionPlan p;
    p.cut = cut;
    p.peak_memory = std::numeric_limits<std::int64_t>::max();
    return p;
  }
}

}  // namespace

ContractionPlan plan_contraction(const NetworkShape& shape, const PlanOptions& opts) {
  if (opts.memory_budget > 0) {
    std::int64_t biggest = 0;
    for (const auto& node : shape.nodes) biggest = std::max(biggest, node.bytes());
    if (opts.memory_budget < biggest) throw std::invalid_argument("memory budget below the largest node tensor");
  }
  if (opts.memory_budget <= 0) return greedy_plan(shape, Cut{});
  ContractionPlan plan = greedy_plan_or_huge(shape, Cut{});
  if (plan.peak_memory <= opts.memory_budget) return plan;

  Cut cut;
  while (static_cast<int>(cut.labels.size()) < opts.max_cut_labels) {
    std::set<Label> taken(cut.labels.begin(), cut.labels.end()), candidates;
    for (const auto& b : shape.bonds)
      if (!taken.count(b.label)) candidates.insert(b.label);
    bool found = false;
    ContractionPlan best;
    Label best_label;
    for (const auto& l : candidates) {
      Cut trial = cut;
      trial.labels.push_back(l);
      ContractionPlan p = greedy_plan_or_huge(shape, trial);
      if (!found || p.peak_memory < best.peak_memory) {
        found = true;
        best = std::move(p);
        best_label = l;
      }
    }
    if (!found || best.peak_memory >= plan.peak_memory)
      throw std::runtime_error("no plan found under the memory budget; add cuts");
    cut.labels.push_back(best_label);
    plan = std::move(best);
    if (plan.peak_memory <= opts.memory_budget) break;
  }
  if (plan.peak_memory > opts.memory_budget) throw std::runtime_error("no plan found under the memory budget; add cuts");
  while (!cut.labels.empty()) {
    Cut trial = cut;
    // Each round multiplies the group by the last cut label's extent
    // (proj/src/plan.cpp:341-351).
    trial.group *= label_extent(shape, trial.labels.back());
    ContractionPlan p = greedy_plan_or_huge(shape, trial);
    if (p.peak_memory > opts.memory_budget) break;
    cut = trial;
    plan = std::move(p);
    if (cut_fixed_count(shape, cut) == 0) break;
  }
  return plan;
}

std::string plan_to_json(const ContractionPlan& plan) {
  using json::Value;
  auto int_array = [](const auto& v) {
    Value a = Value::make_array();
    for (auto x : v) a.push(Value::make_int(static_cast<std::int64_t>(x)));
    return a;
  };
  auto str_array = [](const std::vector<Label>& v) {
    Value a = Value::make_array();
    for (const auto& x : v) a.push(Value::make_string(x));
    return a;
  };
  Value j = Value::make_object();
  j.set("version", Value::make_int(1));
  j.set("open_qubits", int_array(plan.open_qubits));
  Value cut = Value::make_object();
  cut.set("labels", str_array(plan.cut.labels));
  cut.set("group", Value::make_int(plan.cut.group));
  j.set("cut", cut);
  j.set("slices", Value::make_int(plan.num_slices));
  Value order = Value::make_array();
  for (const auto& s : plan.steps) {
    Value pair = Value::make_array();
    pair.push(Value::make_string(s.lhs));
    pair.push(Value::make_string(s.rhs));
    order.push(pair);
  }
  j.set("order", order);
  Value steps = Value::make_array();
  for (const auto& s : plan.steps) {
    Value o = Value::make_object();
    o.set("out", Value::make_string(s.out));
    o.set("lhs", Value::make_string(s.lhs));
    o.set("rhs", Value::make_string(s.rhs));
    o.set("out_labels", str_array(s.out_labels));
    o.set("volume", Value::make_int(s.out_volume));
    o.set("flops", Value::make_int(static_cast<std::int64_t>(s.flops)));
    o.set("intensity", Value::make_double(s.intensity));
    o.set("working_set", Value::make_int(s.working_set));
    steps.push(o);
  }
  j.set("steps", steps);
  Value per = Value::make_object();
  per.set("flops", Value::make_int(static_cast<std::int64_t>(plan.flops_per_slice)));
  per.set("peak_memory", Value::make_int(plan.peak_memory));
  per.set("max_rank", Value::make_int(plan.max_rank));
  j.set("per_slice", per);
  return json::dump(j) + "\n";
}

std::vector<int> plan_json_open_qubits(const std::string& text) {
  const json::Value j = json::parse(text);
  std::vector<int> open;
  if (j.has("open_qubits"))
    for (const auto& v : j.at("open_qubits").arr) open.push_back(static_cast<int>(v.as_int()));
  return open;
}

ContractionPlan plan_from_json(const std::string& text, const NetworkShape& shape) {
  const json::Value j = json::parse(text);
  ContractionPlan plan;
  if (j.has("cut")) {
    for (const auto& v : j.at("cut").at("labels").arr) plan.cut.labels.push_back(v.as_string());
    if (j.at("cut").has("group")) plan.cut.group = j.at("cut").at("group").as_int();
  }
  if (j.has("open_qubits")) {
    std::vector<int> open;
    for (const auto& v : j.at("open_qubits").arr) open.push_back(static_cast<int>(v.as_int()));
    if (open != shape.open_qubits) throw std::invalid_argument("plan open qubits do not match the network");
  }
  int idx = 0;
  for (const auto& pair : j.at("order").arr) {
    PlanStep s;
    s.lhs = pair.at(0).as_string();
    s.rhs = pair.at(1).as_string();
    s.out = step_name(idx++);
    plan.steps.push_back(std::move(s));
  }
  annotate_plan(shape, plan);
  if (j.has("slices") && j.at("slices").as_int() != plan.num_slices)
    throw std::invalid_argument("plan slice count does not match its cut");
  return plan;
}

std::vector<int> reference_open_qubits_7x7() { return {33, 34, 40, 41, 47, 48}; }

ContractionPlan reference_plan_7x7(const NetworkShape& shape) {
  if (shape.rows != 7 || shape.cols != 7) throw std::invalid_argument("reference plan: network is not a 7x7 grid");
  if (shape.open_qubits != reference_open_qubits_7x7())
    throw std::invalid_argument("reference plan: open qubits must be the corner region");
  auto first_bonds = [&](int a, int b, std::size_t k) {
    std::vector<BondRef> on_edge;
    for (const auto& bond : shape.bonds)
      if ((bond.q0 == a && bond.q1 == b) || (bond.q0 == b && bond.q1 == a)) on_edge.push_back(bond);
    std::sort(on_edge.begin(), on_edge.end(), [](const BondRef& x, const BondRef& y) { return x.cycle < y.cycle; });
    if (on_edge.size() < k) throw std::invalid_argument("reference plan: edge has too few bonds");
    std::vector<Label> out;
    for (std::size_t i = 0; i < k; ++i) out.push_back(on_edge[i].label);
    return out;
  };
  ContractionPlan plan;
  for (auto [a, b, k] : {std::tuple{21, 28, 3}, std::tuple{22, 29, 2}, std::tuple{3, 4, 5}})
    for (const auto& l : first_bonds(a, b, static_cast<std::size_t>(k))) plan.cut.labels.push_back(l);

  // Regions: A = cols 0..3 x rows 0..3 column-major, D = cols 6..4 x rows
  // 0..3, merge; B = rows 4..6 of cols 0..2 column-major then col 3
  // bottom-up, merge; then the column-4 strip and the open corner.
  const std::vector<int> region_a = {0, 7, 14, 21, 1, 8, 15, 22, 2, 9, 16, 23, 3, 10, 17, 24};
  const std::vector<int> region_d = {6, 13, 20, 27, 5, 12, 19, 26, 4, 11, 18, 25};
  const std::vector<int> region_b = {28, 35, 42, 29, 36, 43, 30, 37, 44, 45, 38, 31};
  const std::vector<int> tail = {32, 39, 46, 33, 34, 40, 41, 47, 48};
  int idx = 0;
  auto push = [&](const std::string& l, const std::string& r) {
    PlanStep s;
    s.lhs = l;
    s.rhs = r;
    s.out = step_name(idx++);
    plan.steps.push_back(s);
    return s.out;
  };
  auto chain = [&](const std::vector<int>& nodes) {
    std::string acc = node_name(nodes[0]);
    for (std::size_t i = 1; i < nodes.size(); ++i) acc = push(acc, node_name(nodes[i]));
    return acc;
  };
  const std::string a = chain(region_a);
  const std::string d = chain(region_d);
  const std::string ad = push(a, d);
  const std::string b = chain(region_b);
  std::string acc = push(ad, b);
  for (int q : tail) acc = push(acc, node_name(q));
  annotate_plan(shape, plan);
  return plan;
}

Fraction parse_fraction(const std::string& text) {
  const auto slash = text.find('/');
  if (slash == std::string::npos) throw std::invalid_argument("fraction must look like k/K: " + text);
  Fraction f;
  f.num = std::stoll(text.substr(0, slash));
  f.den = std::stoll(text.substr(slash + 1));
  if (f.den < 1 || f.num < 1 || f.num > f.den) throw std::invalid_argument("fraction out of range: " + text);
  return f;
}

std::vector<std::int64_t> select_slices(Fraction f, std::int64_t num_slices, std::uint64_t seed) {
  if (f.den != num_slices)
    throw std::invalid_argument("fraction denominator " + std::to_string(f.den) + " does not match the plan's " +
                                std::to_string(num_slices) + " slices");
  const auto offset = static_cast<std::int64_t>(mix_seed(seed, 0x51ce) % static_cast<std::uint64_t>(num_slices));
  std::vector<std::int64_t> ids;
  for (std::int64_t i = 0; i < f.num; ++i) ids.push_back((offset + i) % num_slices);
  std::sort(ids.begin(), ids.end());
  return ids;
}

std::string merge_bits(const std::vector<int>& x1_bits, const std::vector<int>& open_sorted,
                       std::size_t batch_index) {
  std::string s(x1_bits.size(), '0');
  for (std::size_t q = 0; q < x1_bits.size(); ++q)
    if (x1_bits[q] >= 0) s[q] = static_cast<char>('0' + x1_bits[q]);
  const std::size_t k = open_sorted.size();
  for (std::size_t r = 0; r < k; ++r)
    s[static_cast<std::size_t>(open_sorted[r])] = static_cast<char>('0' + ((batch_index >> (k - 1 - r)) & 1));
  return s;
}

}  // namespace qsg
