// integration/qsg_backend.hpp -> proj/include/qsim/qsg_backend.hpp (new file in the reference tree;
// compiled against the reference headers and linked by tests/test_abi.py)
#pragma once
#include <qsg.h>

#include <cstdint>
#include <map>
#include <stdexcept>
#include <vector>

#include "qsim/tensor.hpp"
#include "qsim/contraction.hpp"
namespace qsim::qsg_backend {
inline void check(int rc) {
  if (rc == QSG_OK) return;
  const char* m = qsg_last_error();
  switch (rc) {
    case QSG_ERR_INVALID_ARGUMENT: throw std::invalid_argument(m);
    case QSG_ERR_LENGTH: throw std::length_error(m);
    case QSG_ERR_OUT_OF_RANGE: throw std::out_of_range(m);
    default: throw std::runtime_error(m);
  }
}
// Drop-in for contract_ttgt (contraction.hpp:186), followed by
// normalize_inplace (tensor.hpp:209) when `normalize`, on host tensors:
// labels -> small ints; the contraction runs on the GPU.
inline Tensorf contract(const Tensorf& l, const Tensorf& r, const std::vector<Label>& out_labels, FlopCounter* fc,
                        bool normalize) {
  std::map<Label, int> id;
  auto ids = [&](const std::vector<Label>& ls) { std::vector<int> v; for (auto& x : ls) v.push_back(id.emplace(x, id.size()).first->second); return v; };
  auto li = ids(l.labels()), ri = ids(r.labels()), oi = ids(out_labels);
  std::vector<std::int64_t> od; for (auto& x : out_labels) od.push_back(l.has_label(x) ? l.dim(x) : r.dim(x));
  std::vector<cfloat> out(Tensorf::volume_from_dims(od));
  double scale = 0; std::uint64_t flops = 0;
  check(qsg_contract(l.rank(), li.data(), l.dims().data(), reinterpret_cast<const float*>(l.data().data()), l.log_scale(),
                     r.rank(), ri.data(), r.dims().data(), reinterpret_cast<const float*>(r.data().data()), r.log_scale(),
                     (int)oi.size(), oi.data(), reinterpret_cast<float*>(out.data()), &scale, &flops, normalize ? 1 : 0));
  if (fc) fc->add(flops);
  return Tensorf(out_labels, od, std::move(out), scale);
}
inline Tensorf contract_normalized(const Tensorf& l, const Tensorf& r, const std::vector<Label>& out_labels,
                                   FlopCounter* fc) {
  return contract(l, r, out_labels, fc, true);
}
}  // namespace qsim::qsg_backend
