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
// Drop-in for contract_ttgt + normalize_inplace on host tensors
// (contraction.hpp:186 / tensor.hpp:209): labels -> small ints.
inline Tensorf contract_normalized(const Tensorf& l, const Tensorf& r, const std::vector<Label>& out_labels,
                                   FlopCounter* fc) {
  std::map<Label, int> id;
  auto ids = [&](const std::vector<Label>& ls) { std::vector<int> v; for (auto& x : ls) v.push_back(id.emplace(x, id.size()).first->second); return v; };
  auto li = ids(l.labels()), ri = ids(r.labels()), oi = ids(out_labels);
  std::vector<std::int64_t> od; for (auto& x : out_labels) od.push_back(l.has_label(x) ? l.dim(x) : r.dim(x));
  std::vector<cfloat> out(Tensorf::volume_from_dims(od));
  double scale = 0; std::uint64_t flops = 0;
  check(qsg_contract(l.rank(), li.data(), l.dims().data(), reinterpret_cast<const float*>(l.data().data()), l.log_scale(),
                     r.rank(), ri.data(), r.dims().data(), reinterpret_cast<const float*>(r.data().data()), r.log_scale(),
                     (int)oi.size(), oi.data(), reinterpret_cast<float*>(out.data()), &scale, &flops, 1));
  if (fc) fc->add(flops);
  return Tensorf(out_labels, od, std::move(out), scale);
}
}  // namespace qsim::qsg_backend
