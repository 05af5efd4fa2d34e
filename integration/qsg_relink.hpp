// integration/qsg_relink.hpp -- relinks the reference's UNMODIFIED
// execute_slice (proj/src/engine.cpp:182-245) onto the B200 contraction.
//
// Force-included ahead of proj/src/engine.cpp (`g++ -include qsg_relink.hpp`,
// oracle/Makefile target libqsim_relink.so): the non-template overload
// below is an exact match for the call `contract_ttgt(a, b, spec,
// opts.counter)` at src/engine.cpp:227 (and the pipeline's at :144), so
// overload resolution prefers it to the header template
// (include/qsim/contraction.hpp:186) and every contraction of the
// reference's own step loop runs through qsg_contract on the GPU, while
// the fold, cut, live map and normalize_inplace stay the reference's.
#pragma once
#include "qsim/contraction.hpp"
#include "qsim/tensor.hpp"
#include "qsg_backend.hpp"

namespace qsim {
inline Tensorf contract_ttgt(const Tensorf& l, const Tensorf& r, const ContractionSpec& spec, FlopCounter* fc) {
  return qsg_backend::contract(l, r, spec.output_labels, fc, /*normalize=*/false);
}
}  // namespace qsim
