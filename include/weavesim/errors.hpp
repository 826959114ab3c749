// weavesim/errors.hpp -- drop-in exception taxonomy of the reference operator
// API (same names and bases as proj/include/weavesim/errors.hpp:8-31).  The
// C-ABI status codes of include/tw/tw.h map onto these one to one.
#pragma once

#include <stdexcept>
#include <string>

namespace weavesim {

#define WEAVESIM_DEFINE_ERROR(Name)                                    \
  struct Name : std::runtime_error {                                   \
    explicit Name(const std::string& what) : std::runtime_error(what) {} \
  }

WEAVESIM_DEFINE_ERROR(DimensionError);    // shapes, weight length, shard shapes
WEAVESIM_DEFINE_ERROR(NumericError);      // NaN/Inf inputs, negative epsilon
WEAVESIM_DEFINE_ERROR(ConfigError);       // world size < 2, bad profile/policy
WEAVESIM_DEFINE_ERROR(ContractError);     // malformed shard maps
WEAVESIM_DEFINE_ERROR(CalibrationError);  // (kept for source compatibility)
WEAVESIM_DEFINE_ERROR(ParseError);        // (kept for source compatibility)
// B200 build only: CUDA/driver failure or a cross-rank barrier timeout.
WEAVESIM_DEFINE_ERROR(DeviceError);

#undef WEAVESIM_DEFINE_ERROR

}  // namespace weavesim
