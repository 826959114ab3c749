// weavesim/scheduler.hpp -- drop-in subset of the reference scheduler API
// (proj/include/weavesim/scheduler.hpp:15-19): the baseline modes a caller
// selects.  The analytic event simulator itself is not re-implemented -- the
// B200 build RUNS layers (include/tw/tw_weave.h).
#pragma once

#include <string>

namespace weavesim {

enum class BaselineMode { Default, Multimem, NoComm, FuseOnly, TokenWeave };

const char* to_string(BaselineMode mode);
// ConfigError on an unknown name (proj/src/scheduler.cpp:38-45).
BaselineMode baseline_mode_from_string(const std::string& name);

}  // namespace weavesim
