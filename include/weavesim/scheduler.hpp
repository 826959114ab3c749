// weavesim/scheduler.hpp -- drop-in subset of the reference scheduler API
// (proj/include/weavesim/scheduler.hpp:15-19): the baseline modes a caller
// selects.  The analytic event simulator itself is not re-implemented -- the
// B200 build RUNS layers (include/tw/tw_weave.h).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "weavesim/splitter.hpp"
#include "weavesim/wavemodel.hpp"

namespace weavesim {

enum class BaselineMode { Default, Multimem, NoComm, FuseOnly, TokenWeave };

const char* to_string(BaselineMode mode);
// ConfigError on an unknown name (proj/src/scheduler.cpp:38-45).
BaselineMode baseline_mode_from_string(const std::string& name);

// Shape of one iteration's batch (proj/include/weavesim/scheduler.hpp:46-52).
struct BatchShape {
  std::int64_t total_tokens = 0;
  std::int64_t kv_context = 0;  // prior-context tokens (sum over sequences)
  bool decode_only = false;
  std::vector<std::int64_t> sequence_lengths;  // optional; empty = single sequence
};

// The reference's signature (scheduler.hpp:79-81).  B200 build: the layer is
// RUN on this GPU (one GPU's share at spec.tp_degree; the mode mapping and
// the TokenWeave degrade rules of simulate_throughput, workloads.hpp) and the
// result is the measured per-layer time x spec.num_layers, in seconds.
double iteration_latency(const BatchShape& batch, const LayerSpec& spec, const HardwareProfile& profile,
                         BaselineMode mode, const SplitPolicy& policy);

}  // namespace weavesim
