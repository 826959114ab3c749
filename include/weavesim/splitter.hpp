// weavesim/splitter.hpp -- drop-in token-split planner of the weave
// (proj/include/weavesim/splitter.hpp:11-56): same types, semantics and
// errors.  smart_offset_sweep's callback is, on B200, a MEASURED weaved-layer
// time (tw::weave::LayerRunner), the paper's Algorithm 1.
#pragma once

#include <cstdint>
#include <functional>
#include <vector>

#include "weavesim/wavemodel.hpp"

namespace weavesim {

enum class SplitMode { NoSplit, FusedOnly, Overlap };

struct SplitPlan {
  std::int64_t total_tokens = 0;
  std::int64_t prefix_tokens = 0;
  std::int64_t suffix_tokens = 0;
  std::int64_t offset = 0;  // signed, relative to T/2
  SplitMode mode = SplitMode::NoSplit;
  std::vector<std::int64_t> prefix_len_per_sequence;
};

struct SplitPolicy {
  std::int64_t threshold_tokens = 1024;  // 1K dense, 4K MoE
  std::vector<std::int64_t> offset_grid = {0, 64, 128, 192, 256, 512};
};

SplitMode select_mode(std::int64_t num_tokens, const SplitPolicy& policy);
std::int64_t smart_offset_analytic(std::int64_t num_tokens, const HardwareProfile& profile);
std::int64_t smart_offset_sweep(std::int64_t num_tokens, const SplitPolicy& policy,
                                const std::function<double(std::int64_t, std::int64_t)>& forward);
SplitPlan make_split_plan(std::int64_t num_tokens, const HardwareProfile& profile, const SplitPolicy& policy);
SplitPlan place_sequence_boundaries(const std::vector<std::int64_t>& sequence_lengths, SplitPlan plan);

}  // namespace weavesim
