// weavesim_splitter.cpp -- the weave's token-split planner (host C++), same
// semantics and errors as the reference planner:
//   cta_count / wave_count          proj/src/wavemodel.cpp:38-49
//   HardwareProfile::validate       proj/src/wavemodel.cpp:8-21
//   select_mode                     proj/src/splitter.cpp:11-14
//   smart_offset_analytic           proj/src/splitter.cpp:16-53
//   smart_offset_sweep (Alg. 1)     proj/src/splitter.cpp:55-69
//   make_split_plan                 proj/src/splitter.cpp:71-88
//   place_sequence_boundaries       proj/src/splitter.cpp:90-105
// Parity: tests/test_weave.py checks every plan against the oracle
// restatement and the golden plans generated from the reference.
#include <algorithm>
#include <cstdlib>
#include <limits>

#include "weavesim/errors.hpp"
#include "weavesim/splitter.hpp"
#include "weavesim/wavemodel.hpp"

namespace weavesim {

void HardwareProfile::validate() const {
  if (num_sms < 1) throw ConfigError("HardwareProfile: num_sms must be >= 1");
  if (collective_sms >= num_sms) throw ConfigError("HardwareProfile: collective_sms must be < num_sms");
  if (tile_tokens < 1 || cta_columns < 1) throw ConfigError("HardwareProfile: tile geometry must be positive");
  const bool rates_ok = sm_flops > 0 && hbm_bandwidth_effective > 0 && collective_per_token_time > 0 &&
                        collective_base_latency > 0;
  if (!rates_ok) throw ConfigError("HardwareProfile: rates and latencies must be positive");
}

HardwareProfile b200_geometry() {
  HardwareProfile p;
  p.name = "b200";
  p.num_sms = 148;
  p.sm_flops = 8.4e12;
  return p;
}

std::int64_t cta_count(std::int64_t num_tokens, const HardwareProfile& profile) {
  if (num_tokens < 0) throw DimensionError("cta_count: negative token count");
  const std::int64_t tiles = (num_tokens + profile.tile_tokens - 1) / profile.tile_tokens;
  return tiles * profile.cta_columns;
}

std::int64_t wave_count(std::int64_t ctas, std::int64_t sms_available) {
  if (sms_available < 1) throw ConfigError("wave_count: sms_available must be >= 1");
  if (ctas < 0) throw DimensionError("wave_count: negative CTA count");
  return ctas == 0 ? 0 : (ctas - 1) / sms_available + 1;
}

SplitMode select_mode(std::int64_t num_tokens, const SplitPolicy& policy) {
  if (policy.threshold_tokens < 1) throw ConfigError("SplitPolicy: threshold must be >= 1");
  return num_tokens < policy.threshold_tokens ? SplitMode::FusedOnly : SplitMode::Overlap;
}

namespace {

std::int64_t split_waves(std::int64_t prefix, std::int64_t total, const HardwareProfile& p) {
  return wave_count(cta_count(prefix, p), p.num_sms) + wave_count(cta_count(total - prefix, p), p.num_sms);
}

}  // namespace

std::int64_t smart_offset_analytic(std::int64_t num_tokens, const HardwareProfile& profile) {
  profile.validate();
  if (num_tokens < 0) throw DimensionError("smart_offset_analytic: negative token count");
  const std::int64_t half = num_tokens / 2;
  const std::int64_t degenerate = num_tokens - half;  // everything in the prefix
  const std::int64_t tiles = (num_tokens + profile.tile_tokens - 1) / profile.tile_tokens;
  if (wave_count(cta_count(num_tokens, profile), profile.num_sms) <= 1 || tiles < 2) return degenerate;

  // Candidates: the equal split first, then every row-tile boundary.  Keep the
  // fewest total waves; on a tie prefer the candidate closest to T/2 (the
  // earliest such candidate wins, so an equal-wave result stays balanced).
  struct Best {
    std::int64_t prefix, waves, imbalance;
  } best{half, std::numeric_limits<std::int64_t>::max(), std::numeric_limits<std::int64_t>::max()};
  auto try_prefix = [&](std::int64_t prefix) {
    if (prefix <= 0 || prefix >= num_tokens) return;
    const Best cand{prefix, split_waves(prefix, num_tokens, profile), std::llabs(prefix - half)};
    if (cand.waves < best.waves || (cand.waves == best.waves && cand.imbalance < best.imbalance)) best = cand;
  };
  try_prefix(half);
  for (std::int64_t t = 1; t < tiles; ++t) try_prefix(std::min(t * profile.tile_tokens, num_tokens - 1));
  return best.prefix - half;
}

std::int64_t smart_offset_sweep(std::int64_t num_tokens, const SplitPolicy& policy,
                                const std::function<double(std::int64_t, std::int64_t)>& forward) {
  const std::int64_t half = num_tokens / 2;
  std::int64_t chosen = 0;
  double fastest = std::numeric_limits<double>::infinity();
  for (const std::int64_t off : policy.offset_grid) {
    if (off >= half) continue;  // the prefix must stay < T
    const double t = forward(half + off, num_tokens - half - off);
    if (t < fastest) {  // strict: ties keep the earlier (smaller) offset
      fastest = t;
      chosen = off;
    }
  }
  return chosen;
}

SplitPlan make_split_plan(std::int64_t num_tokens, const HardwareProfile& profile, const SplitPolicy& policy) {
  SplitPlan plan;
  plan.total_tokens = num_tokens;
  plan.mode = select_mode(num_tokens, policy);
  if (plan.mode == SplitMode::Overlap) {
    plan.offset = smart_offset_analytic(num_tokens, profile);
    plan.prefix_tokens = num_tokens / 2 + plan.offset;
    plan.suffix_tokens = num_tokens - plan.prefix_tokens;
    if (plan.suffix_tokens == 0) plan.mode = SplitMode::FusedOnly;
  } else {
    plan.prefix_tokens = num_tokens;
  }
  return plan;
}

SplitPlan place_sequence_boundaries(const std::vector<std::int64_t>& sequence_lengths, SplitPlan plan) {
  std::int64_t total = 0;
  for (std::int64_t n : sequence_lengths) total += n;
  if (total != plan.total_tokens) throw ContractError("place_sequence_boundaries: sequence lengths must sum to T");
  plan.prefix_len_per_sequence.clear();
  std::int64_t left = plan.prefix_tokens;
  for (std::int64_t n : sequence_lengths) {
    const std::int64_t take = std::max<std::int64_t>(0, std::min(left, n));
    plan.prefix_len_per_sequence.push_back(take);
    left -= take;
  }
  return plan;
}

}  // namespace weavesim

// ---- C-ABI (include/tw/tw_split.h) ------------------------------------------------

#include "tw/tw_split.h"

namespace {

template <class F>
tw_status guarded(F&& f) {
  try {
    f();
    return TW_OK;
  } catch (const weavesim::DimensionError&) {
    return TW_ERR_DIMENSION;
  } catch (const weavesim::NumericError&) {
    return TW_ERR_NUMERIC;
  } catch (const weavesim::ConfigError&) {
    return TW_ERR_CONFIG;
  } catch (const weavesim::ContractError&) {
    return TW_ERR_CONTRACT;
  } catch (...) {
    return TW_ERR_CUDA;
  }
}

weavesim::HardwareProfile geometry(int num_sms, int tile_tokens, int cta_columns) {
  weavesim::HardwareProfile p = weavesim::b200_geometry();
  p.num_sms = num_sms;
  p.tile_tokens = tile_tokens;
  p.cta_columns = cta_columns;
  if (p.collective_sms >= num_sms) p.collective_sms = num_sms > 1 ? num_sms - 1 : 0;
  return p;
}

}  // namespace

extern "C" {

tw_status tw_make_split_plan(int64_t num_tokens, int num_sms, int tile_tokens, int cta_columns,
                             int64_t threshold_tokens, int64_t* prefix, int64_t* suffix, int64_t* offset, int* mode) {
  return guarded([&] {
    weavesim::SplitPolicy pol;
    pol.threshold_tokens = threshold_tokens;
    const weavesim::SplitPlan plan =
        weavesim::make_split_plan(num_tokens, geometry(num_sms, tile_tokens, cta_columns), pol);
    if (prefix) *prefix = plan.prefix_tokens;
    if (suffix) *suffix = plan.suffix_tokens;
    if (offset) *offset = plan.offset;
    if (mode) *mode = static_cast<int>(plan.mode);
  });
}

tw_status tw_smart_offset_analytic(int64_t num_tokens, int num_sms, int tile_tokens, int cta_columns,
                                   int64_t* offset) {
  return guarded([&] {
    *offset = weavesim::smart_offset_analytic(num_tokens, geometry(num_sms, tile_tokens, cta_columns));
  });
}

tw_status tw_smart_offset_sweep(int64_t num_tokens, const int64_t* offset_grid, int n,
                                double (*forward)(int64_t, int64_t, void*), void* ctx, int64_t* offset) {
  return guarded([&] {
    weavesim::SplitPolicy pol;
    pol.offset_grid.assign(offset_grid, offset_grid + n);
    *offset = weavesim::smart_offset_sweep(num_tokens, pol,
                                           [&](std::int64_t a, std::int64_t b) { return forward(a, b, ctx); });
  });
}

tw_status tw_place_sequence_boundaries(const int64_t* lengths, int n, int64_t total_tokens, int64_t prefix_tokens,
                                       int64_t* prefix_len_out) {
  return guarded([&] {
    weavesim::SplitPlan plan;
    plan.total_tokens = total_tokens;
    plan.prefix_tokens = prefix_tokens;
    plan = weavesim::place_sequence_boundaries(std::vector<std::int64_t>(lengths, lengths + n), plan);
    std::copy(plan.prefix_len_per_sequence.begin(), plan.prefix_len_per_sequence.end(), prefix_len_out);
  });
}

}  // extern "C"
