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

enum class OpKind { Attention, Ffn, FusedARNorm, AllReduce, RmsNorm, AllGatherOp, Misc };
enum class SplitId { Prefix, Suffix, Whole };
enum class StreamId { Compute, Comm };
enum class BaselineMode { Default, Multimem, NoComm, FuseOnly, TokenWeave };

const char* to_string(BaselineMode mode);
const char* to_string(OpKind op);
// ConfigError on an unknown name (proj/src/scheduler.cpp:38-45).
BaselineMode baseline_mode_from_string(const std::string& name);

// Shape of one iteration's batch (proj/include/weavesim/scheduler.hpp:46-52).
struct BatchShape {
  std::int64_t total_tokens = 0;
  std::int64_t kv_context = 0;  // prior-context tokens (sum over sequences)
  bool decode_only = false;
  std::vector<std::int64_t> sequence_lengths;  // optional; empty = single sequence
};

// One event of a layer's two-stream DAG (scheduler.hpp:20-35).  B200 build:
// start / end are MEASURED (CUDA events, seconds from the layer's first op);
// the work-description fields of the reference's simulator stay 0.
struct StreamEvent {
  int id = 0;
  OpKind op = OpKind::Misc;
  SplitId split = SplitId::Whole;
  StreamId stream = StreamId::Compute;
  std::vector<int> depends_on;  // ids of earlier events only
  double scalable_seconds = 0.0;
  double fixed_seconds = 0.0;
  double start = 0.0;
  double end = 0.0;
};

struct Timeline {
  std::vector<StreamEvent> events;
  double iteration_latency = 0.0;  // seconds

  // The reference's JSON schema (scheduler.cpp:301-317).
  std::string to_json() const;
  void to_json_file(const std::string& path) const;
};

// The reference's signature (scheduler.hpp:74-77).  B200 build: the batch's
// layer is RUN (as iteration_latency) and the timeline holds the measured
// events of ONE layer with the DAG's dependency edges; iteration_latency is
// that layer's time x spec.num_layers.  plan_override selects the TokenWeave
// split (else make_split_plan).
Timeline iteration_timeline(const BatchShape& batch, const LayerSpec& spec, const HardwareProfile& profile,
                            BaselineMode mode, const SplitPolicy& policy, const SplitPlan* plan_override = nullptr);

// The reference's signature (scheduler.hpp:79-81).  B200 build: the layer is
// RUN on this GPU (one GPU's share at spec.tp_degree; the mode mapping and
// the TokenWeave degrade rules of simulate_throughput, workloads.hpp) and the
// result is the measured per-layer time x spec.num_layers, in seconds.
double iteration_latency(const BatchShape& batch, const LayerSpec& spec, const HardwareProfile& profile,
                         BaselineMode mode, const SplitPolicy& policy);

}  // namespace weavesim
