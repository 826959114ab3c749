// weavesim_models.cpp -- drop-in model presets, baseline modes and the
// throughput entry point of the reference API (host C++):
//   LayerSpec::validate            proj/src/wavemodel.cpp:23-36
//   to_string / baseline_mode_from_string   proj/src/scheduler.cpp:16-46
//   model_preset / builtin_profile proj/src/presets.cpp:53-110 (geometry only)
//   iteration_latency              proj/src/scheduler.cpp:387-392, the layer RUN
//   simulate_throughput            proj/src/workloads.cpp:111-141, every batch
//                                  RUN through the layer runner
// The runner lives in libtw_weave.so, which links this library; it is loaded
// here with dlopen from this library's own directory (no link cycle).
#include <dlfcn.h>

#include <algorithm>
#include <vector>
#include <fstream>
#include <charconv>
#include <cstdint>
#include <string>

#include "tw/tw_weave.h"
#include "weavesim/errors.hpp"
#include "weavesim/presets.hpp"
#include "weavesim/scheduler.hpp"
#include "weavesim/workloads.hpp"

namespace weavesim {

void LayerSpec::validate() const {
  if (hidden < 1 || intermediate < 1 || num_layers < 1) throw ConfigError("LayerSpec: dimensions must be positive");
  if (num_attention_heads < 1 || num_kv_heads < 1 || head_dim < 1 || num_attention_heads % num_kv_heads != 0)
    throw ConfigError("LayerSpec: head structure invalid");
  if (experts < 1 || top_k < 1 || top_k > experts) throw ConfigError("LayerSpec: experts >= top_k >= 1 required");
  if (tp_degree < 2) throw ConfigError("LayerSpec: tp_degree must be >= 2");
}

const char* to_string(BaselineMode mode) {
  switch (mode) {
    case BaselineMode::Default: return "default";
    case BaselineMode::Multimem: return "multimem";
    case BaselineMode::NoComm: return "nocomm";
    case BaselineMode::FuseOnly: return "fuseonly";
    case BaselineMode::TokenWeave: return "tokenweave";
  }
  return "?";
}

const char* to_string(OpKind op) {
  switch (op) {
    case OpKind::Attention: return "attention";
    case OpKind::Ffn: return "ffn";
    case OpKind::FusedARNorm: return "fused_ar_norm";
    case OpKind::AllReduce: return "allreduce";
    case OpKind::RmsNorm: return "rmsnorm";
    case OpKind::AllGatherOp: return "allgather";
    case OpKind::Misc: return "misc";
  }
  return "?";
}

BaselineMode baseline_mode_from_string(const std::string& name) {
  if (name == "default") return BaselineMode::Default;
  if (name == "multimem") return BaselineMode::Multimem;
  if (name == "nocomm") return BaselineMode::NoComm;
  if (name == "fuseonly") return BaselineMode::FuseOnly;
  if (name == "tokenweave") return BaselineMode::TokenWeave;
  throw ConfigError("unknown baseline mode: " + name);
}

ModelPreset model_preset(const std::string& name) {
  ModelPreset preset;
  preset.name = name;
  LayerSpec& s = preset.spec;
  if (name == "llama-70b" || name == "qwen-72b") {
    s.hidden = 8192;
    s.intermediate = name == "llama-70b" ? 28672 : 29568;
    s.num_attention_heads = 64;
    s.num_kv_heads = 8;
    s.head_dim = 128;
    s.num_layers = 80;
    preset.policy.threshold_tokens = 1024;
  } else if (name == "mixtral-8x22b") {
    s.hidden = 6144;
    s.intermediate = 16384;
    s.num_attention_heads = 48;
    s.num_kv_heads = 8;
    s.head_dim = 128;
    s.num_layers = 56;
    s.experts = 8;
    s.top_k = 2;
    preset.policy.threshold_tokens = 4096;
  } else {
    throw ConfigError("unknown model preset: " + name);
  }
  s.tp_degree = 8;
  s.validate();
  return preset;
}

std::vector<std::string> model_preset_names() { return {"llama-70b", "qwen-72b", "mixtral-8x22b"}; }

HardwareProfile builtin_profile(const std::string& name) {
  if (name == "h100") return HardwareProfile{};  // defaults describe the H100 geometry
  if (name == "b200") return b200_geometry();
  throw ConfigError("unknown profile: " + name + " (expected h100 or b200)");
}

namespace {

// The layer runner's entry points, resolved from libtw_weave.so next to this library.
struct WeaveApi {
  decltype(&tw_weave_create) create = nullptr;
  decltype(&tw_weave_destroy) destroy = nullptr;
  decltype(&tw_weave_run_batch) run_batch = nullptr;
  decltype(&tw_weave_last_error) last_error = nullptr;
  decltype(&tw_weave_trace) trace = nullptr;
};

const WeaveApi& weave_api() {
  static WeaveApi api = [] {
    WeaveApi a;
    Dl_info info{};
    std::string dir;
    if (dladdr(reinterpret_cast<void*>(&weave_api), &info) && info.dli_fname) {
      dir = info.dli_fname;
      dir = dir.substr(0, dir.find_last_of('/') + 1);
    }
    void* h = dlopen((dir + "libtw_weave.so").c_str(), RTLD_NOW | RTLD_LOCAL);
    if (!h) return a;
    a.create = reinterpret_cast<decltype(a.create)>(dlsym(h, "tw_weave_create"));
    a.destroy = reinterpret_cast<decltype(a.destroy)>(dlsym(h, "tw_weave_destroy"));
    a.run_batch = reinterpret_cast<decltype(a.run_batch)>(dlsym(h, "tw_weave_run_batch"));
    a.last_error = reinterpret_cast<decltype(a.last_error)>(dlsym(h, "tw_weave_last_error"));
    a.trace = reinterpret_cast<decltype(a.trace)>(dlsym(h, "tw_weave_trace"));
    return a;
  }();
  return api;
}

[[noreturn]] void runner_error(const WeaveApi& api, tw_status st, const std::string& where) {
  const std::string msg = where + ": " + (api.last_error ? api.last_error() : "");
  if (st == TW_ERR_CONFIG) throw ConfigError(msg);
  if (st == TW_ERR_DIMENSION) throw DimensionError(msg);
  if (st == TW_ERR_CONTRACT) throw ContractError(msg);
  throw DeviceError(msg);
}

// One runner per process, reused while the layer shape matches and it is
// large enough (creating one allocates the layer's weights and activations).
struct RunnerCache {
  tw_weave_t w = nullptr;
  tw_layer_spec spec{};
  std::int64_t max_tokens = 0;
};

tw_weave_t runner_for(const WeaveApi& api, const LayerSpec& spec, std::int64_t tokens) {
  static RunnerCache cache;  // intentionally not destroyed at exit (CUDA may be torn down first)
  const tw_layer_spec ls{spec.hidden, spec.intermediate, spec.num_attention_heads, spec.num_kv_heads, spec.head_dim,
                         spec.experts, spec.top_k, spec.tp_degree};
  const bool same = cache.w && cache.spec.hidden == ls.hidden && cache.spec.intermediate == ls.intermediate &&
                    cache.spec.heads == ls.heads && cache.spec.kv_heads == ls.kv_heads &&
                    cache.spec.head_dim == ls.head_dim && cache.spec.experts == ls.experts &&
                    cache.spec.top_k == ls.top_k && cache.spec.tp == ls.tp;
  if (same && cache.max_tokens >= tokens) return cache.w;
  if (cache.w) api.destroy(cache.w);
  cache.w = nullptr;
  const std::int64_t cap = std::max<std::int64_t>(tokens, same ? 2 * cache.max_tokens : tokens);
  tw_weave_t w = nullptr;
  const tw_status st = api.create(&ls, cap, 0, &w);
  if (st != TW_OK) runner_error(api, st, "weavesim: layer runner");
  cache.w = w;
  cache.spec = ls;
  cache.max_tokens = cap;
  return w;
}

const WeaveApi& require_api() {
  const WeaveApi& api = weave_api();
  if (!api.create || !api.destroy || !api.run_batch)
    throw DeviceError("weavesim: libtw_weave.so not found next to libweavesim_b200.so");
  return api;
}

// The runner mode and split for a batch: the mode mapping and TokenWeave
// degrade rules (decode-only and non-Overlap batches run fuse-only,
// scheduler.cpp:333-341).
tw_weave_mode runner_mode(const BatchShape& batch, const HardwareProfile& profile, BaselineMode mode,
                          const SplitPolicy& policy, const SplitPlan* plan_override, std::int64_t* prefix) {
  *prefix = 0;
  switch (mode) {
    case BaselineMode::Default:
    case BaselineMode::Multimem: return TW_MODE_UNFUSED;
    case BaselineMode::NoComm: return TW_MODE_NO_COMM;
    case BaselineMode::FuseOnly: return TW_MODE_FUSE_ONLY;
    case BaselineMode::TokenWeave: break;
  }
  if (batch.decode_only) return TW_MODE_FUSE_ONLY;
  const SplitPlan plan = plan_override ? *plan_override : make_split_plan(batch.total_tokens, profile, policy);
  if (plan.mode != SplitMode::Overlap || plan.suffix_tokens <= 0) return TW_MODE_FUSE_ONLY;
  *prefix = plan.prefix_tokens;
  return TW_MODE_WEAVE;
}

// One measured layer of the batch (us).  Weaved layers take the fused op's SM
// budget that schedules best on this box (16/32/64); `best_budget` reports it.
float measured_layer_us(const WeaveApi& api, tw_weave_t w, const BatchShape& batch, tw_weave_mode m,
                        std::int64_t prefix, int* best_budget) {
  float us = 0.0f;
  *best_budget = 0;
  if (m == TW_MODE_WEAVE) {
    for (int cand : {16, 32, 64}) {
      float t = 0.0f;
      const tw_status st = api.run_batch(w, batch.total_tokens, prefix, batch.kv_context, m, cand, 0, 2, 0u, &t);
      if (st != TW_OK) runner_error(api, st, "weavesim: measured iteration");
      if (us == 0.0f || t < us) {
        us = t;
        *best_budget = cand;
      }
    }
  } else {
    const tw_status st = api.run_batch(w, batch.total_tokens, prefix, batch.kv_context, m, 0, 0, 2, 0u, &us);
    if (st != TW_OK) runner_error(api, st, "weavesim: measured iteration");
  }
  return us;
}

double measured_iteration(const WeaveApi& api, tw_weave_t w, const BatchShape& batch, const LayerSpec& spec,
                          const HardwareProfile& profile, BaselineMode mode, const SplitPolicy& policy) {
  std::int64_t prefix = 0;
  const tw_weave_mode m = runner_mode(batch, profile, mode, policy, nullptr, &prefix);
  int budget = 0;
  return 1e-6 * static_cast<double>(measured_layer_us(api, w, batch, m, prefix, &budget)) * spec.num_layers;
}

// JSON number text: shortest round trip, as nlohmann::json::dump writes it.
std::string json_number(double v) {
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof(buf), v);
  std::string s(buf, r.ptr);
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  return s;
}

}  // namespace

double iteration_latency(const BatchShape& batch, const LayerSpec& spec, const HardwareProfile& profile,
                         BaselineMode mode, const SplitPolicy& policy) {
  spec.validate();
  profile.validate();
  if (batch.total_tokens < 0 || batch.kv_context < 0) throw DimensionError("iteration_latency: negative batch shape");
  if (batch.total_tokens == 0) return 0.0;
  const WeaveApi& api = require_api();
  return measured_iteration(api, runner_for(api, spec, batch.total_tokens), batch, spec, profile, mode, policy);
}

Timeline iteration_timeline(const BatchShape& batch, const LayerSpec& spec, const HardwareProfile& profile,
                            BaselineMode mode, const SplitPolicy& policy, const SplitPlan* plan_override) {
  spec.validate();
  profile.validate();
  if (batch.total_tokens < 0 || batch.kv_context < 0) throw DimensionError("iteration_timeline: negative batch shape");
  Timeline tl;
  if (batch.total_tokens == 0) return tl;
  const WeaveApi& api = require_api();
  if (!api.trace) throw DeviceError("weavesim: libtw_weave.so lacks tw_weave_trace");
  tw_weave_t w = runner_for(api, spec, batch.total_tokens);
  std::int64_t prefix = 0;
  const tw_weave_mode m = runner_mode(batch, profile, mode, policy, plan_override, &prefix);
  int budget = 0;
  float us = measured_layer_us(api, w, batch, m, prefix, &budget);
  if (m == TW_MODE_WEAVE) {  // re-run at the best budget so the trace shows that schedule
    const tw_status st = api.run_batch(w, batch.total_tokens, prefix, batch.kv_context, m, budget, 0, 2, 0u, &us);
    if (st != TW_OK) runner_error(api, st, "weavesim: measured iteration");
  }
  int n = 0;
  int op[16], sp[16], stm[16];
  float a[16], b[16];
  const tw_status st = api.trace(w, 16, &n, op, sp, stm, a, b);
  if (st != TW_OK) runner_error(api, st, "weavesim: trace");
  float t0 = n ? a[0] : 0.0f;
  for (int i = 0; i < n; ++i) t0 = std::min(t0, a[i]);
  for (int i = 0; i < n; ++i) {
    StreamEvent e;
    e.id = i;
    e.op = op[i] == TW_OP_ATTENTION ? OpKind::Attention : op[i] == TW_OP_FFN ? OpKind::Ffn : OpKind::FusedARNorm;
    e.split = sp[i] == 0 ? SplitId::Prefix : sp[i] == 1 ? SplitId::Suffix : SplitId::Whole;
    // the reference's DAG puts every collective on the comm stream, sequential
    // modes included (ordered by edges); the runner serialises those on the
    // compute stream, so the label follows the op
    e.stream = (stm[i] || e.op == OpKind::FusedARNorm) ? StreamId::Comm : StreamId::Compute;
    // the DAG edges of build_layer_graph (scheduler.cpp:119-147 weave, :150-181 chains)
    if (n == 8) {
      static const std::vector<int> deps[8] = {{}, {0}, {0}, {2, 1}, {1}, {4, 3}, {3}, {6, 5}};
      e.depends_on = deps[i];
    } else if (i > 0) {
      e.depends_on = {i - 1};
    }
    e.start = 1e-6 * static_cast<double>(a[i] - t0);
    e.end = 1e-6 * static_cast<double>(b[i] - t0);
    tl.events.push_back(e);
  }
  tl.iteration_latency = 1e-6 * static_cast<double>(us) * spec.num_layers;
  return tl;
}

std::string Timeline::to_json() const {
  // the reference's Timeline::to_json layout (json dump(2): sorted keys,
  // two-space indent, id lists inline)
  std::string o = "{\n  \"events\": [";
  for (size_t i = 0; i < events.size(); ++i) {
    const StreamEvent& e = events[i];
    o += i ? ",\n    {\n" : "\n    {\n";
    o += "      \"depends_on\": [";  // the reference build prints id lists inline: [2,1]
    for (size_t k = 0; k < e.depends_on.size(); ++k) o += (k ? "," : "") + std::to_string(e.depends_on[k]);
    o += "],\n";
    o += "      \"end\": " + json_number(e.end) + ",\n";
    o += "      \"id\": " + std::to_string(e.id) + ",\n";
    o += std::string("      \"op\": \"") + to_string(e.op) + "\",\n";
    o += std::string("      \"split\": \"") +
         (e.split == SplitId::Prefix ? "prefix" : e.split == SplitId::Suffix ? "suffix" : "whole") + "\",\n";
    o += "      \"start\": " + json_number(e.start) + ",\n";
    o += std::string("      \"stream\": \"") + (e.stream == StreamId::Comm ? "comm" : "compute") + "\"\n    }";
  }
  o += events.empty() ? "],\n" : "\n  ],\n";
  o += "  \"iteration_latency\": " + json_number(iteration_latency) + "\n}";
  return o;
}

void Timeline::to_json_file(const std::string& path) const {
  std::ofstream out(path);
  if (!out) throw ParseError("cannot write timeline: " + path);
  out << to_json() << "\n";
}

ThroughputResult simulate_throughput(const std::vector<Request>& requests, const LayerSpec& spec,
                                     const HardwareProfile& profile, BaselineMode mode, const SplitPolicy& policy,
                                     std::int64_t chunk_size) {
  spec.validate();
  profile.validate();
  const std::vector<IterationBatch> batches = form_batches(requests, chunk_size);
  ThroughputResult result;
  if (batches.empty()) return result;
  const WeaveApi& api = require_api();
  std::int64_t max_t = 0;
  for (const IterationBatch& b : batches) max_t = std::max(max_t, b.total_tokens);
  tw_weave_t w = runner_for(api, spec, max_t);
  for (const IterationBatch& b : batches) {
    BatchShape shape;
    shape.total_tokens = b.total_tokens;
    shape.kv_context = b.kv_context;
    shape.decode_only = b.decode_only();
    const double latency = measured_iteration(api, w, shape, spec, profile, mode, policy);
    result.iteration_latencies.push_back(latency);
    result.total_seconds += latency;
    result.total_tokens += b.total_tokens;
  }
  result.iterations = static_cast<std::int64_t>(batches.size());
  if (result.total_seconds > 0.0) result.tokens_per_sec = result.total_tokens / result.total_seconds;
  result.mean_iteration_latency = result.total_seconds / static_cast<double>(result.iterations);
  return result;
}

}  // namespace weavesim
