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

// One measured iteration: the mode mapping and TokenWeave degrade rules
// (decode-only and non-Overlap batches run fuse-only, scheduler.cpp:333-341).
double measured_iteration(const WeaveApi& api, tw_weave_t w, const BatchShape& batch, const LayerSpec& spec,
                          const HardwareProfile& profile, BaselineMode mode, const SplitPolicy& policy) {
  tw_weave_mode m = TW_MODE_UNFUSED;
  std::int64_t prefix = 0;
  switch (mode) {
    case BaselineMode::Default:
    case BaselineMode::Multimem: m = TW_MODE_UNFUSED; break;
    case BaselineMode::NoComm: m = TW_MODE_NO_COMM; break;
    case BaselineMode::FuseOnly: m = TW_MODE_FUSE_ONLY; break;
    case BaselineMode::TokenWeave: {
      m = TW_MODE_FUSE_ONLY;
      if (!batch.decode_only) {
        const SplitPlan plan = make_split_plan(batch.total_tokens, profile, policy);
        if (plan.mode == SplitMode::Overlap && plan.suffix_tokens > 0) {
          m = TW_MODE_WEAVE;
          prefix = plan.prefix_tokens;
        }
      }
      break;
    }
  }
  float us = 0.0f;
  if (m == TW_MODE_WEAVE) {
    // the fused op's SM budget that schedules best on this box, over 16/32/64
    float best = 0.0f;
    for (int cand : {16, 32, 64}) {
      float t = 0.0f;
      const tw_status st = api.run_batch(w, batch.total_tokens, prefix, batch.kv_context, m, cand, 0, 2, 0u, &t);
      if (st != TW_OK) runner_error(api, st, "weavesim: measured iteration");
      if (best == 0.0f || t < best) best = t;
    }
    us = best;
  } else {
    const tw_status st = api.run_batch(w, batch.total_tokens, prefix, batch.kv_context, m, 0, 0, 2, 0u, &us);
    if (st != TW_OK) runner_error(api, st, "weavesim: measured iteration");
  }
  return 1e-6 * static_cast<double>(us) * spec.num_layers;
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
