// ref_capi.cpp -- extern "C" adapter over the UNMODIFIED reference sources
// (/root/reference/proj/src/*.cpp), compiled by oracle/Makefile into
// oracle/_ref/libweavesim_ref.so.  TEST INFRASTRUCTURE ONLY: used by tests/
// to pin the C restatement (tw_oracle.c) and golden fixtures, and by bench.py
// as the reference CPU arm.  Never linked by the product.
//
// Exceptions from the reference API are mapped to tw.h status codes:
// DimensionError 1, NumericError 2, ConfigError 3, ContractError 4, other 9.
#include <algorithm>
#include <chrono>
#include <malloc.h>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

#include "weavesim/calibration.hpp"
#include "weavesim/commands.hpp"
#include "weavesim/collectives.hpp"
#include "weavesim/errors.hpp"
#include "weavesim/numerics.hpp"
#include "weavesim/presets.hpp"
#include "weavesim/scheduler.hpp"
#include "weavesim/splitter.hpp"
#include "weavesim/wavemodel.hpp"
#include "weavesim/workloads.hpp"

using namespace weavesim;

namespace {

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const DimensionError&) {
    return 1;
  } catch (const NumericError&) {
    return 2;
  } catch (const ConfigError&) {
    return 3;
  } catch (const ContractError&) {
    return 4;
  } catch (...) {
    return 9;
  }
}

TokenMatrix make_matrix(const float* v, std::int64_t T, std::int64_t H) {
  TokenMatrix m;
  m.num_tokens = T;
  m.hidden = H;
  m.values.assign(v, v + T * H);
  return m;
}

}  // namespace

extern "C" {

int ref_rmsnorm_residual(const float* input, const float* residual, const float* weight,
                         std::int64_t T, std::int64_t H, float eps, float* output,
                         float* residual_out) {
  return guarded([&] {
    NormParams p;
    p.weight.assign(weight, weight + H);
    p.epsilon = eps;
    NormResult r = rmsnorm_residual(make_matrix(input, T, H), make_matrix(residual, T, H), p);
    std::memcpy(output, r.output.values.data(), sizeof(float) * T * H);
    std::memcpy(residual_out, r.residual_out.values.data(), sizeof(float) * T * H);
  });
}

int ref_token_shard_map(std::int64_t T, int world, std::int64_t* ranges) {
  return guarded([&] {
    ShardMap m = token_shard_map(T, world);
    for (int r = 0; r < world; ++r) {
      ranges[2 * r] = m.ranges[r].begin;
      ranges[2 * r + 1] = m.ranges[r].end;
    }
  });
}

int ref_shard_map_validate(const std::int64_t* ranges, int world, std::int64_t total) {
  return guarded([&] {
    ShardMap m;
    for (int r = 0; r < world; ++r) m.ranges.push_back({ranges[2 * r], ranges[2 * r + 1]});
    m.validate(total);
  });
}

int ref_all_reduce(int world, const float* const* inputs, std::int64_t T, std::int64_t H,
                   float* out) {
  return guarded([&] {
    RankGroup g;
    g.world_size = world;
    for (int r = 0; r < world; ++r) g.inputs.push_back(make_matrix(inputs[r], T, H));
    TokenMatrix s = all_reduce(g);
    std::memcpy(out, s.values.data(), sizeof(float) * T * H);
  });
}

// ranges == nullptr -> token_shard_map(T, world).  residual_shards[r] is
// [T_r, H] and receives r' (the reference overwrites its shards).
int ref_fused_allreduce_rmsnorm(int world, const float* const* inputs, float* const* residual_shards,
                                const std::int64_t* ranges, const float* weight, std::int64_t T,
                                std::int64_t H, float eps, int parallel, float* output) {
  return guarded([&] {
    RankGroup g;
    g.world_size = world;
    for (int r = 0; r < world; ++r) g.inputs.push_back(make_matrix(inputs[r], T, H));
    ShardMap shards;
    if (ranges) {
      for (int r = 0; r < world; ++r) shards.ranges.push_back({ranges[2 * r], ranges[2 * r + 1]});
    } else {
      shards = token_shard_map(T, world);
    }
    for (int r = 0; r < world; ++r) {
      const std::int64_t len = std::max<std::int64_t>(0, shards.ranges[r].size());
      g.residual_shards.push_back(make_matrix(residual_shards[r], len, H));
    }
    NormParams p;
    p.weight.assign(weight, weight + H);
    p.epsilon = eps;
    TokenMatrix out = fused_allreduce_rmsnorm(g, p, shards, parallel != 0);
    std::memcpy(output, out.values.data(), sizeof(float) * T * H);
    for (int r = 0; r < world; ++r) {
      std::memcpy(residual_shards[r], g.residual_shards[r].values.data(),
                  sizeof(float) * g.residual_shards[r].values.size());
    }
  });
}

// The acceptance-test draw order (proj/tests/acceptance.cpp:45-66):
// mt19937_64(seed); N rank inputs U(-1,1); residual shards U(-1,1) in shard
// order; weight U(0.5,1.5).  inputs: world*T*H, residual: T*H (shards
// concatenated in token order), weight: H.
void ref_fill_group(std::uint64_t seed, int world, std::int64_t T, std::int64_t H, float* inputs,
                    float* residual, float* weight) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<float> dist(-1.0f, 1.0f);
  for (std::int64_t i = 0; i < static_cast<std::int64_t>(world) * T * H; ++i) inputs[i] = dist(rng);
  for (std::int64_t i = 0; i < T * H; ++i) residual[i] = dist(rng);
  std::uniform_real_distribution<float> wdist(0.5f, 1.5f);
  for (std::int64_t j = 0; j < H; ++j) weight[j] = wdist(rng);
}

std::uint64_t ref_acceptance_seed(int world, std::int64_t T, std::int64_t H, int i) {
  return (static_cast<std::uint64_t>(world) << 48) ^ (static_cast<std::uint64_t>(T) << 24) ^
         (static_cast<std::uint64_t>(H) << 8) ^ static_cast<std::uint64_t>(i);
}

// Wave model and split planner (proj/src/wavemodel.cpp:38-49, splitter.cpp).
std::int64_t ref_cta_count(std::int64_t tokens, int tile_tokens, int cta_columns) {
  HardwareProfile p;
  p.tile_tokens = tile_tokens;
  p.cta_columns = cta_columns;
  return cta_count(tokens, p);
}

std::int64_t ref_smart_offset_analytic(std::int64_t tokens, int num_sms, int tile_tokens,
                                       int cta_columns) {
  HardwareProfile p;
  p.num_sms = num_sms;
  p.tile_tokens = tile_tokens;
  p.cta_columns = cta_columns;
  return smart_offset_analytic(tokens, p);
}

// Builtin profile + model preset plan (Appendix A of SURVEY.md).
// out4 = {prefix, suffix, offset, mode}.  Also returns the profile geometry
// in geom3 = {num_sms, tile_tokens, cta_columns} and the policy threshold.
int ref_make_split_plan(const char* profile, const char* model, std::int64_t T, std::int64_t* out4,
                        std::int64_t* geom4) {
  return guarded([&] {
    HardwareProfile hp = builtin_profile(profile);
    ModelPreset mp = model_preset(model);
    SplitPlan plan = make_split_plan(T, hp, mp.policy);
    out4[0] = plan.prefix_tokens;
    out4[1] = plan.suffix_tokens;
    out4[2] = plan.offset;
    out4[3] = static_cast<std::int64_t>(plan.mode);
    if (geom4) {
      geom4[0] = hp.num_sms;
      geom4[1] = hp.tile_tokens;
      geom4[2] = hp.cta_columns;
      geom4[3] = mp.policy.threshold_tokens;
    }
  });
}

// Modeled per-layer latency (seconds) of build_layer_graph + simulate for
// one layer, no tail: the reference's "predicted" column.  mode is a
// BaselineMode name ("multimem", "fuseonly", "tokenweave", ...).
int ref_layer_latency(const char* profile, const char* model, std::int64_t T, const char* mode,
                      double* seconds) {
  return guarded([&] {
    HardwareProfile hp = builtin_profile(profile);
    ModelPreset mp = model_preset(model);
    BaselineMode m = baseline_mode_from_string(mode);
    SplitPlan plan = make_split_plan(T, hp, mp.policy);
    if (m == BaselineMode::TokenWeave && plan.mode != SplitMode::Overlap) m = BaselineMode::FuseOnly;
    std::vector<StreamEvent> g = build_layer_graph(plan, mp.spec, hp, m, 0);
    *seconds = simulate(g, hp).iteration_latency;
  });
}

// The reference's own calibrate() (proj/src/calibration.cpp:98-192) on a
// CalibrationTable JSON file: out6 = {AR intercept us, AR slope us/token,
// RMSNorm intercept us, RMSNorm slope us/token, hbm_bandwidth_effective B/s,
// fused_extra_latency s}.
int ref_calibrate_file(const char* path, double* out6) {
  return guarded([&] {
    const CalibrationTable table = CalibrationTable::from_json_file(path);
    HardwareProfile base;
    base.name = "b200";
    base.num_sms = 148;
    base.sm_flops = 8.4e12;
    const HardwareProfile p = calibrate(table, base);
    out6[0] = p.collective_base_latency * 1e6;
    out6[1] = p.collective_per_token_time * 1e6;
    out6[2] = p.rmsnorm_base_latency * 1e6;
    out6[3] = p.hbm_bandwidth_effective > 0 ? 3.0 * table.hidden * table.bytes_per_element /
                                                  p.hbm_bandwidth_effective * 1e6
                                            : 0.0;
    out6[4] = p.hbm_bandwidth_effective;
    out6[5] = p.fused_extra_latency;
  });
}

// --- CPU-baseline timers (the reference path as shipped, incl. its validation).

// Times fused_allreduce_rmsnorm on a fixed group `iters` times; returns the
// median milliseconds.  Residual shards are restored (outside the timed
// region) before every call so each call sees the same inputs.
// each_ms (optional, iters entries): every iteration's time, so a caller can
// drop warm-up iterations without regenerating the inputs.
int ref_time_fused(int world, std::int64_t T, std::int64_t H, int parallel, int iters,
                   double* median_ms, double* each_ms) {
  mallopt(M_MMAP_MAX, 0);  // heap reuse across iterations (see ref_time_rmsnorm)
  mallopt(M_TRIM_THRESHOLD, 1 << 30);
  return guarded([&] {
    RankGroup g;
    g.world_size = world;
    std::mt19937_64 rng(1234);
    std::uniform_real_distribution<float> dist(-1.0f, 1.0f);
    for (int r = 0; r < world; ++r) {
      TokenMatrix m = TokenMatrix::zeros(T, H);
      for (float& v : m.values) v = dist(rng);
      g.inputs.push_back(std::move(m));
    }
    const ShardMap shards = token_shard_map(T, world);
    for (const TokenRange& range : shards.ranges) {
      TokenMatrix m = TokenMatrix::zeros(range.size(), H);
      for (float& v : m.values) v = dist(rng);
      g.residual_shards.push_back(std::move(m));
    }
    NormParams p;
    p.weight.assign(H, 1.0f);
    const std::vector<TokenMatrix> saved = g.residual_shards;
    std::vector<double> ms;
    for (int i = 0; i < iters; ++i) {
      g.residual_shards = saved;
      const auto t0 = std::chrono::steady_clock::now();
      TokenMatrix out = fused_allreduce_rmsnorm(g, p, shards, parallel != 0);
      const auto t1 = std::chrono::steady_clock::now();
      ms.push_back(std::chrono::duration<double, std::milli>(t1 - t0).count());
      if (each_ms) each_ms[i] = ms.back();
    }
    std::sort(ms.begin(), ms.end());
    *median_ms = ms[ms.size() / 2];
  });
}

// Times rmsnorm_residual over T x H with `threads` host threads, each calling
// the reference rmsnorm_residual on a contiguous token chunk (the reference
// op is single-threaded; chunking across cores is the caller-level
// parallelism a host deployment would use).  Returns median milliseconds.
int ref_time_rmsnorm(std::int64_t T, std::int64_t H, int threads, int iters, double* median_ms,
                     double* each_ms) {
  // heap reuse across iterations, as tools/dropin_bench.cpp (the drop-in arm) sets
  mallopt(M_MMAP_MAX, 0);
  mallopt(M_TRIM_THRESHOLD, 1 << 30);
  return guarded([&] {
    if (threads < 1) threads = 1;
    std::mt19937_64 rng(4321);
    std::uniform_real_distribution<float> dist(-1.0f, 1.0f);
    std::vector<TokenMatrix> ins, ress;
    const std::int64_t chunk = (T + threads - 1) / threads;
    for (int c = 0; c < threads; ++c) {
      const std::int64_t rows = std::max<std::int64_t>(0, std::min(T, (c + 1) * chunk) - c * chunk);
      TokenMatrix a = TokenMatrix::zeros(rows, H), b = TokenMatrix::zeros(rows, H);
      for (float& v : a.values) v = dist(rng);
      for (float& v : b.values) v = dist(rng);
      ins.push_back(std::move(a));
      ress.push_back(std::move(b));
    }
    NormParams p;
    p.weight.assign(H, 1.0f);
    std::vector<double> ms;
    for (int i = 0; i < iters; ++i) {
      const auto t0 = std::chrono::steady_clock::now();
      std::vector<std::thread> pool;
      for (int c = 0; c < threads; ++c) {
        pool.emplace_back([&, c] { NormResult r = rmsnorm_residual(ins[c], ress[c], p); (void)r; });
      }
      for (auto& th : pool) th.join();
      const auto t1 = std::chrono::steady_clock::now();
      ms.push_back(std::chrono::duration<double, std::milli>(t1 - t0).count());
      if (each_ms) each_ms[i] = ms.back();
    }
    std::sort(ms.begin(), ms.end());
    *median_ms = ms[ms.size() / 2];
  });
}

// --- Workloads (proj/src/workloads.cpp): traces, form_batches, the modeled
// throughput (simulate_throughput) that the measured run is printed beside.
// Requests are flat int64 triples {prompt, output, arrival_us} (id = index).

namespace {
std::vector<Request> make_requests(const std::int64_t* r3, const double* arrival, std::int64_t n) {
  std::vector<Request> v;
  for (std::int64_t i = 0; i < n; ++i) v.push_back({i, r3[2 * i], r3[2 * i + 1], arrival ? arrival[i] : 0.0});
  return v;
}
}  // namespace

// out rows: {total_tokens, decode_token_count, kv_context, num_slices}; slices
// rows: {request_id, start, len}.  counts[2] = {batches, slices} (always set);
// returns 1 (DimensionError) if the arrays are too small.
int ref_form_batches(const std::int64_t* r2, const double* arrival, std::int64_t n, std::int64_t chunk,
                     std::int64_t* out4, std::int64_t max_batches, std::int64_t* slices3, std::int64_t max_slices,
                     std::int64_t* counts) {
  return guarded([&] {
    const std::vector<IterationBatch> b = form_batches(make_requests(r2, arrival, n), chunk);
    std::int64_t ns = 0;
    for (const auto& x : b) ns += static_cast<std::int64_t>(x.prefill_token_slices.size());
    counts[0] = static_cast<std::int64_t>(b.size());
    counts[1] = ns;
    if (counts[0] > max_batches || ns > max_slices) throw DimensionError("too small");
    std::int64_t s = 0;
    for (std::size_t k = 0; k < b.size(); ++k) {
      out4[4 * k + 0] = b[k].total_tokens;
      out4[4 * k + 1] = b[k].decode_token_count;
      out4[4 * k + 2] = b[k].kv_context;
      out4[4 * k + 3] = static_cast<std::int64_t>(b[k].prefill_token_slices.size());
      for (const auto& p : b[k].prefill_token_slices) {
        slices3[3 * s + 0] = p.request_id;
        slices3[3 * s + 1] = p.start;
        slices3[3 * s + 2] = p.len;
        ++s;
      }
    }
  });
}

int ref_save_trace(const std::int64_t* r2, const double* arrival, std::int64_t n, const char* path) {
  return guarded([&] { save_trace(make_requests(r2, arrival, n), path); });
}

// counts = number of requests; r2/arrival filled up to cap.  ParseError -> 5.
int ref_load_trace(const char* path, std::int64_t* r2, double* arrival, std::int64_t cap, std::int64_t* count) {
  try {
    const std::vector<Request> v = load_trace(path);
    *count = static_cast<std::int64_t>(v.size());
    for (std::int64_t i = 0; i < std::min<std::int64_t>(cap, *count); ++i) {
      r2[2 * i] = v[i].prompt_tokens;
      r2[2 * i + 1] = v[i].output_tokens;
      arrival[i] = v[i].arrival_s;
    }
    return 0;
  } catch (const ParseError&) {
    return 5;
  } catch (...) {
    return 9;
  }
}

// simulate_throughput on a builtin profile/model preset: out4 = {tokens_per_sec,
// iterations, total_tokens, total_seconds}.
int ref_simulate_throughput(const char* profile, const char* model, const char* mode, const std::int64_t* r2,
                            std::int64_t n, std::int64_t chunk, double* out4) {
  return guarded([&] {
    const HardwareProfile hp = builtin_profile(profile);
    const ModelPreset mp = model_preset(model);
    const ThroughputResult r = simulate_throughput(make_requests(r2, nullptr, n), mp.spec, hp,
                                                   baseline_mode_from_string(mode), mp.policy, chunk);
    out4[0] = r.tokens_per_sec;
    out4[1] = static_cast<double>(r.iterations);
    out4[2] = static_cast<double>(r.total_tokens);
    out4[3] = r.total_seconds;
  });
}

// The reference CLI's `throughput` command (proj/src/commands.cpp:432-480),
// run as shipped: its CSV (modeled tokens/s of the fixed-2048x128 and
// chatlike traces, every mode) into buf.  Returns the CSV length.
long long ref_cmd_throughput_csv(const char* model, const char* profile, std::int64_t chunk, std::uint64_t seed,
                                 char* buf, long long cap) {
  long long n = -1;
  guarded([&] {
    RunConfig c;
    c.model = model;
    c.profile = profile;
    c.chunk_size = chunk;
    c.seed = seed;
    const CommandResult r = cmd_throughput(c);
    n = static_cast<long long>(r.csv.size());
    if (buf && cap > 0) {
      const long long m = std::min<long long>(n, cap - 1);
      std::memcpy(buf, r.csv.data(), static_cast<size_t>(m));
      buf[m] = '\0';
    }
  });
  return n;
}

// Restatement of the CLI's chatlike_trace (proj/src/commands.cpp:59-75,
// anonymous there): lognormal prompts / replies from std::mt19937_64(seed),
// clamped.  Test infrastructure: pinned by feeding it to simulate_throughput
// and matching ref_cmd_throughput_csv's chatlike rows.  out2 = {prompt, output}.
int ref_chatlike_trace(std::int64_t count, std::uint64_t seed, std::int64_t* out2) {
  return guarded([&] {
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> prompt_log(6.8, 0.9);
    std::normal_distribution<double> output_log(4.0, 0.7);
    for (std::int64_t i = 0; i < count; ++i) {
      out2[2 * i] = std::clamp<std::int64_t>(std::llround(std::exp(prompt_log(rng))), 32, 8192);
      out2[2 * i + 1] = std::clamp<std::int64_t>(std::llround(std::exp(output_log(rng))), 16, 256);
    }
  });
}

// The reference's Timeline JSON (proj/src/scheduler.cpp:301-317) of one
// iteration_timeline call on a builtin profile / model preset: the schema
// fixture the measured C++ iteration_timeline is compared with.
long long ref_timeline_json(const char* profile, const char* model, std::int64_t T, const char* mode, char* buf,
                            long long cap) {
  long long n = -1;
  guarded([&] {
    const HardwareProfile hp = builtin_profile(profile);
    const ModelPreset mp = model_preset(model);
    BatchShape b;
    b.total_tokens = T;
    const std::string j = iteration_timeline(b, mp.spec, hp, baseline_mode_from_string(mode), mp.policy).to_json();
    n = static_cast<long long>(j.size());
    if (buf && cap > 0) {
      const long long m = std::min<long long>(n, cap - 1);
      std::memcpy(buf, j.data(), static_cast<size_t>(m));
      buf[m] = '\0';
    }
  });
  return n;
}

}  // extern "C"
