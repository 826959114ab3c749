// test_dropin.cpp -- the reference's own test cases for the hot-path API,
// restated against the drop-in build (libweavesim_b200.so): the same source a
// reference user compiles, linked against the B200 library instead.
//
//   test_dropin host   -> validation / exception / planner cases (no GPU)
//   test_dropin gpu    -> + numerical cases that run the sm_100a kernels
//
// Cases follow proj/tests/test_numerics.cpp, test_collectives.cpp,
// test_splitter.cpp and acceptance.cpp check 1 (cited per case).
#include <chrono>
#include <fstream>
#include <cmath>
#include <tuple>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>

#include "weavesim/collectives.hpp"
#include "weavesim/errors.hpp"
#include "weavesim/numerics.hpp"
#include "weavesim/splitter.hpp"
#include "weavesim/workloads.hpp"
#include "weavesim/presets.hpp"
#include "weavesim/scheduler.hpp"
#include <numeric>

using namespace weavesim;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                          \
  do {                                                                       \
    if (cond) {                                                              \
      ++g_pass;                                                              \
    } else {                                                                 \
      ++g_fail;                                                              \
      std::printf("FAIL %s:%d  %s\n", __FILE__, __LINE__, #cond);            \
    }                                                                        \
  } while (0)
#define CHECK_THROWS_AS(expr, Type)                                          \
  do {                                                                       \
    bool ok_ = false;                                                        \
    try {                                                                    \
      (void)(expr);                                                          \
    } catch (const Type&) {                                                  \
      ok_ = true;                                                            \
    } catch (...) {                                                          \
    }                                                                        \
    CHECK(ok_ && #Type);                                                     \
  } while (0)

namespace {

TokenMatrix random_matrix(std::int64_t t, std::int64_t h, std::mt19937_64& rng, float lo, float hi) {
  std::uniform_real_distribution<float> d(lo, hi);
  TokenMatrix m = TokenMatrix::zeros(t, h);
  for (float& v : m.values) v = d(rng);
  return m;
}

RankGroup random_group(int world, std::int64_t tokens, std::int64_t hidden, std::uint64_t seed) {
  std::mt19937_64 rng(seed);
  RankGroup g;
  g.world_size = world;
  for (int r = 0; r < world; ++r) g.inputs.push_back(random_matrix(tokens, hidden, rng, -1.f, 1.f));
  for (const TokenRange& range : token_shard_map(tokens, world).ranges)
    g.residual_shards.push_back(random_matrix(range.size(), hidden, rng, -1.f, 1.f));
  return g;
}

NormParams unit_norm(std::int64_t h) {
  NormParams p;
  p.weight.assign(static_cast<size_t>(h), 1.0f);
  return p;
}

void host_cases() {
  // test_numerics.cpp:39-60
  TokenMatrix m = TokenMatrix::zeros(7, 5);
  CHECK(m.values.size() == 35);
  TokenMatrix bad = TokenMatrix::zeros(2, 3);
  bad.values.pop_back();
  CHECK_THROWS_AS(bad.validate(), DimensionError);
  TokenMatrix nan = TokenMatrix::zeros(2, 3);
  nan.values[1] = std::nanf("");
  CHECK_THROWS_AS(nan.validate(), NumericError);
  // test_numerics.cpp:117-126
  NormParams p8 = unit_norm(8);
  CHECK_THROWS_AS(rmsnorm_residual(TokenMatrix::zeros(2, 8), TokenMatrix::zeros(3, 8), p8), DimensionError);
  NormParams p7 = unit_norm(7);
  CHECK_THROWS_AS(rmsnorm_residual(TokenMatrix::zeros(2, 8), TokenMatrix::zeros(2, 8), p7), DimensionError);
  // test_collectives.cpp:40-70
  for (std::int64_t T : {0, 1, 7, 8, 100, 1023}) {
    for (int W : {2, 3, 4, 8}) {
      ShardMap map = token_shard_map(T, W);
      CHECK(map.world_size() == W && map.total_tokens() == T);
      bool ok = true;
      for (const TokenRange& r : map.ranges) ok = ok && r.size() >= T / W && r.size() <= T / W + 1;
      CHECK(ok);
      map.validate(T);
    }
  }
  CHECK_THROWS_AS(token_shard_map(16, 1), ConfigError);
  CHECK_THROWS_AS(token_shard_map(-1, 4), DimensionError);
  ShardMap sm = token_shard_map(16, 4);
  CHECK_THROWS_AS(sm.validate(17), ContractError);
  ShardMap ov = sm;
  ov.ranges[2].begin -= 1;
  CHECK_THROWS_AS(ov.validate(16), ContractError);
  CHECK_THROWS_AS(ShardMap{}.validate(0), ContractError);
  // test_collectives.cpp:129-161 (validation precedes any device work)
  RankGroup g = random_group(4, 8, 8, 3);
  const ShardMap shards = token_shard_map(8, 4);
  RankGroup wrong_count = g;
  wrong_count.inputs.pop_back();
  CHECK_THROWS_AS(all_reduce(wrong_count), DimensionError);
  RankGroup bad_res = g;
  bad_res.residual_shards[1] = TokenMatrix::zeros(5, 8);
  CHECK_THROWS_AS(fused_allreduce_rmsnorm(bad_res, unit_norm(8), shards), DimensionError);
  ShardMap corrupt = shards;
  corrupt.ranges[1].begin -= 1;
  CHECK_THROWS_AS(fused_allreduce_rmsnorm(g, unit_norm(8), corrupt), ContractError);
  CHECK_THROWS_AS(fused_allreduce_rmsnorm(g, unit_norm(7), shards), DimensionError);
  const ShardMap s10 = token_shard_map(10, 2);
  std::vector<TokenMatrix> wrong = {TokenMatrix::zeros(5, 4), TokenMatrix::zeros(4, 4)};
  CHECK_THROWS_AS(all_gather(wrong, s10), DimensionError);
  // test_splitter.cpp:21-32, 34-47, 128-150
  SplitPolicy dense;
  CHECK(select_mode(1023, dense) == SplitMode::FusedOnly);
  CHECK(select_mode(1024, dense) == SplitMode::Overlap);
  HardwareProfile p;
  p.tile_tokens = 128;
  p.cta_columns = 4;
  const std::int64_t T = 9600, prefix = T / 2 + smart_offset_analytic(T, p);
  CHECK(cta_count(prefix, p) == 132);
  CHECK(wave_count(cta_count(prefix, p), p.num_sms) + wave_count(cta_count(T - prefix, p), p.num_sms) == 3);
  SplitPlan plan;
  plan.total_tokens = 100;
  plan.prefix_tokens = 55;
  plan = place_sequence_boundaries({30, 40, 30}, plan);
  CHECK((plan.prefix_len_per_sequence == std::vector<std::int64_t>{30, 25, 0}));
  CHECK_THROWS_AS(place_sequence_boundaries({30, 40}, plan), ContractError);
  // SURVEY.md Appendix A (B200 geometry, dense threshold 1024)
  const SplitPlan b = make_split_plan(4096, b200_geometry(), dense);
  CHECK(b.prefix_tokens == 1152 && b.suffix_tokens == 2944 && b.offset == -896 && b.mode == SplitMode::Overlap);
  CHECK(make_split_plan(512, b200_geometry(), dense).mode == SplitMode::FusedOnly);
  // Alg. 1 sweep tie rules (test_splitter.cpp:83-101)
  SplitPolicy grid;
  CHECK(smart_offset_sweep(4096, grid, [](std::int64_t, std::int64_t) { return 1.0; }) == 0);
  CHECK(smart_offset_sweep(4096, grid, [](std::int64_t a, std::int64_t) { return a == 2048 + 128 ? 0.5 : 1.0; }) ==
        128);
  CHECK(smart_offset_sweep(64, grid, [](std::int64_t, std::int64_t) { return 1.0; }) == 0);
}

void gpu_cases() {
  // test_numerics.cpp:62-89 -- vs an independent double-precision restatement
  std::mt19937_64 rng(7);
  // 2049 x 4096 fp32 (32 MiB per matrix): the result vectors are
  // value-initialised on helper threads overlapped with the pipeline (ragged
  // against both the 512-row pipeline chunk and the 256-row fill step)
  for (auto [T, H] : {std::pair<std::int64_t, std::int64_t>{1, 8}, {5, 16}, {17, 33}, {64, 128}, {2049, 4096}}) {
    const TokenMatrix in = random_matrix(T, H, rng, -2.f, 2.f);
    const TokenMatrix res = random_matrix(T, H, rng, -2.f, 2.f);
    NormParams params;
    std::uniform_real_distribution<float> wd(0.5f, 1.5f);
    params.weight.resize(static_cast<size_t>(H));
    for (float& w : params.weight) w = wd(rng);
    const NormResult r = rmsnorm_residual(in, res, params);
    bool ok = true;
    for (std::int64_t t = 0; t < T; ++t) {
      double ss = 0;
      for (std::int64_t j = 0; j < H; ++j) {
        const double v = double(in.at(t, j)) + res.at(t, j);
        ss += v * v;
      }
      const double inv = 1.0 / std::sqrt(ss / H + params.epsilon);
      for (std::int64_t j = 0; j < H; ++j) {
        const double want = (double(in.at(t, j)) + res.at(t, j)) * inv * params.weight[j];
        ok = ok && std::abs(r.output.at(t, j) - want) <= 1e-5;
        ok = ok && r.residual_out.at(t, j) == in.at(t, j) + res.at(t, j);
      }
    }
    CHECK(ok);
  }
  {
    // a NaN on the overlapped-fill path: NumericError, helper threads joined,
    // and the next call on the same path is correct
    TokenMatrix in = random_matrix(1500, 4096, rng, -1.f, 1.f);
    const TokenMatrix res = random_matrix(1500, 4096, rng, -1.f, 1.f);
    NormParams p = unit_norm(4096);
    in.at(1400, 7) = std::nanf("");
    CHECK_THROWS_AS(rmsnorm_residual(in, res, p), NumericError);
    in.at(1400, 7) = 0.5f;
    const NormResult r = rmsnorm_residual(in, res, p);
    bool same = r.output.values.size() == in.values.size() && r.residual_out.values.size() == in.values.size();
    for (size_t i = 0; same && i < in.values.size(); ++i) same = r.residual_out.values[i] == in.values[i] + res.values[i];
    CHECK(same);
  }
  // test_numerics.cpp:91-98
  NormParams p8 = unit_norm(8);
  const NormResult z = rmsnorm_residual(TokenMatrix::zeros(3, 8), TokenMatrix::zeros(3, 8), p8);
  bool zero = true;
  for (float v : z.output.values) zero = zero && v == 0.0f;
  CHECK(zero);
  // test_collectives.cpp:72-92
  RankGroup g = random_group(4, 9, 12, 5);
  const TokenMatrix sum = all_reduce(g);
  bool exact = true;
  for (std::int64_t i = 0; i < 9 * 12; ++i) {
    float e = 0.0f;
    for (const TokenMatrix& m : g.inputs) e += m.values[i];
    exact = exact && sum.values[i] == e;
  }
  CHECK(exact);
  RankGroup wide = random_group(13, 9, 12, 6);  // wider than a communicator
  const TokenMatrix wsum = all_reduce(wide);
  bool wexact = true;
  for (std::int64_t i = 0; i < 9 * 12; ++i) {
    float e = 0.0f;
    for (const TokenMatrix& m : wide.inputs) e += m.values[i];
    wexact = wexact && wsum.values[i] == e;
  }
  CHECK(wexact);
  for (std::int64_t tokens : {1, 7, 64, 129}) {
    RankGroup gg = random_group(8, tokens, 16, 1000 + tokens);
    const ShardMap shards = token_shard_map(tokens, 8);
    CHECK(all_reduce(gg).values == all_gather(reduce_scatter(gg, shards), shards).values);
  }
  // test_collectives.cpp:94-114 -- fused vs unfused composition
  // worlds above TW_MAX_RANKS take the drop-in's chained path (the reference
  // accepts any N >= 2); 1027 x 4096 (16 MiB outputs) takes the helper-thread
  // output fill in all_reduce, reduce_scatter and fused_allreduce_rmsnorm
  for (auto [world, tokens, hidden] : {std::tuple<int, std::int64_t, std::int64_t>{2, 1, 32}, {2, 3, 32},
                                       {2, 17, 32}, {2, 40, 32}, {4, 1, 32}, {4, 3, 32}, {4, 17, 32}, {4, 40, 32},
                                       {8, 1, 32}, {8, 3, 32}, {8, 17, 32}, {8, 40, 32}, {12, 1, 32}, {12, 3, 32},
                                       {12, 17, 32}, {12, 40, 32}, {16, 1, 32}, {16, 3, 32}, {16, 17, 32},
                                       {16, 40, 32}, {2, 1027, 4096}, {3, 1027, 4096}, {12, 1027, 4096}}) {
    {
      RankGroup group = random_group(world, tokens, hidden, 77 * world + tokens);
      const ShardMap shards = token_shard_map(tokens, world);
      const NormParams params = unit_norm(hidden);
      const TokenMatrix reduced = all_reduce(group);
      const TokenMatrix residual = all_gather(group.residual_shards, shards);
      const NormResult oracle = rmsnorm_residual(reduced, residual, params);
      const TokenMatrix fused = fused_allreduce_rmsnorm(group, params, shards);
      bool ok = fused.values.size() == oracle.output.values.size();
      for (size_t i = 0; ok && i < fused.values.size(); ++i)
        ok = std::abs(fused.values[i] - oracle.output.values[i]) <= 1e-5;
      CHECK(ok);
      CHECK(all_gather(group.residual_shards, shards).values == oracle.residual_out.values);
      if (hidden == 4096) {  // the large outputs: rank-ascending fp32 sum, RS o AG == AR, bitwise
        bool exact = true;
        for (size_t i = 0; exact && i < reduced.values.size(); ++i) {
          float e = 0.0f;
          for (const TokenMatrix& m : group.inputs) e += m.values[i];
          exact = reduced.values[i] == e;
        }
        CHECK(exact);
        CHECK(all_gather(reduce_scatter(group, shards), shards).values == reduced.values);
      }
    }
  }
  // test_collectives.cpp:116-127 -- parallel flag is bitwise neutral
  RankGroup seq = random_group(8, 53, 24, 99);
  RankGroup par = seq;
  const ShardMap s53 = token_shard_map(53, 8);
  const TokenMatrix a = fused_allreduce_rmsnorm(seq, unit_norm(24), s53, false);
  const TokenMatrix b = fused_allreduce_rmsnorm(par, unit_norm(24), s53, true);
  CHECK(a.values == b.values);
  for (int r = 0; r < 8; ++r) CHECK(seq.residual_shards[r].values == par.residual_shards[r].values);
  // NaN/Inf anywhere in the group -> NumericError with the residual shards
  // untouched (the drop-in scans while staging the copies; the reference
  // validates first), and a structural error still wins over a NaN wherever
  // the reference checks structure first
  for (int world : {2, 8}) {
    RankGroup clean = random_group(world, 40, 64, 5 + world);
    const ShardMap sh = token_shard_map(40, world);
    RankGroup nan_in = clean;
    nan_in.inputs[world - 1].values[64 * 17 + 3] = std::nanf("");
    CHECK_THROWS_AS(fused_allreduce_rmsnorm(nan_in, unit_norm(64), sh), NumericError);
    CHECK(nan_in.residual_shards[0].values == clean.residual_shards[0].values);
    RankGroup inf_res = clean;
    inf_res.residual_shards[1].values.back() = -INFINITY;
    CHECK_THROWS_AS(fused_allreduce_rmsnorm(inf_res, unit_norm(64), sh), NumericError);
    CHECK(inf_res.residual_shards[0].values == clean.residual_shards[0].values);
    CHECK_THROWS_AS(fused_allreduce_rmsnorm(nan_in, unit_norm(63), sh), NumericError);  // validate() precedes the weight check
    RankGroup nan_bad_shard = nan_in;
    nan_bad_shard.residual_shards[0] = TokenMatrix::zeros(3, 64);
    CHECK_THROWS_AS(fused_allreduce_rmsnorm(nan_bad_shard, unit_norm(64), sh), NumericError);  // inputs first
    RankGroup bad_shard = clean;
    bad_shard.residual_shards[0] = TokenMatrix::zeros(3, 64);
    CHECK_THROWS_AS(fused_allreduce_rmsnorm(bad_shard, unit_norm(64), sh), DimensionError);
    CHECK_THROWS_AS(all_reduce(nan_in), NumericError);
    CHECK_THROWS_AS(reduce_scatter(nan_in, sh), NumericError);
    ShardMap bad_map = sh;
    bad_map.ranges[0].end += 1;
    CHECK_THROWS_AS(reduce_scatter(nan_in, bad_map), NumericError);  // the group before the shard map
    CHECK_THROWS_AS(reduce_scatter(clean, bad_map), ContractError);
    // and the same group without the NaN still computes (the cached state is intact)
    RankGroup again = clean;
    const TokenMatrix out = fused_allreduce_rmsnorm(again, unit_norm(64), sh);
    CHECK(out.values.size() == static_cast<size_t>(40 * 64));
  }
}

// acceptance.cpp:37-86 -- the fused op vs the unfused chain over the
// acceptance grid (full grid: N{2,4,8} x T{1,3,17,256,1024} x H{16,64,1024}
// x 50 seeds = 2250 instances, <= 1e-5, < 60 s).
void acceptance_cases(bool full) {
  const auto t0 = std::chrono::steady_clock::now();
  const std::vector<std::int64_t> token_grid =
      full ? std::vector<std::int64_t>{1, 3, 17, 256, 1024} : std::vector<std::int64_t>{1, 3, 17, 256};
  const int seeds = full ? 50 : 2;
  double max_err = 0;
  long instances = 0;
  for (int world : {2, 4, 8})
    for (std::int64_t tokens : token_grid)
      for (std::int64_t hidden : {16, 64, 1024})
        for (int seed = 0; seed < seeds; ++seed) {
          ++instances;
          std::mt19937_64 r2((std::uint64_t(world) << 48) ^ (std::uint64_t(tokens) << 24) ^
                             (std::uint64_t(hidden) << 8) ^ std::uint64_t(seed));
          std::uniform_real_distribution<float> d(-1.f, 1.f);
          RankGroup grp;
          grp.world_size = world;
          for (int q = 0; q < world; ++q) {
            TokenMatrix m = TokenMatrix::zeros(tokens, hidden);
            for (float& v : m.values) v = d(r2);
            grp.inputs.push_back(std::move(m));
          }
          const ShardMap sh = token_shard_map(tokens, world);
          for (const TokenRange& rg : sh.ranges) {
            TokenMatrix m = TokenMatrix::zeros(rg.size(), hidden);
            for (float& v : m.values) v = d(r2);
            grp.residual_shards.push_back(std::move(m));
          }
          NormParams prm;
          prm.weight.resize(static_cast<size_t>(hidden));
          std::uniform_real_distribution<float> wd(0.5f, 1.5f);
          for (float& w : prm.weight) w = wd(r2);
          const NormResult orc = rmsnorm_residual(all_reduce(grp), all_gather(grp.residual_shards, sh), prm);
          const TokenMatrix fused = fused_allreduce_rmsnorm(grp, prm, sh);
          for (size_t i = 0; i < fused.values.size(); ++i)
            max_err = std::max(max_err, double(std::abs(fused.values[i] - orc.output.values[i])));
        }
  const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::printf("acceptance%s instances=%ld max_abs_err=%.3g runtime=%.1fs\n", full ? "" : "-slice", instances, max_err,
              secs);
  CHECK(max_err <= 1e-5);
  if (full) CHECK(secs < 60.0);
}

// proj/tests/test_workloads.cpp:14-125, restated (host only).
void workload_cases() {
  {  // :14-26 trace JSONL round trip
    const std::string path = "test_trace_roundtrip.jsonl";
    std::vector<Request> requests = {{0, 100, 10, 0.0}, {1, 2048, 128, 0.5}, {2, 1, 0, 1.25}};
    save_trace(requests, path);
    const std::vector<Request> loaded = load_trace(path);
    CHECK(loaded.size() == 3);
    for (size_t i = 0; i < 3 && i < loaded.size(); ++i) {
      CHECK(loaded[i].prompt_tokens == requests[i].prompt_tokens);
      CHECK(loaded[i].output_tokens == requests[i].output_tokens);
      CHECK(loaded[i].arrival_s == requests[i].arrival_s);
    }
    std::remove(path.c_str());
  }
  {  // :28-54 parse errors name the line
    const std::string path = "test_trace_bad.jsonl";
    {
      std::ofstream out(path);
      out << R"({"prompt_tokens": 10, "output_tokens": 2})" << "\n";
      out << "not json\n";
    }
    bool named = false;
    try {
      load_trace(path);
    } catch (const ParseError& e) {
      named = std::string(e.what()).find("line 2") != std::string::npos;
    }
    CHECK(named);
    {
      std::ofstream out(path);
      out << R"({"prompt_tokens": 10})" << "\n";
    }
    CHECK_THROWS_AS(load_trace(path), ParseError);
    {
      std::ofstream out(path);
      out << R"({"prompt_tokens": 0, "output_tokens": 2})" << "\n";
    }
    CHECK_THROWS_AS(load_trace(path), ParseError);
    std::remove(path.c_str());
    CHECK_THROWS_AS(load_trace("missing_trace.jsonl"), ParseError);
  }
  {  // :56-70 conservation
    std::int64_t prefill = 0, decode = 0;
    for (const IterationBatch& b : form_batches(synth_trace(16, 1000, 37), 512)) {
      std::int64_t slice_sum = 0;
      for (const PrefillSlice& s : b.prefill_token_slices) slice_sum += s.len;
      CHECK(b.total_tokens == slice_sum + b.decode_token_count);
      prefill += slice_sum;
      decode += b.decode_token_count;
    }
    CHECK(prefill == 16 * 1000);
    CHECK(decode == 16 * 37);
  }
  {  // :72-80 budget
    bool ok = true;
    for (const IterationBatch& b : form_batches(synth_trace(8, 4096, 64), 1024)) {
      std::int64_t slice_sum = 0;
      for (const PrefillSlice& s : b.prefill_token_slices) slice_sum += s.len;
      ok = ok && slice_sum <= 1024 && b.total_tokens <= 1024 + b.decode_token_count;
    }
    CHECK(ok);
  }
  {  // :82-98 FCFS, decode-only tail
    const std::vector<IterationBatch> b = form_batches(synth_trace(4, 100, 5), 250);
    CHECK(!b.empty() && b[0].prefill_token_slices.size() == 3);
    if (!b.empty() && b[0].prefill_token_slices.size() == 3) {
      CHECK(b[0].prefill_token_slices[0].request_id == 0);
      CHECK(b[0].prefill_token_slices[2].request_id == 2);
      CHECK(b[0].prefill_token_slices[2].len == 50);
      CHECK(b[0].decode_token_count == 0);
      CHECK(b[1].decode_token_count == 2);
      CHECK(b.back().decode_only());
    }
  }
  {  // :100-106 arrival ties
    const std::vector<IterationBatch> b = form_batches({{0, 100, 0, 2.0}, {1, 100, 0, 0.0}, {2, 100, 0, 2.0}}, 100);
    CHECK(b.size() == 3 && b[0].prefill_token_slices[0].request_id == 1 &&
          b[1].prefill_token_slices[0].request_id == 0 && b[2].prefill_token_slices[0].request_id == 2);
  }
  {  // :108-119 kv context
    const std::vector<IterationBatch> b = form_batches(synth_trace(1, 300, 3), 100);
    CHECK(b.size() == 6);
    const std::int64_t want[6] = {0, 100, 200, 300, 301, 302};
    for (size_t i = 0; i < 6 && i < b.size(); ++i) CHECK(b[i].kv_context == want[i]);
  }
  // :121-125 bad arguments
  CHECK_THROWS_AS(form_batches({}, 0), ConfigError);
  CHECK_THROWS_AS(synth_trace(0, 100, 10), ConfigError);
  CHECK_THROWS_AS(synth_trace(4, 0, 10), ConfigError);
  // presets / modes / LayerSpec (proj/src/presets.cpp:68-110, scheduler.cpp:16-46, wavemodel.cpp:23-36)
  CHECK(model_preset("llama-70b").spec.num_layers == 80 && model_preset("mixtral-8x22b").spec.experts == 8);
  CHECK(model_preset("mixtral-8x22b").policy.threshold_tokens == 4096 && model_preset_names().size() == 3);
  CHECK_THROWS_AS(model_preset("gpt-5"), ConfigError);
  CHECK(builtin_profile("b200").num_sms == 148 && builtin_profile("h100").num_sms == 132);
  CHECK_THROWS_AS(builtin_profile("a100"), ConfigError);
  for (BaselineMode m : {BaselineMode::Default, BaselineMode::Multimem, BaselineMode::NoComm, BaselineMode::FuseOnly,
                         BaselineMode::TokenWeave})
    CHECK(baseline_mode_from_string(to_string(m)) == m);
  CHECK_THROWS_AS(baseline_mode_from_string("magic"), ConfigError);
  {
    LayerSpec bad = model_preset("llama-70b").spec;
    bad.tp_degree = 1;
    CHECK_THROWS_AS(bad.validate(), ConfigError);
    bad = model_preset("llama-70b").spec;
    bad.num_kv_heads = 7;
    CHECK_THROWS_AS(bad.validate(), ConfigError);
  }
  // simulate_throughput validates before touching a device
  const ModelPreset pr = model_preset("llama-70b");
  CHECK_THROWS_AS(simulate_throughput(synth_trace(2, 10, 1), pr.spec, builtin_profile("b200"),
                                      BaselineMode::TokenWeave, pr.policy, 0),
                  ConfigError);
  {
    BatchShape neg;
    neg.total_tokens = -1;
    CHECK_THROWS_AS(iteration_latency(neg, pr.spec, builtin_profile("b200"), BaselineMode::FuseOnly, pr.policy),
                    DimensionError);
    BatchShape empty;
    CHECK(iteration_latency(empty, pr.spec, builtin_profile("b200"), BaselineMode::FuseOnly, pr.policy) == 0.0);
  }
}

// proj/tests/test_workloads.cpp:127-147 on the measured (B200) simulate_throughput.
void throughput_gpu_cases() {
  const ModelPreset preset = model_preset("llama-70b");
  const HardwareProfile profile = builtin_profile("b200");
  const std::vector<Request> requests = synth_trace(4, 512, 3);
  const ThroughputResult r =
      simulate_throughput(requests, preset.spec, profile, BaselineMode::TokenWeave, preset.policy, 1024);
  CHECK(r.total_tokens == 4 * (512 + 3));
  CHECK(r.iterations == static_cast<std::int64_t>(r.iteration_latencies.size()));
  const double sum = std::accumulate(r.iteration_latencies.begin(), r.iteration_latencies.end(), 0.0);
  CHECK(std::abs(r.total_seconds - sum) <= 1e-12 * sum + 1e-15);
  CHECK(std::abs(r.tokens_per_sec - r.total_tokens / r.total_seconds) <= 1e-9 * r.tokens_per_sec);
  const double nocomm =
      simulate_throughput(requests, preset.spec, profile, BaselineMode::NoComm, preset.policy, 1024).tokens_per_sec;
  const double multimem =
      simulate_throughput(requests, preset.spec, profile, BaselineMode::Multimem, preset.policy, 1024).tokens_per_sec;
  CHECK(nocomm >= multimem);
  // iteration_latency: measured layer x num_layers; communication costs time
  BatchShape b;
  b.total_tokens = 2048;
  const double nc = iteration_latency(b, preset.spec, profile, BaselineMode::NoComm, preset.policy);
  const double fo = iteration_latency(b, preset.spec, profile, BaselineMode::FuseOnly, preset.policy);
  const double mm = iteration_latency(b, preset.spec, profile, BaselineMode::Multimem, preset.policy);
  const double tw = iteration_latency(b, preset.spec, profile, BaselineMode::TokenWeave, preset.policy);
  CHECK(nc > 0 && nc < fo && fo < mm && tw > nc);
  std::printf("iteration_latency (llama-70b, T=2048, 80 layers): nocomm %.2f ms, fuseonly %.2f, multimem %.2f, "
              "tokenweave %.2f\n", 1e3 * nc, 1e3 * fo, 1e3 * mm, 1e3 * tw);
}

}  // namespace

// test_dropin timeline <dir>: the measured iteration_timeline JSON of one
// Llama-3.3-70B layer (T = 8192, TP = 8 shapes) for TokenWeave and FuseOnly,
// written to <dir>/timeline_<mode>.json (schema-checked by tests/test_dropin.py).
void timeline_cases(const std::string& dir) {
  const ModelPreset preset = model_preset("llama-70b");
  BatchShape b;
  b.total_tokens = 8192;
  for (BaselineMode m : {BaselineMode::TokenWeave, BaselineMode::FuseOnly}) {
    const Timeline t = iteration_timeline(b, preset.spec, builtin_profile("b200"), m, preset.policy);
    CHECK(!t.events.empty() && t.iteration_latency > 0);
    t.to_json_file(dir + "/timeline_" + to_string(m) + ".json");
  }
}

// usage: test_dropin host | gpu | acceptance | timeline <dir>
int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "host";
  host_cases();
  workload_cases();
  if (mode == "gpu") {
    gpu_cases();
    throughput_gpu_cases();
    acceptance_cases(false);
  }
  if (mode == "acceptance") acceptance_cases(true);
  if (mode == "timeline") timeline_cases(argc > 2 ? argv[2] : ".");
  std::printf("%s: %d passed, %d failed\n", mode.c_str(), g_pass, g_fail);
  return g_fail ? 1 : 0;
}
