// weavesim/wavemodel.hpp -- drop-in subset of the reference wave model
// (proj/include/weavesim/wavemodel.hpp:11-95) that the token-split planner
// needs: the hardware/tile geometry and the CTA / wave counts.  The analytic
// time model (gemm_time, collective_time, ...) is the reference simulator's
// job and is not re-implemented: the B200 weave runner MEASURES layer times.
#pragma once

#include <cstdint>
#include <string>

namespace weavesim {

struct HardwareProfile {
  std::string name = "h100";
  int num_sms = 132;
  int tile_tokens = 128;   // tokens per CTA row tile of a GEMM
  int cta_columns = 32;    // CTA columns per GEMM
  int collective_sms = 8;  // SMs the fused collective occupies while overlapping
  int bytes_per_element = 2;
  double sm_flops = 4.2e12;
  double hbm_bandwidth_effective = 2.24e12;
  double collective_base_latency = 13.5e-6;
  double collective_per_token_time = 6.0e-8;
  double fused_extra_latency = 0.9e-6;
  double rmsnorm_base_latency = 5.8e-6;
  double rs_base_latency = 12.0e-6;
  double rs_per_token_time = 3.0e-8;
  double ag_base_latency = 12.0e-6;
  double ag_per_token_time = 3.0e-8;
  double ring_collective_scale = 1.4;
  double launch_overhead = 2.0e-6;
  double nonlayer_overhead = 20.0e-3;
  double sm_saturation_coeff = 0.35;
  std::int64_t calib_hidden = 8192;

  // ConfigError on impossible geometry (proj/src/wavemodel.cpp:8-21).
  void validate() const;
};

// Transformer layer shape; per-GPU work is derived via tp_degree
// (proj/include/weavesim/wavemodel.hpp:48-60).
struct LayerSpec {
  std::int64_t hidden = 8192;
  std::int64_t intermediate = 28672;
  int num_attention_heads = 64;
  int num_kv_heads = 8;
  int head_dim = 128;
  int num_layers = 80;
  int experts = 1;  // 1 = dense
  int top_k = 1;    // active experts per token
  int tp_degree = 8;

  // ConfigError on an impossible shape (proj/src/wavemodel.cpp:23-36).
  void validate() const;
};

// B200 geometry (148 SMs, the reference's default tile geometry).  Replaces the
// geometry part of builtin_profile("b200") (proj/src/presets.cpp:58-64).
HardwareProfile b200_geometry();

std::int64_t cta_count(std::int64_t num_tokens, const HardwareProfile& profile);
std::int64_t wave_count(std::int64_t ctas, std::int64_t sms_available);

}  // namespace weavesim
