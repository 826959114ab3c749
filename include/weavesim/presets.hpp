// weavesim/presets.hpp -- drop-in model presets and built-in profiles
// (proj/include/weavesim/presets.hpp:12-33, proj/src/presets.cpp:53-110).
// builtin_profile returns the GEOMETRY of the named GPU (SM count, tile
// shape) -- what the split planner and the measured layer runner use; the
// reference's calibrated analytic rates belong to its simulator (out of
// scope), so the rate fields keep their defaults.
#pragma once

#include <string>
#include <vector>

#include "weavesim/splitter.hpp"
#include "weavesim/wavemodel.hpp"

namespace weavesim {

struct ModelPreset {
  std::string name;
  LayerSpec spec;
  SplitPolicy policy;
};

// llama-70b, qwen-72b, mixtral-8x22b (proj/src/presets.cpp:68-104).
ModelPreset model_preset(const std::string& name);
std::vector<std::string> model_preset_names();

// "h100" (132 SMs) and "b200" (148 SMs); ConfigError otherwise.
HardwareProfile builtin_profile(const std::string& name);

}  // namespace weavesim
