// Synthetic data: the reference generator behind sgnn_gen_synthetic / sgnn_gen_model,
//     reproduced output-for-output (proj/src/core/synth.hpp:14-58,
//     synth.cpp:18-165): std::mt19937_64, the same float construction and the
//     same file layout, so a dataset generated through this library is
//     byte-identical to one generated through the reference.
//     (The R-MAT benchmark inputs are harness code: tools/rmat_gen.hpp.)
#pragma once

#include <random>
#include <string>
#include <vector>

#include "common.hpp"
#include "host_graph.hpp"
#include "model.hpp"

namespace sgb {

class Rng {  // reference synth.hpp:14-24
 public:
  explicit Rng(uint64_t seed) : eng_(seed) {}
  uint64_t next_u64() { return eng_(); }
  uint32_t below(uint32_t n) { return static_cast<uint32_t>(next_u64() % n); }
  float unit() { return static_cast<float>(next_u64() >> 40) * (1.0f / 16777216.0f); }
  float range(float lo, float hi) { return flush_zero(lo + (hi - lo) * unit()); }

 private:
  std::mt19937_64 eng_;
};

struct GenConfig {
  uint32_t num_nodes = 1000;
  double avg_degree = 8.0;
  uint32_t feature_len = 16;
  uint32_t stream_len = 200;
  uint64_t seed = 1;
  double insert_fraction = 0.6;
};

void write_dataset(const GenConfig& cfg, const std::string& dir);

struct ModelGenConfig {
  std::string kind;
  uint32_t feature_len = 16, hidden = 16, layers = 2;
  uint64_t seed = 1;
  float epsilon = 0.1f;
};

void make_model(const ModelGenConfig& cfg, ModelSpec& spec, WeightSet& ws);
void write_model(const ModelGenConfig& cfg, const std::string& dir);

void make_directories(const std::string& dir);

}  // namespace sgb
