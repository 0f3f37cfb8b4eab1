// Model description, weights and binding.
//
// The description grammar, weight manifest and dimension/hook validation are
// the reference's (proj/src/core/model.hpp:28-115, model.cpp:29-218,
// hooks.cpp:38-62), re-implemented so the same files load with the same error
// codes. A bound model is lowered to a per-partition op program that the device
// engine executes (device/combine.cuh); the arithmetic contract of every op is
// pinned in that file.
#pragma once

#include <map>
#include <string>
#include <vector>

#include "common.hpp"

namespace sgb {

enum class OpKind : uint8_t { Aggregate, Linear, Relu, UserApply };

struct ModelOp {
  OpKind kind = OpKind::Relu;
  std::string weight;  // Linear
  std::string bias;    // Linear, empty = none
  std::string hook;    // UserApply
};

struct Partition {
  uint32_t begin = 0, end = 0, aggregate = 0;
};

struct ModelSpec {
  std::vector<ModelOp> ops;
  std::vector<Partition> partitions;
  Agg agg = Agg::Min;

  static ModelSpec parse(const std::string& text);
  std::string serialize() const;
  int num_layers() const { return static_cast<int>(partitions.size()); }
  bool has_user_ops() const;
  bool has_prefix_ops() const { return partitions[0].aggregate > 0; }
};

struct Matrix {
  uint32_t rows = 0, cols = 0;
  std::vector<float> data;
};

struct WeightSet {
  std::map<std::string, Matrix> matrices;
  std::map<std::string, std::vector<float>> vectors;
  std::map<uint32_t, float> epsilon;
};

WeightSet load_weights(const std::string& manifest_path);
void save_weights(const WeightSet& ws, const std::string& manifest_path);

// One executable step of a partition's combination (after its aggregate) or of
// the prefix (before the first aggregate).
struct ProgramOp {
  enum Kind : uint8_t { Linear, Relu, SageSelf, GinSelf } kind;
  const Matrix* w = nullptr;                // Linear: W; SageSelf: W2_<p>
  const std::vector<float>* bias = nullptr;  // Linear only
  float gin_scale = 0.0f;                   // 1.0f + epsilon_p, computed in float (hooks.cpp:33)
  uint32_t in_dim = 0, out_dim = 0;         // running-value dims before/after the op
};

// A spec bound to weights and an input length, with every stage dimension
// validated (reference Model ctor, model.cpp:184-218).
class BoundModel {
 public:
  BoundModel(const ModelSpec& spec, const WeightSet& ws, uint32_t input_dim);
  BoundModel(const BoundModel&) = delete;  // programs point into ws_
  BoundModel& operator=(const BoundModel&) = delete;

  Agg agg() const { return spec_.agg; }
  int num_layers() const { return spec_.num_layers(); }
  uint32_t input_dim() const { return input_dim_; }
  bool has_prefix() const { return spec_.has_prefix_ops(); }
  bool has_user_ops() const { return spec_.has_user_ops(); }
  // Message length feeding layer 1..k; k+1 = output (model.cpp:220-224).
  uint32_t message_dim(int layer) const;
  // Self-message reads performed per combination of partition p (one per
  // user_apply op; EngineApplyContext::self_message, engine.cpp:125-128).
  int user_ops_in(int partition) const { return user_ops_[partition]; }
  const std::vector<ProgramOp>& program(int partition) const { return programs_[partition]; }
  const std::vector<ProgramOp>& prefix() const { return prefix_; }

 private:
  ModelSpec spec_;
  WeightSet ws_;
  uint32_t input_dim_;
  std::vector<uint32_t> stage_dims_;
  std::vector<std::vector<ProgramOp>> programs_;
  std::vector<ProgramOp> prefix_;
  std::vector<int> user_ops_;
};

}  // namespace sgb
