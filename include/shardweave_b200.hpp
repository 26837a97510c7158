// Header-only C++ face of the C ABI, for reference (shardweave) code that wants to run its
// transformer training step on B200s. The names follow the reference's own API so a call site
// changes by namespace only:
//   shardweave::parse_model_spec        -> shardweave::b200::parse_model_spec
//   shardweave::derive_plan / validate_plan / serialize_plan / parse_plan
//                                        -> shardweave::b200::{derive_plan, ...}
//   shardweave::build_mesh              -> shardweave::b200::Mesh
//   shard_params + spmd_forward_backward + dp_sync_grads + adamw_step (Trainer::fit inner step,
//   pipeline.hpp:388-449)               -> shardweave::b200::Model::{forward_backward, dp_sync,
//                                          adamw_step, train_step}
// Errors are rethrown as exceptions named like the reference's (ConfigError, PartitionError,
// ShapeError, NonFiniteError; errors.hpp:10-35, tensor.hpp:37-45).
#pragma once

#include <cstdint>
#include <cstdlib>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "shardweave_b200.h"

namespace shardweave {
namespace b200 {

struct Error : std::runtime_error {
  sw_status status;
  Error(sw_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};
struct ConfigError : Error {
  using Error::Error;
};
struct PartitionError : Error {
  using Error::Error;
};
struct ShapeError : Error {
  using Error::Error;
};
struct NonFiniteError : Error {
  using Error::Error;
};
// CheckpointError (errors.hpp:23-35): the message ends with "(at byte offset N)".
struct CheckpointError : Error {
  using Error::Error;
};

/// A named RNG stream captured in a snapshot (RngSnapshot, checkpoint.hpp:190-191).
struct RngState {
  std::string name;
  uint64_t seed = 0, stream_id = 0, counter = 0;
};

inline void check(sw_status s) {
  if (s == SW_OK) return;
  const std::string msg = sw_last_error();
  switch (s) {
    case SW_ERR_CONFIG: throw ConfigError(s, msg);
    case SW_ERR_PARTITION: throw PartitionError(s, msg);
    case SW_ERR_SHAPE: throw ShapeError(s, msg);
    case SW_ERR_NONFINITE: throw NonFiniteError(s, msg);
    case SW_ERR_CHECKPOINT: throw CheckpointError(s, msg);
    default: throw Error(s, msg);
  }
}

inline std::string take(char* p) {
  std::string s = p ? p : "";
  sw_free(p);
  return s;
}

using Shape = std::vector<int64_t>;
using ShapeMap = std::vector<std::pair<std::string, Shape>>;  // params.hpp:88
struct RoleOverride {
  std::string pattern, role;
};

namespace detail {
struct Encoded {
  std::vector<const char*> names;
  std::vector<int32_t> ranks;
  std::vector<int64_t> dims;
  explicit Encoded(const ShapeMap& shapes) {
    for (const auto& [n, s] : shapes) {
      names.push_back(n.c_str());
      ranks.push_back(static_cast<int32_t>(s.size()));
      dims.insert(dims.end(), s.begin(), s.end());
    }
  }
};
struct EncodedOverrides {
  std::vector<const char*> pats, roles;
  explicit EncodedOverrides(const std::vector<RoleOverride>& o) {
    for (const auto& x : o) {
      pats.push_back(x.pattern.c_str());
      roles.push_back(x.role.c_str());
    }
  }
};
}  // namespace detail

class ModelSpec {
 public:
  explicit ModelSpec(const std::string& text) { check(sw_model_spec_parse(text.c_str(), &h_)); }
  ~ModelSpec() { sw_model_spec_free(h_); }
  ModelSpec(const ModelSpec&) = delete;
  ModelSpec& operator=(const ModelSpec&) = delete;
  const sw_model_spec* get() const { return h_; }
  ShapeMap param_shapes() const {  // transformer_param_shapes (model.hpp:17-43)
    char* t = nullptr;
    check(sw_transformer_param_shapes(h_, &t));
    ShapeMap out;
    const std::string s = take(t);
    size_t pos = 0;
    while (pos < s.size()) {
      const size_t nl = s.find('\n', pos), tab = s.find('\t', pos);
      Shape sh;
      std::string dims = s.substr(tab + 1, nl - tab - 1);
      size_t p = 0;
      while (p < dims.size()) {
        size_t c = dims.find(',', p);
        if (c == std::string::npos) c = dims.size();
        sh.push_back(std::stoll(dims.substr(p, c - p)));
        p = c + 1;
      }
      out.emplace_back(s.substr(pos, tab - pos), sh);
      pos = nl + 1;
    }
    return out;
  }
  std::vector<RoleOverride> overrides() const {
    char* t = nullptr;
    check(sw_model_spec_overrides(h_, &t));
    std::vector<RoleOverride> out;
    const std::string s = take(t);
    size_t pos = 0;
    while (pos < s.size()) {
      const size_t nl = s.find('\n', pos), tab = s.find('\t', pos);
      out.push_back({s.substr(pos, tab - pos), s.substr(tab + 1, nl - tab - 1)});
      pos = nl + 1;
    }
    return out;
  }

 private:
  sw_model_spec* h_ = nullptr;
};

inline std::unique_ptr<ModelSpec> parse_model_spec(const std::string& text) {
  return std::make_unique<ModelSpec>(text);
}

class ShardingPlan {
 public:
  explicit ShardingPlan(sw_plan* h) : h_(h) {}
  ~ShardingPlan() { sw_plan_free(h_); }
  ShardingPlan(const ShardingPlan&) = delete;
  ShardingPlan& operator=(const ShardingPlan&) = delete;
  const sw_plan* get() const { return h_; }
  std::string serialize() const {
    char* t = nullptr;
    check(sw_plan_serialize(h_, &t));
    return take(t);
  }
  std::string warnings() const {
    char* t = nullptr;
    check(sw_plan_warnings(h_, &t));
    return take(t);
  }
  std::vector<std::pair<std::string, std::string>> entries() const {
    size_t n = 0;
    int shards = 0;
    check(sw_plan_size(h_, &n, &shards));
    std::vector<std::pair<std::string, std::string>> out;
    for (size_t i = 0; i < n; ++i) {
      const char* name = nullptr;
      int kind = 0;
      int64_t dim = -1;
      check(sw_plan_entry(h_, i, &name, &kind, &dim));
      out.emplace_back(name, kind ? "split:" + std::to_string(dim) : "replicated");
    }
    return out;
  }

 private:
  sw_plan* h_ = nullptr;
};

// derive_plan(params, n_shards, overrides) (plan.hpp:40-47)
inline std::unique_ptr<ShardingPlan> derive_plan(const ShapeMap& shapes, int n_shards,
                                                 const std::vector<RoleOverride>& overrides = {}) {
  detail::Encoded e(shapes);
  detail::EncodedOverrides o(overrides);
  sw_plan* h = nullptr;
  check(sw_plan_derive(e.names.data(), e.ranks.data(), e.dims.data(), shapes.size(), o.pats.data(),
                       o.roles.data(), overrides.size(), n_shards, &h));
  return std::make_unique<ShardingPlan>(h);
}

inline std::unique_ptr<ShardingPlan> parse_plan(const std::string& text, int n_shards) {
  sw_plan* h = nullptr;
  check(sw_plan_parse(text.c_str(), n_shards, &h));
  return std::make_unique<ShardingPlan>(h);
}

inline std::vector<std::string> validate_plan(const ShardingPlan& plan, const ShapeMap& shapes) {
  detail::Encoded e(shapes);
  char* t = nullptr;
  check(sw_plan_validate(plan.get(), e.names.data(), e.ranks.data(), e.dims.data(), shapes.size(), &t));
  const std::string s = take(t);
  std::vector<std::string> out;
  size_t pos = 0;
  while (!s.empty() && pos <= s.size()) {
    const size_t nl = s.find('\n', pos);
    out.push_back(s.substr(pos, nl == std::string::npos ? std::string::npos : nl - pos));
    if (nl == std::string::npos) break;
    pos = nl + 1;
  }
  return out;
}

// build_mesh(dp, mp, n_hosts) (mesh.hpp:47-52). world == 1 emulates the whole mesh on one GPU.
class Mesh {
 public:
  Mesh(int dp, int mp, int n_hosts = 1, int rank = 0, int world = 1, const uint8_t* nccl_id = nullptr,
       int cuda_device = 0) {
    check(sw_mesh_create(dp, mp, n_hosts, rank, world, nccl_id, cuda_device, &h_));
  }
  ~Mesh() { sw_mesh_free(h_); }
  Mesh(const Mesh&) = delete;
  Mesh& operator=(const Mesh&) = delete;
  sw_mesh* get() { return h_; }
  std::string comm_report_csv() const {  // CommReport::to_csv (mesh.cpp:128-138)
    char* t = nullptr;
    check(sw_mesh_comm_report(h_, &t));
    return take(t);
  }

 private:
  sw_mesh* h_ = nullptr;
};

struct AdamWConfig {  // train_state.hpp:172-178
  double lr = 1e-3, beta1 = 0.9, beta2 = 0.999, eps = 1e-8, weight_decay = 0.0;
  sw_adamw_cfg c() const { return {lr, beta1, beta2, eps, weight_decay}; }
};

// transformer_loss program on the mesh + its sharded TrainState in HBM.
class Model {
 public:
  /// inference = true: the Predictor-only model (sw_model_create_inference): bf16 weight shards
  /// and the K/V cache, no gradients or optimizer state.
  Model(const ModelSpec& spec, const ShardingPlan& plan, Mesh& mesh, int batch, int seq_len, bool inference = false) {
    check(inference ? sw_model_create_inference(spec.get(), plan.get(), mesh.get(), batch, seq_len, &h_)
                    : sw_model_create(spec.get(), plan.get(), mesh.get(), batch, seq_len, &h_));
    batch_ = batch;
  }
  ~Model() { sw_model_free(h_); }
  Model(const Model&) = delete;
  Model& operator=(const Model&) = delete;

  void init_params(uint64_t seed, const std::string& stream = "model-init") {
    check(sw_model_init_params(h_, seed, stream.c_str()));
  }
  void set_param(const std::string& name, const std::vector<float>& full) {
    check(sw_model_set_param(h_, name.c_str(), full.data(), static_cast<int64_t>(full.size())));
  }
  std::vector<float> param(const std::string& name, int64_t numel) { return get(name, 0, numel); }
  std::vector<float> grad(const std::string& name, int64_t numel) { return get(name, 1, numel); }
  // collate_fn output (tokens / targets as ids, weights) for the global batch (dp * batch rows)
  void stage_batch(const std::vector<int32_t>& tokens, const std::vector<int32_t>& targets,
                   const std::vector<float>* weights = nullptr) {
    check(sw_model_stage_batch(h_, tokens.data(), targets.data(), weights ? weights->data() : nullptr));
  }
  void forward_backward(bool accumulate = false) { check(sw_model_forward_backward(h_, accumulate)); }
  void scale_grads(double f) { check(sw_model_scale_grads(h_, f)); }
  void dp_sync() { check(sw_model_dp_sync(h_)); }
  void adamw_step(const AdamWConfig& cfg, bool check_finite = true) {
    const sw_adamw_cfg c = cfg.c();
    check(sw_model_adamw_step(h_, &c, check_finite));
  }
  void train_step(const AdamWConfig& cfg) {
    const sw_adamw_cfg c = cfg.c();
    check(sw_model_train_step(h_, &c));
  }
  double loss() {
    double x = 0;
    check(sw_model_last_loss(h_, &x));
    return x;
  }
  /// save_checkpoint(path, state, mesh, rngs) (checkpoint.hpp:193-220).
  void save_checkpoint(const std::string& path, const std::vector<RngState>& rngs = {}) {
    std::vector<const char*> names;
    std::vector<uint64_t> seeds, ids, ctrs;
    for (const RngState& r : rngs) {
      names.push_back(r.name.c_str());
      seeds.push_back(r.seed);
      ids.push_back(r.stream_id);
      ctrs.push_back(r.counter);
    }
    check(sw_model_save_checkpoint(h_, path.c_str(), static_cast<uint32_t>(rngs.size()), names.data(),
                                   seeds.data(), ids.data(), ctrs.data()));
  }
  /// load_checkpoint(path, plan, mesh) onto this model (checkpoint.hpp:233-298); returns the
  /// stored RNG streams.
  std::vector<RngState> load_checkpoint(const std::string& path) {
    uint32_t n = 0;
    check(sw_model_load_checkpoint(h_, path.c_str(), &n));
    std::vector<RngState> out(n);
    for (uint32_t i = 0; i < n; ++i) {
      char buf[4096];
      check(sw_model_checkpoint_rng(h_, i, buf, sizeof(buf), &out[i].seed, &out[i].stream_id, &out[i].counter));
      out[i].name = buf;
    }
    return out;
  }
  /// The Predictor's greedy next-token loop (cli.cpp:425-447): prompts [batch * P] -> [batch * n_new].
  std::vector<int32_t> generate(const std::vector<int32_t>& prompts, int P, int n_new) {
    if (P < 1 || n_new < 1 || prompts.size() != static_cast<size_t>(batch_) * static_cast<size_t>(P)) {
      throw std::invalid_argument("generate: prompts must hold batch * P tokens, P and n_new positive");
    }
    std::vector<int32_t> out(static_cast<size_t>(batch_) * static_cast<size_t>(n_new));
    check(sw_model_generate(h_, prompts.data(), P, n_new, out.data()));
    return out;
  }
  uint64_t step() {
    uint64_t st = 0, sd = 0;
    check(sw_model_state_info(h_, &st, &sd));
    return st;
  }

 private:
  std::vector<float> get(const std::string& name, int which, int64_t numel) {
    std::vector<float> out(static_cast<size_t>(numel));
    check(sw_model_get_tensor(h_, name.c_str(), which, out.data(), numel));
    return out;
  }
  sw_model* h_ = nullptr;
  int batch_ = 0;
};

}  // namespace b200
}  // namespace shardweave
