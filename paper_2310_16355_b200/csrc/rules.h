// Host rule engine: parameter-role inference, the two sharding rules, plan validation and the
// plan text format, plus the model-spec parser and the transformer parameter tree.
//
// Contract: for every input, the entries, their order, warnings and error messages are
// identical to the reference (roles.cpp, plan.cpp, model_spec.cpp, model.hpp:17-43). The
// golden cases in tests/golden/rules.json are produced by the reference itself.
#pragma once

#include <cstdint>
#include <string>
#include <utility>
#include <vector>

namespace sw {

using Dims = std::vector<int64_t>;

struct NamedShape {
  std::string name;
  Dims dims;
};

enum class Role : uint8_t { kQKV, kOut, kFC, kEmbedding, kNorm, kBias, kOther };

const char* role_name(Role r);
Role parse_role(const std::string& text);  // throws Error(SW_ERR_CONFIG)

struct RoleOverride {
  std::string pattern;
  Role role;
};

struct RoleOf {
  std::string name;
  Role role = Role::kOther;
  int seq = -1;  // position among fully-connected kernels of the same block
};

struct RoleResult {
  std::vector<RoleOf> roles;
  std::vector<std::string> warnings;
};

RoleResult infer_roles(const std::vector<NamedShape>& shapes,
                       const std::vector<RoleOverride>& overrides);

struct Layout {
  enum Kind : uint8_t { kReplicated = 0, kSplit = 1 };
  Kind kind = kReplicated;
  int64_t dim = -1;
  bool operator==(const Layout& o) const {
    return kind == o.kind && (kind != kSplit || dim == o.dim);
  }
};

struct Plan {
  int n_shards = 1;
  std::vector<std::pair<std::string, Layout>> entries;
  std::vector<std::string> warnings;
  const Layout* find(const std::string& name) const;
  const Layout& at(const std::string& name) const;  // throws Error(SW_ERR_CONFIG)
};

Plan derive_plan(const std::vector<RoleOf>& roles, const std::vector<NamedShape>& shapes,
                 int n_shards);
std::vector<std::string> validate_plan(const Plan& plan, const std::vector<NamedShape>& shapes);
std::string serialize_plan(const Plan& plan);
Plan parse_plan(const std::string& text, int n_shards);
int64_t expected_state_elements(const Plan& plan, const std::vector<NamedShape>& shapes,
                                int mp_size);

std::string dims_str(const Dims& d);  // "[a,b]"

struct ModelSpec {
  int64_t vocab_size = 0;
  int n_layers = 0;
  int64_t d_model = 0;
  int n_heads = 0;
  int64_t d_ff = 0;
  int64_t max_seq_len = 0;
  bool tie_embeddings = false;
  // Extension (not in the reference's spec language): `mlp = swiglu` gives the
  // LLaMA MLP down(silu(gate x) * up x) with gate named block_i/mlp/fc1/gate/kernel (gate:0,
  // up:0, down:1 under the reference rules, no MLP biases); `norm = rmsnorm` makes every
  // LayerNorm an RMSNorm (scale only).
  bool swiglu = false;
  bool rmsnorm = false;
  // Extension (BASELINE cfg4): `arch = t5` selects a T5 encoder-decoder
  // (T5 v1.0 layer: RMSNorm, unscaled attention with bucketed relative-position bias shared by a
  // stack's layers, ReLU MLP, no biases, separate lm_head) named with the reference's scopes
  // (attn / cross_attn / mlp), so the reference rules plan it: n_layers encoder and n_dec_layers
  // decoder blocks, head dim d_kv (inner width n_heads * d_kv), rel_buckets / rel_max_distance.
  bool t5 = false;
  int n_dec_layers = 0;
  int64_t d_kv = 0;
  int rel_buckets = 32;
  int rel_max_distance = 128;
  std::vector<RoleOverride> overrides;
};

// T5 relative-position bucket (the HF T5 `_relative_position_bucket` rule): rp = key - query;
// bidirectional (encoder) halves the buckets between rp < 0 and rp > 0; unidirectional
// (decoder) buckets only rp <= 0. Small |rp| map exactly, larger ones log-spaced up to
// max_distance. Evaluated in double with a 1e-9 guard before truncation so host and oracle
// agree at the log-spaced boundaries.
int t5_rel_bucket(int64_t rp, bool bidirectional, int num_buckets, int max_distance);

ModelSpec parse_model_spec(const std::string& text);
std::vector<NamedShape> transformer_param_shapes(const ModelSpec& spec);

}  // namespace sw
