// C ABI of the host rule engine (include/shardweave_b200.h, "Rule engine" section).
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "rules.h"
#include "status.h"

struct sw_model_spec {
  sw::ModelSpec spec;
};
struct sw_plan {
  sw::Plan plan;
};

namespace {

char* dup_string(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  if (p == nullptr) sw::fail(SW_ERR_INTERNAL, "out of host memory");
  std::memcpy(p, s.data(), s.size());
  p[s.size()] = '\0';
  return p;
}

std::string join_lines(const std::vector<std::string>& v) {
  std::string s;
  for (size_t i = 0; i < v.size(); ++i) {
    if (i) s += '\n';
    s += v[i];
  }
  return s;
}

std::vector<sw::NamedShape> read_shapes(const char* const* names, const int32_t* ranks,
                                        const int64_t* dims, size_t n) {
  std::vector<sw::NamedShape> out(n);
  size_t k = 0;
  for (size_t i = 0; i < n; ++i) {
    if (names == nullptr || names[i] == nullptr) sw::fail(SW_ERR_CONFIG, "null parameter name");
    out[i].name = names[i];
    if (ranks[i] < 0) sw::fail(SW_ERR_SHAPE, "negative rank for '" + out[i].name + "'");
    out[i].dims.assign(dims + k, dims + k + ranks[i]);
    k += static_cast<size_t>(ranks[i]);
  }
  return out;
}

std::vector<sw::RoleOverride> read_overrides(const char* const* patterns, const char* const* roles,
                                             size_t n) {
  std::vector<sw::RoleOverride> out;
  for (size_t i = 0; i < n; ++i) out.push_back({patterns[i], sw::parse_role(roles[i])});
  return out;
}

void require(const void* p, const char* what) {
  if (p == nullptr) sw::fail(SW_ERR_CONFIG, std::string(what) + " is NULL");
}

}  // namespace

extern "C" {

sw_status sw_model_spec_parse(const char* text, sw_model_spec** out) {
  return sw::guarded([&] {
    require(text, "text");
    require(out, "out");
    *out = new sw_model_spec{sw::parse_model_spec(text)};
  });
}

sw_status sw_model_spec_dims(const sw_model_spec* spec, int64_t out[7]) {
  return sw::guarded([&] {
    require(spec, "spec");
    const sw::ModelSpec& s = spec->spec;
    const int64_t v[7] = {s.vocab_size, s.n_layers, s.d_model, s.n_heads,
                          s.d_ff,       s.max_seq_len, s.tie_embeddings ? 1 : 0};
    std::memcpy(out, v, sizeof(v));
  });
}

sw_status sw_model_spec_variant(const sw_model_spec* spec, int* swiglu, int* rmsnorm) {
  return sw::guarded([&] {
    require(spec, "spec");
    if (swiglu) *swiglu = spec->spec.swiglu ? 1 : 0;
    if (rmsnorm) *rmsnorm = spec->spec.rmsnorm ? 1 : 0;
  });
}

sw_status sw_model_spec_t5(const sw_model_spec* spec, int64_t out[5]) {
  return sw::guarded([&] {
    require(spec, "spec");
    const sw::ModelSpec& s = spec->spec;
    const int64_t v[5] = {s.t5 ? 1 : 0, s.n_dec_layers, s.d_kv, s.rel_buckets, s.rel_max_distance};
    std::memcpy(out, v, sizeof(v));
  });
}

sw_status sw_t5_rel_buckets(int64_t tq, int64_t tk, int bidirectional, int num_buckets, int max_distance,
                            int32_t* out) {
  return sw::guarded([&] {
    require(out, "out");
    for (int64_t i = 0; i < tq; ++i)
      for (int64_t j = 0; j < tk; ++j) out[i * tk + j] = sw::t5_rel_bucket(j - i, bidirectional != 0, num_buckets, max_distance);
  });
}

sw_status sw_model_spec_overrides(const sw_model_spec* spec, char** text_out) {
  return sw::guarded([&] {
    require(spec, "spec");
    std::string s;
    for (const auto& o : spec->spec.overrides) s += o.pattern + "\t" + sw::role_name(o.role) + "\n";
    *text_out = dup_string(s);
  });
}

void sw_model_spec_free(sw_model_spec* spec) { delete spec; }

sw_status sw_transformer_param_shapes(const sw_model_spec* spec, char** text_out) {
  return sw::guarded([&] {
    require(spec, "spec");
    std::string s;
    for (const auto& p : sw::transformer_param_shapes(spec->spec)) {
      s += p.name + "\t";
      for (size_t i = 0; i < p.dims.size(); ++i) s += (i ? "," : "") + std::to_string(p.dims[i]);
      s += "\n";
    }
    *text_out = dup_string(s);
  });
}

sw_status sw_infer_roles(const char* const* names, const int32_t* ranks, const int64_t* dims,
                         size_t n, const char* const* override_patterns,
                         const char* const* override_roles, size_t n_overrides, char** roles_out,
                         char** warnings_out) {
  return sw::guarded([&] {
    const auto shapes = read_shapes(names, ranks, dims, n);
    const auto res = sw::infer_roles(shapes, read_overrides(override_patterns, override_roles,
                                                             n_overrides));
    std::string s;
    for (const auto& r : res.roles) {
      s += r.name + "\t" + sw::role_name(r.role) + "\t" + std::to_string(r.seq) + "\n";
    }
    *roles_out = dup_string(s);
    if (warnings_out != nullptr) *warnings_out = dup_string(join_lines(res.warnings));
  });
}

sw_status sw_plan_derive(const char* const* names, const int32_t* ranks, const int64_t* dims,
                         size_t n, const char* const* override_patterns,
                         const char* const* override_roles, size_t n_overrides, int n_shards,
                         sw_plan** out) {
  return sw::guarded([&] {
    require(out, "out");
    const auto shapes = read_shapes(names, ranks, dims, n);
    const auto roles = sw::infer_roles(shapes, read_overrides(override_patterns, override_roles,
                                                              n_overrides));
    sw::Plan plan = sw::derive_plan(roles.roles, shapes, n_shards);
    plan.warnings.insert(plan.warnings.begin(), roles.warnings.begin(), roles.warnings.end());
    *out = new sw_plan{std::move(plan)};
  });
}

sw_status sw_plan_parse(const char* text, int n_shards, sw_plan** out) {
  return sw::guarded([&] {
    require(text, "text");
    require(out, "out");
    *out = new sw_plan{sw::parse_plan(text, n_shards)};
  });
}

sw_status sw_plan_serialize(const sw_plan* plan, char** text_out) {
  return sw::guarded([&] {
    require(plan, "plan");
    *text_out = dup_string(sw::serialize_plan(plan->plan));
  });
}

sw_status sw_plan_validate(const sw_plan* plan, const char* const* names, const int32_t* ranks,
                           const int64_t* dims, size_t n, char** violations_out) {
  return sw::guarded([&] {
    require(plan, "plan");
    *violations_out =
        dup_string(join_lines(sw::validate_plan(plan->plan, read_shapes(names, ranks, dims, n))));
  });
}

sw_status sw_plan_warnings(const sw_plan* plan, char** text_out) {
  return sw::guarded([&] {
    require(plan, "plan");
    *text_out = dup_string(join_lines(plan->plan.warnings));
  });
}

sw_status sw_plan_size(const sw_plan* plan, size_t* n_entries, int* n_shards) {
  return sw::guarded([&] {
    require(plan, "plan");
    if (n_entries) *n_entries = plan->plan.entries.size();
    if (n_shards) *n_shards = plan->plan.n_shards;
  });
}

sw_status sw_plan_entry(const sw_plan* plan, size_t i, const char** name, int* kind, int64_t* dim) {
  return sw::guarded([&] {
    require(plan, "plan");
    if (i >= plan->plan.entries.size()) sw::fail(SW_ERR_CONFIG, "sw_plan_entry: index out of range");
    const auto& e = plan->plan.entries[i];
    if (name) *name = e.first.c_str();
    if (kind) *kind = e.second.kind;
    if (dim) *dim = e.second.dim;
  });
}

void sw_plan_free(sw_plan* plan) { delete plan; }

sw_status sw_shard_range(const int64_t* global_dims, int32_t rank_of_tensor, int kind, int64_t dim,
                         int n_shards, int shard_rank, int64_t* local_dims_out, int64_t* begin_out,
                         int64_t* end_out) {
  // local_shape / shard (sharded_tensor.hpp:20-36, :52-74): even contiguous chunks.
  return sw::guarded([&] {
    if (n_shards < 1) sw::fail(SW_ERR_PARTITION, "shard: need at least one shard, got " + std::to_string(n_shards));
    if (shard_rank < 0 || shard_rank >= n_shards) sw::fail(SW_ERR_PARTITION, "shard: rank out of range");
    sw::Dims g(global_dims, global_dims + rank_of_tensor);
    for (int32_t i = 0; i < rank_of_tensor; ++i) local_dims_out[i] = g[i];
    if (kind == 0) {
      *begin_out = 0;
      *end_out = rank_of_tensor > 0 ? g[0] : 1;
      return;
    }
    if (dim < 0 || dim >= rank_of_tensor) {
      sw::fail(SW_ERR_PARTITION, "local_shape: split dim " + std::to_string(dim) +
                                     " out of range for " + sw::dims_str(g));
    }
    if (g[dim] % n_shards != 0) {
      sw::fail(SW_ERR_PARTITION, "local_shape: dim " + std::to_string(dim) + " of " +
                                     sw::dims_str(g) + " is not divisible by " +
                                     std::to_string(n_shards) + " shards");
    }
    const int64_t chunk = g[dim] / n_shards;
    local_dims_out[dim] = chunk;
    *begin_out = chunk * shard_rank;
    *end_out = chunk * (shard_rank + 1);
  });
}

sw_status sw_expected_state_elements(const sw_plan* plan, const char* const* names,
                                     const int32_t* ranks, const int64_t* dims, size_t n,
                                     int mp_size, int64_t* out) {
  return sw::guarded([&] {
    require(plan, "plan");
    *out = sw::expected_state_elements(plan->plan, read_shapes(names, ranks, dims, n), mp_size);
  });
}

}  // extern "C"
