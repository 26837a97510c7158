// Host rule engine (see rules.h). Behaviour follows, case by case:
//   role heuristics          roles.cpp:36-102      override resolution   roles.cpp:157-166
//   FC numbering per block   roles.cpp:107-116,181-187
//   the two sharding rules   plan.cpp:13-20        derive_plan           plan.cpp:39-91
//   validate_plan            plan.cpp:93-179       text format           plan.cpp:181-239
//   model spec parser        model_spec.cpp:44-119 parameter tree        model.hpp:17-43
#include "rules.h"

#include <algorithm>
#include <cmath>
#include <array>
#include <cctype>
#include <map>
#include <sstream>
#include <string_view>
#include <unordered_map>

#include "status.h"

namespace sw {

namespace {

std::string ascii_lower(std::string s) {
  for (char& c : s) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
  return s;
}

// '/'-separated segments; empty segments are kept ("a//b" has three).
std::vector<std::string> segments_of(const std::string& path) {
  std::vector<std::string> out(1);
  for (char c : path) {
    if (c == '/') {
      out.emplace_back();
    } else {
      out.back().push_back(c);
    }
  }
  return out;
}

bool has_prefix(std::string_view s, std::string_view p) { return s.substr(0, p.size()) == p; }

template <size_t N>
bool one_of(std::string_view s, const std::array<std::string_view, N>& set) {
  return std::find(set.begin(), set.end(), s) != set.end();
}

constexpr std::array<std::string_view, 7> kAttentionScope = {
    "attn", "attention", "self_attn", "self_attention", "mha", "cross_attn", "cross_attention"};
constexpr std::array<std::string_view, 13> kProjectionIn = {
    "q", "k", "v", "query", "key", "value", "qkv", "wq", "wk", "wv", "q_proj", "k_proj", "v_proj"};
constexpr std::array<std::string_view, 6> kProjectionOut = {"o",      "out",    "out_proj",
                                                           "output", "o_proj", "wo"};
constexpr std::array<std::string_view, 4> kNormLeaf = {"scale", "gamma", "weight", "g"};

bool fc_segment(std::string_view s) {
  return s == "mlp" || s == "ffn" || has_prefix(s, "fc") || has_prefix(s, "dense");
}

// Role from the name alone. `matched` is false when a rank>=2 tensor fell through to kOther.
Role classify(const std::string& name, size_t rank, bool& matched) {
  matched = true;
  const std::vector<std::string> seg = segments_of(ascii_lower(name));
  const std::string& leaf = seg.back();
  if (rank < 2) {
    if (leaf.find("bias") != std::string::npos || leaf == "beta" || leaf == "b") return Role::kBias;
    if (one_of(leaf, kNormLeaf)) return Role::kNorm;
    for (const auto& s : seg) {
      if (has_prefix(s, "ln") || s.find("norm") != std::string::npos) return Role::kNorm;
    }
    return Role::kBias;
  }
  for (const auto& s : seg) {
    if (s.find("embed") != std::string::npos) return Role::kEmbedding;
  }
  const bool attention = std::any_of(seg.begin(), seg.end(),
                                     [](const std::string& s) { return one_of(s, kAttentionScope); });
  if (attention) {
    for (auto it = seg.rbegin(); it != seg.rend(); ++it) {  // innermost name decides
      if (one_of(*it, kProjectionIn)) return Role::kQKV;
      if (one_of(*it, kProjectionOut)) return Role::kOut;
    }
  }
  if (std::any_of(seg.begin(), seg.end(), [](const std::string& s) { return fc_segment(s); })) {
    return Role::kFC;
  }
  matched = false;
  return Role::kOther;
}

// Block grouping key for FC numbering: the path without its last two segments.
std::string fc_block(const std::string& path) {
  const std::vector<std::string> seg = segments_of(path);
  if (seg.size() <= 2) return "";
  std::string key = seg[0];
  for (size_t i = 1; i + 2 < seg.size(); ++i) key += "/" + seg[i];
  return key;
}

int64_t rule_dim(const RoleOf& r) {
  if (r.role == Role::kQKV) return 0;
  if (r.role == Role::kOut) return 1;
  if (r.role == Role::kFC) return (r.seq % 2 == 0) ? 0 : 1;
  return -1;
}

std::string quote(const std::string& s) { return "'" + s + "'"; }

std::string trim_ws(const std::string& s) {
  const size_t b = s.find_first_not_of(" \t\r");
  if (b == std::string::npos) return "";
  const size_t e = s.find_last_not_of(" \t\r");
  return s.substr(b, e - b + 1);
}

// std::stoll with the "whole string consumed" requirement; returns false on any failure.
bool full_stoll(const std::string& text, int64_t& out) {
  size_t used = 0;
  try {
    out = std::stoll(text, &used);
  } catch (const std::exception&) {
    used = 0;
  }
  return used != 0 && used == text.size();
}

}  // namespace

std::string dims_str(const Dims& d) {
  std::string s = "[";
  for (size_t i = 0; i < d.size(); ++i) {
    if (i) s += ",";
    s += std::to_string(d[i]);
  }
  return s + "]";
}

const char* role_name(Role r) {
  switch (r) {
    case Role::kQKV: return "attention_qkv";
    case Role::kOut: return "attention_out";
    case Role::kFC: return "fully_connected";
    case Role::kEmbedding: return "embedding";
    case Role::kNorm: return "norm";
    case Role::kBias: return "bias";
    case Role::kOther: return "other";
  }
  return "other";
}

Role parse_role(const std::string& text) {
  static const std::map<std::string, Role> kByName = {
      {"attention_qkv", Role::kQKV}, {"attention_out", Role::kOut},
      {"fully_connected", Role::kFC}, {"embedding", Role::kEmbedding},
      {"norm", Role::kNorm},          {"bias", Role::kBias},
      {"other", Role::kOther}};
  const auto it = kByName.find(ascii_lower(text));
  if (it == kByName.end()) fail(SW_ERR_CONFIG, "parse_role: unknown role " + quote(text));
  return it->second;
}

RoleResult infer_roles(const std::vector<NamedShape>& shapes,
                       const std::vector<RoleOverride>& overrides) {
  RoleResult res;
  res.roles.reserve(shapes.size());
  for (const NamedShape& p : shapes) {
    const std::string path = ascii_lower(p.name);
    const RoleOverride* chosen = nullptr;
    for (const RoleOverride& o : overrides) {
      if (path.find(ascii_lower(o.pattern)) == std::string::npos) continue;
      if (chosen == nullptr || o.pattern.size() > chosen->pattern.size()) {
        chosen = &o;
      } else if (o.pattern.size() == chosen->pattern.size() && o.role != chosen->role) {
        fail(SW_ERR_CONFIG, "infer_roles: overrides " + quote(chosen->pattern) + " and " +
                                quote(o.pattern) + " conflict for parameter " + quote(p.name));
      }
    }
    RoleOf r;
    r.name = p.name;
    if (chosen != nullptr) {
      r.role = chosen->role;
    } else {
      bool matched = true;
      r.role = classify(p.name, p.dims.size(), matched);
      if (!matched && p.dims.size() >= 2) {
        res.warnings.push_back("parameter " + quote(p.name) + " matched no role; treating as other");
      }
    }
    res.roles.push_back(std::move(r));
  }
  std::unordered_map<std::string, int> counter;
  for (RoleOf& r : res.roles) {
    if (r.role == Role::kFC) r.seq = counter[fc_block(ascii_lower(r.name))]++;
  }
  return res;
}

const Layout* Plan::find(const std::string& name) const {
  for (const auto& e : entries) {
    if (e.first == name) return &e.second;
  }
  return nullptr;
}

const Layout& Plan::at(const std::string& name) const {
  const Layout* l = find(name);
  if (l == nullptr) fail(SW_ERR_CONFIG, "ShardingPlan: no entry for parameter " + quote(name));
  return *l;
}

Plan derive_plan(const std::vector<RoleOf>& roles, const std::vector<NamedShape>& shapes,
                 int n_shards) {
  if (n_shards < 1) {
    fail(SW_ERR_CONFIG, "derive_plan: n_shards must be positive, got " + std::to_string(n_shards));
  }
  std::unordered_map<std::string, const RoleOf*> by_name;
  for (const RoleOf& r : roles) by_name[r.name] = &r;

  if (n_shards > 1) {
    bool splittable = false;
    for (const NamedShape& p : shapes) {
      const auto it = by_name.find(p.name);
      if (it == by_name.end()) continue;
      const int64_t d = rule_dim(*it->second);
      if (d >= 0 && static_cast<size_t>(d) < p.dims.size() && p.dims[d] >= n_shards) {
        splittable = true;
        break;
      }
    }
    if (!splittable) {
      fail(SW_ERR_CONFIG, "derive_plan: model cannot be split this many ways (n_shards=" +
                              std::to_string(n_shards) + ")");
    }
  }

  Plan plan;
  plan.n_shards = n_shards;
  for (const NamedShape& p : shapes) {
    const auto it = by_name.find(p.name);
    if (it == by_name.end()) {
      fail(SW_ERR_CONFIG, "derive_plan: no role assigned for parameter " + quote(p.name));
    }
    const int64_t d = rule_dim(*it->second);
    Layout l;
    if (d >= 0) {
      if (static_cast<size_t>(d) >= p.dims.size()) {
        plan.warnings.push_back("parameter " + quote(p.name) + ": split dim " + std::to_string(d) +
                                " out of range for " + dims_str(p.dims) + "; replicated instead");
      } else if (p.dims[d] % n_shards != 0) {
        plan.warnings.push_back("parameter " + quote(p.name) + ": dim " + std::to_string(d) +
                                " size " + std::to_string(p.dims[d]) + " not divisible by " +
                                std::to_string(n_shards) + " shards; replicated instead");
      } else {
        l.kind = Layout::kSplit;
        l.dim = d;
      }
    }
    plan.entries.emplace_back(p.name, l);
  }
  return plan;
}

std::vector<std::string> validate_plan(const Plan& plan, const std::vector<NamedShape>& shapes) {
  std::vector<std::string> out;
  std::unordered_map<std::string, const Dims*> dims_of;
  for (const NamedShape& p : shapes) dims_of[p.name] = &p.dims;
  const std::string n = std::to_string(plan.n_shards);

  // 1. structural checks of every split entry
  for (const auto& [name, l] : plan.entries) {
    const auto it = dims_of.find(name);
    if (it == dims_of.end()) {
      out.push_back("parameter " + quote(name) + " not present in the shape map");
      continue;
    }
    if (l.kind != Layout::kSplit) continue;
    const Dims& d = *it->second;
    if (l.dim < 0 || static_cast<size_t>(l.dim) >= d.size()) {
      out.push_back("parameter " + quote(name) + ": dim out of range (split:" +
                    std::to_string(l.dim) + " on " + dims_str(d) + ")");
      continue;
    }
    if (d[l.dim] % plan.n_shards != 0) {
      out.push_back("parameter " + quote(name) + ": dim " + std::to_string(l.dim) + " size " +
                    std::to_string(d[l.dim]) + " not divisible by " + n + " shards");
    }
  }

  // 2. rule invariants against default-heuristic roles
  const RoleResult roles = infer_roles(shapes, {});
  std::unordered_map<std::string, const RoleOf*> role_of;
  for (const RoleOf& r : roles.roles) role_of[r.name] = &r;
  std::unordered_map<std::string, std::pair<int, Layout>> prev_fc;
  for (const auto& [name, l] : plan.entries) {
    const auto rit = role_of.find(name);
    if (rit == role_of.end()) continue;
    const auto dit = dims_of.find(name);
    if (dit == dims_of.end()) continue;
    const RoleOf& r = *rit->second;
    const Dims& d = *dit->second;
    const bool split = l.kind == Layout::kSplit;
    if (r.role == Role::kQKV && split && l.dim != 0) {
      out.push_back("parameter " + quote(name) + ": attention qkv split along dim " +
                    std::to_string(l.dim) + ", expected dim 0");
    }
    if (r.role == Role::kOut && split && l.dim != 1) {
      out.push_back("parameter " + quote(name) + ": attention output split along dim " +
                    std::to_string(l.dim) + ", expected dim 1");
    }
    if (plan.n_shards > 1 && !split && d.size() >= 2 &&
        (r.role == Role::kQKV || r.role == Role::kOut)) {
      const int64_t want = rule_dim(r);
      if (d[want] % plan.n_shards == 0) {
        out.push_back("parameter " + quote(name) + ": replicated " + role_name(r.role) +
                      " although dim " + std::to_string(want) + " is divisible by " + n +
                      " shards");
      }
    }
    if (r.role == Role::kFC && split) {
      // block key: the name cut at its second-to-last '/'
      std::string key;
      int cuts = 0;
      for (size_t i = name.size(); i-- > 0;) {
        if (name[i] == '/' && ++cuts == 2) {
          key = name.substr(0, i);
          break;
        }
      }
      const auto pit = prev_fc.find(key);
      if (pit != prev_fc.end() && pit->second.first == r.seq - 1 && pit->second.second == l) {
        out.push_back("parameter " + quote(name) + ": consecutive FC kernels share split dim " +
                      std::to_string(l.dim));
      }
      prev_fc[key] = {r.seq, l};
    }
  }
  return out;
}

std::string serialize_plan(const Plan& plan) {
  std::ostringstream os;
  for (const auto& [name, l] : plan.entries) {
    os << name << '\t';
    if (l.kind == Layout::kSplit) {
      os << "split:" << l.dim;
    } else {
      os << "replicated";
    }
    os << '\n';
  }
  return os.str();
}

Plan parse_plan(const std::string& text, int n_shards) {
  if (n_shards < 1) {
    fail(SW_ERR_CONFIG, "parse_plan: n_shards must be positive, got " + std::to_string(n_shards));
  }
  Plan plan;
  plan.n_shards = n_shards;
  std::istringstream in(text);
  std::string line;
  for (int no = 1; std::getline(in, line); ++no) {
    if (line.empty()) continue;
    const std::string where = "parse_plan: line " + std::to_string(no) + ": ";
    const size_t tab = line.find('\t');
    if (tab == std::string::npos || tab == 0) {
      fail(SW_ERR_CONFIG, where + "expected `name<TAB>replicated|split:<dim>`");
    }
    const std::string layout = line.substr(tab + 1);
    Layout l;
    if (layout == "replicated") {
      l.kind = Layout::kReplicated;
    } else if (has_prefix(layout, "split:")) {
      const std::string dim_text = layout.substr(6);
      int64_t dim = -1;
      if (!full_stoll(dim_text, dim) || dim < 0) {
        fail(SW_ERR_CONFIG, where + "bad split dim " + quote(dim_text));
      }
      l.kind = Layout::kSplit;
      l.dim = dim;
    } else {
      fail(SW_ERR_CONFIG, where + "unknown layout " + quote(layout));
    }
    plan.entries.emplace_back(line.substr(0, tab), l);
  }
  return plan;
}

int64_t expected_state_elements(const Plan& plan, const std::vector<NamedShape>& shapes,
                                int mp_size) {
  int64_t total = 0;
  for (const NamedShape& p : shapes) {
    int64_t n = 1;
    for (int64_t d : p.dims) n *= d;
    total += plan.at(p.name).kind == Layout::kSplit ? n / mp_size : n;
  }
  return 3 * total;
}

ModelSpec parse_model_spec(const std::string& text) {
  ModelSpec spec;
  std::vector<std::string> seen;
  std::istringstream in(text);
  std::string raw;
  for (int no = 1; std::getline(in, raw); ++no) {
    const std::string where = "model spec: line " + std::to_string(no) + ": ";
    const size_t hash = raw.find('#');
    if (hash != std::string::npos) raw.resize(hash);
    const std::string line = trim_ws(raw);
    if (line.empty()) continue;
    const size_t eq = line.find('=');
    const std::string key = eq == std::string::npos ? "" : trim_ws(line.substr(0, eq));
    const std::string value = eq == std::string::npos ? "" : trim_ws(line.substr(eq + 1));
    if (eq == std::string::npos || key.empty() || value.empty()) {
      fail(SW_ERR_CONFIG, where + "expected `key = value`, got " + quote(line));
    }
    if (has_prefix(key, "role ")) {
      const std::string pattern = trim_ws(key.substr(5));
      if (pattern.empty()) fail(SW_ERR_CONFIG, where + "role override needs a pattern");
      spec.overrides.push_back({pattern, parse_role(value)});
      continue;
    }
    if (std::find(seen.begin(), seen.end(), key) != seen.end()) {
      fail(SW_ERR_CONFIG, where + "duplicate key " + quote(key));
    }
    seen.push_back(key);
    auto as_int = [&]() {
      int64_t v = 0;
      if (!full_stoll(value, v)) {
        fail(SW_ERR_CONFIG, where + quote(key) + " needs an integer, got " + quote(value));
      }
      return v;
    };
    if (key == "vocab_size") {
      spec.vocab_size = as_int();
    } else if (key == "n_layers") {
      spec.n_layers = static_cast<int>(as_int());
    } else if (key == "d_model") {
      spec.d_model = as_int();
    } else if (key == "n_heads") {
      spec.n_heads = static_cast<int>(as_int());
    } else if (key == "d_ff") {
      spec.d_ff = as_int();
    } else if (key == "max_seq_len") {
      spec.max_seq_len = as_int();
    } else if (key == "tie_embeddings") {
      if (value == "true" || value == "yes" || value == "1") {
        spec.tie_embeddings = true;
      } else if (value == "false" || value == "no" || value == "0") {
        spec.tie_embeddings = false;
      } else {
        fail(SW_ERR_CONFIG, where + quote(key) + " needs true or false, got " + quote(value));
      }
    } else if (key == "mlp") {  // extension key
      if (value == "gelu") {
        spec.swiglu = false;
      } else if (value == "swiglu") {
        spec.swiglu = true;
      } else {
        fail(SW_ERR_CONFIG, where + quote(key) + " needs gelu or swiglu, got " + quote(value));
      }
    } else if (key == "norm") {  // extension key
      if (value == "layernorm") {
        spec.rmsnorm = false;
      } else if (value == "rmsnorm") {
        spec.rmsnorm = true;
      } else {
        fail(SW_ERR_CONFIG, where + quote(key) + " needs layernorm or rmsnorm, got " + quote(value));
      }
    } else if (key == "arch") {  // extension key (T5 encoder-decoder, BASELINE cfg4)
      if (value == "decoder") {
        spec.t5 = false;
      } else if (value == "t5") {
        spec.t5 = true;
      } else {
        fail(SW_ERR_CONFIG, where + quote(key) + " needs decoder or t5, got " + quote(value));
      }
    } else if (key == "n_dec_layers") {
      spec.n_dec_layers = static_cast<int>(as_int());
    } else if (key == "d_kv") {
      spec.d_kv = as_int();
    } else if (key == "rel_buckets") {
      spec.rel_buckets = static_cast<int>(as_int());
    } else if (key == "rel_max_distance") {
      spec.rel_max_distance = static_cast<int>(as_int());
    } else {
      fail(SW_ERR_CONFIG, where + "unknown key " + quote(key));
    }
  }
  for (const char* k : {"vocab_size", "n_layers", "d_model", "n_heads", "d_ff", "max_seq_len"}) {
    if (std::find(seen.begin(), seen.end(), k) == seen.end()) {
      fail(SW_ERR_CONFIG, std::string("model spec: missing required key '") + k + "'");
    }
  }
  if (spec.vocab_size < 1 || spec.n_layers < 1 || spec.d_model < 1 || spec.n_heads < 1 ||
      spec.d_ff < 1 || spec.max_seq_len < 1) {
    fail(SW_ERR_CONFIG, "model spec: all dimensions must be positive");
  }
  if (spec.d_model % spec.n_heads != 0) {
    fail(SW_ERR_CONFIG, "model spec: d_model " + std::to_string(spec.d_model) +
                            " is not divisible by n_heads " + std::to_string(spec.n_heads));
  }
  const bool t5_keys = std::find(seen.begin(), seen.end(), "n_dec_layers") != seen.end() ||
                       std::find(seen.begin(), seen.end(), "d_kv") != seen.end() ||
                       std::find(seen.begin(), seen.end(), "rel_buckets") != seen.end() ||
                       std::find(seen.begin(), seen.end(), "rel_max_distance") != seen.end();
  if (spec.t5) {
    if (spec.n_dec_layers < 1 || spec.d_kv < 1 || spec.rel_buckets < 4 || spec.rel_buckets % 2 != 0 ||
        spec.rel_max_distance < spec.rel_buckets) {
      fail(SW_ERR_CONFIG, "model spec: arch = t5 needs n_dec_layers >= 1, d_kv >= 1, an even rel_buckets >= 4 "
                          "and rel_max_distance >= rel_buckets");
    }
    if (spec.tie_embeddings || spec.swiglu) {
      fail(SW_ERR_CONFIG, "model spec: arch = t5 has its own lm_head and a ReLU MLP "
                          "(tie_embeddings / mlp = swiglu are not supported)");
    }
    spec.rmsnorm = true;  // T5LayerNorm: scale only, no centring
  } else if (t5_keys) {
    fail(SW_ERR_CONFIG, "model spec: n_dec_layers / d_kv / rel_buckets / rel_max_distance need arch = t5");
  }
  return spec;
}

int t5_rel_bucket(int64_t rp, bool bidirectional, int num_buckets, int max_distance) {
  int ret = 0;
  int64_t n = 0;
  if (bidirectional) {
    num_buckets /= 2;
    if (rp > 0) ret += num_buckets;
    n = rp < 0 ? -rp : rp;
  } else {
    n = rp < 0 ? -rp : 0;
  }
  const int max_exact = num_buckets / 2;
  if (n < max_exact) return ret + static_cast<int>(n);
  const double x = std::log(static_cast<double>(n) / max_exact) / std::log(static_cast<double>(max_distance) / max_exact) *
                   (num_buckets - max_exact);
  int large = max_exact + static_cast<int>(std::floor(x + 1e-9));
  if (large > num_buckets - 1) large = num_buckets - 1;
  return ret + large;
}

static std::vector<NamedShape> t5_param_shapes(const ModelSpec& spec) {
  const int64_t d = spec.d_model, inner = spec.n_heads * spec.d_kv;
  std::vector<NamedShape> out;
  out.push_back({"embed/tok/kernel", {spec.vocab_size, d}});
  auto attn = [&](const std::string& b, const char* scope) {
    for (const char* proj : {"q", "k", "v"}) out.push_back({b + scope + "/" + proj + "/kernel", {inner, d}});
    out.push_back({b + scope + "/o/kernel", {d, inner}});
  };
  auto stack = [&](const std::string& st, int layers, bool decoder) {
    for (int l = 0; l < layers; ++l) {
      const std::string b = st + "/block_" + std::to_string(l) + "/";
      out.push_back({b + "ln1/scale", {d}});
      attn(b, "attn");
      if (l == 0) out.push_back({b + "attn/rel_bias/kernel", {spec.rel_buckets, spec.n_heads}});
      if (decoder) {
        out.push_back({b + "ln_x/scale", {d}});
        attn(b, "cross_attn");
      }
      out.push_back({b + "ln2/scale", {d}});
      out.push_back({b + "mlp/fc1/kernel", {spec.d_ff, d}});
      out.push_back({b + "mlp/fc2/kernel", {d, spec.d_ff}});
    }
    out.push_back({st + "/final_ln/scale", {d}});
  };
  stack("enc", spec.n_layers, false);
  stack("dec", spec.n_dec_layers, true);
  out.push_back({"lm_head/kernel", {spec.vocab_size, d}});
  return out;
}

std::vector<NamedShape> transformer_param_shapes(const ModelSpec& spec) {
  if (spec.t5) return t5_param_shapes(spec);
  // model.hpp:17-43 tree order; the mlp/norm extension keys swap in the SwiGLU / RMSNorm leaves
  const int64_t d = spec.d_model;
  std::vector<NamedShape> out;
  auto norm = [&](const std::string& p) {
    out.push_back({p + "/scale", {d}});
    if (!spec.rmsnorm) out.push_back({p + "/bias", {d}});
  };
  out.push_back({"embed/tok/kernel", {spec.vocab_size, d}});
  out.push_back({"embed/pos/kernel", {spec.max_seq_len, d}});
  for (int l = 0; l < spec.n_layers; ++l) {
    const std::string b = "block_" + std::to_string(l) + "/";
    norm(b + "ln1");
    for (const char* proj : {"q", "k", "v", "o"}) {
      out.push_back({b + "attn/" + proj + "/kernel", {d, d}});
      out.push_back({b + "attn/" + proj + "/bias", {d}});
    }
    norm(b + "ln2");
    if (spec.swiglu) {
      out.push_back({b + "mlp/fc1/gate/kernel", {spec.d_ff, d}});
      out.push_back({b + "mlp/fc1/kernel", {spec.d_ff, d}});
      out.push_back({b + "mlp/fc2/kernel", {d, spec.d_ff}});
    } else {
      out.push_back({b + "mlp/fc1/kernel", {spec.d_ff, d}});
      out.push_back({b + "mlp/fc1/bias", {spec.d_ff}});
      out.push_back({b + "mlp/fc2/kernel", {d, spec.d_ff}});
      out.push_back({b + "mlp/fc2/bias", {d}});
    }
  }
  norm("final_ln");
  if (!spec.tie_embeddings) out.push_back({"lm_head/kernel", {spec.vocab_size, d}});
  return out;
}

}  // namespace sw
