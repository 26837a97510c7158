// ORACLE TEST INFRASTRUCTURE — not product code.
//
// Driver linked against the UNMODIFIED reference sources under /root/reference/proj (built by
// oracle/Makefile into oracle/_ref/, with oracle/eigen_shim standing in for Eigen3). It replaces
// the reference CLI (cli.cpp needs CLI11, which is absent) with direct calls to the same
// functions cmd_plan / cmd_audit_t use (cli.cpp:122-288), and emits golden data for the tests:
//
//   shapes <spec>                                    transformer_param_shapes (model.hpp:17-43)
//   plan <spec> <n_shards>                           infer_roles + derive_plan + validate_plan
//   plan-shapes <shapes.tsv> <n_shards> [ovr.tsv]    same, over an arbitrary name/shape list
//   validate <shapes.tsv> <plan.txt> <n_shards>      parse_plan + validate_plan
//   golden <spec> <f32|f64> <seed> <dp> <mp> <global_batch> <seq> <steps> <lr> <wd> <out>
//                                                    audit-style trajectory dump (cli.cpp:179-240)
//   bench <spec> <mp> <batch> <seq> <steps> <threads>   CPU timing of spmd_forward_backward+AdamW
//   trainer <spec> <seed> <dp> <mp> <pdb> <accum> <epochs> <n_ex> <seq> <lr> <wd> <warmup> <dir>
//                                                    Trainer::fit step losses / lrs / run.log
#include <chrono>
#include <cstdlib>
#include <mutex>
#include <new>
#include <unordered_map>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "shardweave/audit.hpp"
#include "shardweave/checkpoint.hpp"
#include "shardweave/model.hpp"
#include "shardweave/model_spec.hpp"
#include "shardweave/pipeline.hpp"
#include "shardweave/plan.hpp"
#include "shardweave/roles.hpp"
#include "shardweave/spmd.hpp"
#include "shardweave/train_state.hpp"

using namespace shardweave;

// The reference allocates a fresh std::vector for every op result (tensor.hpp value semantics);
// at full model width that is hundreds of MB per op, and glibc returns every such block to the
// OS (mmap/munmap + page faults dominated the CPU time). Real deployments would sit on a
// caching allocator, so this driver provides one: large blocks are kept in per-size free
// lists and reused. Arithmetic is untouched.
namespace {
constexpr std::size_t kCacheMin = 1 << 20;
struct BlockCache {
  std::mutex mu;
  std::unordered_map<std::size_t, std::vector<void*>> free_;
};
BlockCache& block_cache() {
  static BlockCache* c = new BlockCache();
  return *c;
}
}  // namespace

void* operator new(std::size_t n) {
  const std::size_t total = n + 64;
  if (n >= kCacheMin) {
    BlockCache& c = block_cache();
    std::lock_guard<std::mutex> lock(c.mu);
    auto it = c.free_.find(total);
    if (it != c.free_.end() && !it->second.empty()) {
      void* p = it->second.back();
      it->second.pop_back();
      return static_cast<char*>(p) + 64;
    }
  }
  void* p = std::malloc(total);
  if (p == nullptr) throw std::bad_alloc();
  *static_cast<std::size_t*>(p) = total;
  return static_cast<char*>(p) + 64;
}

void operator delete(void* q) noexcept {
  if (q == nullptr) return;
  void* p = static_cast<char*>(q) - 64;
  const std::size_t total = *static_cast<std::size_t*>(p);
  if (total - 64 >= kCacheMin) {
    BlockCache& c = block_cache();
    std::lock_guard<std::mutex> lock(c.mu);
    c.free_[total].push_back(p);
    return;
  }
  std::free(p);
}

void operator delete(void* q, std::size_t) noexcept { operator delete(q); }

namespace {

std::string slurp(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw ConfigError("cannot open '" + path + "'");
  std::ostringstream s;
  s << in.rdbuf();
  return s.str();
}

struct Dump {
  std::ofstream bin, idx;
  std::uint64_t offset = 0;
  explicit Dump(const std::string& dir)
      : bin(dir + "/data.bin", std::ios::binary), idx(dir + "/index.tsv") {}
  template <typename S>
  void put(const std::string& name, const Tensor<S>& t) {
    std::vector<double> v(t.vec().begin(), t.vec().end());
    bin.write(reinterpret_cast<const char*>(v.data()), v.size() * sizeof(double));
    idx << name << '\t' << shape_str(t.shape()) << '\t' << offset << '\t' << v.size() << '\n';
    offset += v.size();
  }
  void scalar(const std::string& name, double x) {
    bin.write(reinterpret_cast<const char*>(&x), sizeof(double));
    idx << name << "\t[]\t" << offset << "\t1\n";
    offset += 1;
  }
};

void print_plan(const ShardingPlan& plan, const ShapeMap& shapes) {
  for (const auto& w : plan.warnings) std::cout << "WARN\t" << w << '\n';
  std::cout << serialize_plan(plan);
  for (const auto& v : validate_plan(plan, shapes)) std::cout << "VIOL\t" << v << '\n';
  std::cout << "STATE\t" << expected_state_elements(plan, shapes, plan.n_shards) << '\n';
}

template <typename Scalar>
InputMap<Scalar> audit_batch(std::uint64_t seed, int step, std::int64_t batch, std::int64_t seq,
                             std::int64_t vocab) {
  // cli.cpp:211-228
  RngStream rng = RngStream(seed, "audit-batch").child(static_cast<std::uint64_t>(step));
  Tensor<Scalar> tokens = Tensor<Scalar>::zeros({batch, seq});
  Tensor<Scalar> targets = Tensor<Scalar>::zeros({batch, seq});
  for (std::int64_t i = 0; i < tokens.numel(); ++i)
    tokens[i] = static_cast<Scalar>(rng.next_below(static_cast<std::uint64_t>(vocab)));
  for (std::int64_t i = 0; i < targets.numel(); ++i)
    targets[i] = static_cast<Scalar>(rng.next_below(static_cast<std::uint64_t>(vocab)));
  InputMap<Scalar> in;
  in.emplace("tokens", std::move(tokens));
  in.emplace("targets", std::move(targets));
  in.emplace("weights", Tensor<Scalar>::full({batch, seq}, Scalar(1)));
  return in;
}

template <typename Scalar>
int golden(const ModelSpec& spec, std::uint64_t seed, int dp, int mp, std::int64_t global_batch,
           std::int64_t seq, int steps, double lr, double wd, const std::string& out) {
  Dump dump(out);
  const std::int64_t rows = global_batch / dp;
  const ParamTree<Scalar> init = init_transformer_params<Scalar>(spec, RngStream(seed, "model-init"));
  for (const auto& [name, t] : init.entries()) dump.put("init/" + name, t);

  // logits of step 0's first replica slice (transformer_logits)
  {
    GraphBuilder<Scalar> lb;
    auto logits = transformer_logits(lb, spec, rows, seq);
    InputMap<Scalar> batch = audit_batch<Scalar>(seed, 0, global_batch, seq, spec.vocab_size);
    InputMap<Scalar> slice = dp == 1 ? batch : slice_batch_inputs(batch, dp, 0);
    dump.put("logits0", evaluate_one(lb.graph(), slice, init, logits.id));
  }

  GraphBuilder<Scalar> builder;
  auto loss = transformer_loss(builder, spec, rows, seq);
  const auto grad_nodes = grad(builder, loss, shapes_of(init));
  const ShardingPlan plan = derive_plan(init, mp, spec.overrides);
  const DeviceMesh mesh = build_mesh(dp, mp, 1);
  AdamWConfig opt;
  opt.lr = lr;
  opt.weight_decay = wd;

  // single-device reference trajectory (audit.hpp:104-118) and the sharded one.
  const DeviceMesh solo = build_mesh(1, 1, 1);
  TrainState<Scalar> ref = shard_params(init, plan, solo);
  TrainState<Scalar> state = shard_params(init, plan, mesh, seed);
  CommReport comm;
  for (int step = 0; step < steps; ++step) {
    const InputMap<Scalar> global = audit_batch<Scalar>(seed, step, global_batch, seq, spec.vocab_size);
    ParamTree<Scalar> ref_params = gather_params(ref, solo);
    DeviceGrads<Scalar> ref_grads = zero_grads_like(ref);
    std::vector<int> outs{loss.id};
    for (const auto& [name, id] : grad_nodes) outs.push_back(id);
    double ref_loss = 0;
    for (int r = 0; r < dp; ++r) {
      const InputMap<Scalar> slice = dp == 1 ? global : slice_batch_inputs(global, dp, r);
      auto vals = evaluate(builder.graph(), slice, ref_params, outs);
      ref_loss += static_cast<double>(vals[0].item());
      for (std::size_t i = 0; i < grad_nodes.size(); ++i) {
        ref_grads[ref.param_index(grad_nodes[i].first)][0].arr() += vals[i + 1].arr();
      }
    }
    ref_loss /= dp;
    if (dp > 1) scale_grads(ref_grads, 1.0 / dp);
    dump.scalar("ref_loss/" + std::to_string(step), ref_loss);
    if (step == 0) {
      for (std::size_t p = 0; p < ref.names.size(); ++p) dump.put("ref_grad0/" + ref.names[p], ref_grads[p][0]);
    }

    DeviceGrads<Scalar> acc = zero_grads_like(state);
    double loss_sum = 0;
    for (int r = 0; r < dp; ++r) {
      const InputMap<Scalar> replica = dp == 1 ? global : slice_batch_inputs(global, dp, r);
      SpmdParamMap<Scalar> views = replica_param_views(state, mesh, r);
      auto res = spmd_forward_backward(builder.graph(), loss.id, grad_nodes, replica, views, mesh,
                                       mesh.mp_group(r), &comm);
      loss_sum += static_cast<double>(res.loss);
      add_replica_grads(acc, state, mesh, r, res.grads);
    }
    dp_sync_grads(acc, mesh, &comm);
    dump.scalar("spmd_loss/" + std::to_string(step), loss_sum / dp);
    if (step == 0) {
      for (std::size_t p = 0; p < state.names.size(); ++p) {
        ShardedTensor<Scalar> g;
        g.global = state.shapes[p];
        g.partition = state.partitions[p];
        for (int j = 0; j < mesh.mp_size(); ++j) g.shards.push_back(acc[p][static_cast<std::size_t>(mesh.device_id(0, j))]);
        dump.put("spmd_grad0/" + state.names[p], gather(g));
      }
    }
    adamw_step(ref, ref_grads, opt);
    adamw_step(state, acc, opt);
  }
  ParamTree<Scalar> final_ref = gather_params(ref, solo);
  ParamTree<Scalar> final_spmd = gather_params(state, mesh);
  for (const auto& [name, t] : final_ref.entries()) dump.put("ref_final/" + name, t);
  for (const auto& [name, t] : final_spmd.entries()) dump.put("spmd_final/" + name, t);
  std::ofstream(out + "/comm_report.csv") << comm.to_csv();
  // optional SWCK snapshot of the sharded state (checkpoint.hpp:193-220), with a "train" stream
  // advanced 17 draws like tests/test_checkpoint.cpp:97-102
  if (const char* ck = std::getenv("SW_REF_CKPT")) {
    RngStream train(seed, "train");
    for (int i = 0; i < 17; ++i) train.next_u64();
    save_checkpoint(ck, state, mesh, {{"train", train}});
  }
  return 0;
}

template <typename Scalar>
int bench(const ModelSpec& spec, int mp, std::int64_t batch, std::int64_t seq, int steps,
          bool threads) {
  const ParamTree<Scalar> init = init_transformer_params<Scalar>(spec, RngStream(42, "model-init"));
  GraphBuilder<Scalar> builder;
  auto loss = transformer_loss(builder, spec, batch, seq);
  const auto grad_nodes = grad(builder, loss, shapes_of(init));
  const ShardingPlan plan = derive_plan(init, mp, spec.overrides);
  const DeviceMesh mesh = build_mesh(1, mp, 1);
  TrainState<Scalar> state = shard_params(init, plan, mesh);
  SpmdOptions options;
  options.worker_threads = threads;
  AdamWConfig opt;
  CommReport comm;
  double total = 0;
  for (int step = 0; step < steps; ++step) {
    const InputMap<Scalar> in = audit_batch<Scalar>(42, step, batch, seq, spec.vocab_size);
    const auto t0 = std::chrono::steady_clock::now();
    SpmdParamMap<Scalar> views = replica_param_views(state, mesh, 0);
    auto res = spmd_forward_backward(builder.graph(), loss.id, grad_nodes, in, views, mesh,
                                     mesh.mp_group(0), &comm, options);
    DeviceGrads<Scalar> acc = zero_grads_like(state);
    add_replica_grads(acc, state, mesh, 0, res.grads);
    adamw_step(state, acc, opt);
    const auto t1 = std::chrono::steady_clock::now();
    const double s = std::chrono::duration<double>(t1 - t0).count();
    total += s;
    std::printf("STEP\t%d\t%.6f\t%.9g\n", step, s, static_cast<double>(res.loss));
  }
  std::printf("TOTAL\t%.6f\t%lld\n", total, static_cast<long long>(batch * seq * steps));
  return 0;
}

// Trainer::fit (pipeline.hpp:351-454) on the transformer: examples are token windows drawn from
// RngStream(seed, "examples") (seq+1 ids each, one stream in order); collate gives tokens /
// targets (shifted) / weights = 1; loss_fn traces transformer_loss at the collated batch size.
template <typename Scalar>
int trainer_golden(const ModelSpec& spec, std::uint64_t seed, int dp, int mp, std::int64_t pdb, int accum,
                   int epochs, int n_examples, std::int64_t seq, double lr, double wd, double warmup,
                   const std::string& workdir) {
  using Example = std::vector<int>;
  DeployerConfig dc;
  dc.n_hosts = 1;
  dc.devices_per_host = dp * mp;
  dc.n_model_shards = mp;
  dc.seed = seed;
  dc.workdir = workdir;
  Deployer<Scalar> dep(dc);
  RngStream ex_rng(seed, "examples");
  std::vector<Example> examples(static_cast<std::size_t>(n_examples));
  for (auto& e : examples) {
    e.resize(static_cast<std::size_t>(seq + 1));
    for (auto& t : e) t = static_cast<int>(ex_rng.next_below(static_cast<std::uint64_t>(spec.vocab_size)));
  }
  PipelineSpec<Scalar, Example> ps;
  ps.collate_fn = [seq](const std::vector<Example>& batch) {
    const auto rows = static_cast<std::int64_t>(batch.size());
    Tensor<Scalar> tokens = Tensor<Scalar>::zeros({rows, seq});
    Tensor<Scalar> targets = Tensor<Scalar>::zeros({rows, seq});
    for (std::int64_t r = 0; r < rows; ++r) {
      for (std::int64_t t = 0; t < seq; ++t) {
        tokens[r * seq + t] = static_cast<Scalar>(batch[static_cast<std::size_t>(r)][static_cast<std::size_t>(t)]);
        targets[r * seq + t] = static_cast<Scalar>(batch[static_cast<std::size_t>(r)][static_cast<std::size_t>(t + 1)]);
      }
    }
    InputMap<Scalar> in;
    in.emplace("tokens", std::move(tokens));
    in.emplace("targets", std::move(targets));
    in.emplace("weights", Tensor<Scalar>::full({rows, seq}, Scalar(1)));
    return in;
  };
  ps.loss_fn = [&spec, seq](GraphBuilder<Scalar>& b, const ShapeMap& shapes) {
    return transformer_loss(b, spec, shapes[0].second[0], seq);
  };
  RunConfig rc;
  rc.n_epochs = epochs;
  rc.per_device_batch_size = pdb;
  rc.accumulate_grad_batches = accum;
  rc.optimizer.lr = lr;
  rc.optimizer.weight_decay = wd;
  rc.warmup_rate = warmup;
  const ParamTree<Scalar> init = init_transformer_params<Scalar>(spec, RngStream(seed, "model-init"));
  Trainer<Scalar, Example> tr(dep, ps, rc, init, spec.overrides);
  const TrainResult res = tr.fit(examples, {});
  for (std::size_t i = 0; i < res.step_losses.size(); ++i) {
    std::printf("STEP\t%zu\t%.17g\t%.17g\n", i, res.step_losses[i], res.step_lrs[i]);
  }
  std::printf("LOG\n%s", slurp(res.log_path).c_str());
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    if (argc < 2) throw ConfigError("usage: sw_ref_driver <cmd> ...");
    const std::string cmd = argv[1];
    if (cmd == "shapes" && argc == 3) {
      const ModelSpec spec = parse_model_spec(slurp(argv[2]));
      for (const auto& [name, shape] : transformer_param_shapes(spec))
        std::cout << name << '\t' << shape_str(shape) << '\n';
      return 0;
    }
    if (cmd == "plan" && argc == 4) {
      const ModelSpec spec = parse_model_spec(slurp(argv[2]));
      const ShapeMap shapes = transformer_param_shapes(spec);
      RoleInference inf = infer_roles(shapes, spec.overrides);
      ShardingPlan plan = derive_plan(inf.roles, shapes, std::atoi(argv[3]));
      plan.warnings.insert(plan.warnings.begin(), inf.warnings.begin(), inf.warnings.end());
      print_plan(plan, shapes);
      return 0;
    }
    if (cmd == "plan-shapes" && (argc == 4 || argc == 5)) {
      // shapes.tsv: name<TAB>d0,d1,...   overrides.tsv: pattern<TAB>role
      ShapeMap shapes;
      std::istringstream in(slurp(argv[2]));
      std::string line;
      while (std::getline(in, line)) {
        if (line.empty()) continue;
        const auto tab = line.find('\t');
        Shape s;
        std::string dims = line.substr(tab + 1);
        std::istringstream ds(dims);
        std::string tok;
        while (std::getline(ds, tok, ',')) {
          if (!tok.empty()) s.push_back(std::stoll(tok));
        }
        shapes.emplace_back(line.substr(0, tab), s);
      }
      std::vector<RoleOverride> ovr;
      if (argc == 5) {
        std::istringstream oi(slurp(argv[4]));
        while (std::getline(oi, line)) {
          if (line.empty()) continue;
          const auto tab = line.find('\t');
          ovr.push_back({line.substr(0, tab), parse_role(line.substr(tab + 1))});
        }
      }
      RoleInference inf = infer_roles(shapes, ovr);
      for (const auto& [name, a] : inf.roles)
        std::cout << "ROLE\t" << name << '\t' << role_name(a.role) << '\t' << a.sequence_index << '\n';
      ShardingPlan plan = derive_plan(inf.roles, shapes, std::atoi(argv[3]));
      plan.warnings.insert(plan.warnings.begin(), inf.warnings.begin(), inf.warnings.end());
      print_plan(plan, shapes);
      return 0;
    }
    if (cmd == "validate" && argc == 5) {
      // validate <shapes.tsv> <plan.txt> <n_shards>: parse_plan + validate_plan
      ShapeMap shapes;
      std::istringstream in(slurp(argv[2]));
      std::string line;
      while (std::getline(in, line)) {
        if (line.empty()) continue;
        const auto tab = line.find('\t');
        Shape s;
        std::istringstream ds(line.substr(tab + 1));
        std::string tok;
        while (std::getline(ds, tok, ',')) {
          if (!tok.empty()) s.push_back(std::stoll(tok));
        }
        shapes.emplace_back(line.substr(0, tab), s);
      }
      const ShardingPlan plan = parse_plan(slurp(argv[3]), std::atoi(argv[4]));
      std::cout << serialize_plan(plan);
      for (const auto& v : validate_plan(plan, shapes)) std::cout << "VIOL\t" << v << '\n';
      return 0;
    }
    if (cmd == "golden" && argc == 13) {
      const ModelSpec spec = parse_model_spec(slurp(argv[2]));
      const std::string dtype = argv[3];
      const auto seed = static_cast<std::uint64_t>(std::stoull(argv[4]));
      const int dp = std::atoi(argv[5]), mp = std::atoi(argv[6]);
      const std::int64_t gb = std::atoll(argv[7]), seq = std::atoll(argv[8]);
      const int steps = std::atoi(argv[9]);
      const double lr = std::atof(argv[10]), wd = std::atof(argv[11]);
      if (dtype == "f64") return golden<double>(spec, seed, dp, mp, gb, seq, steps, lr, wd, argv[12]);
      return golden<float>(spec, seed, dp, mp, gb, seq, steps, lr, wd, argv[12]);
    }
    if (cmd == "ckload" && argc == 6) {
      // ckload <spec> <dtype f32|f64> <mp> <file>: load_checkpoint (checkpoint.hpp:233-298) with the
      // rule plan at mp; prints "ok <step> <seed> <records>" or the CheckpointError text.
      const ModelSpec spec = parse_model_spec(slurp(argv[2]));
      const std::string dtype = argv[3];
      const int mp = std::atoi(argv[4]);
      const auto shapes = transformer_param_shapes(spec);
      ParamTree<double> tree;
      for (const auto& [name, shape] : shapes) tree.add(name, Tensor<double>::zeros(shape));
      const ShardingPlan plan = derive_plan(tree, mp, spec.overrides);
      const DeviceMesh mesh = build_mesh(1, mp, 1);
      try {
        if (dtype == "f64") {
          auto l = load_checkpoint<double>(argv[5], plan, mesh);
          std::cout << "ok " << l.state.step << " " << l.state.seed << " " << l.state.names.size() << "\n";
        } else {
          auto l = load_checkpoint<float>(argv[5], plan, mesh);
          std::cout << "ok " << l.state.step << " " << l.state.seed << " " << l.state.names.size() << "\n";
        }
      } catch (const CheckpointError& e) {
        std::cout << e.what() << "\n";
      }
      return 0;
    }
    if (cmd == "trainer" && argc == 15) {
      // trainer <spec> <seed> <dp> <mp> <per_device_batch> <accumulate> <epochs> <n_examples> <seq>
      //         <lr> <weight_decay> <warmup_rate> <workdir>
      const ModelSpec spec = parse_model_spec(slurp(argv[2]));
      return trainer_golden<float>(spec, std::stoull(argv[3]), std::atoi(argv[4]), std::atoi(argv[5]),
                                   std::atoll(argv[6]), std::atoi(argv[7]), std::atoi(argv[8]), std::atoi(argv[9]),
                                   std::atoll(argv[10]), std::atof(argv[11]), std::atof(argv[12]),
                                   std::atof(argv[13]), argv[14]);
    }
    if (cmd == "bench" && argc == 8) {
      const ModelSpec spec = parse_model_spec(slurp(argv[2]));
      return bench<float>(spec, std::atoi(argv[3]), std::atoll(argv[4]), std::atoll(argv[5]),
                          std::atoi(argv[6]), std::atoi(argv[7]) != 0);
    }
    throw ConfigError("bad arguments for '" + cmd + "'");
  } catch (const std::exception& e) {
    std::cout << "ERR\t" << e.what() << '\n';
    return 2;
  }
}
