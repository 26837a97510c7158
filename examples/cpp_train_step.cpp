// A reference-style C++ caller of the B200 step through include/shardweave_b200.hpp:
// parse a model spec, derive the rule plan (bit-exact with the reference), and (with --run)
// take optimizer steps of the transformer on an emulated dp x mp mesh on GPU 0.
//   cpp_train_step <spec> <mp> [--run <batch> <seq> <steps>]
#include <cstdio>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>

#include "shardweave_b200.hpp"

namespace b2 = shardweave::b200;

int main(int argc, char** argv) {
  if (argc < 3) {
    std::cerr << "usage: cpp_train_step <spec> <mp> [--run <batch> <seq> <steps>]\n";
    return 2;
  }
  try {
    std::ifstream in(argv[1]);
    std::stringstream ss;
    ss << in.rdbuf();
    auto spec = b2::parse_model_spec(ss.str());
    const int mp = std::atoi(argv[2]);
    const auto shapes = spec->param_shapes();
    auto plan = b2::derive_plan(shapes, mp, spec->overrides());
    if (argc == 3) {
      for (const auto& w : {plan->warnings()}) if (!w.empty()) std::cout << "WARN\t" << w << '\n';
      std::cout << plan->serialize();
      for (const auto& v : b2::validate_plan(*plan, shapes)) std::cout << "VIOL\t" << v << '\n';
      return 0;
    }
    const int batch = std::atoi(argv[4]), seq = std::atoi(argv[5]), steps = std::atoi(argv[6]);
    b2::Mesh mesh(1, mp);
    b2::Model model(*spec, *plan, mesh, batch, seq);
    model.init_params(42);
    std::vector<int32_t> tokens(static_cast<size_t>(batch) * seq), targets(tokens.size());
    uint64_t x = 88172645463325252ull;
    const int64_t vocab = static_cast<int64_t>(shapes[0].second[0]);
    for (size_t i = 0; i < tokens.size(); ++i) {
      x ^= x << 13, x ^= x >> 7, x ^= x << 17;
      tokens[i] = static_cast<int32_t>(x % static_cast<uint64_t>(vocab));
      targets[i] = static_cast<int32_t>((x >> 20) % static_cast<uint64_t>(vocab));
    }
    b2::AdamWConfig cfg;
    cfg.lr = 1e-3;
    cfg.weight_decay = 0.01;
    model.stage_batch(tokens, targets);
    for (int s = 0; s < steps; ++s) {
      model.train_step(cfg);
      std::printf("step=%d loss=%.9g\n", s, model.loss());
    }
    std::cout << mesh.comm_report_csv();
  } catch (const b2::Error& e) {
    std::cerr << "error: " << e.what() << '\n';
    return 1;
  }
  return 0;
}
