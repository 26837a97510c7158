"""LLaMA-7B width (2 layers, 512 tokens) at mp = 8 on the emulated mesh: loss and gradient
rel-L2 of the bf16 all-reduce payloads (SW_AR_BF16=1) against fp32 payloads and against mp = 1."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2310_16355_b200 import engine, rules  # noqa: E402

NAMES = ("block_0/attn/q/kernel", "block_0/attn/o/kernel", "block_0/mlp/fc1/kernel", "block_1/mlp/fc2/kernel",
         "block_0/ln1/scale", "block_1/ln2/bias", "lm_head/kernel", "embed/tok/kernel")


def run(mp, bf16, spec):
    os.environ["SW_AR_BF16"] = "1" if bf16 else "0"
    shapes = rules.transformer_param_shapes(spec)
    plan = rules.derive_plan(shapes, mp, spec.overrides)
    mesh = engine.Mesh(1, mp)
    m = engine.Model(spec, plan, mesh, 2, 256)
    m.init_params(42, "model-init")
    rng = np.random.default_rng(3)
    m.stage_batch(rng.integers(0, spec.vocab_size, (2, 256), dtype=np.int32),
                  rng.integers(0, spec.vocab_size, (2, 256), dtype=np.int32), None)
    m.forward_backward()
    out = (m.loss(), {n: m.get_grad(n).astype(np.float64) for n in NAMES})
    m.close()
    mesh.close()
    return out


def rl2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def main():
    text = open("oracle/specs/llama7b_vocab_parallel.spec").read().replace("n_layers = 32", "n_layers = 2")
    spec = rules.parse_model_spec(text)
    ref, f32, b16 = run(1, False, spec), run(8, False, spec), run(8, True, spec)
    out = {"loss": [ref[0], f32[0], b16[0]]}
    for n in NAMES:
        out[n] = {"fp32_vs_mp1": round(rl2(f32[1][n], ref[1][n]), 5), "bf16_vs_mp1": round(rl2(b16[1][n], ref[1][n]), 5)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
