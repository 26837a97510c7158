"""Greedy-decode timing (KV-cached steps) at the LLaMA-7B shape: python tools/decode_bench.py
[spec] [batch] [prompt] [n_new] [inference 0/1] [mp] [seq]. Reports ms per generated position and
the HBM roofline of a step (bf16 weights + the cached K/V read once per step). inference=1 builds
the inference-only model (no train state: the full OPT-66B shape fits one GPU); mp > 1 emulates
the tensor-parallel ranks on one GPU (they run one after another, so the time is the sum)."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2310_16355_b200 import engine, rules  # noqa: E402


def main(spec_path="oracle/specs/llama7b.spec", batch=4, prompt=512, n_new=64, inference=0, mp=1, seq=0):
    batch, prompt, n_new, inference, mp, seq = int(batch), int(prompt), int(n_new), int(inference), int(mp), int(seq)
    spec = rules.read_model_spec(spec_path)
    seq = seq or spec.max_seq_len
    plan = rules.derive_plan(rules.transformer_param_shapes(spec), mp, spec.overrides)
    t0 = time.perf_counter()
    model = engine.Model(spec, plan, engine.Mesh(1, mp), batch, seq, inference=bool(inference))
    model.init_params(1, "model-init")
    t_build = time.perf_counter() - t0
    prompts = np.random.default_rng(0).integers(0, spec.vocab_size, (batch, prompt)).astype(np.int32)
    model.generate(prompts, 2)  # warm-up (prefill + one cached step)
    t0 = time.perf_counter()
    model.generate(prompts, 1)
    t_prefill = time.perf_counter() - t0
    t0 = time.perf_counter()
    model.generate(prompts, n_new)
    t_all = time.perf_counter() - t0
    step_ms = (t_all - t_prefill) / (n_new - 1) * 1e3
    shapes = rules.transformer_param_shapes(spec)
    n_w = sum(int(np.prod(d)) for n, d in shapes if len(d) == 2 and not n.startswith("embed/"))
    hd = spec.d_model // spec.n_heads
    kv = 2 * spec.n_layers * batch * (prompt + n_new / 2) * spec.d_model * 2
    byts = 2 * n_w + kv
    print(json.dumps({"spec": spec_path, "batch": batch, "prompt": prompt, "n_new": n_new,
                      "prefill_ms": round(t_prefill * 1e3, 2), "decode_ms_per_token": round(step_ms, 3),
                      "tokens_per_s": round(batch * 1e3 / step_ms, 1), "bytes_per_step": int(byts),
                      "achieved_gbs": round(byts / step_ms / 1e6, 1), "hd": hd, "inference": bool(inference),
                      "mp": mp, "seq": seq, "device_gb": round(model.device_bytes() / 1e9, 2),
                      "build_s": round(t_build, 1)}))


if __name__ == "__main__":
    main(*sys.argv[1:])
