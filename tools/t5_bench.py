"""T5-11B-width encoder-decoder train step on one GPU (BASELINE cfg4 is TP=8 on 8 GPUs: here
the depth is truncated so the full-width state fits 180 GB at TP=1). Prints tokens/s (decoder
tokens), the per-category device-time breakdown and the algorithmic TFLOP/s.
Usage: python tools/t5_bench.py [enc_layers dec_layers batch enc_len dec_len steps]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import t5_ref  # noqa: E402
from paper_2310_16355_b200 import engine, rules  # noqa: E402


def main(le=2, ld=2, batch=4, te=512, td=512, steps=3):
    text = open(os.path.join("oracle", "specs", "t5_11b.spec")).read()
    text = text.replace("n_layers = 24", f"n_layers = {le}").replace("n_dec_layers = 24", f"n_dec_layers = {ld}")
    spec = rules.parse_model_spec(text)
    shapes = rules.transformer_param_shapes(spec)
    plan = rules.derive_plan(shapes, 1, spec.overrides)
    mesh = engine.Mesh(1, 1)
    model = engine.T5Model(spec, plan, mesh, batch, te, td)
    model.init_params(42, "model-init")
    enc, dec, tgt, w = t5_ref.t5_batch(1, 0, batch, te, td, spec.vocab_size)
    model.stage_batch(enc, dec, tgt, w)
    cfg = engine.AdamWConfig(lr=1e-4, weight_decay=0.01)
    stream = torch.cuda.ExternalStream(model.stream())
    model.train_step(cfg)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        model.train_step(cfg)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    model.set_profiling(True)
    model.train_step(cfg)
    prof = model.read_profile()
    n_params = sum(int(np.prod(d)) for _, d in shapes)
    d, H, dk = spec.d_model, spec.n_heads, spec.d_kv
    # matmul FLOPs: 6 * (params touched per token) per stack + attention (4*T*dk per head-token, x3)
    enc_p = sum(int(np.prod(dd)) for n, dd in shapes if n.startswith("enc/") and len(dd) == 2 and "rel_bias" not in n)
    dec_p = sum(int(np.prod(dd)) for n, dd in shapes if n.startswith("dec/") and len(dd) == 2 and "rel_bias" not in n)
    head_p = spec.vocab_size * d
    flops = 6 * (enc_p * batch * te + dec_p * batch * td + head_p * batch * td)
    flops += 3 * 4 * batch * H * dk * (le * te * te + ld * (td * td / 2 + td * te))
    print(json.dumps({"workload": f"T5-11B width ({le}+{ld} layers of 24+24), batch {batch}, enc {te} / dec {td}",
                      "params": n_params, "ms_per_step": round(ms, 2),
                      "dec_tokens_per_s": round(batch * td / ms * 1e3, 1),
                      "tflops": round(flops / ms / 1e9, 1), "loss": model.loss(),
                      "breakdown_ms": {k: round(v["ms"], 2) for k, v in prof.items() if v["launches"]},
                      "device_gb": round(model.device_bytes() / 1e9, 1)}))


if __name__ == "__main__":
    main(*[int(a) for a in sys.argv[1:]])
