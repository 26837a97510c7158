"""T5-11B width, 1+1 layers: one forward/backward with the tcgen05 attention (SW_T5_TC=1) and with
the CUDA-core kernels (SW_T5_TC=0) from the same weights and batch; prints loss and per-gradient
rel-L2 between the two paths. Usage: python tools/t5_path_compare.py [T] [batch]"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, ".")
from oracle import t5_ref  # noqa: E402
from paper_2310_16355_b200 import engine, rules  # noqa: E402


def run(tc, T, batch):
    os.environ["SW_T5_TC"] = tc
    text = open("oracle/specs/t5_11b.spec").read().replace("n_layers = 24", "n_layers = 1")
    text = text.replace("n_dec_layers = 24", "n_dec_layers = 1")
    spec = rules.parse_model_spec(text)
    shapes = rules.transformer_param_shapes(spec)
    plan = rules.derive_plan(shapes, 1, spec.overrides)
    mesh = engine.Mesh(1, 1)
    m = engine.T5Model(spec, plan, mesh, batch, T, T)
    m.init_params(42, "model-init")
    for n in m.shapes:
        if n.endswith("attn/q/kernel"):
            m.set_param(n, m.get_param(n) / np.sqrt(spec.d_kv))
    enc, dec, tgt, w = t5_ref.t5_batch(1, 0, batch, T, T, spec.vocab_size)
    m.stage_batch(enc, dec, tgt, w)
    m.forward_backward()
    out = (m.loss(), {n: m.get_grad(n) for n in m.shapes})
    m.close()
    mesh.close()
    return out


def main(T=512, batch=2):
    a, b = run("1", T, batch), run("0", T, batch)
    res = {"loss_tc": a[0], "loss_cuda_core": b[0]}
    for n in a[1]:
        x, y = a[1][n].astype(np.float64), b[1][n].astype(np.float64)
        res[n] = round(float(np.linalg.norm(x - y) / max(np.linalg.norm(y), 1e-30)), 5)
    print(json.dumps(res))


if __name__ == "__main__":
    main(*[int(v) for v in sys.argv[1:]])
