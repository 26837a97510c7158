"""Per-parameter rel-L2 of the T5 head-dim-128 step (tcgen05 or CUDA-core attention) vs the oracle."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from oracle import t5_ref  # noqa: E402
from paper_2310_16355_b200 import engine, rules  # noqa: E402
import test_t5_gpu as T5  # noqa: E402


def main(mp=1, T=160):
    spec = rules.read_model_spec(os.path.join(T5.SPECS, "mini_t5_hd128.spec"))
    shapes = rules.transformer_param_shapes(spec)
    plan = rules.derive_plan(shapes, mp, spec.overrides)
    mesh = engine.Mesh(1, mp)
    model = engine.T5Model(spec, plan, mesh, 2, T, T)
    model.init_params(11, "model-init")
    T5.t5_init_scaling(model, spec)
    enc, dec, tgt, w = t5_ref.t5_batch(11, 0, 2, T, T, spec.vocab_size)
    model.stage_batch(enc, dec, tgt, w)
    model.forward_backward()
    params = {n: model.get_param(n) for n in model.shapes}
    wl, want, _ = t5_ref.forward_backward(T5.gemm_view(params), T5.spec_dict(spec), enc, dec, tgt, w, bf16_acts=True,
                                         round_p=os.environ.get("SW_T5_TC", "1") == "1")
    out = {"tc": os.environ.get("SW_T5_TC", "1"), "loss": [model.loss(), wl]}
    for n in want:
        out[n] = round(T5.rel_l2(model.get_grad(n).astype(np.float64), want[n]), 5)
    print(json.dumps(out))


if __name__ == "__main__":
    main(*[int(a) for a in sys.argv[1:]])
