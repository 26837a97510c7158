"""Per-parameter rel-L2 of the T5 GPU gradients against the oracle (diagnostics)."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from oracle import t5_ref  # noqa: E402
import test_t5_gpu as T  # noqa: E402


def main(mp=1, bf16_acts=1):
    model, mesh, spec = T.make(mp)
    model.init_params(42, "model-init")
    T.t5_init_scaling(model, spec)
    sd = T.spec_dict(spec)
    enc, dec, tgt, w = t5_ref.t5_batch(42, 0, T.B, T.TE, T.TD, spec.vocab_size)
    model.stage_batch(enc, dec, tgt, w)
    model.forward_backward()
    loss = model.loss()
    params = {n: model.get_param(n) for n in model.shapes}
    wl, want, logits = t5_ref.forward_backward(T.gemm_view(params), sd, enc, dec, tgt, w, bf16_acts=bool(bf16_acts))
    out = {"loss": [loss, wl]}
    for n in want:
        g = model.get_grad(n).astype(np.float64)
        out[n] = round(T.rel_l2(g, want[n]), 5)
    print(json.dumps(out, indent=0))


if __name__ == "__main__":
    main(*[int(a) for a in sys.argv[1:]])
