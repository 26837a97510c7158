"""Per-parameter parity report of the GPU step vs the numpy oracle (both oracle modes)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import model_ref, rng_ref  # noqa: E402
from tests.test_model_gpu import gemm_rounded, make, oracle_params, rel_l2, spec_dict, spec_of  # noqa: E402


def main(spec_name="tiny.spec", dp=1, mp=2, batch=4, seq=128):
    spec = spec_of(spec_name)
    model, mesh, _ = make(spec, dp, mp, batch, seq)
    model.init_params(42, "model-init")
    tokens, targets, weights = rng_ref.audit_batch(42, 0, dp * batch, seq, spec.vocab_size)
    model.stage_batch(tokens, targets, weights)
    model.forward_backward()
    model.dp_sync()
    out = {"loss": model.loss()}
    pr = gemm_rounded(oracle_params(spec))
    for mode in (False, True):
        l, g, _ = model_ref.forward_backward(pr, spec_dict(spec), tokens, targets, weights, bf16_acts=mode)
        out[f"oracle_loss_bf16acts={mode}"] = l
        errs = {n: rel_l2(model.get_grad(n).astype(np.float64), g[n]) for n in g}
        out[f"worst_bf16acts={mode}"] = sorted(errs.items(), key=lambda x: -x[1])[:8]
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(*[int(a) if a.isdigit() else a for a in sys.argv[1:]])
