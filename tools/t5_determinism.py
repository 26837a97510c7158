"""Repeatability of the T5 executor's gradients on the mini config: python tools/t5_determinism.py [reps]
Prints the largest rel-L2 between the first run's gradients and each later run's (same model,
same batch, forward_backward only)."""
import sys

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from test_t5_gpu import B, TD, TE, make, rel_l2, t5_init_scaling  # noqa: E402

from oracle import t5_ref  # noqa: E402


def main(reps=6, mp=1):
    model, _, spec = make(int(mp))
    model.init_params(11, "model-init")
    t5_init_scaling(model, spec)
    enc, dec, tgt, w = t5_ref.t5_batch(11, 0, B, TE, TD, spec.vocab_size)
    model.stage_batch(enc, dec, tgt, w)
    ref = None
    worst = []
    for _ in range(int(reps)):
        model.forward_backward()
        g = {n: model.get_grad(n) for n in model.shapes}
        if ref is None:
            ref = g
            continue
        worst.append(max((rel_l2(g[n], ref[n]), n) for n in g))
    print(worst)


if __name__ == "__main__":
    main(*sys.argv[1:])
