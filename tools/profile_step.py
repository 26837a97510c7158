"""One training step of the LLaMA-7B-shape model bracketed by cudaProfilerStart/Stop, for
`ncu --profile-from-start off` (launch lists and single-kernel captures)."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2310_16355_b200 import engine, rules  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--spec", default="oracle/specs/llama7b.spec")
ap.add_argument("--batch", type=int, default=4)
ap.add_argument("--seq", type=int, default=2048)
ap.add_argument("--steps", type=int, default=1)
a = ap.parse_args()
spec = rules.read_model_spec(a.spec)
plan = rules.derive_plan(rules.transformer_param_shapes(spec), 1, spec.overrides)
mesh = engine.Mesh(1, 1)
model = engine.Model(spec, plan, mesh, a.batch, a.seq)
model.init_params(42, "model-init")
rng = np.random.default_rng(0)
tok = rng.integers(0, spec.vocab_size, (a.batch, a.seq), dtype=np.int32)
tgt = rng.integers(0, spec.vocab_size, (a.batch, a.seq), dtype=np.int32)
model.stage_batch(tok, tgt, None)
cfg = engine.AdamWConfig(lr=1e-4, weight_decay=0.01)
model.train_step(cfg)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for _ in range(a.steps):
    model.train_step(cfg)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("loss", model.loss(), "launches/step", model.launch_count())
