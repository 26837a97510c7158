"""One prefill + a few cached decode steps (eager launches) for an ncu launch list:
SW_DECODE_GRAPH=0 ncu --metrics gpu__time_duration.sum ... python tools/decode_profile.py"""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2310_16355_b200 import engine, rules  # noqa: E402

spec = rules.read_model_spec(sys.argv[1] if len(sys.argv) > 1 else "oracle/specs/llama7b.spec")
B = int(sys.argv[2]) if len(sys.argv) > 2 else 1
plan = rules.derive_plan(rules.transformer_param_shapes(spec), 1, spec.overrides)
model = engine.Model(spec, plan, engine.Mesh(1, 1), B, spec.max_seq_len, inference=True)
model.init_params(1, "model-init")
prompts = np.random.default_rng(0).integers(0, spec.vocab_size, (B, 512)).astype(np.int32)
model.generate(prompts, 4)
