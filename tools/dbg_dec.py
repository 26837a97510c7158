import os, sys, numpy as np
sys.path.insert(0, ".")
from oracle import rng_ref
from paper_2310_16355_b200 import engine, rules
txt = open("oracle/specs/mini_hd64.spec").read()
for name, t in (("hd64", txt), ("hd128", txt.replace("d_model = 128", "d_model = 256"))):
    spec = rules.parse_model_spec(t)
    plan = rules.derive_plan(rules.transformer_param_shapes(spec), 1, spec.overrides)
    model = engine.Model(spec, plan, engine.Mesh(1, 1), 2, 16)
    model.init_params(7, "model-init")
    nm = "lm_head/kernel"
    model.set_param(nm, model.get_param(nm) * 24.0)
    prompts = rng_ref.RngStream(3, "prompts").below(2 * 5, spec.vocab_size).reshape(2, 5)
    got = model.generate(prompts, 11)
    ctx = prompts.copy(); rec = []
    for _ in range(11):
        nxt = model.generate(ctx, 1); rec.append(nxt[:, 0]); ctx = np.concatenate([ctx, nxt], 1)
    rec = np.stack(rec, 1)
    print(name, os.environ.get("SW_DECODE_GRAPH"), "\n", got, "\n", rec, np.array_equal(got, rec))
