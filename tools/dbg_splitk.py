import sys, numpy as np
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from test_model_gpu import make, rel_l2
from oracle import rng_ref
from paper_2310_16355_b200 import engine, rules
import tempfile, os
d = tempfile.mkdtemp(); path = os.path.join(d, "s.spec")
open(path, "w").write("vocab_size = 1024\nn_layers = 2\nd_model = 512\nn_heads = 4\nd_ff = 1376\nmax_seq_len = 512\n")
spec = rules.read_model_spec(path)
seq, batch, mp = 512, 4, 2
fused, _, _ = make(spec, 1, mp, batch, seq); plain, _, _ = make(spec, 1, mp, batch, seq)
for m in (fused, plain): m.init_params(42, "model-init")
cfg = engine.AdamWConfig(lr=1e-3, weight_decay=0.01)
tokens, targets, weights = rng_ref.audit_batch(42, 0, batch, seq, spec.vocab_size)
for m in (fused, plain): m.stage_batch(tokens, targets, weights)
fused.train_step(cfg)
plain.forward_backward()
g = {n: plain.get_grad(n) for n in plain.shapes}
plain.adamw_step(cfg)
print("loss", fused.loss(), plain.loss())
for n in plain.shapes:
    a, b = fused.get_param(n), plain.get_param(n)
    dd = np.abs(a - b)
    print(n, "maxdiff", float(dd.max()), "n_off", int((dd > 1e-6 + 1e-5*np.abs(b)).sum()), "size", a.size, "gmax", float(np.abs(g[n]).max()))
