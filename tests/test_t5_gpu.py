"""GPU parity of the T5 encoder-decoder extension (BASELINE cfg4): the step
through the C ABI (sw_t5_*) against the numpy f64 oracle (oracle/t5_ref.py, pinned by finite
differences in test_oracle_t5.py) on the same bf16-rounded GEMM weights, at mp = 1 / 2 / 4 on
the emulated mesh. Tolerances as the decoder's (north_star: rel-L2 <= 1e-2 in bf16), with the
attention-score path (q/k kernels and what only they feed) at 2e-2."""
import os

import numpy as np
import pytest

from oracle import t5_ref
from paper_2310_16355_b200 import engine, rules

pytestmark = pytest.mark.gpu

SPECS = os.path.join(os.path.dirname(__file__), "..", "oracle", "specs")
B, TE, TD = 2, 16, 16


def spec_dict(spec):
    return dict(vocab_size=spec.vocab_size, n_layers=spec.n_layers, n_dec_layers=spec.n_dec_layers,
                d_model=spec.d_model, n_heads=spec.n_heads, d_kv=spec.d_kv, d_ff=spec.d_ff,
                max_seq_len=spec.max_seq_len, rel_buckets=spec.rel_buckets,
                rel_max_distance=spec.rel_max_distance, arch="t5")


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-6 * np.sqrt(b.size)))


def make(mp):
    spec = rules.read_model_spec(os.path.join(SPECS, "mini_t5.spec"))
    shapes = rules.transformer_param_shapes(spec)
    plan = rules.derive_plan(shapes, mp, spec.overrides)
    mesh = engine.Mesh(1, mp)
    return engine.T5Model(spec, plan, mesh, B, TE, TD), mesh, spec


def gemm_view(params):
    """What the device computes with: GEMM weights as their bf16 shadow; the embedding table and
    the relative-position bias are read in fp32."""
    return {k: (t5_ref.bf16_round(v) if v.ndim == 2 and not k.startswith("embed/") and "rel_bias" not in k
                else v.astype(np.float64)) for k, v in params.items()}


def t5_init_scaling(model, spec):
    """T5's own initialisation folds the 1/sqrt(d_kv) attention scale into the query weights
    (Mesh-TF T5: q ~ N(0, (d_model * d_kv)^-1/2)). The reference rule N(0, 1/fan_in) leaves the
    unscaled T5 scores ~sqrt(d_kv) times sharper than trained T5 runs see, which amplifies bf16
    rounding of q/k into the probabilities; the parity tests use T5's regime."""
    for n in model.shapes:
        if n.endswith("attn/q/kernel"):
            model.set_param(n, model.get_param(n) / np.sqrt(spec.d_kv))


SCORE = ("attn/q/kernel", "attn/k/kernel", "ln1/scale", "ln_x/scale", "rel_bias/kernel")


def test_t5_init_matches_reference_rules():
    model, _, spec = make(2)
    model.init_params(42, "model-init")
    want = t5_ref.init_params(spec_dict(spec), seed=42, dtype=np.float32)
    for n in want:
        assert np.array_equal(model.get_param(n), want[n]), n


@pytest.mark.parametrize("mp", [1, 2, 4])
def test_t5_forward_backward_matches_oracle(mp):
    model, mesh, spec = make(mp)
    model.init_params(42, "model-init")
    t5_init_scaling(model, spec)
    sd = spec_dict(spec)
    enc, dec, tgt, w = t5_ref.t5_batch(42, 0, B, TE, TD, spec.vocab_size)
    w[:, -3:] = 0.5  # non-uniform weights
    model.stage_batch(enc, dec, tgt, w)
    model.forward_backward()
    loss = model.loss()
    params = {n: model.get_param(n) for n in model.shapes}
    want_loss, want, logits = t5_ref.forward_backward(gemm_view(params), sd, enc, dec, tgt, w, bf16_acts=True)
    assert abs(loss - want_loss) / want_loss < 2e-3, (loss, want_loss)
    worst = ("", 0.0)
    for n in want:
        r = rel_l2(model.get_grad(n).astype(np.float64), want[n])
        worst = max(worst, (n, r), key=lambda x: x[1])
        assert r < (2e-2 if n.endswith(SCORE) else 1e-2), (n, r)
    got_logits = model.forward_logits()
    assert rel_l2(got_logits.astype(np.float64), logits) < 1e-2
    if mp == 2:
        ar = mesh.comm_report().splitlines()[1].split(",")
        L = spec.n_layers + spec.n_dec_layers
        # fwd: 2 AR per encoder layer, 3 per decoder layer; bwd: the same plus one for the
        # encoder-output gradient and one per rel_bias table (counted over fwd+bwd+logits fwd)
        fwd = 2 * spec.n_layers + 3 * spec.n_dec_layers
        assert int(ar[1]) == 2 * fwd + 3 + fwd, (ar, L)


def test_t5_tensor_parallel_invariance_and_training():
    """mp = 2 gradients equal mp = 1 ones; a few AdamW steps lower the loss on a fixed batch."""
    res = {}
    for mp in (1, 2):
        model, _, spec = make(mp)
        model.init_params(7, "model-init")
        enc, dec, tgt, w = t5_ref.t5_batch(7, 0, B, TE, TD, spec.vocab_size)
        model.stage_batch(enc, dec, tgt, w)
        model.forward_backward()
        res[mp] = (model.loss(), {n: model.get_grad(n) for n in model.shapes})
        if mp == 2:
            cfg = engine.AdamWConfig(lr=3e-3, weight_decay=0.0)
            losses = []
            for _ in range(4):
                model.train_step(cfg)
                losses.append(model.loss())
            assert losses[-1] < losses[0], losses
    assert abs(res[2][0] - res[1][0]) / res[1][0] < 2e-4
    for n in res[1][1]:
        assert rel_l2(res[2][1][n].astype(np.float64), res[1][1][n].astype(np.float64)) < 1e-2, n


@pytest.mark.parametrize("tc", ["1", "0"])
@pytest.mark.parametrize("mp,T,Td", [(1, 160, 160), (2, 128, 128), (1, 192, 128), (2, 128, 200)])
def test_t5_head_dim_128_attention_paths(tc, mp, T, Td, monkeypatch):
    """d_kv = 128 runs the tcgen05 attention (relative bias as a per-head LUT over key - query,
    non-causal encoder, the bias gradient summed along diagonals of dS; cross-attention over fused
    q|k|v when enc_len == dec_len, over separate decoder q and encoder k|v rows otherwise -- the
    last two cases); SW_T5_TC=0 forces the CUDA-core kernels. Both match
    the oracle (which models the tensor-core kernels' bf16 P / dS operands); T = 160 exercises the
    sequence tails. Tolerance 3e-2 (score path 4e-2): in this d_model = 64 / inner = 256 shape the
    bf16 forward noise flips ReLU masks below the last MLP, so both attention paths sit at 1-2.5%
    rel-L2 there (measured: CUDA-core worst 2.3%, tensor-core 2.6%); mini_t5.spec keeps 1e-2."""
    monkeypatch.setenv("SW_T5_TC", tc)
    spec = rules.read_model_spec(os.path.join(SPECS, "mini_t5_hd128.spec"))
    shapes = rules.transformer_param_shapes(spec)
    plan = rules.derive_plan(shapes, mp, spec.overrides)
    mesh = engine.Mesh(1, mp)
    model = engine.T5Model(spec, plan, mesh, 2, T, Td)
    model.init_params(11, "model-init")
    t5_init_scaling(model, spec)
    enc, dec, tgt, w = t5_ref.t5_batch(11, 0, 2, T, Td, spec.vocab_size)
    model.stage_batch(enc, dec, tgt, w)
    model.forward_backward()
    loss = model.loss()
    params = {n: model.get_param(n) for n in model.shapes}
    want_loss, want, _ = t5_ref.forward_backward(gemm_view(params), spec_dict(spec), enc, dec, tgt, w, bf16_acts=True,
                                                 round_p=tc == "1")
    assert abs(loss - want_loss) / want_loss < 2e-3, (loss, want_loss)
    for n in want:
        got = model.get_grad(n).astype(np.float64)
        if "rel_bias" in n:
            # sum_j dS_ij = 0 for every query row, so a bucket covering most of a row is a sum that
            # nearly cancels: relative norms are ill-conditioned; use the reference audit metric
            # max|a-b| / max(|b|, 1) (cli.cpp:234) as for the analytically-zero attn/k/bias
            assert np.max(np.abs(got - want[n]) / np.maximum(np.abs(want[n]), 1.0)) < 1e-3, n
            continue
        r = rel_l2(got, want[n])
        assert r < (4e-2 if n.endswith(SCORE) else 3e-2), (n, r)


@pytest.mark.parametrize("mp", [1, 2])
def test_t5_fused_optimizer_matches_two_pass_step(mp):
    """train_step applies AdamW inside the weight-gradient GEMM epilogues (GEMM weights) and one
    flat AdamW over the rest; forward_backward + adamw_step is the two-pass step. Same init, same
    batch, two steps. Two backward passes of this executor differ by up to ~2e-3 rel-L2 in the
    first encoder layer's attention gradients and ~1.3% in its norm-scale gradient (order-
    dependent fp32 reductions, amplified by the cancellation in dS = P (dP - delta) at this
    near-uniform init; tools/t5_determinism.py), and AdamW turns such noise on near-zero
    gradients into full-size updates of either sign, so the check is: Adam first moments close,
    and all but a sliver of the parameter updates equal."""
    lr, steps = 1e-3, 2
    out = {}
    for fused in (True, False):
        model, _, spec = make(mp)
        model.init_params(11, "model-init")
        t5_init_scaling(model, spec)
        p0 = {n: model.get_param(n) for n in model.shapes}
        enc, dec, tgt, w = t5_ref.t5_batch(11, 0, B, TE, TD, spec.vocab_size)
        model.stage_batch(enc, dec, tgt, w)
        cfg = engine.AdamWConfig(lr=lr, weight_decay=0.01)
        for _ in range(steps):
            if fused:
                model.train_step(cfg)
            else:
                model.forward_backward()
                model.adamw_step(cfg)
        out[fused] = (model.loss(), {n: model.get_param(n) - p0[n] for n in model.shapes},
                      {n: model.get_adam(n)[0] for n in model.shapes})
    assert abs(out[True][0] - out[False][0]) <= 1e-4 * abs(out[False][0])
    for n in out[True][1]:
        m_f, m_u = out[True][2][n].astype(np.float64), out[False][2][n].astype(np.float64)
        assert rel_l2(m_f, m_u) < 5e-2, n
        diff = np.abs(out[True][1][n] - out[False][1][n])
        assert diff.max() <= 2 * lr * steps + 1e-6, n
        # the attention-score kernels carry the noisiest gradients (~1% of their elements flip)
        assert (diff > 1e-4).sum() <= max(2, 0.05 * diff.size), (n, int((diff > 1e-4).sum()))


def test_t5_fused_step_nonfinite_loss_leaves_state_unchanged():
    """A non-finite loss gates every fused AdamW epilogue: train_step raises NonFiniteError and
    every parameter and moment is exactly as before the step (the model stays usable)."""
    model, _, spec = make(1)
    model.init_params(5, "model-init")
    enc, dec, tgt, w = t5_ref.t5_batch(5, 0, B, TE, TD, spec.vocab_size)
    tok = model.get_param("embed/tok/kernel")
    bad = tok.copy()
    bad[int(dec[0, 0])] = np.inf  # a decoder input row: the logits, hence the loss, go non-finite
    model.set_param("embed/tok/kernel", bad)
    model.stage_batch(enc, dec, tgt, w)
    before = {n: (model.get_param(n), *model.get_adam(n)) for n in model.shapes}
    with pytest.raises(engine._lib.NonFiniteError, match="non-finite loss"):
        model.train_step(engine.AdamWConfig(lr=1e-3))
    for n, (p, m, v) in before.items():
        p2, m2, v2 = model.get_param(n), *model.get_adam(n)
        assert np.array_equal(p, p2, equal_nan=True) and np.array_equal(m, m2) and np.array_equal(v, v2), n
    model.set_param("embed/tok/kernel", tok)
    model.train_step(engine.AdamWConfig(lr=1e-3))
    assert np.isfinite(model.loss())
