"""Greedy generation: the Predictor's next-token loop (cli.cpp:425-447) with a
KV cache. The cached steps must pick exactly the tokens a full re-run of the reference's window
picks (checked on the device against the window recompute, and against the f64 oracle wherever
the oracle's top-2 margin is not a near-tie), including the switch to the sliding window once the
context outgrows seq_len."""
import os

import numpy as np
import pytest

from oracle import model_ref, rng_ref
from paper_2310_16355_b200 import engine, rules

pytestmark = pytest.mark.gpu
SPECS = os.path.join(os.path.dirname(__file__), "..", "oracle", "specs")


def build(spec_name, mp, batch, seq):
    spec = rules.read_model_spec(os.path.join(SPECS, spec_name))
    plan = rules.derive_plan(rules.transformer_param_shapes(spec), mp, spec.overrides)
    model = engine.Model(spec, plan, engine.Mesh(1, mp), batch, seq)
    model.init_params(7, "model-init")
    # a confident head: random-init logits are nearly flat, so argmax would sit on near-ties
    name = "embed/tok/kernel" if spec.tie_embeddings else "lm_head/kernel"
    model.set_param(name, model.get_param(name) * 24.0)
    return model, spec


def spec_dict(spec):
    return dict(vocab_size=spec.vocab_size, n_layers=spec.n_layers, d_model=spec.d_model, n_heads=spec.n_heads,
                d_ff=spec.d_ff, max_seq_len=spec.max_seq_len, tie_embeddings=spec.tie_embeddings, mlp=spec.mlp,
                norm=spec.norm)


def oracle_check(model, spec, prompts, got, seq):
    """Teacher-forced: at every step the f64 oracle runs the reference's window over the device's
    own context and must pick the device's token unless its top two logits are within a few bf16
    ulps (relative margin < 2%). Returns the number of decisive steps."""
    params = {n: model.get_param(n).astype(np.float64) for n in model.shapes}
    for n, v in params.items():  # the device's GEMMs read bf16 weights
        if v.ndim == 2 and not n.startswith("embed/"):
            params[n] = model_ref.bf16_round(v)
    ctx = np.asarray(prompts)
    decisive = 0
    for i in range(got.shape[1]):
        take = min(ctx.shape[1], seq)
        win = np.zeros((ctx.shape[0], seq), np.int64)
        win[:, :take] = ctx[:, -take:]
        _, _, logits = model_ref.forward_backward(params, spec_dict(spec), win, win, np.ones(win.shape),
                                                  need_grads=False)
        row = logits[:, take - 1]
        srt = np.sort(row, -1)
        margin = (srt[:, -1] - srt[:, -2]) / np.maximum(np.abs(srt[:, -1]), 1.0)
        for b in range(ctx.shape[0]):
            if margin[b] >= 0.02:
                assert got[b, i] == row[b].argmax(), (i, b, got[b, i], row[b].argmax(), margin[b])
                decisive += 1
        ctx = np.concatenate([ctx, got[:, i:i + 1]], 1)
    return decisive


@pytest.mark.parametrize("spec_name,mp", [("mini.spec", 1), ("mini.spec", 2), ("mini_vocab_parallel.spec", 2),
                                          ("mini_swiglu.spec", 2), ("mini_hd64.spec", 1)])
def test_kv_cached_greedy_matches_window_recompute_and_oracle(spec_name, mp):
    batch, seq, P, n_new = 2, 16, 5, 20  # 5 + 20 > 16: the last steps run the sliding window
    model, spec = build(spec_name, mp, batch, seq)
    prompts = rng_ref.RngStream(3, "prompts").below(batch * P, spec.vocab_size).reshape(batch, P)
    got = model.generate(prompts, n_new)
    assert got.shape == (batch, n_new) and got.min() >= 0 and got.max() < spec.vocab_size

    # the reference's loop on the device: every step re-runs the window (n_new = 1 calls)
    ctx = prompts.copy()
    recompute = []
    for _ in range(n_new):
        nxt = model.generate(ctx[:, -seq:] if ctx.shape[1] > seq else ctx, 1)
        recompute.append(nxt[:, 0])
        ctx = np.concatenate([ctx, nxt], 1)
    recompute = np.stack(recompute, 1)
    assert np.array_equal(got, recompute), (got, recompute)

    decisive = oracle_check(model, spec, prompts, got, seq)
    assert decisive >= got.size // 2, decisive


def test_generate_rejects_bad_prompts():
    model, _ = build("mini.spec", 1, 2, 16)
    with pytest.raises(engine._lib.ShapeError, match="prompt length"):
        model.generate(np.zeros((2, 17), np.int32), 3)


@pytest.mark.parametrize("hd,mp,batch,extra", [(64, 2, 2, ""), (128, 1, 3, ""),
                                             (64, 2, 2, "role lm_head/kernel = fully_connected\n"),
                                             (128, 2, 2, "mlp = swiglu\nnorm = rmsnorm\n")])
def test_trimmed_prefill_matches_full_window(tmp_path, hd, mp, batch, extra):
    """A prompt much shorter than seq_len is prefilled over its first 128-row tile only, one
    sequence at a time (window_forward); the cached steps then cross that tile. Every generated
    token must be the argmax of the untrimmed full-window forward over the same context
    (teacher-forced, one device forward) except at near-ties."""
    path = tmp_path / "long.spec"
    path.write_text(f"vocab_size = 96\nn_layers = 2\nd_model = {2 * hd}\nn_heads = 2\nd_ff = {4 * hd}\n"
                    "max_seq_len = 384\n" + extra)
    spec = rules.read_model_spec(str(path))
    plan = rules.derive_plan(rules.transformer_param_shapes(spec), mp, spec.overrides)
    model = engine.Model(spec, plan, engine.Mesh(1, mp), batch, 384, inference=True)
    model.init_params(5, "model-init")
    head = "embed/tok/kernel" if spec.tie_embeddings else "lm_head/kernel"
    model.set_param(head, model.get_param(head) * 24.0)
    P, n_new = 40, 100
    prompts = rng_ref.RngStream(9, "prompts").below(batch * P, spec.vocab_size).reshape(batch, P)
    got = model.generate(prompts, n_new)
    ctx = np.concatenate([prompts, got], 1)
    win = np.zeros((batch, 384), np.int32)
    win[:, :P + n_new - 1] = ctx[:, :P + n_new - 1]
    model.stage_batch(win, win)
    logits = model.forward_logits()[:, P - 1:P + n_new - 1]
    srt = np.sort(logits, -1)
    margin = (srt[..., -1] - srt[..., -2]) / np.maximum(np.abs(srt[..., -1]), 1.0)
    pred = logits.argmax(-1)
    decisive = margin >= 0.02
    assert np.array_equal(pred[decisive], got[decisive])
    assert decisive.mean() > 0.5
