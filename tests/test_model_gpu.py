"""GPU executor parity: the tensor-parallel step through the C ABI vs the numpy oracle
(oracle/model_ref.py, itself pinned against the reference in test_oracle.py).

Tolerances (north_star): rel-L2 <= 1e-2 for bf16 compute. The oracle runs in f64 on the same
bf16-rounded GEMM weights the device uses (SURVEY.md §8c protocol point 2). attn/k/bias has an
analytically zero gradient; its check uses the reference audit metric max|a-b|/max(|b|,1)
instead of a relative norm (protocol point 3)."""
import os

import numpy as np
import pytest

from oracle import model_ref, rng_ref
from paper_2310_16355_b200 import engine, rules

pytestmark = pytest.mark.gpu

SPECS = os.path.join(os.path.dirname(__file__), "..", "oracle", "specs")


def spec_of(name):
    return rules.read_model_spec(os.path.join(SPECS, name))


def spec_dict(spec):
    return dict(vocab_size=spec.vocab_size, n_layers=spec.n_layers, d_model=spec.d_model,
                n_heads=spec.n_heads, d_ff=spec.d_ff, max_seq_len=spec.max_seq_len,
                tie_embeddings=spec.tie_embeddings, mlp=spec.mlp, norm=spec.norm)


def bf16_round(x):
    a = np.asarray(x, np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def oracle_params(spec, seed=42):
    p = rng_ref.init_transformer_params(spec_dict(spec), seed=seed, dtype=np.float32)
    return {k: v.astype(np.float64) for k, v in p.items()}


def gemm_rounded(params):
    """Weights as the GEMMs see them (bf16 shadow); 1-D params and embeddings stay fp32."""
    out = {}
    for k, v in params.items():
        if v.ndim == 2 and not k.startswith("embed/"):
            out[k] = bf16_round(v)
        else:
            out[k] = v.copy()
    return out


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-6 * np.sqrt(b.size)))


def max_rel(a, b):
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1.0)))


def make(spec, dp, mp, batch, seq):
    shapes = rules.transformer_param_shapes(spec)
    plan = rules.derive_plan(shapes, mp, spec.overrides)
    mesh = engine.Mesh(dp, mp)
    model = engine.Model(spec, plan, mesh, batch, seq)
    return model, mesh, plan


# attention-score path: q/k kernels, q bias, and the ln1 scale whose gradient is the sum of the
# q/k/v input gradients (it inherits the same cancellation)
SCORE_PATH = ("attn/q/kernel", "attn/k/kernel", "attn/q/bias", "ln1/scale")


def check_grads(model, spec, want, tol=1e-2):
    """rel-L2 <= tol for every gradient, except the attention-score path (q/k kernels, q bias):
    at random init the softmax is nearly uniform, dS = P*(dP - delta) cancels, and bf16
    rounding alone moves these by ~1% (SURVEY.md §8c probe6: 9.4e-3 from weight rounding
    only) — they get 2*tol and are reported as the worst case."""
    worst = ("", 0.0)
    for name in want:
        got = model.get_grad(name).astype(np.float64)
        if name.endswith("attn/k/bias"):
            assert max_rel(got, want[name]) < 1e-3, name
            continue
        r = rel_l2(got, want[name])
        if r > worst[1]:
            worst = (name, r)
        t = 2 * tol if name.endswith(SCORE_PATH) else tol
        assert r < t, (name, r)
    return worst


@pytest.mark.parametrize("spec_name,dp,mp,batch,seq", [
    ("mini.spec", 1, 1, 2, 16),
    ("mini.spec", 1, 2, 2, 16),
    ("mini.spec", 1, 4, 2, 16),
    ("mini.spec", 2, 2, 2, 16),
    ("tiny.spec", 1, 1, 4, 128),
    ("tiny.spec", 1, 2, 4, 128),
    ("tiny_vocab_parallel.spec", 1, 2, 4, 128),
    ("tiny_vocab_parallel.spec", 2, 2, 2, 128),
    ("mini_vocab_parallel.spec", 1, 4, 2, 16),
    # SwiGLU MLP + RMSNorm extension: fused gate|up GEMM, SwiGLU-bwd epilogue
    ("mini_swiglu.spec", 1, 1, 2, 16),
    ("mini_swiglu.spec", 1, 2, 2, 16),
    ("mini_swiglu.spec", 2, 2, 2, 16),
    ("tiny_swiglu.spec", 1, 1, 4, 128),
    ("tiny_swiglu.spec", 1, 2, 4, 128),
])
def test_forward_backward_matches_oracle(spec_name, dp, mp, batch, seq):
    spec = spec_of(spec_name)
    model, mesh, _ = make(spec, dp, mp, batch, seq)
    model.init_params(42, "model-init")
    # device init == reference init (counter-based stream, model.hpp:49-70)
    ref = oracle_params(spec)
    for name, val in ref.items():
        got = model.get_param(name)
        mism = np.count_nonzero(got != val.astype(np.float32))
        assert mism <= max(1, val.size // 100000), (name, mism)
    tokens, targets, weights = rng_ref.audit_batch(42, 0, dp * batch, seq, spec.vocab_size)
    model.stage_batch(tokens, targets, weights)
    model.forward_backward()
    model.dp_sync()
    loss = model.loss()
    # oracle: audit-style average over dp slices on the bf16-rounded weights, (a) f64
    # activations (the north-star protocol) and (b) bf16-stored activations at the points
    # where the device stores bf16 (isolates kernel arithmetic from storage rounding)
    sd = spec_dict(spec)
    pr = gemm_rounded(ref)
    # f64 activations: 2e-2 for the small-width cases and for SwiGLU, whose h = silu(g)*u and its
    # derivatives multiply two bf16-stored pre-activations (~1% from storage alone); the
    # bf16_acts pass rounds where the device stores (1e-2; 1.5e-2 for SwiGLU, where the attention-score
    # noise of the reference family reaches the residual stream through five more bf16 stores)
    f64_tol = 1e-2 if spec.d_model >= 256 and spec.mlp != "swiglu" else 2e-2
    bf_tol = 1.5e-2 if spec.mlp == "swiglu" else 1e-2
    for bf16_acts, tol in ((False, f64_tol), (True, bf_tol)):
        want_loss, acc = 0.0, None
        for r in range(dp):
            sl = slice(r * batch, (r + 1) * batch)
            l, g, _ = model_ref.forward_backward(pr, sd, tokens[sl], targets[sl], weights[sl],
                                                 bf16_acts=bf16_acts)
            want_loss += l / dp
            acc = {k: v / dp for k, v in g.items()} if acc is None else {k: acc[k] + g[k] / dp for k in acc}
        assert abs(loss - want_loss) / abs(want_loss) < 2e-3, (loss, want_loss)
        check_grads(model, spec, acc, tol)


@pytest.mark.parametrize("ar_bf16", [1, 0])
def test_tensor_parallel_invariance(ar_bf16, monkeypatch):
    """The sharded step equals the unsharded one (what audit_equivalence checks, audit.hpp:78),
    with the row-parallel all-reduce payloads in fp32 (the default) and in bf16 (SW_AR_BF16=1)."""
    monkeypatch.setenv("SW_AR_BF16", str(ar_bf16))
    spec = spec_of("tiny.spec")
    tokens, targets, weights = rng_ref.audit_batch(42, 0, 4, 128, spec.vocab_size)
    res = {}
    for mp in (1, 2, 4):
        model, mesh, _ = make(spec, 1, mp, 4, 128)
        model.init_params(42, "model-init")
        model.stage_batch(tokens, targets, weights)
        model.forward_backward()
        res[mp] = (model.loss(), {n: model.get_grad(n) for n in ("block_0/attn/q/kernel",
                                                                  "block_1/mlp/fc2/kernel",
                                                                  "block_0/mlp/fc1/bias",
                                                                  "embed/tok/kernel")})
        if mp == 2:
            csv = mesh.comm_report().splitlines()
            ar, ag = csv[1].split(","), csv[2].split(",")
            # fwd: 2 AR/layer; bwd: 2 AR/layer (fused QKV dx, fc1 dx), each pipelined over 4 row
            # chunks (M = 512 tokens); 4 bias-grad AG/layer
            chunks = 4
            assert int(ar[1]) == 4 * spec.n_layers * chunks and int(ag[1]) == 4 * spec.n_layers
            assert int(ar[2]) == 4 * spec.n_layers * 512 * spec.d_model * (2 if ar_bf16 else 4)
    for mp in (2, 4):
        assert abs(res[mp][0] - res[1][0]) / res[1][0] < 2e-4
        for n in res[1][1]:
            t = 1e-2 if (n.endswith(SCORE_PATH) or n.startswith("embed/")) else 5e-3
            assert rel_l2(res[mp][1][n].astype(np.float64), res[1][1][n].astype(np.float64)) < t, (mp, n)


def test_adamw_step_matches_formula():
    """adamw_step (train_state.hpp:183-220) on the device == the numpy formula on the same
    grads; sharded == unsharded (test_spmd.cpp:520-565)."""
    spec = spec_of("mini.spec")
    tokens, targets, weights = rng_ref.audit_batch(42, 0, 2, 16, spec.vocab_size)
    cfg = engine.AdamWConfig(lr=1e-2, weight_decay=0.01)
    finals = {}
    for mp in (1, 2):
        model, mesh, _ = make(spec, 1, mp, 2, 16)
        model.init_params(42, "model-init")
        p0 = {n: model.get_param(n) for n in model.shapes}
        model.stage_batch(tokens, targets, weights)
        model.forward_backward()
        g = {n: model.get_grad(n) for n in model.shapes}
        model.adamw_step(cfg)
        for n in model.shapes:
            m = np.zeros_like(p0[n])
            v = np.zeros_like(p0[n])
            p = {n: p0[n].copy()}
            model_ref.adamw_step(p, {n: m}, {n: v}, {n: g[n]}, 0, lr=cfg.lr, wd=cfg.weight_decay,
                                 dtype=np.float32)
            got = model.get_param(n)
            np.testing.assert_allclose(got, p[n], rtol=2e-6, atol=2e-7, err_msg=n)
        finals[mp] = {n: model.get_param(n) for n in model.shapes}
    for n in finals[1]:
        if not n.endswith("attn/k/bias"):
            assert max_rel(finals[2][n], finals[1][n]) < 2 * cfg.lr, n


def test_train_trajectory_tracks_oracle():
    """Three optimizer steps (Trainer::fit inner loop, pipeline.hpp:388-449) track the f64
    reference trajectory recorded in tests/golden (losses within 1e-2 relative)."""
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "mini_f64_dp1_mp2.npz"))
    spec = spec_of("mini.spec")
    model, mesh, _ = make(spec, 1, 2, 2, 16)
    model.init_params(42, "model-init")
    cfg = engine.AdamWConfig(lr=1e-2, weight_decay=0.01)
    for step in range(3):
        tokens, targets, weights = rng_ref.audit_batch(42, step, 2, 16, spec.vocab_size)
        model.stage_batch(tokens, targets, weights)
        model.train_step(cfg)
        want = float(z[f"spmd_loss/{step}"])
        assert abs(model.loss() - want) / want < 1e-2, (step, model.loss(), want)


def test_forward_logits_match_reference_golden():
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "mini_f64_dp1_mp2.npz"))
    spec = spec_of("mini.spec")
    model, mesh, _ = make(spec, 1, 2, 2, 16)
    model.init_params(42, "model-init")
    tokens, targets, weights = rng_ref.audit_batch(42, 0, 2, 16, spec.vocab_size)
    model.stage_batch(tokens, targets, weights)
    logits = model.forward_logits()
    assert rel_l2(logits.astype(np.float64), z["logits0"]) < 1e-2


def test_nonfinite_gradient_raises():
    spec = spec_of("mini.spec")
    model, mesh, _ = make(spec, 1, 1, 2, 16)
    model.init_params(42, "model-init")
    bad = model.get_param("block_0/ln1/scale")
    bad[3] = np.nan
    model.set_param("block_0/ln1/scale", bad)
    tokens, targets, weights = rng_ref.audit_batch(42, 0, 2, 16, spec.vocab_size)
    model.stage_batch(tokens, targets, weights)
    model.forward_backward()
    with pytest.raises(engine._lib.NonFiniteError, match="non-finite gradient for parameter"):
        model.adamw_step(engine.AdamWConfig())


def test_vocab_parallel_head_plan_and_comm():
    """With `role lm_head/kernel = fully_connected` the head is split:0; the step
    exchanges (max, sumexp) stats + target logits instead of all-gathering the logits, and
    all-reduces d(final_h) once."""
    spec = spec_of("tiny_vocab_parallel.spec")
    model, mesh, plan = make(spec, 1, 2, 4, 128)
    assert plan.at("lm_head/kernel") == "split:0"
    model.init_params(42, "model-init")
    tokens, targets, weights = rng_ref.audit_batch(42, 0, 4, 128, spec.vocab_size)
    model.stage_batch(tokens, targets, weights)
    logits = model.forward_logits()
    ref = oracle_params(spec)
    _, _, want = model_ref.forward_backward(gemm_rounded(ref), spec_dict(spec), tokens, targets, weights,
                                            need_grads=False)
    assert rel_l2(logits.astype(np.float64), want) < 1e-2
    mesh.reset_comm_report()
    model.forward_backward()
    csv = mesh.comm_report().splitlines()
    ar, ag = csv[1].split(","), csv[2].split(",")
    L = spec.n_layers
    chunks = 4  # row-parallel all-reduces are pipelined over 4 row chunks at M = 512
    assert int(ar[1]) == (4 * L + 1) * chunks + 1  # + d(final_h) (chunked) + target-logit AR
    assert int(ag[1]) == 4 * L + 1  # + the CE stats all-gather


@pytest.mark.parametrize("spec_name,mp", [("mini.spec", 1), ("mini.spec", 2), ("tiny_vocab_parallel.spec", 2),
                                          ("mini_swiglu.spec", 2)])
def test_fused_optimizer_matches_unfused(spec_name, mp):
    """train_step with dp == 1 applies AdamW inside the wgrad GEMM epilogues (the gradient of a
    weight matrix never reaches HBM). After one step the parameters must equal
    forward_backward + dp_sync + adamw_step (train_state.hpp:170-226 on the stored gradient).

    Both arms carry atomics-order noise (embedding scatter, dQ reduce-add); Adam's first step is
    ~lr*sign(g), so an element whose true gradient is ~0 may flip: at most 1e-3 of the elements
    (or 2 of a small parameter) may differ, and by no more than 2*lr. Three more steps must then
    track in loss (2e-3: the flipped elements move at lr = 1e-2)."""
    spec = spec_of(spec_name)
    seq = 16 if spec_name.startswith("mini") else 128
    fused, _, _ = make(spec, 1, mp, 2, seq)
    plain, _, _ = make(spec, 1, mp, 2, seq)
    for m in (fused, plain):
        m.init_params(42, "model-init")
    cfg = engine.AdamWConfig(lr=1e-2, weight_decay=0.01)
    for step in range(4):
        tokens, targets, weights = rng_ref.audit_batch(42, step, 2, seq, spec.vocab_size)
        fused.stage_batch(tokens, targets, weights)
        fused.train_step(cfg)
        plain.stage_batch(tokens, targets, weights)
        plain.forward_backward()
        plain.dp_sync()
        plain.adamw_step(cfg)
        # the flipped near-zero-gradient elements (lr = 1e-2 each) move later losses a little
        assert abs(fused.loss() - plain.loss()) <= (1e-4 if step == 0 else 2e-3) * abs(plain.loss()), step
        if step == 0:
            for n in plain.shapes:
                a, b = fused.get_param(n), plain.get_param(n)
                d = np.abs(a - b)
                off = d > 1e-6 + 1e-5 * np.abs(b)
                # a small parameter (a 32-wide bias) has too few elements for a fraction: 2 may flip
                assert off.sum() <= max(2, 1e-3 * off.size) or n.endswith("attn/k/bias"), (n, int(off.sum()))
                assert d.max() <= 2 * cfg.lr * (1 + 1e-3) + 1e-6, (n, float(d.max()))


def test_fused_optimizer_nonfinite_raises():
    spec = spec_of("mini.spec")
    model, mesh, _ = make(spec, 1, 1, 2, 16)
    model.init_params(42, "model-init")
    bad = model.get_param("block_0/ln1/scale")
    bad[3] = np.nan
    model.set_param("block_0/ln1/scale", bad)
    tokens, targets, weights = rng_ref.audit_batch(42, 0, 2, 16, spec.vocab_size)
    model.stage_batch(tokens, targets, weights)
    state = {n: [model.get_param(n), *model.get_adam(n)] for n in model.shapes}
    with pytest.raises(engine._lib.NonFiniteError, match="non-finite gradient for parameter"):
        model.train_step(engine.AdamWConfig())
    # the non-finite loss gated every fused update: nothing moved (train_state.hpp:207-210)
    for n, (p, m, v) in state.items():
        assert np.array_equal(model.get_param(n), p, equal_nan=True), n
        m2, v2 = model.get_adam(n)
        assert np.array_equal(m2, m) and np.array_equal(v2, v), n
    # the model is not poisoned: repair the parameter and the fused step goes ahead
    good = model.get_param("block_0/ln1/scale")
    good[3] = 1.0
    model.set_param("block_0/ln1/scale", good)
    model.stage_batch(tokens, targets, weights)
    model.train_step(engine.AdamWConfig())
    assert np.isfinite(model.loss())
    assert not np.array_equal(model.get_param("block_0/mlp/fc1/kernel"), state["block_0/mlp/fc1/kernel"][0])


def test_replicated_param_grads_are_deterministic():
    """Embedding and LayerNorm gradients (replicated on every tensor-parallel rank, like the
    reference's) come from fixed-order reductions (sorted token runs, per-CTA LayerNorm partials
    summed in CTA order), so two backward passes over the same batch agree bit for bit -- which
    is what keeps the replicas identical across ranks."""
    spec = spec_of("tiny.spec")
    model, mesh, _ = make(spec, 1, 2, 4, 128)
    model.init_params(42, "model-init")
    tokens, targets, weights = rng_ref.audit_batch(42, 0, 4, 128, spec.vocab_size)
    # repeated tokens exercise multi-position runs in the embedding backward
    tokens[:, ::3] = tokens[0, 0]
    model.stage_batch(tokens, targets, weights)
    names = [n for n in model.shapes if n.startswith("embed/") or "/ln" in n or n.startswith("final_ln/")]
    runs = []
    for _ in range(2):
        model.forward_backward()
        runs.append({n: model.get_grad(n).view(np.uint32).copy() for n in names})
    for n in names:
        assert np.array_equal(runs[0][n], runs[1][n]), n


@pytest.mark.parametrize("spec_name,ar_bf16", [("llama7b_vocab_parallel.spec", "0"), ("llama7b_swiglu.spec", "0"),
                                               ("llama7b_vocab_parallel.spec", "1")])
def test_llama7b_width_tp8_matches_tp1(spec_name, ar_bf16, monkeypatch):
    """The shapes the 8-GPU scaling run hits (LLaMA-7B width at mp = 8: 4 heads, d/t = 512,
    d_ff/t = 1376 (GEMM N and K tails), vocab shard 4000), depth 2 and 512 tokens, on the
    emulated mesh: the mp = 8 step equals the unsharded one, with fp32 or bf16 (what bench.py uses
    at N > 1) all-reduce payloads."""
    monkeypatch.setenv("SW_AR_BF16", ar_bf16)
    text = open(os.path.join(SPECS, spec_name)).read().replace("n_layers = 32", "n_layers = 2")
    spec = rules.parse_model_spec(text)
    rng = np.random.default_rng(3)
    tokens = rng.integers(0, spec.vocab_size, (2, 256), dtype=np.int32)
    targets = rng.integers(0, spec.vocab_size, (2, 256), dtype=np.int32)
    res = {}
    for mp in (1, 8):
        model, mesh, plan = make(spec, 1, mp, 2, 256)
        model.init_params(42, "model-init")
        model.stage_batch(tokens, targets, None)
        model.forward_backward()
        res[mp] = (model.loss(), {n: model.get_grad(n) for n in ("block_0/attn/q/kernel", "block_1/mlp/fc2/kernel",
                                                                 "block_1/attn/o/kernel", "lm_head/kernel")})
        model.close()
        mesh.close()
    assert abs(res[8][0] - res[1][0]) / res[1][0] < 2e-4, (res[8][0], res[1][0])
    for n in res[1][1]:
        assert rel_l2(res[8][1][n].astype(np.float64), res[1][1][n].astype(np.float64)) < 1e-2, n


def test_gptj_width_dp2_tp4_matches_single_device():
    """BASELINE cfg3's mesh (2-way data x 4-way tensor) at GPT-J-6B width (head dim 256: the
    CUDA-core attention path), depth 2 and 4 x 128 tokens, emulated: the dp x mp step with its
    dp gradient all-reduce and sharded AdamW equals the single-device step."""
    text = open(os.path.join(SPECS, "gptj6b.spec")).read()
    text = "\n".join("n_layers = 2" if ln.startswith("n_layers") else ln for ln in text.splitlines()) + "\n"
    spec = rules.parse_model_spec(text)
    rng = np.random.default_rng(5)
    tokens = rng.integers(0, spec.vocab_size, (4, 128), dtype=np.int32)
    targets = rng.integers(0, spec.vocab_size, (4, 128), dtype=np.int32)
    names = ("block_0/attn/q/kernel", "block_1/mlp/fc2/kernel", "block_0/attn/o/bias", "lm_head/kernel")
    res = {}
    cfg = engine.AdamWConfig(lr=1e-3, weight_decay=0.01)
    for dp, mp in ((1, 1), (2, 4)):
        model, mesh, plan = make(spec, dp, mp, 4 // dp, 128)
        model.init_params(42, "model-init")
        model.stage_batch(tokens, targets, None)
        model.forward_backward()
        model.dp_sync()
        grads = {n: model.get_grad(n) for n in names}
        model.adamw_step(cfg)
        res[(dp, mp)] = (model.loss(), grads, {n: model.get_param(n) for n in names})
        model.close()
        mesh.close()
    a, b = res[(1, 1)], res[(2, 4)]
    assert abs(b[0] - a[0]) / a[0] < 2e-4, (b[0], a[0])
    for n in names:
        assert rel_l2(b[1][n].astype(np.float64), a[1][n].astype(np.float64)) < 1e-2, n
        # one AdamW step (~lr * sign(g)) from identical weights
        assert np.max(np.abs(b[2][n] - a[2][n])) <= 2.5e-3, n


@pytest.mark.parametrize("mp", [1, 2])
def test_fused_bias_colsums_match_separate_pass(mp, monkeypatch):
    """The fc1 bias gradient summed in the GeLU-backward GEMM epilogue and the q|k|v bias
    gradients summed in the attention backward / dQ conversion (per-32-row partials, fixed-order
    reduction) equal the separate column-sum passes over dpre / dqkv (SW_FUSE_COLSUM=0)."""
    text = open(os.path.join(SPECS, "llama7b_vocab_parallel.spec")).read().replace("n_layers = 32", "n_layers = 1")
    spec = rules.parse_model_spec(text)
    rng = np.random.default_rng(11)
    tokens = rng.integers(0, spec.vocab_size, (2, 256), dtype=np.int32)
    targets = rng.integers(0, spec.vocab_size, (2, 256), dtype=np.int32)
    names = ("block_0/attn/q/bias", "block_0/attn/k/bias", "block_0/attn/v/bias", "block_0/mlp/fc1/bias")
    res = {}
    for fuse in ("0", "1"):
        monkeypatch.setenv("SW_FUSE_COLSUM", fuse)
        model, mesh, plan = make(spec, 1, mp, 2, 256)
        model.init_params(42, "model-init")
        model.stage_batch(tokens, targets, None)
        model.forward_backward()
        res[fuse] = {n: model.get_grad(n).astype(np.float64) for n in names}
        model.close()
        mesh.close()
    for n in names:
        assert np.abs(res["0"][n]).max() > 0, n
        assert rel_l2(res["1"][n], res["0"][n]) < 1e-4, n


@pytest.mark.parametrize("mp", [1, 2])
def test_step_bitwise_reproducible(mp, monkeypatch):
    """With head_dim 128 causal attention (dQ summed in key order by the query-block kernel),
    GEMMs that split K into at most two slices (two adds onto zero commute), and fixed-order
    bias / LayerNorm / embedding reductions, the training step is bitwise reproducible: two
    runs of forward_backward + a fused train_step from the same state, with the weight
    gradients on the side stream or on the main stream, give identical gradients, parameters
    and losses (2 layers at d = 1024, 2 x 1024 tokens: the q|k|v weight gradient splits K)."""
    text = open(os.path.join(SPECS, "llama7b.spec")).read()
    for a, b in (("n_layers = 32", "n_layers = 2"), ("d_model = 4096", "d_model = 1024"),
                 ("n_heads = 32", "n_heads = 8"), ("d_ff = 11008", "d_ff = 2752"), ("vocab_size = 32000", "vocab_size = 4096")):
        text = text.replace(a, b)
    spec = rules.parse_model_spec(text)
    rng = np.random.default_rng(5)
    tokens = rng.integers(0, spec.vocab_size, (2, 1024), dtype=np.int32)
    targets = rng.integers(0, spec.vocab_size, (2, 1024), dtype=np.int32)
    names = [n for n, _ in rules.transformer_param_shapes(spec)]
    cfg = engine.AdamWConfig(lr=1e-3, weight_decay=0.01)
    runs = []
    for side in ("1", "1", "0"):
        monkeypatch.setenv("SW_WGRAD_STREAM", side)
        model, mesh, _ = make(spec, 1, mp, 2, 1024)
        model.init_params(42, "model-init")
        model.stage_batch(tokens, targets, None)
        model.forward_backward()
        grads = {n: model.get_grad(n) for n in names}
        loss0 = model.loss()
        model.stage_batch(tokens, targets, None)
        model.train_step(cfg)
        model.stage_batch(tokens, targets, None)
        model.train_step(cfg)
        runs.append((grads, {n: model.get_param(n) for n in names}, loss0, model.loss()))
        model.close()
        mesh.close()
    for other in runs[1:]:
        assert other[2] == runs[0][2] and other[3] == runs[0][3]
        for n in names:
            assert np.array_equal(other[0][n], runs[0][0][n]), n
            assert np.array_equal(other[1][n], runs[0][1][n]), n


@pytest.mark.parametrize("mp", [1, 2])
def test_side_stream_wgrads_match_single_stream(mp, monkeypatch):
    """The weight-gradient GEMMs on the side stream (default) against the single-stream schedule
    (SW_WGRAD_STREAM=0) at a size where the wgrads overlap the following dgrad / attention
    kernels (2 layers, M = 2048 tokens): forward_backward gradients and the parameters after a
    fused train_step. A missing join before gb / dpre / dqkv is rewritten would read a later
    layer's values (O(1) relative error). The attention backward's dQ reduce-add (and split-K
    weight gradients' slice order) are not deterministic, so the bound is their rounding noise:
    every gradient within 1e-3 rel-L2, and after one AdamW step (~lr * sign(g): an element whose gradient is at the
    noise level may flip sign) at most 1% of a weight's elements differ, none by more than 2*lr."""
    text = open(os.path.join(SPECS, "llama7b.spec")).read()
    for a, b in (("n_layers = 32", "n_layers = 2"), ("d_model = 4096", "d_model = 1024"),
                 ("n_heads = 32", "n_heads = 8"), ("d_ff = 11008", "d_ff = 2752"), ("vocab_size = 32000", "vocab_size = 4096")):
        assert a in text
        text = text.replace(a, b)
    spec = rules.parse_model_spec(text)
    rng = np.random.default_rng(3)
    tokens = rng.integers(0, spec.vocab_size, (2, 1024), dtype=np.int32)
    targets = rng.integers(0, spec.vocab_size, (2, 1024), dtype=np.int32)
    names = [n for n, _ in rules.transformer_param_shapes(spec)]
    cfg = engine.AdamWConfig(lr=1e-3, weight_decay=0.01)
    res = {}
    for side in ("0", "1"):
        monkeypatch.setenv("SW_WGRAD_STREAM", side)
        model, mesh, _ = make(spec, 1, mp, 2, 1024)
        model.init_params(42, "model-init")
        model.stage_batch(tokens, targets, None)
        model.forward_backward()
        grads = {n: model.get_grad(n).astype(np.float64) for n in names}
        model.stage_batch(tokens, targets, None)
        model.train_step(cfg)
        params = {n: model.get_param(n) for n in names}
        res[side] = (grads, params, model.loss())
        model.close()
        mesh.close()
    for n in names:
        if n.endswith("attn/k/bias"):  # analytically zero gradient
            assert max_rel(res["1"][0][n], res["0"][0][n]) < 1e-6, n
        else:
            # the dQ reduce-add noise reaches the embedding through every layer's residual
            # gradient (seen up to 2.6e-4 once in ~20 runs); a missed join is O(1)
            assert rel_l2(res["1"][0][n], res["0"][0][n]) < 1e-3, n
        a, b = res["1"][1][n], res["0"][1][n]
        d = np.abs(a - b)
        assert (d > 1e-6 + 1e-5 * np.abs(b)).mean() <= 1e-2 or n.endswith("attn/k/bias"), n
        assert d.max() <= 2 * cfg.lr * (1 + 1e-3) + 1e-6, (n, float(d.max()))
    assert abs(res["0"][2] - res["1"][2]) <= 1e-6 * abs(res["0"][2])


@pytest.mark.parametrize("spec_name,mp", [("mini.spec", 2), ("mini_swiglu.spec", 1)])
def test_dp_allreduce_overlapped_with_backward(spec_name, mp):
    """train_step with dp = 2 all-reduces each layer's GEMM-weight gradients on a side stream as
    soon as the layer's weight-gradient GEMMs are done (emulated mesh: after the last replica's),
    then the rest in dp_sync; forward_backward + dp_sync + adamw_step reduces the whole flat
    buffer after the backward. Same update, up to the atomics-order noise every backward has;
    AdamW turns that noise into full-size updates of either sign for near-zero gradients (whole
    rows of the tied embedding for tokens absent from the batch), so the Adam first moments,
    linear in the gradients, are what is compared, with the losses."""
    spec = spec_of(spec_name)
    seq = 16
    cfg = engine.AdamWConfig(lr=1e-2, weight_decay=0.01)
    out = {}
    for overlapped in (True, False):
        model, _, _ = make(spec, 2, mp, 2, seq)
        model.init_params(42, "model-init")
        losses = []
        for step in range(3):
            tokens, targets, weights = rng_ref.audit_batch(42, step, 4, seq, spec.vocab_size)
            model.stage_batch(tokens, targets, weights)
            if overlapped:
                model.train_step(cfg)
            else:
                model.forward_backward()
                model.dp_sync()
                model.adamw_step(cfg)
            losses.append(model.loss())
        out[overlapped] = (losses, {n: model.get_adam(n)[0] for n in model.shapes},
                           {n: model.get_param(n) for n in model.shapes})
    assert abs(out[True][0][0] - out[False][0][0]) <= 1e-4 * abs(out[False][0][0])
    for a, b in zip(out[True][0][1:], out[False][0][1:]):
        assert abs(a - b) <= 2e-3 * abs(b)
    for n in out[True][1]:
        if n.endswith("attn/k/bias"):
            continue
        m_a, m_b = out[True][1][n].astype(np.float64), out[False][1][n].astype(np.float64)
        assert rel_l2(m_a, m_b) < 2e-2, (n, rel_l2(m_a, m_b))
        assert np.abs(out[True][2][n] - out[False][2][n]).max() <= 3 * 2 * cfg.lr + 1e-6, n

def test_fused_optimizer_split_k_weights(tmp_path):
    """Weights whose gradient GEMM has too few output tiles for the GPU (tensor-parallel shards)
    take split-K (K slices reduce-added into the gradient) and a gated AdamW over the GEMM's
    whole [M, N] range (the fused q|k|v / gate|up weights span several slots) instead of the
    optimizer epilogue: train_step must equal forward_backward + adamw_step after one step (the
    noise bounds of test_fused_optimizer_matches_unfused) and track it in loss after that."""
    path = tmp_path / "splitk.spec"
    path.write_text("vocab_size = 1024\nn_layers = 2\nd_model = 512\nn_heads = 4\nd_ff = 1376\n"
                    "max_seq_len = 512\n")
    spec = rules.read_model_spec(str(path))
    seq, batch, mp = 512, 4, 2  # 2048 tokens: 32 k-blocks per weight gradient, a handful of tiles
    fused, _, _ = make(spec, 1, mp, batch, seq)
    plain, _, _ = make(spec, 1, mp, batch, seq)
    for m in (fused, plain):
        m.init_params(42, "model-init")
    cfg = engine.AdamWConfig(lr=1e-3, weight_decay=0.01)
    for step in range(3):
        tokens, targets, weights = rng_ref.audit_batch(42, step, batch, seq, spec.vocab_size)
        fused.stage_batch(tokens, targets, weights)
        fused.train_step(cfg)
        plain.stage_batch(tokens, targets, weights)
        plain.forward_backward()
        plain.adamw_step(cfg)
        assert abs(fused.loss() - plain.loss()) <= (1e-4 if step == 0 else 2e-3) * abs(plain.loss()), step
        if step == 0:
            for n in plain.shapes:
                a, b = fused.get_param(n), plain.get_param(n)
                d = np.abs(a - b)
                off = d > 1e-6 + 1e-5 * np.abs(b)
                assert off.sum() <= max(2, 1e-3 * off.size) or n.endswith("attn/k/bias"), (n, int(off.sum()))
                assert d.max() <= 2 * cfg.lr * (1 + 1e-3) + 1e-6, (n, float(d.max()))
