"""Pins the numpy oracle (oracle/) against the reference's own outputs (tests/golden/*.npz,
produced by the unmodified reference via oracle/_ref/sw_ref_driver; see make_golden.py)."""
import json
import os

import numpy as np
import pytest

from oracle import model_ref, rng_ref

G = os.path.join(os.path.dirname(__file__), "golden")
SPECS = os.path.join(os.path.dirname(__file__), "..", "oracle", "specs")


def load(name):
    z = np.load(os.path.join(G, name + ".npz"))
    meta = json.loads(str(z["__meta__"]))
    return z, meta


def spec_dict(fn):
    out = {"tie_embeddings": False}
    for ln in open(os.path.join(SPECS, fn)):
        ln = ln.split("#")[0].strip()
        if "=" in ln and not ln.startswith("role"):
            k, v = (x.strip() for x in ln.split("="))
            out[k] = (v in ("true", "yes", "1")) if k == "tie_embeddings" else int(v)
    return out


def max_rel(a, b):
    """The reference audit metric (audit.hpp:37-51): max |a-b| / max(|b|, 1)."""
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1.0)))


def test_rng_known_answers():
    # splitmix64 of 0 (first output of the canonical generator seeded with 0)
    assert rng_ref.mix_int(0) == 0xE220A8397B1DCDAF
    assert rng_ref.fnv1a("") == 0xCBF29CE484222325
    r = rng_ref.RngStream(7, "x")
    a = r.draws(5)
    r2 = rng_ref.RngStream(7, "x")
    assert [int(r2.draws(1)[0]) for _ in range(5)] == [int(x) for x in a]


def test_init_matches_reference_bit_exact():
    z, meta = load("mini_f64_dp1_mp2")
    spec = spec_dict(meta["spec"])
    for exact in (True, False):
        params = rng_ref.init_transformer_params(spec, seed=meta["seed"], exact=exact)
        for name, val in params.items():
            ref = z["init/" + name]
            if exact:
                assert np.array_equal(val, ref), name
            else:
                assert max_rel(val, ref) < 1e-15, name


def test_init_tiny_checksums():
    z, meta = load("tiny_f64_dp1_mp2")
    spec = spec_dict(meta["spec"])
    params = rng_ref.init_transformer_params(spec, seed=meta["seed"])
    for name, val in params.items():
        np.testing.assert_allclose(val.reshape(-1)[:16], z["head/init/" + name], rtol=1e-14, atol=0)
        np.testing.assert_allclose(val.sum(), z["sum/init/" + name], rtol=1e-10, atol=1e-12)


@pytest.mark.parametrize("case", ["mini_f64_dp1_mp2", "mini_f64_dp2_mp2", "tiny_f64_dp1_mp2"])
def test_trajectory_matches_reference(case):
    z, meta = load(case)
    spec = spec_dict(meta["spec"])
    params = rng_ref.init_transformer_params(spec, seed=meta["seed"])
    gb, seq = meta["global_batch"], meta["seq"]
    batch = lambda s: rng_ref.audit_batch(meta["seed"], s, gb, seq, spec["vocab_size"])  # noqa: E731
    losses, g0, final = model_ref.audit_trajectory(params, spec, batch, meta["dp"], meta["steps"],
                                                   meta["lr"], meta["weight_decay"])
    full = "ref_grad0/" + next(iter(params)) in z.files
    for s, l in enumerate(losses):
        assert abs(l - float(z[f"ref_loss/{s}"])) < 1e-12
        assert abs(l - float(z[f"spmd_loss/{s}"])) < 1e-12
    for name in params:
        if full:
            assert max_rel(g0[name], z["ref_grad0/" + name]) < 1e-12, name
            assert max_rel(g0[name], z["spmd_grad0/" + name]) < 1e-12, name
            assert max_rel(final[name], z["ref_final/" + name]) < 1e-10, name  # cli.cpp:234 f64 tolerance
            assert max_rel(final[name], z["spmd_final/" + name]) < 1e-10, name
        else:
            np.testing.assert_allclose(g0[name].sum(), z["sum/ref_grad0/" + name], rtol=1e-8, atol=1e-12)
            np.testing.assert_allclose((g0[name] ** 2).sum(), z["sumsq/ref_grad0/" + name], rtol=1e-9, atol=1e-20)
            np.testing.assert_allclose(final[name].reshape(-1)[:16], z["head/spmd_final/" + name],
                                       rtol=1e-10, atol=1e-10)  # attn/k/bias carries AdamW-amplified noise


def test_logits_match_reference():
    z, meta = load("mini_f64_dp1_mp2")
    spec = spec_dict(meta["spec"])
    params = rng_ref.init_transformer_params(spec, seed=meta["seed"])
    tokens, targets, weights = rng_ref.audit_batch(meta["seed"], 0, meta["global_batch"], meta["seq"],
                                                   spec["vocab_size"])
    _, _, logits = model_ref.forward_backward(params, spec, tokens, targets, weights, need_grads=False)
    assert max_rel(logits, z["logits0"]) < 1e-12


def test_comm_report_matches_analytic():
    """cfg1 mp=2 fwd+bwd: 12 AR + 8 AG per step, payload = 6L(B*T*d*8) + L(3d+d_ff)*8 (f64)."""
    z, meta = load("tiny_f64_dp1_mp2")
    csv = str(z["__comm_csv__"]).splitlines()
    ar = csv[1].split(",")
    ag = csv[2].split(",")
    L, B, T, d, dff = 2, 4, 128, 256, 1024
    assert int(ar[1]) == 12 and int(ag[1]) == 8
    assert int(ar[2]) + int(ag[2]) == 6 * L * B * T * d * 8 + L * (3 * d + dff) * 8


def test_extension_ops_equal_reference_op_compositions():
    """RMSNorm and SiLU are exact compositions of reference ops, so the closed forms
    the oracle uses are pinned to the reference's layer_norm / softmax: RMSNorm(x)*g ==
    slice(layer_norm(concat(x, -x)), d)*g and SiLU(x) == x * softmax([x, 0])[0]."""
    rng = np.random.default_rng(3)
    x = rng.standard_normal((5, 7, 48)) * 2.0
    g = rng.standard_normal(48)
    y, _, _ = model_ref.rms_norm(x, g)
    cat = np.concatenate([x, -x], -1)
    ln, _, _ = model_ref.layer_norm(cat, np.ones(96), np.zeros(96))
    assert np.max(np.abs(y - ln[..., :48] * g)) < 1e-12
    z = rng.standard_normal(1000) * 6.0
    two = np.stack([z, np.zeros_like(z)], -1)
    sm = model_ref._softmax(two)[..., 0]
    assert np.max(np.abs(model_ref.silu(z) - z * sm)) < 1e-12


def test_extension_model_gradients_finite_difference():
    """f64 central differences through the SwiGLU / RMSNorm decoder (loss of the oracle step)."""
    spec = dict(vocab_size=16, n_layers=1, d_model=8, n_heads=2, d_ff=12, max_seq_len=4, mlp="swiglu",
                norm="rmsnorm")
    params = rng_ref.init_transformer_params(spec, seed=5)
    rng = np.random.default_rng(1)
    for k in params:  # non-trivial scales so every term of the RMSNorm backward is exercised
        if k.endswith("/scale"):
            params[k] = params[k] + 0.3 * rng.standard_normal(params[k].shape)
    tokens = rng.integers(0, 16, (2, 4))
    targets = rng.integers(0, 16, (2, 4))
    weights = np.ones((2, 4))
    _, grads, _ = model_ref.forward_backward(params, spec, tokens, targets, weights)
    assert set(grads) == {n for n, _ in rng_ref.transformer_param_shapes(spec)}
    for name in ("block_0/mlp/fc1/gate/kernel", "block_0/mlp/fc1/kernel", "block_0/mlp/fc2/kernel",
                 "block_0/ln2/scale", "block_0/ln1/scale", "final_ln/scale", "embed/tok/kernel"):
        flat = params[name].reshape(-1)
        for i in rng.choice(flat.size, size=min(6, flat.size), replace=False):
            old = flat[i]
            flat[i] = old + 1e-6
            lp, _, _ = model_ref.forward_backward(params, spec, tokens, targets, weights, need_grads=False)
            flat[i] = old - 1e-6
            lm, _, _ = model_ref.forward_backward(params, spec, tokens, targets, weights, need_grads=False)
            flat[i] = old
            fd = (lp - lm) / 2e-6
            an = grads[name].reshape(-1)[i]
            assert abs(fd - an) <= 1e-6 * max(1.0, abs(an)) + 1e-8, (name, i, fd, an)
