"""CPU checks of the T5 encoder-decoder extension (BASELINE cfg4): the spec
keys and parameter tree, the relative-position buckets of the host rule engine against the
oracle, and the oracle's backward against central finite differences (the reference's own
autodiff test method, tests/test_autodiff.cpp:34-164 with tests/fd_oracle.hpp:18-52)."""
import os

import numpy as np
import pytest

from oracle import rng_ref, t5_ref
from paper_2310_16355_b200 import rules
from paper_2310_16355_b200._lib import SwError

SPECS = os.path.join(os.path.dirname(__file__), "..", "oracle", "specs")


def spec_dict(spec):
    return dict(vocab_size=spec.vocab_size, n_layers=spec.n_layers, n_dec_layers=spec.n_dec_layers,
                d_model=spec.d_model, n_heads=spec.n_heads, d_kv=spec.d_kv, d_ff=spec.d_ff,
                max_seq_len=spec.max_seq_len, rel_buckets=spec.rel_buckets,
                rel_max_distance=spec.rel_max_distance, arch="t5")


@pytest.mark.parametrize("name", ["mini_t5.spec", "t5_11b.spec"])
def test_t5_spec_tree(name):
    spec = rules.read_model_spec(os.path.join(SPECS, name))
    assert spec.arch == "t5" and spec.norm == "rmsnorm"
    want = rng_ref.transformer_param_shapes(spec_dict(spec))
    got = [(n, tuple(d)) for n, d in rules.transformer_param_shapes(spec)]
    assert got == [(n, tuple(d)) for n, d in want]
    if name == "t5_11b.spec":
        assert len(got) == 510
        assert sum(int(np.prod(d)) for _, d in got) == 11_340_220_416  # enc 4.83 G + dec 6.44 G + embed + lm_head


def test_t5_plan_rules():
    """Under the reference rules: q/k/v (self and cross) split:0, o split:1, fc1 split:0,
    fc2 split:1; rel_bias, embeddings, norms and lm_head replicated (lm_head and rel_bias match
    no role and raise the reference's warning)."""
    spec = rules.read_model_spec(os.path.join(SPECS, "t5_11b.spec"))
    shapes = rules.transformer_param_shapes(spec)
    plan = rules.derive_plan(shapes, 8, spec.overrides)
    for n, _ in shapes:
        layer = n.split("/")[-2]
        if layer in ("q", "k", "v", "fc1"):
            assert plan.at(n) == "split:0", n
        elif layer in ("o", "fc2"):
            assert plan.at(n) == "split:1", n
        else:
            assert plan.at(n) == "replicated", n


def test_t5_spec_errors():
    base = "vocab_size = 8\nn_layers = 1\nd_model = 8\nn_heads = 2\nd_ff = 8\nmax_seq_len = 4\n"
    with pytest.raises(SwError, match="need arch = t5"):
        rules.parse_model_spec(base + "d_kv = 4\n")
    with pytest.raises(SwError, match="arch = t5 needs"):
        rules.parse_model_spec(base + "arch = t5\n")
    with pytest.raises(SwError, match="needs decoder or t5"):
        rules.parse_model_spec(base + "arch = bert\n")
    with pytest.raises(SwError, match="tie_embeddings"):
        rules.parse_model_spec(base + "arch = t5\nn_dec_layers = 1\nd_kv = 4\ntie_embeddings = true\n")


@pytest.mark.parametrize("tq,tk,bidir,nb,md", [(40, 40, True, 32, 128), (40, 40, False, 32, 128),
                                               (300, 300, True, 32, 128), (300, 300, False, 32, 128),
                                               (33, 20, True, 8, 16), (64, 64, False, 8, 16)])
def test_rel_buckets_host_matches_oracle(tq, tk, bidir, nb, md):
    got = rules.t5_rel_buckets(tq, tk, bidir, nb, md)
    assert np.array_equal(got, t5_ref.bucket_table(tq, tk, bidir, nb, md))
    assert got.min() >= 0 and got.max() < nb


def test_rel_bucket_known_values():
    """Values of the HF T5 rule (bidirectional, 32 buckets, max_distance 128)."""
    f = lambda rp: t5_ref.rel_bucket(rp, True, 32, 128)  # noqa: E731
    assert [f(r) for r in (0, 1, 7, 8, 12, 16, 127, 500)] == [0, 17, 23, 24, 25, 26, 31, 31]
    assert [f(-r) for r in (1, 7, 8, 16, 500)] == [1, 7, 8, 10, 15]
    g = lambda rp: t5_ref.rel_bucket(rp, False, 32, 128)  # noqa: E731
    assert [g(r) for r in (5, 0, -1, -15, -16, -32, -1000)] == [0, 0, 1, 15, 16, 21, 31]


TINY = dict(vocab_size=13, n_layers=1, n_dec_layers=1, d_model=8, n_heads=2, d_kv=3, d_ff=10,
            max_seq_len=8, rel_buckets=8, rel_max_distance=16, arch="t5")


def test_t5_oracle_finite_differences():
    """Every parameter class: central differences, h = 1e-6 * max(1, |theta|), rel err < 1e-6
    (fd_oracle.hpp:18-52)."""
    p = t5_ref.init_params(TINY, seed=3)
    rng = np.random.default_rng(0)
    for k in p:  # break the symmetry of unit scales
        p[k] = p[k] + 0.1 * rng.standard_normal(p[k].shape)
    enc, dec, tgt, w = t5_ref.t5_batch(5, 0, 2, 6, 5, TINY["vocab_size"])
    w = w * np.array([[1.0, 0.5, 2.0, 1.0, 0.0]] * 2, np.float32)
    loss, grads, _ = t5_ref.forward_backward(p, TINY, enc, dec, tgt, w)
    checked = 0
    for name in p:
        flat = p[name].reshape(-1)
        for idx in rng.choice(flat.size, size=min(3, flat.size), replace=False):
            h = 1e-6 * max(1.0, abs(flat[idx]))
            old = flat[idx]
            flat[idx] = old + h
            lp = t5_ref.forward_backward(p, TINY, enc, dec, tgt, w, need_grads=False)[0]
            flat[idx] = old - h
            lm = t5_ref.forward_backward(p, TINY, enc, dec, tgt, w, need_grads=False)[0]
            flat[idx] = old
            fd = (lp - lm) / (2 * h)
            an = grads[name].reshape(-1)[idx]
            assert abs(fd - an) <= 1e-6 * max(1.0, abs(fd), abs(an)) + 1e-9, (name, idx, fd, an)
            checked += 1
    assert checked >= 3 * len(p) - 6


def test_t5_attention_matches_reference_composite():
    """T5 attention with the 1/sqrt(d) factor folded into q, no bias, causal == the reference SDPA
    composite as the pinned decoder oracle computes it (softmax(q k^T / sqrt(d) + mask) v)."""
    rng = np.random.default_rng(1)
    q, k, v = (rng.standard_normal((2, 3, 7, 4)) for _ in range(3))
    out, _ = t5_ref.attention_fwd(q / 2.0, k, v, None, True)
    s = q @ k.transpose(0, 1, 3, 2) / 2.0 + np.triu(np.full((7, 7), -1e9), 1)
    e = np.exp(s - s.max(-1, keepdims=True))
    assert np.allclose(out, (e / e.sum(-1, keepdims=True)) @ v, rtol=1e-13, atol=1e-13)
