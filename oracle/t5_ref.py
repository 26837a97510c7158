"""ORACLE (test infrastructure): numpy f64 T5 encoder-decoder step (extension, SURVEY §8f item 3,
BASELINE cfg4). The reference has no encoder-decoder model; this restates one from the
reference's own ops, as SURVEY §8(c) "Extension oracles" prescribes:
  - linear (kernels.hpp:146-161, W is [out, in], no bias), embedding_lookup (graph.hpp:419-433)
  - RMSNorm = the reference-op identity slice(layer_norm(concat(x,-x)))*g (model_ref.rms_norm,
    pinned in tests/test_oracle.py), eps 1e-6 as T5LayerNorm
  - attention = the SDPA composite (graph.hpp:650-661) without the 1/sqrt(d) factor (T5 folds it
    into the init) plus the relative-position bias: embedding_lookup of host-computed bucket ids
    into rel_bias [buckets, H] and a broadcast add (graph.hpp:390-422); causal -1e9 mask in the
    decoder self-attention (model.hpp:100-106); cross-attention = the same composite with k, v
    from the encoder output and no bias / mask
  - ReLU MLP (T5 v1.0 DenseReluDense), softmax_cross_entropy (kernels.hpp:327-363)
  - the backward is the VJP set autodiff.hpp emits for those ops; the rel_bias gradient is the
    embedding scatter-add (kernels.hpp:291-304) of dS summed over the batch.
Parity of the composition is pinned by tests/test_oracle_t5.py: finite differences on every
parameter class, and the attention/CE primitives against model_ref (which is pinned against the
reference's own goldens). Numerics of the T5 *model* are therefore pinned to the reference's
ops, not to a reference T5 (none exists).
"""
from __future__ import annotations

import math

import numpy as np

from .model_ref import _softmax, bf16_round, rms_norm_bwd

EPS_T5 = 1e-6


def rms_norm(x, s, eps=EPS_T5):
    r = 1.0 / np.sqrt((x * x).mean(-1, keepdims=True) + eps)
    xhat = x * r
    return xhat * s, xhat, r


def rel_bucket(rp: int, bidirectional: bool, num_buckets: int, max_distance: int) -> int:
    """HF T5 `_relative_position_bucket` (rp = key - query), evaluated in double with the same
    1e-9 truncation guard as the host rule engine (rules.h t5_rel_bucket)."""
    ret = 0
    if bidirectional:
        num_buckets //= 2
        if rp > 0:
            ret += num_buckets
        n = abs(rp)
    else:
        n = max(-rp, 0)
    max_exact = num_buckets // 2
    if n < max_exact:
        return ret + n
    x = math.log(n / max_exact) / math.log(max_distance / max_exact) * (num_buckets - max_exact)
    return ret + min(max_exact + int(math.floor(x + 1e-9)), num_buckets - 1)


def bucket_table(tq, tk, bidirectional, num_buckets, max_distance):
    return np.array([[rel_bucket(j - i, bidirectional, num_buckets, max_distance) for j in range(tk)]
                     for i in range(tq)], np.int64)


def _heads(x, H):
    B, T, D = x.shape
    return x.reshape(B, T, H, D // H).transpose(0, 2, 1, 3)


def _merge(x):
    B, H, T, dk = x.shape
    return x.transpose(0, 2, 1, 3).reshape(B, T, H * dk)


def attention_fwd(q, k, v, bias=None, causal=False, round_p=False):
    """q [B,H,Tq,dk], k/v [B,H,Tk,dk]; scores unscaled (T5) + bias [H,Tq,Tk] (+ causal mask).
    round_p: the tensor-core kernels' arithmetic -- the max-shifted exponentials enter the P.V
    product as bf16, the row sum stays fp32."""
    s = q @ k.transpose(0, 1, 3, 2)
    if bias is not None:
        s = s + bias[None]
    if causal:
        Tq, Tk = s.shape[-2:]
        s = s + np.triu(np.full((Tq, Tk), -1e9), 1)
    P = _softmax(s)
    if round_p:
        e = np.exp(s - s.max(-1, keepdims=True))
        return (bf16_round(e) @ v) / e.sum(-1, keepdims=True), P
    return P @ v, P


def attention_bwd(q, k, v, P, dout, o_stored=None, round_p=False):
    """delta = rowsum(dP * P); with o_stored (bf16_acts) the flash form rowsum(dO * O) over the
    stored output, as the device computes it (model_ref does the same). round_p: P and dS enter
    the dV / dK / dQ products as bf16 (tensor-core kernels); the bias gradient uses fp32 dS."""
    dP = dout @ v.transpose(0, 1, 3, 2)
    Pm = bf16_round(P) if round_p else P
    dv = Pm.transpose(0, 1, 3, 2) @ dout
    delta = (dP * P).sum(-1, keepdims=True) if o_stored is None else (dout * o_stored).sum(-1, keepdims=True)
    dS = P * (dP - delta)
    dSm = bf16_round(dS) if round_p else dS
    return dSm @ k, dSm.transpose(0, 1, 3, 2) @ q, dv, dSm


def forward_backward(params: dict, spec: dict, enc_tokens, dec_tokens, targets, weights, need_grads=True,
                     bf16_acts=False, round_p=False):
    """Returns (loss, grads, logits). enc_tokens [B,Te], dec_tokens/targets/weights [B,Td].
    bf16_acts rounds what the device stores in bf16 (GEMM inputs/outputs, attention operands)."""
    R = bf16_round if bf16_acts else (lambda x: x)
    p = params
    H, d = spec["n_heads"], spec["d_model"]
    nb, md = spec.get("rel_buckets", 32), spec.get("rel_max_distance", 128)
    B, Te = enc_tokens.shape
    Td = dec_tokens.shape[1]
    emb = p["embed/tok/kernel"]

    def lin(x, name):
        return x @ p[name].T

    def self_bias(st, T, bidir):
        ids = bucket_table(T, T, bidir, nb, md)
        return p[f"{st}/block_0/attn/rel_bias/kernel"][ids].transpose(2, 0, 1), ids  # [H, T, T]

    cache = {}

    def block_attn(x_in, pre, scope, kv_in, bias, causal):
        a, xh, r = rms_norm(x_in, p[pre + ("ln_x" if scope == "cross_attn" else "ln1") + "/scale"])
        a = R(a)
        src = a if kv_in is None else kv_in
        q = _heads(R(lin(a, pre + f"{scope}/q/kernel")), H)
        k = _heads(R(lin(src, pre + f"{scope}/k/kernel")), H)
        v = _heads(R(lin(src, pre + f"{scope}/v/kernel")), H)
        o, P = attention_fwd(q, k, v, bias, causal, round_p)
        om = R(_merge(o))
        cache[(pre, scope)] = (a, xh, r, q, k, v, P, om)
        return x_in + lin(om, pre + f"{scope}/o/kernel")

    def block_mlp(x_in, pre):
        m, xh, r = rms_norm(x_in, p[pre + "ln2/scale"])
        m = R(m)
        up = R(lin(m, pre + "mlp/fc1/kernel"))
        act = R(np.maximum(up, 0.0))
        cache[(pre, "mlp")] = (m, xh, r, up, act)
        return x_in + lin(act, pre + "mlp/fc2/kernel")

    # encoder
    h = emb[enc_tokens]
    ebias, eids = self_bias("enc", Te, True)
    for l in range(spec["n_layers"]):
        pre = f"enc/block_{l}/"
        h = block_attn(h, pre, "attn", None, ebias, False)
        h = block_mlp(h, pre)
    eout, exh, er = rms_norm(h, p["enc/final_ln/scale"])
    eout = R(eout)
    # decoder
    g = emb[dec_tokens]
    dbias, dids = self_bias("dec", Td, False)
    for l in range(spec["n_dec_layers"]):
        pre = f"dec/block_{l}/"
        g = block_attn(g, pre, "attn", None, dbias, True)
        g = block_attn(g, pre, "cross_attn", eout, None, False)
        g = block_mlp(g, pre)
    f, fxh, fr = rms_norm(g, p["dec/final_ln/scale"])
    f = R(f)
    W_head = bf16_round(p["lm_head/kernel"]) if bf16_acts else p["lm_head/kernel"]
    logits = R(f @ W_head.T)
    mx = logits.max(-1, keepdims=True)
    lse = mx[..., 0] + np.log(np.exp(logits - mx).sum(-1))
    ce = lse - np.take_along_axis(logits, targets[..., None], -1)[..., 0]
    wsum = weights.sum()
    loss = float((ce * weights).sum() / wsum)
    if not need_grads:
        return loss, None, logits

    grads = {k: np.zeros_like(v) for k, v in p.items()}
    dlogits = _softmax(logits)
    np.put_along_axis(dlogits, targets[..., None], np.take_along_axis(dlogits, targets[..., None], -1) - 1.0, -1)
    dlogits = R(dlogits * (weights / wsum)[..., None])
    V = logits.shape[-1]
    grads["lm_head/kernel"] = dlogits.reshape(-1, V).T @ f.reshape(-1, d)
    dg, grads["dec/final_ln/scale"] = rms_norm_bwd(fxh, fr, p["dec/final_ln/scale"], dlogits @ W_head)
    d_eout = np.zeros_like(eout)

    def scatter_bias(st, ids, dS):
        tbl = grads[f"{st}/block_0/attn/rel_bias/kernel"]
        ds = dS.sum(0)  # [H, T, T]
        for hh in range(H):
            np.add.at(tbl[:, hh], ids.reshape(-1), ds[hh].reshape(-1))

    def mlp_bwd(dy, pre):
        m, xh, r, up, act = cache[(pre, "mlp")]
        dyf = R(dy.reshape(-1, d))
        grads[pre + "mlp/fc2/kernel"] = dyf.T @ act.reshape(-1, act.shape[-1])
        dact = dyf.reshape(dy.shape) @ p[pre + "mlp/fc2/kernel"]
        dup = R(dact * (up > 0))
        grads[pre + "mlp/fc1/kernel"] = dup.reshape(-1, dup.shape[-1]).T @ m.reshape(-1, d)
        dm = dup @ p[pre + "mlp/fc1/kernel"]
        dx, grads[pre + "ln2/scale"] = rms_norm_bwd(xh, r, p[pre + "ln2/scale"], dm)
        return dy + dx

    def attn_bwd(dy, pre, scope, kv_in, st, ids):
        a, xh, r, q, k, v, P, om = cache[(pre, scope)]
        dyf = R(dy.reshape(-1, d))
        grads[pre + f"{scope}/o/kernel"] = dyf.T @ om.reshape(-1, om.shape[-1])
        dom = R(dyf.reshape(dy.shape) @ p[pre + f"{scope}/o/kernel"])
        dq, dk, dv, dS = attention_bwd(q, k, v, P, _heads(dom, H), _heads(om, H) if bf16_acts else None, round_p)
        if ids is not None:
            scatter_bias(st, ids, dS)
        dqf, dkf, dvf = (R(_merge(t)) for t in (dq, dk, dv))
        src = a if kv_in is None else kv_in
        for name, t, x in (("q", dqf, a), ("k", dkf, src), ("v", dvf, src)):
            grads[pre + f"{scope}/{name}/kernel"] = t.reshape(-1, t.shape[-1]).T @ x.reshape(-1, d)
        da = dqf @ p[pre + f"{scope}/q/kernel"]
        dsrc = dkf @ p[pre + f"{scope}/k/kernel"] + dvf @ p[pre + f"{scope}/v/kernel"]
        if kv_in is None:
            da = da + dsrc
            dsrc = None
        ln = pre + ("ln_x" if scope == "cross_attn" else "ln1") + "/scale"
        dx, grads[ln] = rms_norm_bwd(xh, r, p[ln], da)
        return dy + dx, dsrc

    for l in reversed(range(spec["n_dec_layers"])):
        pre = f"dec/block_{l}/"
        dg = mlp_bwd(dg, pre)
        dg, dsrc = attn_bwd(dg, pre, "cross_attn", eout, None, None)
        d_eout += dsrc
        dg, _ = attn_bwd(dg, pre, "attn", None, "dec", dids)
    dh, grads["enc/final_ln/scale"] = rms_norm_bwd(exh, er, p["enc/final_ln/scale"], d_eout)
    for l in reversed(range(spec["n_layers"])):
        pre = f"enc/block_{l}/"
        dh = mlp_bwd(dh, pre)
        dh, _ = attn_bwd(dh, pre, "attn", None, "enc", eids)
    np.add.at(grads["embed/tok/kernel"], enc_tokens.reshape(-1), dh.reshape(-1, d))
    np.add.at(grads["embed/tok/kernel"], dec_tokens.reshape(-1), dg.reshape(-1, d))
    return loss, grads, logits


def init_params(spec: dict, seed: int = 42, name: str = "model-init", dtype=np.float64) -> dict:
    """Same rules as init_transformer_params (model.hpp:49-70) applied to the T5 tree."""
    from .rng_ref import init_transformer_params

    return init_transformer_params(dict(spec, arch="t5"), seed, name, dtype)


def t5_batch(seed: int, step: int, batch: int, te: int, td: int, vocab: int):
    """Synthetic encoder/decoder batch: enc tokens, dec tokens, then targets, from
    RngStream(seed, "t5-batch").child(step) (the audit-batch convention of cli.cpp:211-228)."""
    from .rng_ref import RngStream

    r = RngStream(seed, "t5-batch").child(step)
    enc = r.below(batch * te, vocab).reshape(batch, te).astype(np.int32)
    dec = r.below(batch * td, vocab).reshape(batch, td).astype(np.int32)
    tgt = r.below(batch * td, vocab).reshape(batch, td).astype(np.int32)
    return enc, dec, tgt, np.ones((batch, td), np.float32)
