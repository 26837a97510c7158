"""ORACLE (test infrastructure): numpy f64 restatement of the reference transformer step.

  forward   transformer_logits / transformer_loss        model.hpp:76-152
            ops: linear kernels.hpp:146-161 (W is [out,in]); layer_norm (biased variance,
            eps 1e-5) kernels.hpp:184-271, graph.hpp:401-416; tanh-GeLU kernels.hpp:97-129;
            scaled_dot_product_attention with the -1e9 causal mask graph.hpp:650-661,
            model.hpp:100-106; softmax_cross_entropy kernels.hpp:327-363
  backward  the VJPs autodiff.hpp emits (linear :124-139, layer norm :186-211, softmax :222-229,
            cross entropy :230-238, embedding scatter-add kernels.hpp:291-304)
  optimizer adamw_step train_state.hpp:183-220 (c1, c2 in double; decay on every parameter)
  audit     audit_equivalence's single-device trajectory audit.hpp:78-159
  extension mlp = swiglu / norm = rmsnorm: RMSNorm and SiLU written as the
            reference-op identities slice(layer_norm(concat(x,-x)))*g and x*softmax([x,0])[0];
            tests/test_oracle.py checks the closed forms here against those compositions.
"""
from __future__ import annotations

import math

import numpy as np

EPS_LN = 1e-5
GELU_A = 0.7978845608028654
GELU_B = 0.044715


def gelu(x):
    return 0.5 * x * (1.0 + np.tanh(GELU_A * (x + GELU_B * x * x * x)))


def gelu_grad(x):
    t = np.tanh(GELU_A * (x + GELU_B * x * x * x))
    return 0.5 * (1.0 + t) + 0.5 * x * (1.0 - t * t) * GELU_A * (1.0 + 3.0 * GELU_B * x * x)


def layer_norm(x, s, b, eps=EPS_LN):
    mean = x.mean(-1, keepdims=True)
    var = ((x - mean) ** 2).mean(-1, keepdims=True)
    xhat = (x - mean) / np.sqrt(var + eps)
    return xhat * s + b, xhat, 1.0 / np.sqrt(var + eps)


def layer_norm_bwd(xhat, rstd, s, dy):
    g = dy * s
    dx = rstd * (g - g.mean(-1, keepdims=True) - xhat * (g * xhat).mean(-1, keepdims=True))
    return dx, (dy * xhat).reshape(-1, dy.shape[-1]).sum(0), dy.reshape(-1, dy.shape[-1]).sum(0)


def rms_norm(x, s, eps=EPS_LN):
    """Extension: slice(layer_norm(concat(x, -x)), d) * s: the concatenation has
    zero mean and variance mean(x^2), so xhat = x / sqrt(mean(x^2) + eps)."""
    r = 1.0 / np.sqrt((x * x).mean(-1, keepdims=True) + eps)
    xhat = x * r
    return xhat * s, xhat, r


def rms_norm_bwd(xhat, rstd, s, dy):
    g = dy * s
    dx = rstd * (g - xhat * (g * xhat).mean(-1, keepdims=True))
    return dx, (dy * xhat).reshape(-1, dy.shape[-1]).sum(0)


def silu(x):
    """Extension: x * softmax([x, 0])[0] = x * sigmoid(x)."""
    return x / (1.0 + np.exp(-x))


def silu_grad(x):
    sg = 1.0 / (1.0 + np.exp(-x))
    return sg * (1.0 + x * (1.0 - sg))


def _softmax(x):
    m = x.max(-1, keepdims=True)
    e = np.exp(x - m)
    return e / e.sum(-1, keepdims=True)


def bf16_round(x):
    """Round-to-nearest-even to bfloat16, returned as float64."""
    a = np.asarray(x, np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def forward_backward(params: dict, spec: dict, tokens, targets, weights, need_grads=True,
                     bf16_acts=False):
    """Returns (loss, grads dict, logits). tokens/targets int [B,T], weights [B,T].

    bf16_acts=True rounds every GEMM operand that a bf16 tensor-core implementation stores in
    bf16 (LayerNorm outputs, q/k/v, attention output, GeLU input/output, logits and the
    backward's dlogits / residual-gradient / dpre / d(attn out) / dqkv), so a bf16 device run
    can be checked at a tolerance set by accumulation order rather than storage rounding."""
    R = bf16_round if bf16_acts else (lambda x: x)
    swiglu = spec.get("mlp", "gelu") == "swiglu"
    rms = spec.get("norm", "layernorm") == "rmsnorm"

    def norm(x, prefix):
        if rms:
            y, xh, r = rms_norm(x, p[prefix + "/scale"])
            return y, xh, r
        return layer_norm(x, p[prefix + "/scale"], p[prefix + "/bias"])

    def norm_bwd(xh, r, prefix, dy, grads):
        if rms:
            dx, grads[prefix + "/scale"] = rms_norm_bwd(xh, r, p[prefix + "/scale"], dy)
        else:
            dx, grads[prefix + "/scale"], grads[prefix + "/bias"] = layer_norm_bwd(xh, r, p[prefix + "/scale"], dy)
        return dx

    B, T = tokens.shape
    d, H, L = spec["d_model"], spec["n_heads"], spec["n_layers"]
    hd = d // H
    tied = spec.get("tie_embeddings", False)
    p = params
    h = p["embed/tok/kernel"][tokens] + p["embed/pos/kernel"][np.arange(T)][None]
    mask = np.triu(np.full((T, T), -1e9), 1)
    cache = []
    for l in range(L):
        pre = f"block_{l}/"
        a, xh1, r1 = norm(h, pre + "ln1")
        a = R(a)

        def proj(name):
            y = R(a @ p[pre + f"attn/{name}/kernel"].T + p[pre + f"attn/{name}/bias"])
            return y.reshape(B, T, H, hd).transpose(0, 2, 1, 3)

        q, k, v = proj("q"), proj("k"), proj("v")
        s = q @ k.transpose(0, 1, 3, 2) * (1.0 / math.sqrt(hd)) + mask
        P = _softmax(s)
        att = P @ v
        merged = R(att.transpose(0, 2, 1, 3).reshape(B, T, d))
        h_mid = h + merged @ p[pre + "attn/o/kernel"].T + p[pre + "attn/o/bias"]
        m, xh2, r2 = norm(h_mid, pre + "ln2")
        m = R(m)
        if swiglu:
            gate = R(m @ p[pre + "mlp/fc1/gate/kernel"].T)   # pre-activations, stored bf16 on device
            upv = R(m @ p[pre + "mlp/fc1/kernel"].T)
            g = R(silu(gate) * upv)           # h = silu(gate x) * (up x)
            up = (gate, upv)
            h_out = h_mid + g @ p[pre + "mlp/fc2/kernel"].T
        else:
            up_full = m @ p[pre + "mlp/fc1/kernel"].T + p[pre + "mlp/fc1/bias"]
            g = R(gelu(up_full))
            up = R(up_full)
            h_out = h_mid + g @ p[pre + "mlp/fc2/kernel"].T + p[pre + "mlp/fc2/bias"]
        cache.append((a, xh1, r1, q, k, v, P, merged, m, xh2, r2, up, g))
        h = h_out
    f, xhf, rf = norm(h, "final_ln")
    f = R(f)
    W_head = p["embed/tok/kernel"] if tied else p["lm_head/kernel"]
    if bf16_acts:
        W_head = bf16_round(W_head)
    logits = R(f @ W_head.T)
    mx = logits.max(-1, keepdims=True)
    lse = mx[..., 0] + np.log(np.exp(logits - mx).sum(-1))
    ce = lse - np.take_along_axis(logits, targets[..., None], -1)[..., 0]
    wsum = weights.sum()
    loss = float((ce * weights).sum() / wsum)
    if not need_grads:
        return loss, None, logits

    grads = {}
    dlogits = _softmax(logits)
    np.put_along_axis(dlogits, targets[..., None],
                      np.take_along_axis(dlogits, targets[..., None], -1) - 1.0, -1)
    dlogits *= (weights / wsum)[..., None]
    dlogits = R(dlogits)
    V = logits.shape[-1]
    dW_head = dlogits.reshape(-1, V).T @ f.reshape(-1, d)
    df = dlogits @ W_head
    dh = norm_bwd(xhf, rf, "final_ln", df, grads)
    for l in reversed(range(L)):
        pre = f"block_{l}/"
        a, xh1, r1, q, k, v, P, merged, m, xh2, r2, up, g = cache[l]
        dflat = R(dh.reshape(-1, d))
        grads[pre + "mlp/fc2/kernel"] = dflat.T @ g.reshape(-1, g.shape[-1])
        dhid = dflat.reshape(dh.shape) @ p[pre + "mlp/fc2/kernel"]
        if swiglu:
            gate, upv = up
            dgate = R(dhid * upv * silu_grad(gate))
            dupv = R(dhid * silu(gate))
            grads[pre + "mlp/fc1/gate/kernel"] = dgate.reshape(-1, dgate.shape[-1]).T @ m.reshape(-1, d)
            grads[pre + "mlp/fc1/kernel"] = dupv.reshape(-1, dupv.shape[-1]).T @ m.reshape(-1, d)
            dm = dgate @ p[pre + "mlp/fc1/gate/kernel"] + dupv @ p[pre + "mlp/fc1/kernel"]
        else:
            grads[pre + "mlp/fc2/bias"] = dh.reshape(-1, d).sum(0)
            dup = R(dhid * gelu_grad(up))
            grads[pre + "mlp/fc1/kernel"] = dup.reshape(-1, dup.shape[-1]).T @ m.reshape(-1, d)
            grads[pre + "mlp/fc1/bias"] = dup.reshape(-1, dup.shape[-1]).sum(0)
            dm = dup @ p[pre + "mlp/fc1/kernel"]
        dx = norm_bwd(xh2, r2, pre + "ln2", dm, grads)
        dh = dh + dx
        dflat = R(dh.reshape(-1, d))
        grads[pre + "attn/o/kernel"] = dflat.T @ merged.reshape(-1, d)
        grads[pre + "attn/o/bias"] = dh.reshape(-1, d).sum(0)
        datt = R(dflat.reshape(dh.shape) @ p[pre + "attn/o/kernel"]).reshape(B, T, H, hd).transpose(0, 2, 1, 3)
        dP = datt @ v.transpose(0, 1, 3, 2)
        dv = P.transpose(0, 1, 3, 2) @ datt
        if bf16_acts:  # flash-style: delta = rowsum(dO * O) with the stored (bf16) O
            delta = (datt * merged.reshape(B, T, H, hd).transpose(0, 2, 1, 3)).sum(-1, keepdims=True)
        else:
            delta = (dP * P).sum(-1, keepdims=True)
        dS = P * (dP - delta) * (1.0 / math.sqrt(hd))
        dq = dS @ k
        dk = dS.transpose(0, 1, 3, 2) @ q
        da = np.zeros_like(a)
        for name, dy in (("q", dq), ("k", dk), ("v", dv)):
            dyf = R(dy.transpose(0, 2, 1, 3).reshape(-1, d))
            grads[pre + f"attn/{name}/kernel"] = dyf.T @ a.reshape(-1, d)
            grads[pre + f"attn/{name}/bias"] = dyf.sum(0)
            da += (dyf @ p[pre + f"attn/{name}/kernel"]).reshape(B, T, d)
        dx = norm_bwd(xh1, r1, pre + "ln1", da, grads)
        dh = dh + dx
    dtok = np.zeros_like(p["embed/tok/kernel"])
    np.add.at(dtok, tokens.reshape(-1), dh.reshape(-1, d))
    dpos = np.zeros_like(p["embed/pos/kernel"])
    dpos[:T] = dh.sum(0)
    if tied:
        dtok = dtok + dW_head
    else:
        grads["lm_head/kernel"] = dW_head
    grads["embed/tok/kernel"] = dtok
    grads["embed/pos/kernel"] = dpos
    return loss, grads, logits


def adamw_step(params, m, v, grads, step, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, wd=0.0,
               dtype=np.float64):
    """train_state.hpp:183-220 for one replica; step is the pre-increment counter."""
    t = float(step + 1)
    c1 = dtype(1.0 - beta1 ** t)
    c2 = dtype(1.0 - beta2 ** t)
    b1, b2, lr_, eps_, wd_ = (dtype(x) for x in (beta1, beta2, lr, eps, wd))
    for k in params:
        g = grads[k]
        m[k] = b1 * m[k] + (dtype(1) - b1) * g
        v[k] = b2 * v[k] + (dtype(1) - b2) * (g * g)
        params[k] = params[k] - lr_ * ((m[k] / c1) / (np.sqrt(v[k] / c2) + eps_) + wd_ * params[k])


def audit_trajectory(params, spec, batch_for_step, dp, steps, lr, wd):
    """Single-device audit trajectory (audit.hpp:100-159): each step averages loss and grads of
    the dp batch slices, then AdamW. Returns (losses, grads of step 0, final params)."""
    params = {k: v.astype(np.float64).copy() for k, v in params.items()}
    m = {k: np.zeros_like(v) for k, v in params.items()}
    vv = {k: np.zeros_like(v) for k, v in params.items()}
    losses, g0 = [], None
    for step in range(steps):
        tokens, targets, weights = batch_for_step(step)
        rows = tokens.shape[0] // dp
        loss_sum, acc = 0.0, {k: np.zeros_like(v) for k, v in params.items()}
        for r in range(dp):
            sl = slice(r * rows, (r + 1) * rows)
            loss, grads, _ = forward_backward(params, spec, tokens[sl], targets[sl], weights[sl])
            loss_sum += loss
            for k in acc:
                acc[k] += grads[k]
        if dp > 1:
            for k in acc:
                acc[k] *= 1.0 / dp
        losses.append(loss_sum / dp)
        if step == 0:
            g0 = {k: x.copy() for k, x in acc.items()}
        adamw_step(params, m, vv, acc, step, lr=lr, wd=wd)
    return losses, g0, params
