"""Kernel-level parity of the non-GEMM kernels vs plain PyTorch fp32 references of the same op
(same bf16 inputs, upcast)."""
import math

import pytest
import torch

from paper_2310_16355_b200 import _lib

pytestmark = pytest.mark.gpu
DEV = "cuda"


def rel(a, b):
    return ((a.float() - b.float()).norm() / b.float().norm().clamp_min(1e-30)).item()


def ref_attention(qkv, B, T, Hl, hd):
    Dl = Hl * hd
    x = qkv.float().view(B, T, 3, Hl, hd)
    q, k, v = (x[:, :, i].permute(0, 2, 1, 3) for i in range(3))
    s = q @ k.transpose(-1, -2) / math.sqrt(hd)
    mask = torch.triu(torch.ones(T, T, dtype=torch.bool, device=DEV), 1)
    s = s.masked_fill(mask, float("-inf"))
    lse = torch.logsumexp(s, -1)
    o = torch.softmax(s, -1) @ v
    return o.permute(0, 2, 1, 3).reshape(B * T, Dl), lse


@pytest.mark.parametrize("B,T,Hl,hd", [(2, 64, 2, 8), (2, 128, 2, 64), (1, 256, 2, 128), (2, 200, 3, 64),
                                        (2, 200, 2, 128), (1, 1000, 3, 128), (2, 96, 1, 128), (1, 2048, 2, 128),
                                        (1, 160, 2, 256),
                                        # more work items than SMs: the persistent kernels walk
                                        # several items per CTA (T = 640: an odd query-block count,
                                        # so the last pair has one tile)
                                        (4, 640, 48, 128), (2, 1024, 40, 128),
                                        # head_dim 256 (GPT-J): tcgen05 forward, 64-key blocks
                                        (2, 1000, 4, 256), (1, 2048, 3, 256)])
def test_attention_fwd_bwd(B, T, Hl, hd):
    L = _lib.lib()
    g = torch.Generator(device=DEV).manual_seed(B * 1000 + T + hd)
    Dl = Hl * hd
    qkv = torch.randn(B * T, 3 * Dl, generator=g, device=DEV).bfloat16()
    o = torch.empty(B * T, Dl, device=DEV, dtype=torch.bfloat16)
    lse = torch.empty(B, Hl, T, device=DEV)
    _lib.check(L.sw_k_attention_fwd(qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), B, T, Hl, hd, None))
    torch.cuda.synchronize()
    want_o, want_lse = ref_attention(qkv, B, T, Hl, hd)
    assert rel(o, want_o) < 1e-2
    assert (lse - want_lse).abs().max().item() < 1e-3

    # backward vs autograd through the fp32 reference on the same bf16 inputs
    dout = torch.randn(B * T, Dl, generator=g, device=DEV).bfloat16()
    dqkv = torch.empty_like(qkv)
    scratch = torch.empty(L.sw_k_attention_bwd_scratch(B, T, Hl, hd), device=DEV)
    _lib.check(L.sw_k_attention_bwd(qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), dout.data_ptr(),
                                    dqkv.data_ptr(), scratch.data_ptr(), B, T, Hl, hd, None))
    torch.cuda.synchronize()
    x = qkv.float().requires_grad_(True)
    ro, _ = ref_attention(x, B, T, Hl, hd)
    # the device uses the stored (bf16) o for delta = rowsum(dO * O); so does this reference
    (ro * dout.float()).sum().backward()
    assert rel(dqkv, x.grad) < 2e-2, rel(dqkv, x.grad)
    for i in range(3):
        blk = slice(i * Dl, (i + 1) * Dl)
        assert rel(dqkv[:, blk], x.grad[:, blk]) < 2e-2, (i, rel(dqkv[:, blk], x.grad[:, blk]))


@pytest.mark.parametrize("M,d", [(64, 32), (300, 256), (257, 4096), (33, 9216), (10, 100)])
def test_layernorm_fwd_bwd(M, d):
    L = _lib.lib()
    g = torch.Generator(device=DEV).manual_seed(M + d)
    x = torch.randn(M, d, generator=g, device=DEV) * 3 + 1
    s = torch.randn(d, generator=g, device=DEV)
    b = torch.randn(d, generator=g, device=DEV)
    y = torch.empty(M, d, device=DEV, dtype=torch.bfloat16)
    mean = torch.empty(M, device=DEV)
    rstd = torch.empty(M, device=DEV)
    _lib.check(L.sw_k_layernorm_fwd(x.data_ptr(), s.data_ptr(), b.data_ptr(), y.data_ptr(), mean.data_ptr(),
                                    rstd.data_ptr(), M, d, 1e-5, None))
    torch.cuda.synchronize()
    xr = x.clone().requires_grad_(True)
    sr = s.clone().requires_grad_(True)
    br = b.clone().requires_grad_(True)
    want = torch.nn.functional.layer_norm(xr, (d,), sr, br, 1e-5)
    assert rel(y, want) < 5e-3
    dy = torch.randn(M, d, generator=g, device=DEV)
    want.backward(dy)
    gio = torch.randn(M, d, generator=g, device=DEV)
    g0 = gio.clone()
    gb = torch.empty(M, d, device=DEV, dtype=torch.bfloat16)
    ds = torch.zeros(d, device=DEV)
    db = torch.zeros(d, device=DEV)
    _lib.check(L.sw_k_layernorm_bwd(x.data_ptr(), mean.data_ptr(), rstd.data_ptr(), s.data_ptr(), dy.data_ptr(),
                                    gio.data_ptr(), gb.data_ptr(), ds.data_ptr(), db.data_ptr(), M, d, 1, None))
    torch.cuda.synchronize()
    assert rel(gio - g0, xr.grad) < 1e-4
    assert rel(gb, gio) < 5e-3
    assert rel(ds, sr.grad) < 1e-4
    assert rel(db, br.grad) < 1e-4


@pytest.mark.parametrize("M,V", [(16, 64), (40, 32000), (7, 1000)])
def test_xent(M, V):
    L = _lib.lib()
    g = torch.Generator(device=DEV).manual_seed(M + V)
    logits = (torch.randn(M, V, generator=g, device=DEV) * 2).bfloat16()
    tgt = torch.randint(0, V, (M,), generator=g, device=DEV, dtype=torch.int32)
    w = torch.rand(M, generator=g, device=DEV)
    wsum = w.sum().reshape(1)
    wl = torch.empty(M, device=DEV)
    lg = logits.clone()
    _lib.check(L.sw_k_xent(lg.data_ptr(), V, M, V, tgt.data_ptr(), w.data_ptr(), wsum.data_ptr(), wl.data_ptr(),
                           1, None))
    torch.cuda.synchronize()
    x = logits.float().requires_grad_(True)
    ce = torch.nn.functional.cross_entropy(x, tgt.long(), reduction="none")
    loss = (ce * w).sum() / wsum
    loss.backward()
    assert rel(wl, ce * w) < 1e-5
    assert rel(lg, x.grad) < 1e-2


def test_adamw_kernel():
    L = _lib.lib()
    n = 1003
    g = torch.Generator(device=DEV).manual_seed(0)
    p = torch.randn(n, generator=g, device=DEV)
    m = torch.randn(n, generator=g, device=DEV) * 0.1
    v = torch.rand(n, generator=g, device=DEV) * 0.01
    gr = torch.randn(n, generator=g, device=DEV)
    sh = torch.empty(n, device=DEV, dtype=torch.bfloat16)
    lr, b1, b2, eps, wd, t = 1e-3, 0.9, 0.999, 1e-8, 0.01, 3
    c1, c2 = 1 - b1 ** t, 1 - b2 ** t
    # Scalar = float semantics of train_state.hpp:199-216 (constants cast to float first)
    F = lambda x: torch.tensor(x, dtype=torch.float32, device=DEV)  # noqa: E731
    one = F(1.0)
    want_m = F(b1) * m + (one - F(b1)) * gr
    want_v = F(b2) * v + (one - F(b2)) * (gr * gr)
    want_p = p - F(lr) * ((want_m / F(c1)) / ((want_v / F(c2)).sqrt() + F(eps)) + F(wd) * p)
    _lib.check(L.sw_k_adamw(p.data_ptr(), m.data_ptr(), v.data_ptr(), gr.data_ptr(), sh.data_ptr(), n, lr, b1, b2,
                            eps, wd, c1, c2, None))
    torch.cuda.synchronize()
    assert torch.allclose(p, want_p, rtol=1e-6, atol=1e-7)
    assert torch.allclose(m, want_m, rtol=1e-6, atol=1e-7)
    assert torch.allclose(v, want_v, rtol=1e-6, atol=1e-9)
    assert torch.equal(sh, p.bfloat16())

    # the hand-worked KAT of tests/test_spmd.cpp:474-499: theta=1, g=1, lr=0.1, one step
    one = torch.ones(4, device=DEV)
    pm, mm, vm = one.clone(), torch.zeros(4, device=DEV), torch.zeros(4, device=DEV)
    sh4 = torch.empty(4, device=DEV, dtype=torch.bfloat16)
    _lib.check(L.sw_k_adamw(pm.data_ptr(), mm.data_ptr(), vm.data_ptr(), one.data_ptr(), sh4.data_ptr(), 4, 0.1,
                            0.9, 0.999, 1e-8, 0.0, 1 - 0.9, 1 - 0.999, None))
    torch.cuda.synchronize()
    assert torch.allclose(mm, torch.full_like(mm, 0.1))
    assert torch.allclose(vm, torch.full_like(vm, 0.001))
    assert torch.allclose(pm, torch.full_like(pm, 1 - 0.1 / (1 + 1e-8)))


@pytest.mark.parametrize("M,d", [(64, 32), (300, 256), (257, 4096), (33, 9216), (10, 100)])
def test_rmsnorm_fwd_bwd(M, d):
    """RMSNorm extension vs torch fp32: y = x * rsqrt(mean(x^2) + eps) * g."""
    L = _lib.lib()
    g = torch.Generator(device=DEV).manual_seed(M * 3 + d)
    x = torch.randn(M, d, generator=g, device=DEV) * 3 + 1
    s = torch.randn(d, generator=g, device=DEV)
    y = torch.empty(M, d, device=DEV, dtype=torch.bfloat16)
    rstd = torch.empty(M, device=DEV)
    _lib.check(L.sw_k_rmsnorm_fwd(x.data_ptr(), s.data_ptr(), y.data_ptr(), rstd.data_ptr(), M, d, 1e-5, None))
    xr = x.clone().requires_grad_(True)
    sr = s.clone().requires_grad_(True)
    ref = xr * torch.rsqrt((xr * xr).mean(-1, keepdim=True) + 1e-5) * sr
    torch.cuda.synchronize()
    assert rel(y, ref) < 1e-2
    assert torch.allclose(rstd, torch.rsqrt((x * x).mean(-1) + 1e-5), rtol=1e-5)
    dy = torch.randn(M, d, generator=g, device=DEV)
    gio = torch.randn(M, d, generator=g, device=DEV)
    g0 = gio.clone()
    gb = torch.empty(M, d, device=DEV, dtype=torch.bfloat16)
    ds = torch.zeros(d, device=DEV)
    _lib.check(L.sw_k_rmsnorm_bwd(x.data_ptr(), rstd.data_ptr(), s.data_ptr(), dy.data_ptr(), gio.data_ptr(),
                                  gb.data_ptr(), ds.data_ptr(), M, d, 1, None))
    (ref * dy).sum().backward()
    torch.cuda.synchronize()
    assert rel(gio - g0, xr.grad) < 1e-5
    assert rel(ds, sr.grad) < 1e-5
    assert rel(gb, gio) < 1e-2


@pytest.mark.parametrize("hd", [64, 128])
def test_attention_lazy_rescale_path(hd):
    """Scores that grow along the keys force the online-softmax max to jump by more than 2^8
    between key blocks, so every query row rescales its O accumulator (the warp-collective TMEM
    rewrite) -- the path random inputs almost never take."""
    L = _lib.lib()
    B, T, Hl = 2, 640, 2
    Dl = Hl * hd
    g = torch.Generator(device=DEV).manual_seed(11)
    x = torch.randn(B * T, 3 * Dl, generator=g, device=DEV) * 0.1
    x = x.view(B, T, 3, Hl, hd)
    ramp = torch.arange(T, device=DEV, dtype=torch.float32)[None, :, None, None] / 48.0
    x[:, :, 0] += 0.5                       # q along the ones direction
    x[:, :, 1] += ramp                      # k grows with the key index
    qkv = x.reshape(B * T, 3 * Dl).bfloat16()
    o = torch.empty(B * T, Dl, device=DEV, dtype=torch.bfloat16)
    lse = torch.empty(B, Hl, T, device=DEV)
    _lib.check(L.sw_k_attention_fwd(qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), B, T, Hl, hd, None))
    torch.cuda.synchronize()
    want_o, want_lse = ref_attention(qkv, B, T, Hl, hd)
    assert rel(o, want_o) < 1e-2
    assert ((lse - want_lse).abs() / want_lse.abs().clamp_min(1)).max().item() < 1e-3


@pytest.mark.parametrize("hd", [64, 128, 256])
@pytest.mark.parametrize("p", [0, 5, 17, 200, 1023])
@pytest.mark.parametrize("split", [0, 1])
def test_decode_attention_step(hd, p, split, Hl=4):
    """One KV-cached decode step against torch fp32 attention of the new query over keys 0..p,
    where key / value p are the step's own (written into cache row p by the kernel). With 12
    heads the split kernel uses ceil((p + 1) / 64) splits up to 16 (1, 4 and 16 here)."""
    L = _lib.lib()
    B, T = 3, 1024
    Dl = Hl * hd
    g = torch.Generator(device=DEV).manual_seed(hd * 7 + p)
    cache = torch.randn(B * T, 3 * Dl, generator=g, device=DEV).bfloat16()
    new = torch.randn(B, 3 * Dl, generator=g, device=DEV).bfloat16()
    out = torch.empty(B, Dl, device=DEV, dtype=torch.bfloat16)
    part = torch.empty(B * Hl * 16 * (hd + 2), device=DEV)
    ticket = torch.zeros(B * Hl, device=DEV, dtype=torch.int32)
    want_cache = cache.clone().view(B, T, 3 * Dl)
    want_cache[:, p, Dl:] = new[:, Dl:]
    for rep in range(2):  # the second launch exercises the never-reset split tickets
        c = cache.clone()
        _lib.check(L.sw_k_decode_attention(new.data_ptr(), c.data_ptr(), out.data_ptr(), B, T, p, Hl, hd, split,
                                           part.data_ptr(), ticket.data_ptr(), None))
        torch.cuda.synchronize()
        assert torch.equal(c.view(B, T, 3 * Dl)[:, p, Dl:], new[:, Dl:])
        kv = want_cache[:, : p + 1].float()
        q = new[:, :Dl].float().view(B, Hl, 1, hd)
        k = kv[..., Dl:2 * Dl].view(B, p + 1, Hl, hd).transpose(1, 2)
        v = kv[..., 2 * Dl:].view(B, p + 1, Hl, hd).transpose(1, 2)
        ref = torch.softmax(q @ k.transpose(-1, -2) / math.sqrt(hd), -1) @ v
        assert rel(out, ref.view(B, Dl)) < 1e-2, (rep, rel(out, ref.view(B, Dl)))


@pytest.mark.parametrize("p", [150, 1023])
def test_decode_attention_split_budget(p):
    """192 heads: the launch's CTA budget caps the split count at 3, so a split covers up to 342
    keys (several 2-key unrolled passes per warp); same check as the one-step test."""
    test_decode_attention_step(128, p, 1, Hl=64)
