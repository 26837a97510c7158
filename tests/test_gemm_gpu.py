"""tcgen05 GEMM family vs a plain PyTorch fp32 reference of the same op (same bf16 inputs).

Covers both operand majors (forward / dgrad / wgrad layouts of a [out, in] weight), ragged M/N/K
tails, and every fused epilogue."""
import math

import pytest
import torch

from paper_2310_16355_b200 import _lib

pytestmark = pytest.mark.gpu

DEV = "cuda"


def _gemm(A, a_mn, B, b_mn, M, N, K, epi, C, C2=None, bias=None, aux=None, alpha=1.0, acc=0):
    L = _lib.lib()
    lda = A.stride(0)
    ldb = B.stride(0)
    _lib.check(L.sw_k_gemm_bf16(
        M, N, K, A.data_ptr(), lda, a_mn, B.data_ptr(), ldb, b_mn, epi, C.data_ptr(), C.stride(0),
        C2.data_ptr() if C2 is not None else None, C2.stride(0) if C2 is not None else 0,
        bias.data_ptr() if bias is not None else None,
        aux.data_ptr() if aux is not None else None, aux.stride(0) if aux is not None else 0,
        alpha, acc, None))
    torch.cuda.synchronize()


def _ref_operands(M, N, K, a_mn, b_mn, gen):
    a = torch.randn(M, K, generator=gen, device=DEV).bfloat16()
    b = torch.randn(N, K, generator=gen, device=DEV).bfloat16()
    A = a.t().contiguous() if a_mn else a
    B = b.t().contiguous() if b_mn else b
    ref = a.float() @ b.float().t()
    return A, B, ref


def _rel(x, y):
    return ((x.float() - y.float()).norm() / y.float().norm().clamp_min(1e-30)).item()


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 1), (1, 0)])
@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (256, 512, 256), (200, 136, 72),
                                   (512, 1376, 512), (1000, 776, 1000)])
def test_gemm_layouts_f32(M, N, K, a_mn, b_mn):
    gen = torch.Generator(device=DEV).manual_seed(M * 7 + N * 3 + K + a_mn * 2 + b_mn)
    A, B, ref = _ref_operands(M, N, K, a_mn, b_mn, gen)
    C = torch.full((M, N), float("nan"), device=DEV)
    _gemm(A, a_mn, B, b_mn, M, N, K, 1, C)
    assert _rel(C, ref) < 1e-5


@pytest.mark.parametrize("acc", [0, 1])
@pytest.mark.parametrize("M,N,K,a_mn,b_mn", [(4096, 512, 16384, 1, 1), (1376, 4096, 8192, 1, 1),
                                             (512, 256, 4096, 1, 1), (600, 1000, 3000, 1, 1)])
def test_gemm_split_k_f32(M, N, K, a_mn, b_mn, acc):
    """fp32-store weight-gradient GEMMs with too few 256 x 256 tiles for the GPU (the TP = 8
    shards) run split-K: K slices reduce-added into C by TMA (C zeroed first, or accumulated
    into; accumulating GEMMs stay unsplit). The bound is fp32 summation noise over K = 16384
    (an unsplit 16384-deep accumulation measured 1.9e-5); a lost or doubled slice is O(1)."""
    gen = torch.Generator(device=DEV).manual_seed(M + N + K + acc)
    A, B, ref = _ref_operands(M, N, K, a_mn, b_mn, gen)
    C0 = torch.randn(M, N, generator=gen, device=DEV) if acc else torch.full((M, N), float("nan"), device=DEV)
    C = C0.clone()
    _gemm(A, a_mn, B, b_mn, M, N, K, 1, C, acc=acc)
    want = ref + (C0 if acc else 0)
    assert _rel(C, want) < 5e-5


@pytest.mark.parametrize("M,N,K", [(384, 768, 512), (4096, 4096, 4096)])
def test_gemm_bf16_bias(M, N, K):
    gen = torch.Generator(device=DEV).manual_seed(1)
    A, B, ref = _ref_operands(M, N, K, 0, 0, gen)
    bias = torch.randn(N, generator=gen, device=DEV)
    C = torch.empty(M, N, device=DEV, dtype=torch.bfloat16)
    _gemm(A, 0, B, 0, M, N, K, 0, C, bias=bias)
    assert _rel(C, ref + bias) < 1e-2


def test_gemm_bias_gelu():
    M, N, K = 300, 520, 256
    gen = torch.Generator(device=DEV).manual_seed(2)
    A, B, ref = _ref_operands(M, N, K, 0, 0, gen)
    bias = torch.randn(N, generator=gen, device=DEV)
    pre = torch.empty(M, N, device=DEV, dtype=torch.bfloat16)
    act = torch.empty(M, N, device=DEV, dtype=torch.bfloat16)
    _gemm(A, 0, B, 0, M, N, K, 2, pre, C2=act, bias=bias)
    x = ref + bias
    g = 0.5 * x * (1 + torch.tanh(0.7978845608028654 * (x + 0.044715 * x ** 3)))
    assert _rel(pre, x) < 1e-2
    assert _rel(act, g) < 1e-2


def test_gemm_residual_f32():
    M, N, K = 256, 512, 384
    gen = torch.Generator(device=DEV).manual_seed(3)
    A, B, ref = _ref_operands(M, N, K, 0, 0, gen)
    bias = torch.randn(N, generator=gen, device=DEV)
    h = torch.randn(M, N, generator=gen, device=DEV)
    want = h + ref + bias
    _gemm(A, 0, B, 0, M, N, K, 3, h, bias=bias, aux=h)  # in place on the residual stream
    assert _rel(h, want) < 1e-5


def test_gemm_gelu_bwd_dgrad():
    # d_pre = (dy . W) * gelu'(pre) with W stored [out, in] -> B operand MN-major
    M, Nout, Kin = 256, 512, 384  # dy [M, Nout], W [Nout, Kin], result [M, Kin]
    gen = torch.Generator(device=DEV).manual_seed(4)
    dy = torch.randn(M, Nout, generator=gen, device=DEV).bfloat16()
    W = torch.randn(Nout, Kin, generator=gen, device=DEV).bfloat16()
    pre = torch.randn(M, Kin, generator=gen, device=DEV).bfloat16()
    out = torch.empty(M, Kin, device=DEV, dtype=torch.bfloat16)
    _gemm(dy, 0, W, 1, M, Kin, Nout, 4, out, aux=pre)
    x = pre.float()
    t = torch.tanh(0.7978845608028654 * (x + 0.044715 * x ** 3))
    gp = 0.5 * (1 + t) + 0.5 * x * (1 - t * t) * 0.7978845608028654 * (1 + 3 * 0.044715 * x * x)
    want = (dy.float() @ W.float()) * gp
    assert _rel(out, want) < 1e-2


def test_gemm_wgrad_accumulate():
    # dW[N, K] += dy^T x, both operands MN-major (token dim is the reduction dim)
    T, Nout, Kin = 640, 384, 256
    gen = torch.Generator(device=DEV).manual_seed(5)
    dy = torch.randn(T, Nout, generator=gen, device=DEV).bfloat16()
    x = torch.randn(T, Kin, generator=gen, device=DEV).bfloat16()
    dW = torch.randn(Nout, Kin, generator=gen, device=DEV)
    want = dW + dy.float().t() @ x.float()
    _gemm(dy, 1, x, 1, Nout, Kin, T, 1, dW, acc=1)
    assert _rel(dW, want) < 1e-5


@pytest.mark.parametrize("M,N,K", [(384, 320, 512), (200, 136, 72), (1024, 4096, 2048)])
def test_gemm_adamw_epilogue_matches_store_then_adamw(M, N, K):
    """Epi::kAdamW (optimizer in the backward): the wgrad GEMM with AdamW applied in its
    epilogue equals storing the fp32 gradient and running sw_k_adamw on it (same gradient bits,
    same update code), including ragged tiles; the shadow is the bf16 of the new parameter."""
    L = _lib.lib()
    gen = torch.Generator(device=DEV).manual_seed(M + N + K)
    A, B, ref = _ref_operands(M, N, K, 1, 1, gen)
    # gradients and moments spread over ~40 decades so both the branch-free fast path and the
    # IEEE fallback of the epilogue run
    scale = torch.pow(10.0, torch.empty(M, device=DEV).uniform_(-14, 1, generator=gen))
    A.mul_(scale.bfloat16()[None, :])
    ref = A.float().t() @ B.float()
    p = torch.randn(M, N, generator=gen, device=DEV) * 0.05
    m = torch.randn(M, N, generator=gen, device=DEV) * torch.pow(10.0, torch.empty(M, N, device=DEV).uniform_(-30, -1, generator=gen))
    v = torch.rand(M, N, generator=gen, device=DEV) * torch.pow(10.0, torch.empty(M, N, device=DEV).uniform_(-38, -2, generator=gen))
    m[::7] = 0.0
    v[::7] = 0.0
    sh = torch.empty(M, N, device=DEV, dtype=torch.bfloat16)
    p2, m2, v2, sh2 = p.clone(), m.clone(), v.clone(), sh.clone()
    flag = torch.zeros(1, device=DEV, dtype=torch.int32)
    hp = dict(lr=1e-3, b1=0.9, b2=0.999, eps=1e-8, wd=0.01, c1=1 - 0.9 ** 3, c2=1 - 0.999 ** 3)
    _lib.check(L.sw_k_gemm_bf16_adamw(M, N, K, A.data_ptr(), A.stride(0), 1, B.data_ptr(), B.stride(0), 1,
                                      p.data_ptr(), m.data_ptr(), v.data_ptr(), sh.data_ptr(), N, flag.data_ptr(),
                                      *hp.values(), None))
    G = torch.empty(M, N, device=DEV)
    _gemm(A, 1, B, 1, M, N, K, 1, G)
    assert _rel(G, ref) < 1e-5
    _lib.check(L.sw_k_adamw(p2.data_ptr(), m2.data_ptr(), v2.data_ptr(), G.data_ptr(), sh2.data_ptr(), M * N,
                            *hp.values(), None))
    torch.cuda.synchronize()
    assert int(flag.item()) == 0
    assert torch.equal(p, p2) and torch.equal(m, m2) and torch.equal(v, v2) and torch.equal(sh, sh2)


def test_gemm_adamw_epilogue_flags_nonfinite():
    L = _lib.lib()
    M, N, K = 256, 256, 128
    gen = torch.Generator(device=DEV).manual_seed(5)
    A, B, _ = _ref_operands(M, N, K, 1, 1, gen)
    A[7, 9] = float("inf")
    p, m, v = (torch.zeros(M, N, device=DEV) for _ in range(3))
    sh = torch.empty(M, N, device=DEV, dtype=torch.bfloat16)
    flag = torch.zeros(1, device=DEV, dtype=torch.int32)
    _lib.check(L.sw_k_gemm_bf16_adamw(M, N, K, A.data_ptr(), A.stride(0), 1, B.data_ptr(), B.stride(0), 1,
                                      p.data_ptr(), m.data_ptr(), v.data_ptr(), sh.data_ptr(), N, flag.data_ptr(),
                                      1e-3, 0.9, 0.999, 1e-8, 0.0, 0.1, 0.001, None))
    torch.cuda.synchronize()
    assert int(flag.item()) == 1


@pytest.mark.parametrize("M,N,K", [(256, 256, 128), (1024, 4096, 2048)])
def test_gemm_adamw_epilogue_gated_by_flag(M, N, K):
    """A non-zero flag on entry (set by the loss reduction when the loss is non-finite) gates
    every chunk's update: p, m, v and the shadow keep their bytes."""
    L = _lib.lib()
    gen = torch.Generator(device=DEV).manual_seed(M + K)
    A, B, _ = _ref_operands(M, N, K, 1, 1, gen)
    p = torch.randn(M, N, generator=gen, device=DEV)
    m = torch.randn(M, N, generator=gen, device=DEV) * 1e-3
    v = torch.rand(M, N, generator=gen, device=DEV) * 1e-4
    sh = p.bfloat16()
    before = [t.clone() for t in (p, m, v, sh)]
    flag = torch.full((1,), 2, device=DEV, dtype=torch.int32)
    _lib.check(L.sw_k_gemm_bf16_adamw(M, N, K, A.data_ptr(), A.stride(0), 1, B.data_ptr(), B.stride(0), 1,
                                      p.data_ptr(), m.data_ptr(), v.data_ptr(), sh.data_ptr(), N, flag.data_ptr(),
                                      1e-3, 0.9, 0.999, 1e-8, 0.01, 0.1, 0.001, None))
    torch.cuda.synchronize()
    assert int(flag.item()) == 2
    for a, b in zip((p, m, v, sh), before):
        assert torch.equal(a, b)


@pytest.mark.parametrize("M,N,K", [(256, 128, 64), (300, 200, 136), (1000, 1376, 512), (512, 688, 4096),
                                   # decode sizes: the small-M kernels (tensor-core GEMV; K = 136 the
                                   # register-streamed one)
                                   (1, 1376, 4096), (3, 200, 136), (8, 688, 512),
                                   # batched decode: 2 / 4 activation groups per warp, 2 CTA groups
                                   (16, 688, 512), (29, 1376, 4096), (64, 200, 1376), (128, 1376, 4096)])
def test_gemm_swiglu_fwd_bwd(M, N, K):
    """SwiGLU extension vs torch fp32 on the same bf16 operands: the fused [gate; up]
    GEMM writes h = silu(g)*u and the bf16 pre-activations; the down-projection dgrad epilogue
    writes d(gate) | d(up) from them."""
    L = _lib.lib()
    gen = torch.Generator(device=DEV).manual_seed(M + 7 * N + K)
    x = torch.randn(M, K, generator=gen, device=DEV).bfloat16()
    w = (torch.randn(2 * N, K, generator=gen, device=DEV) / math.sqrt(K)).bfloat16()
    h = torch.full((M, N), float("nan"), device=DEV).bfloat16()
    pre = torch.full((M, 2 * N), float("nan"), device=DEV).bfloat16()
    _lib.check(L.sw_k_gemm_bf16_swiglu(M, N, K, x.data_ptr(), K, w.data_ptr(), K, h.data_ptr(), N, pre.data_ptr(),
                                       2 * N, None))
    torch.cuda.synchronize()
    acc = x.float() @ w.float().t()
    g_ref, u_ref = acc[:, :N], acc[:, N:]
    assert _rel(pre[:, :N], g_ref) < 1e-2 and _rel(pre[:, N:], u_ref) < 1e-2
    gb, ub = pre[:, :N].float(), pre[:, N:].float()
    assert _rel(h, torch.nn.functional.silu(gb) * ub) < 1e-2

    # backward: dh = dY . W_down (dY [M, D], W_down [D, N] used MN-major like the executor)
    D = 96
    dy = torch.randn(M, D, generator=gen, device=DEV).bfloat16()
    wd = (torch.randn(D, N, generator=gen, device=DEV) / math.sqrt(N)).bfloat16()
    dpre = torch.full((M, 2 * N), float("nan"), device=DEV).bfloat16()
    _lib.check(L.sw_k_gemm_bf16_swiglu_bwd(M, N, D, dy.data_ptr(), D, 0, wd.data_ptr(), N, 1, pre.data_ptr(), 2 * N,
                                           dpre.data_ptr(), 2 * N, None))
    torch.cuda.synchronize()
    dh = dy.float() @ wd.float()
    sg = torch.sigmoid(gb)
    want_g = dh * ub * sg * (1 + gb * (1 - sg))
    want_u = dh * torch.nn.functional.silu(gb)
    assert _rel(dpre[:, :N], want_g) < 1e-2 and _rel(dpre[:, N:], want_u) < 1e-2


@pytest.mark.parametrize("M", [1, 3, 8, 12, 16, 29, 32, 47, 64, 65, 100, 128])
@pytest.mark.parametrize("epi", [0, 1, 3])
@pytest.mark.parametrize("N,K", [(200, 136), (4096, 1376), (12288, 4096)])
def test_small_m_gemv_path(M, epi, N, K):
    """Decode-size forward GEMMs take the weight-streaming kernels: M <= 8 the mma.sync one (the
    register-streamed one when K % 32 != 0), 9 <= M <= 128 the tcgen05 swap-AB kernel (weight rows
    as the MMA M, K slices reduced across a cluster through distributed shared memory; ragged M,
    N = 200 in a partial 128-row block, K = 136 / 1376 in partial 64-deep boxes); same epilogues."""
    gen = torch.Generator(device=DEV).manual_seed(M * 10 + epi)
    A, B, ref = _ref_operands(M, N, K, 0, 0, gen)
    bias = torch.randn(N, generator=gen, device=DEV)
    if epi == 0:
        C = torch.empty(M, N, device=DEV, dtype=torch.bfloat16)
        _gemm(A, 0, B, 0, M, N, K, 0, C, bias=bias)
        want = ref + bias
    elif epi == 1:
        C = torch.full((M, N), float("nan"), device=DEV)
        _gemm(A, 0, B, 0, M, N, K, 1, C)
        want = ref
    else:
        aux = torch.randn(M, N, generator=gen, device=DEV)
        C = torch.empty(M, N, device=DEV)
        _gemm(A, 0, B, 0, M, N, K, 3, C, bias=bias, aux=aux)
        want = aux + ref + bias
    assert _rel(C, want) < (1e-2 if epi == 0 else 1e-5)


@pytest.mark.parametrize("Bs,T,H,K", [(2, 320, 4, 384), (1, 2048, 2, 4096)])
def test_gemm_dout_with_attention_delta(Bs, T, H, K):
    """epi 8: the attention-output-gradient GEMM (dO = g x Wo, Wo MN-major) also writes the flash
    backward's delta[b, h, t] = sum_c dO[b*T+t, h*128+c] * O[b*T+t, h*128+c] from the bf16 dO it
    stores (replaces attn_bwd's separate delta pass)."""
    M, N = Bs * T, H * 128
    gen = torch.Generator(device=DEV).manual_seed(T + K)
    g = torch.randn(M, K, generator=gen, device=DEV).bfloat16()
    wo = torch.randn(K, N, generator=gen, device=DEV).bfloat16()  # [d, dl]: B operand MN-major
    O = torch.randn(M, N, generator=gen, device=DEV).bfloat16()
    dO = torch.empty(M, N, device=DEV, dtype=torch.bfloat16)
    delta = torch.full((Bs * H * T,), float("nan"), device=DEV)
    L = _lib.lib()
    _lib.check(L.sw_k_gemm_bf16(M, N, K, g.data_ptr(), K, 0, wo.data_ptr(), N, 1, 8, dO.data_ptr(), N,
                                delta.data_ptr(), T, None, O.data_ptr(), N, 1.0, 0, None))
    torch.cuda.synchronize()
    want = g.float() @ wo.float()
    assert _rel(dO, want) < 1e-2
    ref = (dO.float() * O.float()).view(Bs, T, H, 128).sum(-1).permute(0, 2, 1).reshape(-1)
    assert torch.isfinite(delta).all()
    assert torch.allclose(delta, ref, rtol=1e-5, atol=1e-3)


def test_gemm_dout_delta_rejects_ragged_heads():
    L = _lib.lib()
    x = torch.zeros(256, 200, device=DEV, dtype=torch.bfloat16)
    w = torch.zeros(64, 200, device=DEV, dtype=torch.bfloat16)
    d = torch.zeros(256 * 2, device=DEV)
    st = L.sw_k_gemm_bf16(256, 200, 64, torch.zeros(256, 64, device=DEV, dtype=torch.bfloat16).data_ptr(), 64, 0,
                          w.data_ptr(), 200, 1, 8, x.data_ptr(), 200, d.data_ptr(), 128, None, x.data_ptr(), 200,
                          1.0, 0, None)
    assert st != 0
