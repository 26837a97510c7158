"""Times the attention kernels at the LLaMA-7B shape (B=4, T=2048, H=32, hd=128) with CUDA
events; checks them against torch SDPA (fp32 math on the same bf16 inputs) on a slice."""
import json
import math
import sys

import torch

sys.path.insert(0, ".")
from paper_2310_16355_b200 import _lib  # noqa: E402


def main(B=4, T=2048, Hl=32, hd=128, iters=10):
    L = _lib.lib()
    Dl = Hl * hd
    g = torch.Generator(device="cuda").manual_seed(0)
    qkv = torch.randn(B * T, 3 * Dl, generator=g, device="cuda").bfloat16()
    o = torch.empty(B * T, Dl, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(B, Hl, T, device="cuda")
    dout = torch.randn(B * T, Dl, generator=g, device="cuda").bfloat16()
    dqkv = torch.empty_like(qkv)
    scratch = torch.empty(L.sw_k_attention_bwd_scratch(B, T, Hl, hd), device="cuda")
    s = torch.cuda.current_stream().cuda_stream

    def fwd():
        _lib.check(L.sw_k_attention_fwd(qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), B, T, Hl, hd, s))

    def bwd():
        _lib.check(L.sw_k_attention_bwd(qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), dout.data_ptr(),
                                        dqkv.data_ptr(), scratch.data_ptr(), B, T, Hl, hd, s))

    def timeit(fn):
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / iters

    flops_fwd = 2.0 * B * Hl * T * T * hd  # causal: half of 4*B*H*T^2*hd
    res = {"shape": [B, T, Hl, hd]}
    ms = timeit(fwd)
    res["fwd_ms"] = ms
    res["fwd_tflops"] = flops_fwd / ms / 1e9
    ms = timeit(bwd)
    res["bwd_ms"] = ms
    res["bwd_tflops"] = 2 * flops_fwd / ms / 1e9
    # torch SDPA (flash) for context
    x = qkv.view(B, T, 3, Hl, hd)
    q, k, v = (x[:, :, i].transpose(1, 2).contiguous() for i in range(3))
    sd = lambda: torch.nn.functional.scaled_dot_product_attention(q, k, v, is_causal=True)  # noqa: E731
    ms = timeit(sd)
    res["torch_sdpa_fwd_tflops"] = flops_fwd / ms / 1e9
    qg, kg, vg = (t.detach().requires_grad_(True) for t in (q, k, v))
    og = torch.nn.functional.scaled_dot_product_attention(qg, kg, vg, is_causal=True)
    go = torch.randn_like(og)
    sdb = lambda: torch.autograd.grad(og, (qg, kg, vg), go, retain_graph=True)  # noqa: E731
    ms = timeit(sdb)
    res["torch_sdpa_bwd_tflops"] = 2 * flops_fwd / ms / 1e9
    # correctness on the first (b, h)
    fwd()
    torch.cuda.synchronize()
    ref = torch.nn.functional.scaled_dot_product_attention(q.float(), k.float(), v.float(), is_causal=True)
    got = o.view(B, T, Hl, hd).transpose(1, 2).float()
    res["fwd_rel_err"] = ((got - ref).norm() / ref.norm()).item()
    print(json.dumps(res))


if __name__ == "__main__":
    main(*[int(a) for a in sys.argv[1:]])
