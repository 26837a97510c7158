"""KV-cached decode attention step timing (split-key kernel): python tools/decode_attn_bench.py
Back-to-back launches on one stream, B = 1, T = 2048, head dim 128, LLaMA-7B (32 heads) and
OPT-66B (72 heads) widths at several positions."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2310_16355_b200 import _lib  # noqa: E402


def run(Hl, p, B=1, T=2048, hd=128, iters=200):
    L = _lib.lib()
    Dl = Hl * hd
    cache = torch.randn(B * T, 3 * Dl, device="cuda").bfloat16()
    new = torch.randn(B, 3 * Dl, device="cuda").bfloat16()
    out = torch.empty(B, Dl, device="cuda", dtype=torch.bfloat16)
    part = torch.empty(B * Hl * 64 * (hd + 2), device="cuda")
    ticket = torch.zeros(B * Hl, device="cuda", dtype=torch.int32)
    f = lambda: _lib.check(L.sw_k_decode_attention(  # noqa: E731
        new.data_ptr(), cache.data_ptr(), out.data_ptr(), B, T, p, Hl, hd, 1, part.data_ptr(), ticket.data_ptr(),
        torch.cuda.current_stream().cuda_stream))
    for _ in range(10):
        f()
    torch.cuda.synchronize()
    # one CUDA graph of `iters` launches: the host launch rate (a few us per ctypes call) would
    # otherwise be what is timed, as in the decode step, which is one graph launch too
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(iters):
            f()
    g.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / iters * 1e3
    byts = 2 * B * (p + 1) * Dl * 2
    return {"Hl": Hl, "p": p, "B": B, "us": round(us, 2), "kv_gbs": round(byts / us / 1e3, 1)}


if __name__ == "__main__":
    if len(sys.argv) > 1:  # batched: python tools/decode_attn_bench.py B [Hl p]
        B = int(sys.argv[1])
        Hl = int(sys.argv[2]) if len(sys.argv) > 2 else 32
        for p in ([int(sys.argv[3])] if len(sys.argv) > 3 else (512, 1024)):
            print(json.dumps(run(Hl, p, B=B, iters=50)))
        sys.exit(0)
    for Hl in (32, 72):
        for p in (128, 512, 1024, 2000):
            print(json.dumps(run(Hl, p)))
