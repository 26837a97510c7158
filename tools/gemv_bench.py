"""Weight-streaming small-M GEMM path (decode) bandwidth: python tools/gemv_bench.py"""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2310_16355_b200 import _lib  # noqa: E402


def run(M, N, K, iters=50):
    L = _lib.lib()
    A = torch.randn(M, K, device="cuda").bfloat16()
    # enough weight copies to exceed L2 (126 MB) several times over: every launch streams from HBM
    n_w = max(2, -(-512 * 2**20 // (N * K * 2)))
    Ws = [torch.randn(N, K, device="cuda").bfloat16() for _ in range(n_w)]
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    s = torch.cuda.current_stream().cuda_stream
    it = [0]

    def f():
        W = Ws[it[0] % n_w]
        it[0] += 1
        _lib.check(L.sw_k_gemm_bf16(M, N, K, A.data_ptr(), K, 0, W.data_ptr(), K, 0, 0, C.data_ptr(), N,
                                    None, 0, None, None, 0, 1.0, 0, s))
    for _ in range(5):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(iters):
        f()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    return {"M": M, "N": N, "K": K, "us": round(ms * 1e3, 1), "weight_gbs": round(N * K * 2 / ms / 1e6, 1)}


if __name__ == "__main__":
    if len(sys.argv) > 1:  # M list: the decode projections of LLaMA-7B at each M
        for M in (int(x) for x in sys.argv[1].split(",")):
            for N, K in ((12288, 4096), (4096, 4096), (22016, 4096), (4096, 11008)):
                print(json.dumps(run(M, N, K)))
        sys.exit(0)
    for sh in [(1, 12288, 4096), (1, 4096, 4096), (1, 11008, 4096), (1, 4096, 11008), (1, 32000, 4096),
               (4, 12288, 4096), (8, 4096, 11008)]:
        print(json.dumps(run(*sh)))
