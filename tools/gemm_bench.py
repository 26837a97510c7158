"""Times the tcgen05 GEMM family on the shapes of the LLaMA-7B-shape step (CUDA events)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2310_16355_b200 import _lib  # noqa: E402


def bench(M, N, K, a_mn=0, b_mn=0, epi=1, iters=20):
    L = _lib.lib()
    A = torch.randn((K, M) if a_mn else (M, K), device="cuda").bfloat16()
    B = torch.randn((K, N) if b_mn else (N, K), device="cuda").bfloat16()
    C = torch.empty(M, N, device="cuda", dtype=torch.float32 if epi == 1 else torch.bfloat16)
    s = torch.cuda.current_stream().cuda_stream

    def run():
        _lib.check(L.sw_k_gemm_bf16(M, N, K, A.data_ptr(), A.stride(0), a_mn, B.data_ptr(),
                                    B.stride(0), b_mn, epi, C.data_ptr(), C.stride(0), None, 0,
                                    None, None, 0, 1.0, 0, s))
    for _ in range(3):
        run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(iters):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    tf = 2.0 * M * N * K / ms / 1e9
    # cuBLAS for context
    a = A.t() if a_mn else A
    b = B if b_mn else B.t()
    for _ in range(3):
        torch.matmul(a, b)
    e0.record()
    for _ in range(iters):
        torch.matmul(a, b)
    e1.record()
    torch.cuda.synchronize()
    ms_cb = e0.elapsed_time(e1) / iters
    return {"M": M, "N": N, "K": K, "a_mn": a_mn, "b_mn": b_mn, "epi": epi, "ms": round(ms, 4),
            "tflops": round(tf, 1), "cublas_tflops": round(2.0 * M * N * K / ms_cb / 1e9, 1)}


if __name__ == "__main__" and "--adamw" not in sys.argv:
    shapes = [(8192, 8192, 8192, 0, 0, 0), (8192, 12288, 4096, 0, 0, 0),
              (8192, 11008, 4096, 0, 0, 0), (8192, 4096, 11008, 0, 0, 0),
              (8192, 4096, 11008, 0, 1, 1), (11008, 4096, 8192, 1, 1, 1),
              (8192, 32000, 4096, 0, 0, 0)]
    for sh in shapes:
        print(json.dumps(bench(*sh)), flush=True)


def bench_adamw(M, N, K, iters=10):
    """wgrad layout (both operands MN-major) with the AdamW epilogue vs the fp32-store epilogue
    followed by the flat AdamW kernel: the optimizer-in-backward trade."""
    L = _lib.lib()
    A = torch.randn(K, M, device="cuda").bfloat16()
    B = torch.randn(K, N, device="cuda").bfloat16()
    p, m, v, g = (torch.randn(M, N, device="cuda") * 1e-2 for _ in range(4))
    v.abs_()
    sh = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    flag = torch.zeros(1, device="cuda", dtype=torch.int32)
    s = torch.cuda.current_stream().cuda_stream
    hp = (1e-5, 0.9, 0.999, 1e-8, 0.0, 0.5, 0.5)

    def fused():
        _lib.check(L.sw_k_gemm_bf16_adamw(M, N, K, A.data_ptr(), M, 1, B.data_ptr(), N, 1, p.data_ptr(),
                                          m.data_ptr(), v.data_ptr(), sh.data_ptr(), N, flag.data_ptr(), *hp, s))

    def store():
        _lib.check(L.sw_k_gemm_bf16(M, N, K, A.data_ptr(), M, 1, B.data_ptr(), N, 1, 1, g.data_ptr(), N, None, 0,
                                    None, None, 0, 1.0, 0, s))

    def adamw():
        _lib.check(L.sw_k_adamw(p.data_ptr(), m.data_ptr(), v.data_ptr(), g.data_ptr(), sh.data_ptr(), M * N, *hp, s))

    out = {"M": M, "N": N, "K": K}
    for name, fn in (("fused", fused), ("store", store), ("adamw", adamw)):
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        out[name + "_ms"] = round(e0.elapsed_time(e1) / iters, 4)
    out["fused_tflops"] = round(2.0 * M * N * K / out["fused_ms"] / 1e9, 1)
    out["store_tflops"] = round(2.0 * M * N * K / out["store_ms"] / 1e9, 1)
    return out


if __name__ == "__main__" and "--adamw" in sys.argv:
    for sh in [(12288, 4096, 8192), (4096, 4096, 8192), (11008, 4096, 8192), (4096, 11008, 8192),
               (16000, 4096, 8192)]:
        print(json.dumps(bench_adamw(*sh)), flush=True)
