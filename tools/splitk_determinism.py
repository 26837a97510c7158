"""Run-to-run differences of a split-K weight-gradient GEMM: python tools/splitk_determinism.py"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2310_16355_b200 import _lib  # noqa: E402

L = _lib.lib()
M, N, K = 4096, 1024, 2048
g = torch.Generator(device="cuda").manual_seed(0)
A = (torch.randn(K, M, generator=g, device="cuda") * 1e-3).bfloat16()  # MN-major [K, M]
B = torch.randn(K, N, generator=g, device="cuda").bfloat16()
outs = []
for i in range(4):
    C = torch.empty(M, N, device="cuda")
    _lib.check(L.sw_k_gemm_bf16(M, N, K, A.data_ptr(), M, 1, B.data_ptr(), N, 1, 1, C.data_ptr(), N, None, 0,
                                None, None, 0, 1.0, 0, None))
    torch.cuda.synchronize()
    outs.append(C)
ref = A.float().t() @ B.float()
for C in outs:
    print(((C - outs[0]).norm() / outs[0].norm()).item(), ((C - ref).norm() / ref.norm()).item())
