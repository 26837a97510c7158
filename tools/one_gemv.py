"""One M=1 weight-streaming GEMM (decode GEMV) launch series for ncu: python tools/one_gemv.py N K"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2310_16355_b200 import _lib  # noqa: E402

N, K = (int(x) for x in sys.argv[1:3])
L = _lib.lib()
A = torch.randn(1, K, device="cuda").bfloat16()
Ws = [torch.randn(N, K, device="cuda").bfloat16() for _ in range(4)]  # > L2 together: cold weights
C = torch.empty(1, N, device="cuda", dtype=torch.bfloat16)
for i in range(8):
    W = Ws[i % 4]
    _lib.check(L.sw_k_gemm_bf16(1, N, K, A.data_ptr(), K, 0, W.data_ptr(), K, 0, 0, C.data_ptr(), N, None, 0, None,
                                None, 0, 1.0, 0, None))
torch.cuda.synchronize()
print("ok")
