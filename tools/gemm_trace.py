"""Per-tile phase trace of one CTA of the CTA-pair GEMM (SW_GEMM_TRACE_CTA): mainloop start/end,
cycles the MMA warp waited for operands, epilogue start/end and, for the AdamW epilogue, cycles
waited for the optimizer-state TMA loads. Usage:
  SW_GEMM_TRACE_CTA=<cta> python tools/gemm_trace.py fused|store [M N K]"""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2310_16355_b200 import _lib  # noqa: E402


def main(kind, M=12288, N=4096, K=8192):
    L = _lib.lib()
    A = torch.randn(K, M, device="cuda").bfloat16()
    B = torch.randn(K, N, device="cuda").bfloat16()
    p, m, v, g = (torch.randn(M, N, device="cuda") * 1e-2 for _ in range(4))
    v.abs_()
    sh = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    flag = torch.zeros(1, device="cuda", dtype=torch.int32)
    s = torch.cuda.current_stream().cuda_stream
    hp = (1e-5, 0.9, 0.999, 1e-8, 0.0, 0.5, 0.5)
    aux = torch.randn(M, N, device="cuda")
    outf = torch.empty(M, N, device="cuda")
    A2 = torch.randn(M, K, device="cuda").bfloat16()
    B2 = torch.randn(N, K, device="cuda").bfloat16()
    for _ in range(3):
        if kind in ("gelu", "gelubwd"):  # fc1 forward (pre + act) / fc2 dgrad with the GeLU derivative
            Cb = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
            C2 = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
            pre = torch.randn(M, N, device="cuda").bfloat16()
            bias = torch.randn(N, device="cuda")
            if kind == "gelu":
                _lib.check(L.sw_k_gemm_bf16(M, N, K, A2.data_ptr(), K, 0, B2.data_ptr(), K, 0, 2, Cb.data_ptr(), N,
                                            C2.data_ptr(), N, bias.data_ptr(), None, 0, 1.0, 0, s))
            else:
                B3 = torch.randn(K, N, device="cuda").bfloat16()
                _lib.check(L.sw_k_gemm_bf16(M, N, K, A2.data_ptr(), K, 0, B3.data_ptr(), N, 1, 4, Cb.data_ptr(), N,
                                            None, 0, None, pre.data_ptr(), N, 1.0, 0, s))
        elif kind == "swiglu":  # fused gate|up forward: N = h columns, B = [gate; up] [2N, K]
            Wgu = torch.randn(2 * N, K, device="cuda").bfloat16()
            Hh = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
            PRE = torch.empty(M, 2 * N, device="cuda", dtype=torch.bfloat16)
            _lib.check(L.sw_k_gemm_bf16_swiglu(M, N, K, A2.data_ptr(), K, Wgu.data_ptr(), K, Hh.data_ptr(), N,
                                               PRE.data_ptr(), 2 * N, s))
        elif kind == "resid":  # forward residual epilogue (kResidF32): K-major operands
            _lib.check(L.sw_k_gemm_bf16(M, N, K, A2.data_ptr(), K, 0, B2.data_ptr(), K, 0, 3, outf.data_ptr(), N,
                                        None, 0, None, aux.data_ptr(), N, 1.0, 0, s))
        elif kind == "fused":
            _lib.check(L.sw_k_gemm_bf16_adamw(M, N, K, A.data_ptr(), M, 1, B.data_ptr(), N, 1, p.data_ptr(),
                                              m.data_ptr(), v.data_ptr(), sh.data_ptr(), N, flag.data_ptr(), *hp, s))
        else:
            _lib.check(L.sw_k_gemm_bf16(M, N, K, A.data_ptr(), M, 1, B.data_ptr(), N, 1, 1, g.data_ptr(), N, None, 0,
                                        None, None, 0, 1.0, 0, s))
    torch.cuda.synchronize()
    buf = (C.c_ulonglong * 1024)()
    L.sw_k_gemm_trace.argtypes = [C.c_void_p]
    _lib.check(L.sw_k_gemm_trace(buf))
    t0 = buf[0]
    rows = []
    for i in range(64):
        b = buf[8 * i:8 * i + 8]
        if b[0] == 0 or b[0] < t0:
            break
        rows.append({"mma": [b[0] - t0, b[1] - t0], "mma_wait_full": b[2], "epi": [b[3] - t0, b[4] - t0, b[5] - t0],
                     "epi_wait_opt": b[6]})
    print(json.dumps({"kind": kind, "cta": int(os.environ.get("SW_GEMM_TRACE_CTA", "-1")), "tiles": rows}))


if __name__ == "__main__":
    main(sys.argv[1], *[int(a) for a in sys.argv[2:]])
