"""Phase trace of one attention-backward CTA (clock64 stamps written by attn_bwd_tc2 when
SW_ATTN_TRACE_CTA names a CTA). Prints, per query block n, the cycle offsets of:
  mma:  issue_s wait begin / s_free passed / p_full passed
  sm0/sm1 (warps 4, 8): loop top / s_full passed / math done / mma_done passed / p_full arrived
  dq:   dq_full passed / s_free arrived
Usage: SW_ATTN_TRACE_CTA=<cta> python tools/attn_trace.py [B T Hl]"""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2310_16355_b200 import _lib  # noqa: E402


def main(B=4, T=2048, Hl=32, hd=128):
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
    _lib.check(L.sw_k_attention_fwd(qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), B, T, Hl, hd, s))
    for _ in range(3):
        _lib.check(L.sw_k_attention_bwd(qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), dout.data_ptr(),
                                        dqkv.data_ptr(), scratch.data_ptr(), B, T, Hl, hd, s))
    torch.cuda.synchronize()
    buf = (C.c_ulonglong * 4096)()
    L.sw_k_attention_trace.argtypes = [C.c_void_p]
    L.sw_k_attention_trace.restype = C.c_int
    _lib.check(L.sw_k_attention_trace(buf))
    t0 = buf[4000]
    nq = buf[4001]
    rel = lambda x: int(x - t0) if x else None  # noqa: E731
    out = {"cta": int(os.environ.get("SW_ATTN_TRACE_CTA", "-1")), "nq": nq,
           "kv_full": rel(buf[4002]), "epilogue": rel(buf[4003]), "end": rel(buf[4004]), "blocks": []}
    for n in range(min(nq, 64)):
        b = [rel(buf[n * 16 + i]) for i in range(16)]
        out["blocks"].append({"mma": [b[0], b[1], b[2]], "sm0": b[3:8], "sm1": b[8:13], "dq": [b[13], b[14]], "p_full_last": b[15]})
    print(json.dumps(out))


if __name__ == "__main__":
    main(*[int(a) for a in sys.argv[1:]])
