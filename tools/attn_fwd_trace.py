"""Phase trace of one attention-forward CTA (clock64 stamps written by attn_fwd_tc2 when
SW_ATTN_TRACE_CTA names a CTA). Per tile-block k of the CTA (both tiles, in issue order):
  mma:  p_full wait begin / passed (the P V issue of that tile's block)
  sm:   s_full wait begin / passed / math done / p_full arrived
Per item i: MMA q_full wait begin / passed / kv_full passed; softmax-A O epilogue done.
Slots 4090-4093: clock64 + globaltimer at kernel start / end (gives the SM clock).
Usage: SW_ATTN_TRACE_CTA=<cta> python tools/attn_fwd_trace.py [B T Hl]"""
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
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(4):
        _lib.check(L.sw_k_attention_fwd(qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), B, T, Hl, hd, s))
    torch.cuda.synchronize()
    buf = (C.c_ulonglong * 4096)()
    L.sw_k_attention_trace.argtypes = [C.c_void_p]
    L.sw_k_attention_trace.restype = C.c_int
    _lib.check(L.sw_k_attention_trace(buf))
    t0 = buf[4090]
    mhz = (buf[4092] - buf[4090]) / max(1, (buf[4093] - buf[4091])) * 1e3
    rel = lambda x: int(x - t0) if x else None  # noqa: E731
    out = {"cta": int(os.environ.get("SW_ATTN_TRACE_CTA", "-1")), "sm_mhz": round(mhz, 1),
           "total": rel(buf[4092]), "items": [], "blocks": []}
    for i in range(16):
        it = [rel(buf[4000 + 4 * i + k]) for k in range(4)]
        if any(x is not None for x in it):
            out["items"].append(it)
    for k in range(3900 // 16):
        b = [rel(buf[k * 16 + i]) for i in range(12)]
        if all(x is None for x in b):
            continue
        out["blocks"].append({"k": k, "mmaA": b[0:2], "mmaB": b[2:4], "smA": b[4:8], "smB": b[8:12]})
    print(json.dumps(out))


if __name__ == "__main__":
    main(*[int(a) for a in sys.argv[1:]])
