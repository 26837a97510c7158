"""Phase trace of one head-dim-256 dV-pass CTA: SW_ATTN_TRACE_HD256=1 SW_ATTN_TRACE_DV=1
SW_ATTN_TRACE_CTA=<cta> python tools/attn256_dv_trace.py. Per query block n: MMA (before / after
the p_full wait), softmax warp 4 (s_full wait begin / passed / P stored); slot 2000 = MMA start,
2001 = softmax loop end."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2310_16355_b200 import _lib  # noqa: E402

L = _lib.lib()
B, T, Hl, hd = 4, 2048, 16, 256
Dl = Hl * hd
g = torch.Generator(device="cuda").manual_seed(0)
qkv = torch.randn(B * T, 3 * Dl, generator=g, device="cuda").bfloat16()
o = torch.empty(B * T, Dl, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(B, Hl, T, device="cuda")
dout = torch.randn(B * T, Dl, generator=g, device="cuda").bfloat16()
dqkv = torch.empty_like(qkv)
scr = torch.empty(B * T * Hl + B * T * 2 * Dl, device="cuda")
L.sw_k_attention_fwd(qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), B, T, Hl, hd, None)
for _ in range(3):
    L.sw_k_attention_bwd(qkv.data_ptr(), o.data_ptr(), lse.data_ptr(), dout.data_ptr(), dqkv.data_ptr(),
                         scr.data_ptr(), B, T, Hl, hd, None)
torch.cuda.synchronize()
buf = (C.c_ulonglong * 4096)()
L.sw_k_attention_trace.argtypes = [C.c_void_p]
L.sw_k_attention_trace(buf)
t0 = buf[2000]
print("end", buf[2001] - t0)
for n in range(40):
    b = [buf[16 * n + i] for i in (0, 1, 4, 5, 6)]
    if b[0] == 0:
        break
    print(n, [int(x - t0) if x else None for x in b])
