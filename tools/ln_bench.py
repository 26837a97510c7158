"""Times the LayerNorm kernels at the LLaMA-7B step shape (8192 x 4096) with CUDA events and
reports achieved HBM bandwidth (fwd 12 B/elem: fp32 x in, bf16 y out... as DESIGN §5 counts)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2310_16355_b200 import _lib  # noqa: E402


def main(M=8192, d=4096, iters=20):
    L = _lib.lib()
    x = torch.randn(M, d, device="cuda")
    s = torch.randn(d, device="cuda")
    b = torch.randn(d, device="cuda")
    y = torch.empty(M, d, device="cuda", dtype=torch.bfloat16)
    mean = torch.empty(M, device="cuda")
    rstd = torch.empty(M, device="cuda")
    dy = torch.randn(M, d, device="cuda")
    gio = torch.randn(M, d, device="cuda")
    gb = torch.empty(M, d, device="cuda", dtype=torch.bfloat16)
    ds = torch.zeros(d, device="cuda")
    dbias = torch.zeros(d, device="cuda")

    def fwd():
        _lib.check(L.sw_k_layernorm_fwd(x.data_ptr(), s.data_ptr(), b.data_ptr(), y.data_ptr(), mean.data_ptr(),
                                        rstd.data_ptr(), M, d, 1e-5, None))

    def bwd():
        _lib.check(L.sw_k_layernorm_bwd(x.data_ptr(), mean.data_ptr(), rstd.data_ptr(), s.data_ptr(), dy.data_ptr(),
                                        gio.data_ptr(), gb.data_ptr(), ds.data_ptr(), dbias.data_ptr(), M, d, 1,
                                        None))

    res = {"M": M, "d": d}
    for name, fn, byts in (("fwd", fwd, 6 * M * d), ("bwd", bwd, 18 * M * d)):
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / iters
        res[name + "_us"] = round(ms * 1000, 1)
        res[name + "_gbs"] = round(byts / ms / 1e6, 1)
    print(json.dumps(res))


if __name__ == "__main__":
    main(*[int(a) for a in sys.argv[1:]])
