"""Runs one GEMM flavour (fused AdamW wgrad / store-only wgrad / flat AdamW) back to back for a few
seconds while sampling nvidia-smi SM clock and power: tells power-cap throttling apart from
kernel inefficiency. Usage: python tools/clock_probe.py fused|store|adamw [M N K]"""
import json
import subprocess
import sys
import threading
import time

import torch

sys.path.insert(0, ".")
from paper_2310_16355_b200 import _lib  # noqa: E402


def main(kind, M=12288, N=4096, K=8192, seconds=4.0):
    L = _lib.lib()
    A = torch.randn(K, M, device="cuda").bfloat16()
    B = torch.randn(K, N, device="cuda").bfloat16()
    p, m, v, g = (torch.randn(M, N, device="cuda") * 1e-2 for _ in range(4))
    v.abs_()
    sh = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    flag = torch.zeros(1, device="cuda", dtype=torch.int32)
    s = torch.cuda.current_stream().cuda_stream
    hp = (1e-5, 0.9, 0.999, 1e-8, 0.0, 0.5, 0.5)
    fns = {
        "fused": lambda: L.sw_k_gemm_bf16_adamw(M, N, K, A.data_ptr(), M, 1, B.data_ptr(), N, 1, p.data_ptr(),
                                                m.data_ptr(), v.data_ptr(), sh.data_ptr(), N, flag.data_ptr(), *hp, s),
        "store": lambda: L.sw_k_gemm_bf16(M, N, K, A.data_ptr(), M, 1, B.data_ptr(), N, 1, 1, g.data_ptr(), N, None, 0,
                                          None, None, 0, 1.0, 0, s),
    }
    fn = fns[kind]
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    samples = []
    stop = threading.Event()

    def sampler():
        while not stop.is_set():
            out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits"],
                                 capture_output=True, text=True).stdout.strip().split(",")
            try:
                samples.append((float(out[0]), float(out[1])))
            except (ValueError, IndexError):
                pass
            time.sleep(0.1)

    th = threading.Thread(target=sampler)
    th.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 0
    t0 = time.time()
    e0.record()
    while time.time() - t0 < seconds:
        for _ in range(20):
            fn()
        n += 20
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    stop.set()
    th.join()
    ms = e0.elapsed_time(e1) / n
    mid = samples[len(samples) // 4:] or samples
    print(json.dumps({"kind": kind, "ms": round(ms, 4), "tflops": round(2.0 * M * N * K / ms / 1e9, 1),
                      "sm_mhz": sorted(x[0] for x in mid)[len(mid) // 2],
                      "power_w": sorted(x[1] for x in mid)[len(mid) // 2], "samples": len(samples)}))


if __name__ == "__main__":
    main(sys.argv[1], *[int(a) for a in sys.argv[2:]])
