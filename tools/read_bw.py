import torch
for mb in (32, 100, 1000):
    n = mb * 1024 * 1024 // 4
    x = torch.ones(n, device="cuda", dtype=torch.int32)
    for _ in range(3): x.sum()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(20): x.sum()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(mb, "MB read:", round(ms * 1e3, 1), "us", round(n * 4 / ms / 1e6), "GB/s")
