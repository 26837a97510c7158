"""One fused wgrad+AdamW GEMM launch for ncu captures: python tools/one_gemm_adamw.py [M N K]
(default the QKV wgrad of the bench at 8 x 2048 tokens: M=12288 N=4096 K=16384)."""
import sys

import torch

sys.path.insert(0, ".")
from tools.gemm_bench import bench_adamw  # noqa: E402

if __name__ == "__main__":
    M, N, K = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (12288, 4096, 16384)
    print(bench_adamw(M, N, K, iters=1))
    torch.cuda.synchronize()
