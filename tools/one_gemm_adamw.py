"""One fused wgrad+AdamW GEMM launch (M=12288, N=4096, K=8192) for ncu captures."""
import sys

import torch

sys.path.insert(0, ".")
from tools.gemm_bench import bench_adamw  # noqa: E402

if __name__ == "__main__":
    print(bench_adamw(12288, 4096, 8192, iters=1))
