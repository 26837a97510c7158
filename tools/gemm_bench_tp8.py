"""Per-rank GEMM shapes of the LLaMA-7B step at TP=8 (8 x 2048 tokens): python tools/gemm_bench_tp8.py
(forward, dgrad and wgrad layouts with the plain store epilogues; the fused ones are timed in the step)."""
import json
import sys

sys.path.insert(0, ".")
from tools.gemm_bench import bench  # noqa: E402

if __name__ == "__main__":
    M = 16384
    for sh in [(M, 1536, 4096, 0, 0, 0), (M, 4096, 512, 0, 0, 1), (M, 1376, 4096, 0, 0, 0), (M, 4096, 1376, 0, 0, 1),
               (M, 4096, 1536, 0, 1, 1), (M, 512, 4096, 0, 1, 0), (M, 4096, 1376, 0, 1, 1), (M, 1376, 4096, 0, 1, 0),
               (1536, 4096, M, 1, 1, 1), (4096, 512, M, 1, 1, 1), (1376, 4096, M, 1, 1, 1), (4096, 1376, M, 1, 1, 1),
               (M, 4000, 4096, 0, 0, 0)]:
        print(json.dumps(bench(*sh)), flush=True)
