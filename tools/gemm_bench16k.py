"""The bench's GEMM shapes at 8 x 2048 tokens (M or K = 16384): python tools/gemm_bench16k.py"""
import json
import sys

sys.path.insert(0, ".")
from tools.gemm_bench import bench, bench_adamw  # noqa: E402

if __name__ == "__main__":
    # plain-store epilogues only (bench() passes no bias / aux / second output)
    for sh in [(16384, 12288, 4096, 0, 0, 0), (16384, 11008, 4096, 0, 0, 0), (16384, 4096, 11008, 0, 0, 0),
               (16384, 4096, 4096, 0, 0, 0), (16384, 4096, 11008, 0, 1, 1), (16384, 32000, 4096, 0, 0, 0),
               (11008, 4096, 16384, 1, 1, 1)]:
        print(json.dumps(bench(*sh)), flush=True)
    for sh in [(12288, 4096, 16384), (4096, 11008, 16384)]:
        print(json.dumps(bench_adamw(*sh)), flush=True)
