"""One tcgen05 GEMM shape for ncu captures: python tools/one_gemm.py M N K a_mn b_mn epi"""
import sys

sys.path.insert(0, ".")
from tools.gemm_bench import bench  # noqa: E402

if __name__ == "__main__":
    M, N, K, a, b, e = (int(x) for x in sys.argv[1:7])
    print(bench(M, N, K, a, b, e, iters=2))
