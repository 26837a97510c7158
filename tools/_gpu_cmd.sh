for i in 1 2 3; do for q in 0 1; do echo "dq_first=$q"; SW_ATTN_BWD_DQ_FIRST=$q python tools/attn_bench.py; done; done > gpurun_out/ab.log 2>&1
