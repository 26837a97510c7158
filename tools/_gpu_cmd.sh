timeout 300 python -m pytest tests/test_kernels_gpu.py -x -q -k attention > gpurun_out/t.log 2>&1; echo EXIT $? >> gpurun_out/t.log
for i in 1 2 3; do for v in 0 1; do echo "ts=$v"; SW_ATTN_BWD_TS=$v python tools/attn_bench.py; done; done > gpurun_out/ab.log 2>&1
SW_ATTN_TRACE_CTA=700 python tools/attn_trace.py > gpurun_out/trace.log 2>&1
