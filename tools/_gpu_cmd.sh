for i in 1 2; do
for lib in paper_2310_16355_b200/libshardweave_b200.so variants/libsw_bigbox.so variants/libsw_bigbox8.so; do
  echo "$lib"; SW_LIB_PATH=$lib python -c "
import sys, json; sys.path.insert(0,'.')
from tools.gemm_bench import bench_adamw
for sh in [(12288,4096,8192),(4096,11008,8192)]: print(json.dumps(bench_adamw(*sh)))"
done; done > gpurun_out/bb_ab.log 2>&1
SW_LIB_PATH=variants/libsw_bigbox.so SW_GEMM_TRACE_CTA=0 python tools/gemm_trace.py fused >> gpurun_out/bb_ab.log 2>&1
