SW_LIB_PATH=variants/libsw_direct.so timeout 600 python -m pytest tests/test_model_gpu.py tests/test_kernels_gpu.py tests/test_gemm_gpu.py -q -x -k "adamw or fused" > gpurun_out/t.log 2>&1; echo EXIT $? >> gpurun_out/t.log
for i in 1 2; do for lib in paper_2310_16355_b200/libshardweave_b200.so variants/libsw_direct.so; do
  echo "$lib"; SW_LIB_PATH=$lib python -c "
import sys, json; sys.path.insert(0,'.')
from tools.gemm_bench import bench_adamw
for sh in [(12288,4096,8192),(4096,11008,8192),(4096,4096,8192)]: print(json.dumps(bench_adamw(*sh)))"
done; done > gpurun_out/d_ab.log 2>&1
