for i in 1 2; do for lib in paper_2310_16355_b200/libshardweave_b200.so variants/libsw_nostate.so variants/libsw_noshadow.so; do
  echo "$lib"; SW_LIB_PATH=$lib python -c "
import sys, json; sys.path.insert(0,'.')
from tools.gemm_bench import bench_adamw
for sh in [(12288,4096,8192)]: print(json.dumps(bench_adamw(*sh)))"
done; done > gpurun_out/x_ab.log 2>&1
