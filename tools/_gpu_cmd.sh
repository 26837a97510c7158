for i in 1 2; do for lib in paper_2310_16355_b200/libshardweave_b200.so variants/libsw_noload.so variants/libsw_nostore.so variants/libsw_noboth.so; do
echo "$lib $(SW_LIB_PATH=$lib python -c 'import sys; sys.path.insert(0,"."); from tools.gemm_bench import bench_adamw; print(bench_adamw(12288,4096,8192,iters=10))' 2>&1 | tail -1)"
done; done > gpurun_out/adamw_exp.log 2>&1
