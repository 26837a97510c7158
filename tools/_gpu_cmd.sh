timeout 600 python -m pytest tests -m gpu -q > gpurun_out/t.log 2>&1; echo EXIT $? >> gpurun_out/t.log
timeout 600 python bench.py > gpurun_out/r1c_bench.log 2>&1
rm -f gpurun_out/prof.csv; SW_PROFILE_LOG=gpurun_out/prof.csv timeout 400 python bench.py --spec oracle/specs/llama7b_swiglu.spec --no-cpu-baseline > gpurun_out/r1c_bench_swiglu.log 2>&1
python tools/gemm_shape_report.py gpurun_out/prof.csv 2 > gpurun_out/r1c_swiglu_shapes.log
