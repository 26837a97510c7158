set -x
timeout 600 python bench.py > gpurun_out/r1b_bench.log 2>&1
timeout 300 python bench.py --impl reference > gpurun_out/r1b_bench_ref.log 2>&1
timeout 400 python bench.py --spec oracle/specs/llama7b_swiglu.spec --no-cpu-baseline > gpurun_out/r1b_bench_swiglu.log 2>&1
rm -f gpurun_out/prof.csv; SW_PROFILE_LOG=gpurun_out/prof.csv timeout 400 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/r1b_bench_shapes_run.log 2>&1
python tools/gemm_shape_report.py gpurun_out/prof.csv 2 > gpurun_out/r1b_gemm_shapes.log
python tools/profile_step.py > gpurun_out/plain.log 2>&1 && \
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1b_launches.csv python tools/profile_step.py > gpurun_out/ncu1.log 2>&1
python tools/attn_bench.py > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:attn_bwd_tc2 -s 3 -c 1 -o gpurun_out/r1b_attn_bwd python tools/attn_bench.py > gpurun_out/ncu2.log 2>&1
python tools/one_gemm_adamw.py > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none -k regex:gemm_bf16_2sm -c 1 -o gpurun_out/r1b_gemm_adamw python tools/one_gemm_adamw.py > gpurun_out/ncu3.log 2>&1
echo done
