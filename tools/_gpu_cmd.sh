timeout 900 python -m pytest tests -m gpu -q > gpurun_out/t.log 2>&1; echo EXIT $? >> gpurun_out/t.log
timeout 600 python bench.py > gpurun_out/r1d_bench.log 2>&1
timeout 300 python bench.py --impl reference > gpurun_out/r1d_bench_ref.log 2>&1
rm -f gpurun_out/prof.csv; SW_PROFILE_LOG=gpurun_out/prof.csv timeout 400 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/r1d_run.log 2>&1
python tools/gemm_shape_report.py gpurun_out/prof.csv 2 > gpurun_out/r1d_gemm_shapes.log
python tools/profile_step.py > gpurun_out/plain.log 2>&1 && \
ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1d_launches.csv python tools/profile_step.py > gpurun_out/ncu1.log 2>&1
echo done
