timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t.log 2>&1; echo EXIT $? >> gpurun_out/t.log
SW_GEMM_TRACE_CTA=0 python tools/gemm_trace.py gelu 8192 11008 4096 > gpurun_out/gtr.log 2>&1
SW_GEMM_TRACE_CTA=0 python tools/gemm_trace.py gelubwd 8192 11008 4096 >> gpurun_out/gtr.log 2>&1
for i in 1 2; do for lib in variants/libsw_prev.so paper_2310_16355_b200/libshardweave_b200.so; do
SW_LIB_PATH=$lib timeout 400 python bench.py --no-cpu-baseline --steps 8 > gpurun_out/b.log 2>&1
echo "$lib $(python3 -c "import json; d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]); print(round(d['value']), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['breakdown_ms_per_step']['gemm'])")"
done; done > gpurun_out/ab.log 2>&1
for lib in variants/libsw_prev.so paper_2310_16355_b200/libshardweave_b200.so; do echo "== $lib"; SW_LIB_PATH=$lib timeout 300 python tools/gemm_shape_report.py 2>&1 | grep -E "epi2|epi4" ; done > gpurun_out/shapes.log 2>&1
