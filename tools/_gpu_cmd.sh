timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/t.log 2>&1; echo EXIT $? >> gpurun_out/t.log
for i in 1 2; do for lib in variants/libsw_tanhf.so paper_2310_16355_b200/libshardweave_b200.so; do
rm -f gpurun_out/prof.csv; SW_LIB_PATH=$lib SW_PROFILE_LOG=gpurun_out/prof.csv timeout 400 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/bench2.log 2>&1
echo "== $lib $(python3 -c "import json; d=json.loads(open('gpurun_out/bench2.log').read().strip().splitlines()[-1]); print(round(d['value']), round(d['ms_per_step'],1), d['clocks']['sm_mhz'])")"
python tools/gemm_shape_report.py gpurun_out/prof.csv 2 | grep "epi2\|epi4" | cut -c1-130
done; done > gpurun_out/pf_ab.log 2>&1
