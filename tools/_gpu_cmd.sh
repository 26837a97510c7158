timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t.log 2>&1; echo EXIT $? >> gpurun_out/t.log
for i in 1 2 3; do for lib in variants/libsw_prev.so paper_2310_16355_b200/libshardweave_b200.so; do
SW_LIB_PATH=$lib timeout 400 python bench.py --no-cpu-baseline --steps 8 > gpurun_out/b.log 2>&1
echo "$lib $(python3 -c "import json; d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]); print(round(d['value']), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], round(d['e2e']['value']))")"
done; done > gpurun_out/ab.log 2>&1
