timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t.log 2>&1; echo EXIT $? >> gpurun_out/t.log
for i in 1 2; do for f in 0 1; do
SW_WGRAD_STREAM=$f timeout 400 python bench.py --no-cpu-baseline --steps 8 > gpurun_out/b.log 2>&1
echo "side=$f $(python3 -c "import json; d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]); print(round(d['value']), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['e2e']['value'], d['gpu_launches'], d['loss'])")"
done; done > gpurun_out/ab.log 2>&1
