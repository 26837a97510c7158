for i in 1 2; do for lib in paper_2310_16355_b200/libshardweave_b200.so variants/libsw_tma.so; do
SW_LIB_PATH=$lib timeout 400 python bench.py --no-cpu-baseline --steps 8 > gpurun_out/b.log 2>&1
echo "$lib $(python3 -c "import json; d=json.loads(open('gpurun_out/b.log').read().strip().splitlines()[-1]); print(round(d['value']), round(d['ms_per_step'],2), d['clocks']['sm_mhz'], d['breakdown_ms_per_step']['gemm'])")"
done; done > gpurun_out/tma_ab.log 2>&1
