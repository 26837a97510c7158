for i in 1 2; do for v in base g16 g4; do
if [ $v = base ]; then L=""; else L="SW_LIB_PATH=variants/libsw_$v.so"; fi
env $L python bench.py --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$v', round(d['value']), round(d['ms_per_step'],1), d['clocks']['sm_mhz'], {k:round(v['ms'],1) for k,v in d['breakdown_ms_per_step'].items()})"
done; done
