for i in 1 2 3; do for v in SW_WGRAD_STREAM=0 SW_WGRAD_STREAM=1; do
env $v python bench.py --steps 6 --warmup 3 --batch 4 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$v', round(d['value']), round(d['ms_per_step'],1), d['clocks']['sm_mhz'])"
done; done
