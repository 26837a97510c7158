#!/bin/bash
for i in 1 2 3; do
 for d in oldtree .; do
  (cd $d && python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$d', round(d['value']), round(d['ms_per_step'],1), d['clocks']['sm_mhz'], {k:round(v['ms'],1) for k,v in d['breakdown_ms_per_step'].items()})")
 done
done
