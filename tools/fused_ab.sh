#!/bin/bash
# A/B of the optimizer-in-backward path (SW_FUSED_ADAMW=1) against the unfused step.
for i in 1 2; do for f in 1 0; do
SW_FUSED_ADAMW=$f python bench.py --steps 5 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print($f, round(d['value']), round(d['ms_per_step'],1), d['clocks']['sm_mhz'], {k:round(v['ms'],1) for k,v in d['breakdown_ms_per_step'].items()})"
done; done
