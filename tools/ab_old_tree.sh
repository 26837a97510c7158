#!/bin/bash
# Same-box step A/B of an older revision against the working tree. Prepare the old tree here
# first (the GPU box has no .git): git worktree add oldtree <rev> && make -C oldtree, then
# gpurun -- bash tools/ab_old_tree.sh, then git worktree remove --force oldtree.
for i in 1 2 3; do
 for d in oldtree .; do
  (cd $d && python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$d', round(d['value']), round(d['ms_per_step'],1), d['clocks']['sm_mhz'], {k:round(v['ms'],1) for k,v in d['breakdown_ms_per_step'].items()})")
 done
done
