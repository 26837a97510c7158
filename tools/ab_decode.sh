#!/bin/bash
# Same-box A/B of decode switches: tools/ab_decode.sh <spec> <batch> "ENV=a" "ENV=b" ...
spec=$1; b=$2; shift 2
for i in 1 2 3; do for v in "$@"; do
env $v python tools/decode_bench.py $spec $b 512 64 1 1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$v', d['decode_ms_per_token'])"
done; done
