#!/bin/bash
# Same-box A/B of experiment builds on the decode step: tools/ab_decode_lib.sh <spec> <batch> base v1 v2 ...
spec=$1; b=$2; shift 2
for i in 1 2 3; do for v in "$@"; do
if [ $v = base ]; then L=""; else L="SW_LIB_PATH=variants/libsw_$v.so"; fi
env $L python tools/decode_bench.py $spec $b 512 64 1 1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$v', d['decode_ms_per_token'])"
done; done
