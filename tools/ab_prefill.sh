for i in 1 2 3; do for v in SW_PREFILL_HEAD_ROW=1 SW_PREFILL_HEAD_ROW=0; do
for b in 8 64; do env $v python tools/decode_bench.py oracle/specs/llama7b.spec $b 512 4 1 1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$v', $b, d['prefill_ms'])"; done
done; done
