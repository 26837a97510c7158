timeout 900 python -m pytest tests -m gpu -q > gpurun_out/t.log 2>&1; echo EXIT $? >> gpurun_out/t.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
python bench.py > gpurun_out/bench_end.json 2> gpurun_out/bench_end.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_end.json 2>&1
