# final: smoke, GPU suite, default bench, sweep of configs[0,1,4]
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/smoke73.log 2>&1; echo smoke rc=$?
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu73.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu73.log
timeout 1200 python bench.py > gpurun_out/bench73.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench73.log | cut -c1-300
timeout 2000 python scripts/sweep.py > gpurun_out/sweep73.jsonl 2>&1; echo sweep rc=$?
cut -c1-160 gpurun_out/sweep73.jsonl
