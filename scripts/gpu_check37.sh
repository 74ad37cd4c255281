# merge (parallel header checks + hinted decodes), full GPU suite, default bench, sweep
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/smoke37.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu37.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu37.log
timeout 600 python scripts/merge_bench.py > gpurun_out/merge37.log 2>&1; echo mb rc=$?; cat gpurun_out/merge37.log
timeout 900 python bench.py > gpurun_out/bench37.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench37.log
timeout 1500 python scripts/sweep.py > gpurun_out/sweep37.jsonl 2>&1; echo sweep rc=$?
cat gpurun_out/sweep37.jsonl | cut -c1-250
