mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build41.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "merge" > gpurun_out/pytest_merge41.log 2>&1; echo merge rc=$?
tail -3 gpurun_out/pytest_merge41.log
DELTA_MERGE_TIMING=1 timeout 600 python scripts/merge_bench.py --reps 3 > gpurun_out/merge41.log 2>&1; tail -7 gpurun_out/merge41.log
timeout 1200 python bench.py > gpurun_out/bench41.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench41.log
