mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/smoke26.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu26.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_gpu26.log
timeout 900 python bench.py > gpurun_out/bench26.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench26.log
