mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build33.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "merge" > gpurun_out/pytest_merge33.log 2>&1; echo merge rc=$?
tail -30 gpurun_out/pytest_merge33.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu33.log 2>&1; echo all rc=$?
tail -3 gpurun_out/pytest_gpu33.log
