# final validation of the round's tree: smoke, GPU suite, default bench, reference arm
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/smoke51.log 2>&1; echo smoke rc=$?
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu51.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu51.log
timeout 1200 python bench.py > gpurun_out/bench51.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench51.log
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref51.log 2>&1; echo ref rc=$?
tail -1 gpurun_out/ref51.log
