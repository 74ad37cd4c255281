# re-entry validation of the restored tree on one GPU: smoke, GPU suite, bench N = 1, reference arm
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/smoke78.log 2>&1; echo smoke rc=$?
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu78.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu78.log
timeout 1200 python bench.py > gpurun_out/bench78_n1.log 2>&1; echo "N=1 rc=$?"
tail -1 gpurun_out/bench78_n1.log | cut -c1-600
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref78.log 2>&1; echo ref rc=$?
tail -1 gpurun_out/ref78.log | cut -c1-200
