set -x
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv; free -g | head -2; nproc
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 900 python -m pytest tests -m gpu -x -q -k "not m3 and not u64" > gpurun_out/pytest_small.log 2>&1; echo pytest rc=$?
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --cpu-seconds 5 > gpurun_out/bench1.log 2>&1; echo bench rc=$?
tail -3 gpurun_out/pytest_small.log; tail -2 gpurun_out/bench1.log
