mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu25.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_gpu25.log
bash scripts/gpu_ab.sh
