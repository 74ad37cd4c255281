mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu23.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu23.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b23.log 2>&1
echo "rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/b23.log').read().strip().splitlines()[-1]);k=d['kernel_ms_per_step'];print(d['value'], d['ms_per_step'], d['payload'])")"
