mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu24.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_gpu24.log
for mode in chain sync chain sync; do
  extra=""; [ $mode = sync ] && extra="--sync-step"
  timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline $extra > gpurun_out/b24_$mode.log 2>&1
  echo "$mode rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/b24_$mode.log').read().strip().splitlines()[-1]);k=d['kernel_ms_per_step'];print(d['value'], d['ms_per_step'], round(sum(k.values()),4))")"
done
