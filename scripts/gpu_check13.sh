mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "variants or m1 or ragged or options" > gpurun_out/pytest_gpu13.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu13.log
for cfg in "--scan-kernel 1" "--scan-kernel 4" "--scan-kernel 1" "--scan-kernel 4"; do
  timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline $cfg > gpurun_out/b13.log 2>&1
  echo "[$cfg] rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/b13.log').read().strip().splitlines()[-1]);k=d['kernel_ms_per_step'];print(d['value'], d['ms_per_step'], d['roofline']['achieved'], k['scan_ms'])")"
done
