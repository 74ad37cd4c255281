mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "variants or m1" > gpurun_out/pytest_gpu15.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu15.log
for cfg in "--scan-kernel 1" "--scan-kernel 5" "--scan-kernel 1" "--scan-kernel 5"; do
  timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline $cfg > gpurun_out/b15.log 2>&1
  echo "[$cfg] rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/b15.log').read().strip().splitlines()[-1]);k=d['kernel_ms_per_step'];print(d['value'], d['ms_per_step'], d['roofline']['achieved'], k['scan_ms'])")"
done
timeout 1500 python scripts/sweep.py > gpurun_out/sweep_r1.jsonl 2> gpurun_out/sweep_r1.err; echo sweep rc=$?
cat gpurun_out/sweep_r1.jsonl | cut -c1-300
