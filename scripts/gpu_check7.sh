mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "variants or m1 or ragged or corruption" > gpurun_out/pytest_gpu7.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu7.log
for cfg in "--scan-kernel 1" "--scan-kernel 3" "--scan-kernel 3 --apply-ctas 4" "--scan-kernel 3 --apply-ctas 16" "--scan-kernel 3 --apply-ctas 2"; do
  timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline $cfg > gpurun_out/b7.log 2>&1
  echo "$cfg rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/b7.log').read().strip().splitlines()[-1]);print(d['value'], d['ms_per_step'], d['roofline']['achieved'], d['kernel_ms_per_step'])")"
done
