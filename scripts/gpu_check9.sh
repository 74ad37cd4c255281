mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "m1 or ragged or m3 or options" > gpurun_out/pytest_gpu9.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu9.log
for cfg in "--prefetch-waves 1" "--prefetch-waves 2" "--prefetch-waves 3" "--prefetch-waves 5" "--scatter-order 2" "--scatter-order 2 --scatter-ctas 8"; do
  timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline $cfg > gpurun_out/b9.log 2>&1
  echo "$cfg rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/b9.log').read().strip().splitlines()[-1]);k=d['kernel_ms_per_step'];print(d['value'], d['ms_per_step'], d['roofline']['achieved'], k['scan_ms'], k['scatter_ms'])")"
done
