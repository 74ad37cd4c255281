mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu8.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu8.log
for cfg in "--scatter-ctas 2" "--scatter-ctas 1" "--scatter-ctas 4" "--scatter-ctas 2"; do
  timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline $cfg > gpurun_out/b8.log 2>&1
  echo "$cfg rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/b8.log').read().strip().splitlines()[-1]);print(d['value'], d['ms_per_step'], d['roofline']['achieved'], d['kernel_ms_per_step'])")"
done
