mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "pipelined or async or m1 or corruption" > gpurun_out/pytest_gpu4.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu4.log
for cfg in "--pipeline 1" "--pipeline 4" "--pipeline 8" "--pipeline 8 --apply-ctas 2"; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $cfg > gpurun_out/b4.log 2>&1
  echo "$cfg rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/b4.log').read().strip().splitlines()[-1]);print(d['value'], d['ms_per_step'], d['kernel_ms_per_step'])")"
done
