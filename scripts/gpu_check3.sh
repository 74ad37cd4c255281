mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu3.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/pytest_gpu3.log
for cfg in "--pipeline 1" "--pipeline 4" "--pipeline 8" "--pipeline 16" "--pipeline 8 --apply-ctas 2" "--pipeline 8 --apply-ctas 4"; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $cfg > gpurun_out/b3.log 2>&1
  echo "$cfg rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/b3.log').read().strip().splitlines()[-1]);print(d['value'], d['ms_per_step'], d['kernel_ms_per_step'])")"
done
