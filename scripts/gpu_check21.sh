mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu21.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu21.log
for cfg in "" "" "--rho 0.1 --config M5" "--rho 0.5 --config M5"; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $cfg > gpurun_out/b21.log 2>&1
  echo "[$cfg] rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/b21.log').read().strip().splitlines()[-1]);k=d['kernel_ms_per_step'];print(d['value'], d['ms_per_step'], {a: round(b,3) for a,b in k.items()})")"
done
timeout 300 python scripts/membench.py 2>&1 | head -2
