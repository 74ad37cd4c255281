# A2 double buffering + scatter grid 5/SM: parity, then 1 / 10 / 50 %
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build75.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu75.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu75.log
for r in 0.01 0.1 0.5; do
  timeout 600 python bench.py --config M5 --rho $r --pattern uniform --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/b75.log 2>&1
  echo "rho $r rc=$? $(python -c "import json;d=json.loads(open('/tmp/b75.log').read().strip().splitlines()[-1]);k=d['kernel_ms_per_step'];print(d['value'], d['ms_per_step'], {a: round(b,3) for a,b in k.items()})")"
done
