# scatter grid at 1 / 10 / 50 % uniform
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build74.log 2>&1
for r in 0.5 0.1 0.01; do
  for sc in 4 5 8; do
    timeout 600 python bench.py --config M5 --rho $r --pattern uniform --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --scatter-ctas $sc > /tmp/b74.log 2>&1
    echo "rho $r scatter_ctas $sc rc=$? $(python -c "import json;d=json.loads(open('/tmp/b74.log').read().strip().splitlines()[-1]);k=d['kernel_ms_per_step'];print(d['value'], d['ms_per_step'], k['scatter_ms'])")"
  done
done
