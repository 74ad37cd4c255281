# K1 dense vs sparse compaction at 10 % / 50 % (DELTA_K1_DENSE override)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build56.log 2>&1
for r in 0.1 0.5; do
  for d in 0 1; do
    DELTA_K1_DENSE=$d timeout 600 python bench.py --config M5 --rho $r --pattern uniform --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b56_${r}_$d.log 2>&1
    echo "rho $r dense=$d rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/b56_${r}_$d.log').read().strip().splitlines()[-1]);k=d['kernel_ms_per_step'];print(d['value'], d['ms_per_step'], k['scan_ms'])")"
  done
done
