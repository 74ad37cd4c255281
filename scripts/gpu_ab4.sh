# same-box A/B: K4 without (ab_a) / with (current tree) the next-tile L2 prefetch, 1 %
mkdir -p gpurun_out
for d in ab_a .; do (cd $d && python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1); done
for rep in 1 2 3; do
  for d in ab_a .; do
    (cd $d && timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/ab.log 2>&1)
    echo "rep $rep $d $(python -c "import json;d=json.loads(open('/tmp/ab.log').read().strip().splitlines()[-1]);k=d['kernel_ms_per_step'];print(d['value'], d['ms_per_step'], k['emit_ms'], k['scan_ms'])")"
  done
done
