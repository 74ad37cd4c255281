# same-box A/B/C of the K1 compaction loop variants (ab_a: pointer chains, ab_b: descending
# FLO + indices, current tree: ascending ffs + indices) at 1 % and 10 %
mkdir -p gpurun_out
for d in ab_a ab_b .; do (cd $d && python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1); done
for rep in 1 2; do
for r in 0.01 0.1; do
  for d in ab_a ab_b .; do
    (cd $d && timeout 600 python bench.py --config M5 --rho $r --pattern uniform --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > /tmp/ab.log 2>&1)
    echo "rep $rep rho $r $d $(python -c "import json;d=json.loads(open('/tmp/ab.log').read().strip().splitlines()[-1]);k=d['kernel_ms_per_step'];print(d['value'], d['ms_per_step'], k['scan_ms'])")"
  done
done
done
