# A/B: the tree in ab_old/ (an older commit, built in place) vs the current tree, same box
mkdir -p gpurun_out
for i in 1 2; do
  (cd ab_old && timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > ../gpurun_out/ab_old.log 2>&1)
  echo "old rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/ab_old.log').read().strip().splitlines()[-1]);k=d['kernel_ms_per_step'];print(d['value'], d['ms_per_step'], {a: round(b,3) for a,b in k.items()})")"
  timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_new.log 2>&1
  echo "new rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/ab_new.log').read().strip().splitlines()[-1]);k=d['kernel_ms_per_step'];print(d['value'], d['ms_per_step'], {a: round(b,3) for a,b in k.items()})")"
done
