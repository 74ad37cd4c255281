# launch-shape sweep of the apply kernels at M3 1 %: scatter CTAs/SM and decode CTAs/SM
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build57.log 2>&1
for sc in 2 4 6 8; do
  timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --scatter-ctas $sc > gpurun_out/b57_sc$sc.log 2>&1
  echo "scatter_ctas $sc rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/b57_sc$sc.log').read().strip().splitlines()[-1]);k=d['kernel_ms_per_step'];print(d['value'], d['ms_per_step'], k['scatter_ms'], k['decode_ms'])")"
done
for ac in 4 6 12; do
  timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --apply-ctas $ac > gpurun_out/b57_ac$ac.log 2>&1
  echo "apply_ctas $ac rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/b57_ac$ac.log').read().strip().splitlines()[-1]);k=d['kernel_ms_per_step'];print(d['value'], d['ms_per_step'], k['scatter_ms'], k['decode_ms'])")"
done
