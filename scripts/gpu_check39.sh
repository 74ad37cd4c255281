# emit (register-staged offsets) A/B via bench, merge timing, per-kernel merge launch list
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build39.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu39.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu39.log
for i in 1 2; do
timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b39_$i.log 2>&1
echo "bench rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/b39_$i.log').read().strip().splitlines()[-1]);k=d['kernel_ms_per_step'];print(d['value'], d['ms_per_step'], d['host_synced'], {a: round(b,3) for a,b in k.items()}, d['ops'])")"
done
DELTA_MERGE_TIMING=1 timeout 600 python scripts/merge_bench.py --reps 3 > gpurun_out/merge39.log 2>&1; cat gpurun_out/merge39.log | tail -20
