# K1 emission threshold: vector order everywhere (0) vs dense tiles only (1024) vs per-word only (100000)
OUT=gpurun_out/${1:-tune}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python -m pytest tests -m "gpu and not slow" -q -x > $OUT/pytest_gpu.log 2>&1; echo "tests rc=$?"; tail -1 $OUT/pytest_gpu.log
for T in 0 1024 100000; do
  for P in "0.01 uniform" "0.1 uniform" "0.5 uniform" "0.01 rowblock" "0.1 rowblock" "0.5 rowblock"; do
    set -- $P
    DELTA_K1_DENSE_TILE=$T timeout 600 python bench.py --config M5 --rho $1 --pattern $2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-clocks > $OUT/t${T}_$1_$2.jsonl 2>/dev/null
    python -c "import json;d=json.loads(open('$OUT/t${T}_$1_$2.jsonl').read().strip().splitlines()[-1]);k=d['kernel_ms_per_step'];print('thr',$T,'$1','$2',d['ms_per_step'],'K1',k['scan_ms'],'K4',k['emit_ms'])"
  done
done
