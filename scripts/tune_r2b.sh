OUT=gpurun_out/${1:-tune}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python -m pytest tests -m "gpu and not slow" -q -x > $OUT/pytest_gpu.log 2>&1; echo "tests rc=$?"; tail -1 $OUT/pytest_gpu.log
for S in 5 8 10 12 16 24; do
  timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-clocks --scatter-ctas $S > $OUT/sc_$S.jsonl 2>/dev/null
  python -c "import json;d=json.loads(open('$OUT/sc_$S.jsonl').read().strip().splitlines()[-1]);k=d['kernel_ms_per_step'];print('scatter_ctas',$S,d['ms_per_step'],k['scan_ms'],k['emit_ms'],k['scatter_ms'])"
done
