OUT=gpurun_out/${1:-tune}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for S in 24 32 48 96 180; do
  timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-clocks --scatter-ctas $S > $OUT/sc_$S.jsonl 2>/dev/null
  python -c "import json;d=json.loads(open('$OUT/sc_$S.jsonl').read().strip().splitlines()[-1]);k=d['kernel_ms_per_step'];print('scatter_ctas',$S,d['ms_per_step'],k['scan_ms'],k['decode_ms'],k['scatter_ms'])"
done
for A in 4 16 32 180; do
  timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-clocks --apply-ctas $A --scatter-ctas 24 > $OUT/ac_$A.jsonl 2>/dev/null
  python -c "import json;d=json.loads(open('$OUT/ac_$A.jsonl').read().strip().splitlines()[-1]);k=d['kernel_ms_per_step'];print('apply_ctas',$A,d['ms_per_step'],k['scan_ms'],k['decode_ms'],k['scatter_ms'])"
done
