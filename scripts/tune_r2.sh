# knob sweep on one GPU (M3, 1 %): K1 L2 prefetch distance and scatter CTAs per SM
OUT=gpurun_out/${1:-tune}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for P in 0 1 297 445 593 889; do
  timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-clocks --prefetch-tiles $P > $OUT/pf_$P.jsonl 2>/dev/null
  python -c "import json;d=json.loads(open('$OUT/pf_$P.jsonl').read().strip().splitlines()[-1]);print('prefetch',$P,d['ms_per_step'],d['kernel_ms_per_step']['scan_ms'],d['kernel_ms_per_step']['scatter_ms'])"
done
for S in 4 6 8; do
  timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-clocks --scatter-ctas $S > $OUT/sc_$S.jsonl 2>/dev/null
  python -c "import json;d=json.loads(open('$OUT/sc_$S.jsonl').read().strip().splitlines()[-1]);print('scatter_ctas',$S,d['ms_per_step'],d['kernel_ms_per_step']['scan_ms'],d['kernel_ms_per_step']['scatter_ms'])"
done
