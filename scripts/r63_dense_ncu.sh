# ncu --set full of the dense-regime kernels (configs[4] 50 % uniform, a 40-tensor prefix)
OUT=gpurun_out/r63; mkdir -p $OUT
SMALL="python bench.py --config M5 --rho 0.5 --pattern uniform --tensors 40 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks"
$SMALL > $OUT/plain.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_scan_tiles|k_scatter|k_emit_pair|k_decode_count" \
  -s 4 -c 4 -o $OUT/dense_full $SMALL > $OUT/ncu_full.log 2>&1; echo "full rc=$?"
