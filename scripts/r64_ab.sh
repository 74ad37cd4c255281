# validation + interleaved A/B of the r60 build against the working tree, then dense ncu
OLD=paper_2602_11456_b200/libsparsedelta_r60.so; NEW=paper_2602_11456_b200/libsparsedelta.so
T=${TAG:-r64}; mkdir -p gpurun_out/$T
bash scripts/gpu_run.sh $T tests
bash scripts/ab.sh $T $OLD $NEW 2 > gpurun_out/$T/ab_m3.txt 2>&1
for P in "0.5 uniform" "0.5 rowblock" "0.1 uniform" "0.1 rowblock" "0.01 rowblock"; do
  set -- $P
  bash scripts/ab.sh $T $OLD $NEW 1 --config M5 --rho $1 --pattern $2 --steps 10 >> gpurun_out/$T/ab_dense.txt 2>&1
done
bash scripts/gpu_run.sh $T fullsize
SMALL="python bench.py --config M5 --rho 0.5 --pattern uniform --tensors 40 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scan_tiles|k_scatter|k_emit_pair|k_decode_count" \
  -s 4 -c 4 -o gpurun_out/$T/dense_full $SMALL > gpurun_out/$T/ncu_full.log 2>&1; echo "ncu rc=$?"
cat gpurun_out/$T/ab_m3.txt gpurun_out/$T/ab_dense.txt
