# final ncu evidence for the round's kernels (M3, 1 %): launch list, per-launch DRAM traffic,
# full capture of K1 / K4 / A2 / A4 on a truncated tensor list.  Every ncu run filtered and
# bounded by timeout.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build77.log 2>&1
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks"
$CMD > gpurun_out/plain77.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file gpurun_out/launches77.csv \
    $CMD > gpurun_out/ncu_launch77.log 2>&1
echo launches rc=$?
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:"k_scan_tiles|k_scatter|k_decode_count|k_emit_tiles|k_tiles_gaps" -c 5 --csv --log-file gpurun_out/traffic77.csv \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-clocks > gpurun_out/ncu_traffic77.log 2>&1
echo traffic rc=$?
SMALL="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks --tensors 40"
$SMALL > gpurun_out/plain77_small.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scan_tiles|k_scatter|k_emit_tiles|k_decode_count" -s 1 -c 4 \
    -o gpurun_out/prof77 $SMALL > gpurun_out/ncu_full77.log 2>&1
echo full rc=$?
