# r1b: launch list of the full M3 bench command + full capture of the hot kernels (truncated M3)
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks"
$CMD > gpurun_out/plain_r1b.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file gpurun_out/launches_r1b.csv \
    $CMD > gpurun_out/ncu_launch_r1b.log 2>&1
echo launches rc=$?
SMALL="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks --tensors 40"
$SMALL > gpurun_out/plain_r1b_small.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_scan_tiles|k_scatter|k_emit_tiles|k_decode_count" -s 1 -c 4 \
    -o gpurun_out/prof_r1b $SMALL > gpurun_out/ncu_full_r1b.log 2>&1
echo full rc=$?
