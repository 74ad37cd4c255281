# r1c: launch list (full M3 bench command), full capture of hot kernels (truncated M3),
# and DRAM traffic of one full-size K1 launch (for the bench roofline "traffic" field)
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks"
$CMD > gpurun_out/plain_r1c.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file gpurun_out/launches_r1c.csv \
    $CMD > gpurun_out/ncu_launch_r1c.log 2>&1
echo launches rc=$?
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:"k_scan_tiles|k_scatter|k_decode_count|k_emit_tiles" -c 4 --csv --log-file gpurun_out/traffic_r1c.csv \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-clocks > gpurun_out/ncu_traffic_r1c.log 2>&1
echo traffic rc=$?
SMALL="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks --tensors 40"
$SMALL > gpurun_out/plain_r1c_small.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_scan_tiles|k_scatter|k_emit_tiles|k_decode_count" -s 1 -c 4 \
    -o gpurun_out/prof_r1c $SMALL > gpurun_out/ncu_full_r1c.log 2>&1
echo full rc=$?
