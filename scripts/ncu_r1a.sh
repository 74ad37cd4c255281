# ncu pass 1: launch list (1 metric, whole M3 step) + full capture of each kernel on a truncated M3
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks > gpurun_out/plain_r1a.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file gpurun_out/launches_r1a.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks > gpurun_out/ncu_launch_r1a.log 2>&1
echo launches rc=$?
python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks --tensors 24 > gpurun_out/plain_r1a_small.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_scan_compact|k_scatter|k_emit|k_decode_count|k_entry_lens" -s 9 -c 5 \
    -o gpurun_out/prof_r1a python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks --tensors 24 > gpurun_out/ncu_full_r1a.log 2>&1
echo full rc=$?
