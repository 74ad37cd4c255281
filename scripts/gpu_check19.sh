mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu19.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu19.log
timeout 900 python bench.py > gpurun_out/bench_r1_default.log 2>&1; echo "default rc=$?"; tail -1 gpurun_out/bench_r1_default.log | cut -c1-400
for cfg in "--rho 0.1 --config M5" "--rho 0.5 --config M5" "--rho 0.01 --pattern rowblock --config M5"; do
  timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $cfg > gpurun_out/b19.log 2>&1
  echo "[$cfg] rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/b19.log').read().strip().splitlines()[-1]);k=d['kernel_ms_per_step'];print(d['value'], d['ms_per_step'], {a: round(b,3) for a,b in k.items()})")"
done
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks"
$CMD > gpurun_out/plain_r1d.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file gpurun_out/launches_r1d.csv \
    $CMD > gpurun_out/ncu_launch_r1d.log 2>&1
echo launches rc=$?
T="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks"
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:"k_scan_tiles|k_scatter|k_decode_count|k_emit_tiles" -c 4 --csv --log-file gpurun_out/traffic_r1d.csv \
    $T > gpurun_out/ncu_traffic_r1d.log 2>&1
echo traffic rc=$?
SMALL="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks --tensors 40"
$SMALL > gpurun_out/plain_r1d_small.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_scan_tiles|k_scatter|k_emit_tiles|k_decode_count" -s 1 -c 4 \
    -o gpurun_out/prof_r1d $SMALL > gpurun_out/ncu_full_r1d.log 2>&1
echo full rc=$?
