# final validation of the round's tree (K4 early slot loads): smoke, GPU suite, bench N = 1,
# reference arm, then the ncu launch list + per-launch traffic (each ncu run after its plain run)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/smoke84.log 2>&1; echo smoke rc=$?
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu84.log 2>&1; echo pytest rc=$?
tail -1 gpurun_out/pytest_gpu84.log
timeout 900 python bench.py > gpurun_out/bench84_n1.log 2>&1; echo "N=1 rc=$?"
tail -1 gpurun_out/bench84_n1.log | cut -c1-300
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref84.log 2>&1; echo ref rc=$?
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks"
$CMD > gpurun_out/plain84.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file gpurun_out/launches84.csv \
    $CMD > gpurun_out/ncu_launch84.log 2>&1
echo launches rc=$?
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:"k_scan_tiles|k_scatter|k_decode_count|k_emit_tiles|k_tiles_gaps" -c 5 --csv --log-file gpurun_out/traffic84.csv \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-clocks > gpurun_out/ncu_traffic84.log 2>&1
echo traffic rc=$?
