# parity + bench + ncu (launch list, DRAM traffic, full capture on a truncated set)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/smoke28.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu28.log 2>&1; rc=$?; echo pytest rc=$rc
tail -3 gpurun_out/pytest_gpu28.log
[ $rc = 0 ] || exit 1
timeout 900 python bench.py > gpurun_out/bench28.log 2>&1; echo bench rc=$?
tail -1 gpurun_out/bench28.log
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks"
$CMD > gpurun_out/plain28.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file gpurun_out/launches28.csv \
    $CMD > gpurun_out/ncu_launch28.log 2>&1
echo launches rc=$?
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:"k_scan_tiles|k_scatter|k_decode_count|k_emit_tiles|k_tiles_gaps" -c 5 --csv --log-file gpurun_out/traffic28.csv \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-clocks > gpurun_out/ncu_traffic28.log 2>&1
echo traffic rc=$?
SMALL="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks --tensors 40"
$SMALL > gpurun_out/plain28_small.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_scan_tiles|k_scatter|k_emit_tiles|k_decode_count|k_tiles_gaps" -s 1 -c 5 \
    -o gpurun_out/prof28 $SMALL > gpurun_out/ncu_full28.log 2>&1
echo full rc=$?
