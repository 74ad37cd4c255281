# round 2, call A: the round-1 tree's GPU suite, the scatter probe (plain / windowed / gather /
# sector read / sector write on the same 1 % positions) with DRAM counters, and a same-tree
# section capture of the apply + emit kernels at M3.
mkdir -p gpurun_out/r2a
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/r2a/smoke.log 2>&1; echo smoke rc=$?
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/r2a/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/r2a/pytest_gpu.log
timeout 600 python scripts/scatter_probe.py > gpurun_out/r2a/probe.jsonl 2> gpurun_out/r2a/probe.err; echo probe rc=$?
cat gpurun_out/r2a/probe.jsonl | cut -c1-200
M="dram__bytes_read.sum,dram__bytes_write.sum,dram__cycles_active.avg,dram__cycles_active_read.avg,dram__cycles_active_write.avg,dram__cycles_elapsed.avg,dram__throughput.avg.pct_of_peak_sustained_elapsed,gpu__time_duration.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_read.sum,lts__t_sector_hit_rate.pct"
PROBE_REPS=1 PROBE_ONLY=plain,window_u4,gather,sector timeout 900 ncu --metrics $M --clock-control none -k regex:"k_scatter|k_gather|k_sector" --csv \
   --log-file gpurun_out/r2a/probe_dram.csv python scripts/scatter_probe.py > gpurun_out/r2a/probe_ncu.log 2>&1; echo probe-ncu rc=$?
CMD="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-clocks"
timeout 900 ncu --metrics $M --clock-control none -k regex:"k_scan_tiles|k_scatter|k_decode_count|k_emit_tiles|k_tiles_gaps|k_locate" -c 6 --csv \
   --log-file gpurun_out/r2a/bench_dram.csv $CMD > gpurun_out/r2a/bench_dram.log 2>&1; echo bench-dram rc=$?
timeout 1200 ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --section Occupancy --section WarpStateStats --section LaunchStats \
   --section SchedulerStats --clock-control none -k regex:"k_scatter|k_decode_count|k_emit_tiles" -c 3 -o gpurun_out/r2a/sections \
   $CMD > gpurun_out/r2a/sections.log 2>&1; echo sections rc=$?
