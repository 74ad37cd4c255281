# ncu full capture of K1 / K4 / scatter at 10 % and 50 % uniform (truncated tensor list)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build54.log 2>&1
for r in 0.1 0.5; do
  SMALL="python bench.py --config M5 --rho $r --pattern uniform --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks --tensors 40"
  $SMALL > gpurun_out/plain54_$r.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scan_tiles|k_scatter|k_emit_tiles" -s 3 -c 3 \
      -o gpurun_out/prof54_$r $SMALL > gpurun_out/ncu54_$r.log 2>&1
  echo "rho $r rc=$?"
done
