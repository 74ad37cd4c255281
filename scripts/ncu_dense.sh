# ncu full capture of K1 / emit / decode / scatter at 50 % density on a truncated Qwen3-8B set
mkdir -p gpurun_out
SMALL="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks --config M5 --rho 0.5 --tensors 12"
$SMALL > gpurun_out/plain_dense.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_scan_tiles|k_scatter|k_emit_tiles|k_decode_count" -s 1 -c 4 \
    -o gpurun_out/prof_dense $SMALL > gpurun_out/ncu_full_dense.log 2>&1
echo full rc=$?
