#!/bin/bash
# One parameterised runner for the GPU box (replaces round 1's one-off gpu_check*.sh):
#   bash scripts/gpu_run.sh TAG SUITE [SUITE ...]
# writes everything under gpurun_out/TAG/.  Suites (each bounded by its own timeout; every
# ncu run follows a plain run of the same command that exited 0):
#   smoke      build + __graft_entry__.smoke()
#   tests      pytest -m gpu, without the full-size configs
#   fullsize   pytest tests/test_gpu_fullsize.py (every record of configs[1..4] vs the oracle)
#   bench      bench.py N=1 (default flags) + the reference arm
#   k4tune     bench.py over K4's CTAs per SM (K4_CTAS)
#   k4full     ncu --set full of one kernel (KFULL regex, default K4) on the full M3 step
#   sweep      scripts/sweep.py: configs[0], [1], [4] (0.1/10/50 % uniform + rowblock)
#   launches   ncu launch list of bench.py (gpu__time_duration, cold, serialised)
#   traffic    ncu per-launch DRAM bytes + DRAM activity of the path's kernels at M3
#   sections   ncu SpeedOfLight/Memory/Occupancy/WarpState/Scheduler sections, K4 / A2 / A4 / K1
#   full       ncu --set full of the top kernels on a 40-tensor prefix of M3
#   sanitizer  compute-sanitizer memcheck / racecheck / synccheck / initcheck over the
#              small parity tests — NOTE: closed on this GPU pool (runs left GPUs needing a
#              reset); tests/test_gpu_guard.py (guard bands + fuzz) stands in for memcheck
#   probe      scripts/scatter_probe.py (+ DRAM counters)
#   scale      bench.py --gpus 2 / 4 (as many GPUs as the box has) + dist_check
TAG=${1:?tag}; shift
OUT=gpurun_out/$TAG
mkdir -p $OUT
BENCH_SMALL="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks"
DRAM="dram__bytes_read.sum,dram__bytes_write.sum,dram__cycles_active.avg,dram__cycles_elapsed.avg,dram__throughput.avg.pct_of_peak_sustained_elapsed,gpu__time_duration.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,smsp__issue_active.avg.pct_of_peak_sustained_elapsed"
KERNELS="k_scan_tiles|k_scatter|k_decode_count|k_emit|k_tiles|k_locate|k_apply_scan|k_headers"
for S in "$@"; do
  case $S in
  smoke)
    timeout 600 python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > $OUT/smoke.log 2>&1; echo "smoke rc=$?";;
  tests)
    timeout 1500 python -m pytest tests -m "gpu and not slow" -q -x > $OUT/pytest_gpu.log 2>&1; echo "tests rc=$?"; tail -2 $OUT/pytest_gpu.log;;
  fullsize)
    timeout 2400 python -m pytest tests/test_gpu_fullsize.py -q -x --durations=0 > $OUT/pytest_fullsize.log 2>&1; echo "fullsize rc=$?"; tail -15 $OUT/pytest_fullsize.log;;
  bench)
    timeout 900 python bench.py > $OUT/bench_n1.jsonl 2> $OUT/bench_n1.err; echo "bench rc=$?"; tail -1 $OUT/bench_n1.jsonl | cut -c1-400
    timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref.jsonl 2> $OUT/bench_ref.err; echo "ref rc=$?";;
  k4tune)  # K4 grid: CTAs per SM in K4_CTAS
    for C in ${K4_CTAS:-8 16 24 32}; do
      timeout 600 python bench.py --no-e2e --no-cpu-baseline --emit-ctas $C > $OUT/k4_c${C}.jsonl 2>/dev/null
      echo "C=$C $(tail -1 $OUT/k4_c${C}.jsonl | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["kernel_ms_per_step"]["emit_ms"])' 2>&1 | cut -c1-200)"
    done;;
  k4full)  # ncu --set full of one kernel (regex KFULL, default K4) on the full M3 step (one launch)
    $BENCH_SMALL > $OUT/plain_k4.log 2>&1 && \
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KFULL:-k_emit}" -c 1 -o $OUT/k4full \
      python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-clocks > $OUT/ncu_k4full.log 2>&1; echo "k4full rc=$?";;
  sweep)
    timeout 1800 python scripts/sweep.py > $OUT/sweep.jsonl 2> $OUT/sweep.err; echo "sweep rc=$?";;
  launches)
    $BENCH_SMALL > $OUT/plain_launch.log 2>&1 && \
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv \
      --log-file $OUT/launches.csv $BENCH_SMALL > $OUT/ncu_launches.log 2>&1; echo "launches rc=$?";;
  traffic)
    timeout 900 ncu --metrics $DRAM --clock-control none -k regex:"$KERNELS" -c 20 --csv \
      --log-file $OUT/traffic.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-clocks \
      > $OUT/ncu_traffic.log 2>&1; echo "traffic rc=$?";;
  sections)
    timeout 1500 ncu --section SpeedOfLight --section MemoryWorkloadAnalysis --section Occupancy --section WarpStateStats \
      --section LaunchStats --section SchedulerStats --metrics $DRAM --clock-control none \
      -k regex:"k_scan_tiles|k_scatter|k_decode_count|k_emit|k_locate|k_tiles_scan" -c 12 -o $OUT/sections \
      python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-clocks > $OUT/ncu_sections.log 2>&1
    echo "sections rc=$?";;
  full)
    SMALL="python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks --tensors 40"
    $SMALL > $OUT/plain_full.log 2>&1 && \
    timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_scan_tiles|k_scatter|k_emit|k_decode_count" \
      -s 4 -c 4 -o $OUT/full $SMALL > $OUT/ncu_full.log 2>&1; echo "full rc=$?";;
  sanitizer)
    for T in ${SAN_TOOLS:-memcheck racecheck synccheck initcheck}; do
      timeout ${SAN_TIMEOUT:-2400} compute-sanitizer --tool $T --target-processes all --print-limit 50 --log-file $OUT/san_$T.log \
        python -m pytest tests/test_gpu_parity.py tests/test_gpu_boundary.py -m gpu -q -p no:cacheprovider \
        -k "${SAN_K:-not u64 and not pipelined and not scan_kernel_variants and not scatter_launch_options}" > $OUT/san_${T}_pytest.log 2>&1
      echo "sanitizer $T rc=$? $(grep -c 'ERROR SUMMARY' $OUT/san_$T.log) summaries: $(grep 'ERROR SUMMARY' $OUT/san_$T.log | sort | uniq -c | tr '\n' ' ')"
    done;;
  probe)
    timeout 600 python scripts/scatter_probe.py > $OUT/probe.jsonl 2> $OUT/probe.err; echo "probe rc=$?";;
  scale)
    NG=$(nvidia-smi -L | wc -l)
    for N in 2 4; do
      if [ $N -le $NG ]; then
        timeout 900 python bench.py --gpus $N --no-e2e > $OUT/bench_n$N.jsonl 2> $OUT/bench_n$N.err; echo "bench N=$N rc=$?"
        tail -1 $OUT/bench_n$N.jsonl | cut -c1-300
      fi
    done
    if [ $NG -ge 2 ]; then
      timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29533 \
        scripts/dist_check.py > $OUT/dist_check.log 2>&1; echo "dist_check rc=$?"
    fi;;
  *) echo "unknown suite $S";;
  esac
done
