#!/bin/bash
# A/B of two builds of the library on one box, interleaved (box-to-box variance cancels):
#   bash scripts/ab.sh TAG LIB_A LIB_B REPS [bench.py flags...]
# LIB_A / LIB_B: paths of libsparsedelta.so builds (SPARSEDELTA_LIB override); writes
# gpurun_out/TAG/ab_{a,b}_<rep>.jsonl and prints step / per-kernel ms per run.
TAG=${1:?tag}; A=${2:?lib a}; B=${3:?lib b}; REPS=${4:-3}; shift 4
OUT=gpurun_out/$TAG; mkdir -p $OUT
SUF=$(echo "$*" | tr -d ' -' | tr '.' 'p')
for R in $(seq 1 $REPS); do
  for X in a b; do
    L=$A; [ $X = b ] && L=$B
    SPARSEDELTA_LIB=$L timeout 600 python bench.py --no-e2e --no-cpu-baseline "$@" > $OUT/ab_${SUF}_${X}_$R.jsonl 2>/dev/null
    echo "$X $R $* $(tail -1 $OUT/ab_${SUF}_${X}_$R.jsonl | python -c 'import json,sys; d=json.loads(sys.stdin.read()); k=d["kernel_ms_per_step"]; print(d["ms_per_step"], " ".join("%s=%.3f" % (n[:-3], k[n]) for n in ("scan_ms","lens_ms","emit_ms","decode_ms","apply_scan_ms","scatter_ms")))' 2>&1 | cut -c1-300)"
  done
done
