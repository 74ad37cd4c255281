# One bench.py knob swept on one GPU (M3, 1 % uniform unless more flags follow "--"):
#   bash scripts/tune.sh TAG --scatter-ctas 5 24 96          (a bench.py flag)
#   bash scripts/tune.sh TAG env:DELTA_K1_DENSE_TILE 0 1024 4096 100000   (an environment knob)
# EXTRA="--gpus 4 ..." adds fixed flags.  Writes gpurun_out/TAG/<knob>_<value>.jsonl and prints
# step / kernel times per value.
TAG=${1:?tag}; KNOB=${2:?knob}; shift 2
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
NAME=$(echo "$KNOB" | tr -d '-' | tr ':' '_')
for V in "$@"; do
  if [[ $KNOB == env:* ]]; then
    env "${KNOB#env:}=$V" timeout 600 python bench.py --no-e2e --no-cpu-baseline $EXTRA > $OUT/${NAME}_$V.jsonl 2>/dev/null
  else
    timeout 600 python bench.py --no-e2e --no-cpu-baseline $EXTRA $KNOB $V > $OUT/${NAME}_$V.jsonl 2>/dev/null
  fi
  echo "$KNOB=$V $(tail -1 $OUT/${NAME}_$V.jsonl | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["kernel_ms_per_step"])' 2>&1 | cut -c1-300)"
done
