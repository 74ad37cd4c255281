# multi-GPU validation + scaling on one box: tests, dist_check, bench N=1 and N=2.. (fused and
# nvlink assembly).  Usage: bash scripts/gpu_multi.sh TAG
TAG=${1:?tag}; OUT=gpurun_out/$TAG; mkdir -p $OUT
NG=$(nvidia-smi -L | wc -l); echo "gpus: $NG"
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python -m pytest tests -m "gpu and not slow" -q -x > $OUT/pytest_gpu.log 2>&1; echo "tests rc=$?"; tail -2 $OUT/pytest_gpu.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29533 \
  scripts/dist_check.py > $OUT/dist_check.log 2>&1; echo "dist_check rc=$?"; grep rank $OUT/dist_check.log | head -20
timeout 900 python bench.py --no-e2e --no-cpu-baseline > $OUT/bench_n1.jsonl 2> $OUT/bench_n1.err; echo "bench N=1 rc=$?"
for N in 2 4 8; do
  if [ $N -le $NG ]; then
    for A in fused nvlink; do
      timeout 900 python bench.py --gpus $N --assembly $A --no-e2e > $OUT/bench_n${N}_$A.jsonl 2> $OUT/bench_n${N}_$A.err; echo "bench N=$N $A rc=$?"
    done
  fi
done
python - <<'PY'
import glob, json
for f in sorted(glob.glob("gpurun_out/" + __import__("os").environ.get("TAG", "") + "*/bench_n*.jsonl")):
    pass
PY
for f in $OUT/bench_n*.jsonl; do python -c "
import json,sys
l=[x for x in open('$f') if x.startswith('{')]
d=json.loads(l[-1]) if l else {}
print('$f', d.get('n_gpus'), d.get('value'), d.get('ms_per_step'), d.get('config',{}).get('assembly','-'), d.get('per_rank',{}).get('ms_per_step'))
"; done
