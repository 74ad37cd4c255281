# 4-GPU: the LPT partition (record-granular NVLink assembly) against contiguous ranges.
# Usage: bash scripts/gpu_multi_lpt.sh TAG
TAG=${1:?tag}; OUT=gpurun_out/$TAG; mkdir -p $OUT
NG=$(nvidia-smi -L | wc -l); echo "gpus: $NG"
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29533 \
  scripts/dist_check.py > $OUT/dist_check.log 2>&1; echo "dist_check rc=$?"
run() { timeout 900 python bench.py --no-e2e --no-cpu-baseline "$@" > $OUT/$NAME.jsonl 2> $OUT/$NAME.err; echo "$NAME rc=$?"; }
NAME=n1 run
NAME=n4 run --gpus 4
NAME=n4_lpt run --gpus 4 --partition lpt
NAME=n4_none run --gpus 4 --assembly none
NAME=n4_lpt_none run --gpus 4 --partition lpt --assembly none
NAME=n2 run --gpus 2
NAME=n2_lpt run --gpus 2 --partition lpt
for f in $OUT/*.jsonl; do python -c "
import json
l=[x for x in open('$f') if x.startswith('{')]
d=json.loads(l[-1]) if l else {}
k=d.get('kernel_ms_per_step',{})
pr=d.get('per_rank',{})
print('$f', d.get('n_gpus'), d.get('value'), d.get('ms_per_step'), round(sum(k.values()),3) if k else None, pr.get('ms_per_step'), pr.get('k1_ms'))
"; done
