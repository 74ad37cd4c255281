# Multi-GPU validation + scaling on one box (as many GPUs as it has, up to 4):
# dist_check (every assembly variant byte-equal to the single-GPU body and the oracle), then
# bench.py at N = 1, 2, 4 with the default (auto: contiguous at 2, LPT from 4) and each
# alternative partition / assembly.  Usage: bash scripts/gpu_multi.sh TAG
TAG=${1:?tag}; OUT=gpurun_out/$TAG; mkdir -p $OUT
NG=$(nvidia-smi -L | wc -l); echo "gpus: $NG"
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29533 \
  scripts/dist_check.py > $OUT/dist_check.log 2>&1; echo "dist_check rc=$?"
run() { timeout 900 python bench.py --no-e2e --no-cpu-baseline "$@" > $OUT/$NAME.jsonl 2> $OUT/$NAME.err; echo "$NAME rc=$?"; }
NAME=n1 run
if [ $NG -ge 2 ]; then
  NAME=n2 run --gpus 2
  NAME=n2_lpt run --gpus 2 --partition lpt
  NAME=n2_fused run --gpus 2 --assembly fused
fi
if [ $NG -ge 4 ]; then
  NAME=n4 run --gpus 4
  NAME=n4_contiguous run --gpus 4 --partition contiguous
  NAME=n4_fused run --gpus 4 --assembly fused
  NAME=n4_nccl run --gpus 4 --assembly nccl
  NAME=n4_none run --gpus 4 --assembly none
  NAME=n4_contiguous_none run --gpus 4 --partition contiguous --assembly none
fi
for f in $OUT/*.jsonl; do python -c "
import json
l=[x for x in open('$f') if x.startswith('{')]
d=json.loads(l[-1]) if l else {}
k=d.get('kernel_ms_per_step',{})
pr=d.get('per_rank',{})
print('$f', d.get('n_gpus'), d.get('value'), d.get('ms_per_step'), round(sum(k.values()),3) if k else None, pr.get('ms_per_step'), pr.get('k1_ms'))
"; done
