# 4-GPU scaling of the default path + the assembly variants (nvlink default, fused, nccl, none).  Usage: bash scripts/gpu_multi2.sh TAG
TAG=${1:?tag}; OUT=gpurun_out/$TAG; mkdir -p $OUT
NG=$(nvidia-smi -L | wc -l); echo "gpus: $NG"
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29533 \
  scripts/dist_check.py > $OUT/dist_check.log 2>&1; echo "dist_check rc=$?"
run() { timeout 900 python bench.py --no-e2e --no-cpu-baseline "$@" > $OUT/$NAME.jsonl 2> $OUT/$NAME.err; echo "$NAME rc=$?"; }
NAME=n1 run
NAME=n2 run --gpus 2
NAME=n4 run --gpus 4
NAME=n4_none run --gpus 4 --assembly none
NAME=n2_fused run --gpus 2 --assembly fused
NAME=n4_fused run --gpus 4 --assembly fused
NAME=n4_nccl run --gpus 4 --assembly nccl
for f in $OUT/*.jsonl; do python -c "
import json
l=[x for x in open('$f') if x.startswith('{')]
d=json.loads(l[-1]) if l else {}
k=d.get('kernel_ms_per_step',{})
print('$f', d.get('n_gpus'), d.get('value'), d.get('ms_per_step'), round(sum(k.values()),3) if k else None, d.get('per_rank',{}).get('ms_per_step'))
"; done
