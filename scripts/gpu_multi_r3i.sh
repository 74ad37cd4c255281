OUT=gpurun_out/r3i; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
run() { timeout 900 python bench.py --no-e2e --no-cpu-baseline "$@" > $OUT/$NAME.jsonl 2> $OUT/$NAME.err; echo "$NAME rc=$?"; }
NAME=n4 run --gpus 4
NAME=n4_none run --gpus 4 --assembly none
NAME=n4_e4 run --gpus 4 --emit-ctas 4
NAME=n4_e4_none run --gpus 4 --emit-ctas 4 --assembly none
NAME=n4_c64 run --gpus 4 --assemble-ctas 64
NAME=n4_c16 run --gpus 4 --assemble-ctas 16
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29533 scripts/dist_check.py > $OUT/dist_check.log 2>&1; echo "dist_check rc=$?"
for f in $OUT/*.jsonl; do python -c "
import json
l=[x for x in open('$f') if x.startswith('{')]
d=json.loads(l[-1]) if l else {}
k=d.get('kernel_ms_per_step',{})
print('$f', d.get('n_gpus'), d.get('value'), d.get('ms_per_step'), round(sum(k.values()),3) if k else None, k.get('emit_ms'), d.get('per_rank',{}).get('ms_per_step'))
"; done
