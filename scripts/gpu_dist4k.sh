# flag-based record assembly (LPT): correctness, then N = 4 / 2: flags, flags+LPT, nvlink
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build50.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29711 scripts/dist_check.py > gpurun_out/dist_check50.log 2>&1; rc=$?; echo dist_check4 rc=$rc
grep rank0 gpurun_out/dist_check50.log | tail -4
[ $rc = 0 ] || exit 1
for rep in 1 2; do
for v in "4 flags contiguous" "4 flags lpt" "4 nvlink contiguous" "2 flags lpt"; do
  set -- $v
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port 2972$1 bench.py --gpus $1 --steps 30 --warmup 3 --no-e2e --assembly $2 --shard $3 > gpurun_out/fl50_n$1_$2_$3_$rep.log 2>&1
  echo "rep $rep N=$1 $2 $3 rc=$? $(grep '^{' gpurun_out/fl50_n$1_$2_$3_$rep.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'], d['ms_per_step'], d.get('per_rank',{}).get('ms_per_step'))")"
done
done
