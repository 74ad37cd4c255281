# flag-based assembly: correctness (4 ranks) and N = 2, 4 vs the NCCL-sized NVLink assembly
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build49.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29701 scripts/dist_check.py > gpurun_out/dist_check49.log 2>&1; rc=$?; echo dist_check4 rc=$rc
grep rank0 gpurun_out/dist_check49.log
[ $rc = 0 ] || exit 1
for rep in 1 2; do
for n in 4 2; do
  for a in flags nvlink; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2970$n bench.py --gpus $n --steps 30 --warmup 3 --no-e2e --assembly $a > gpurun_out/fl49_n${n}_${a}_$rep.log 2>&1
    echo "rep $rep N=$n $a rc=$? $(grep '^{' gpurun_out/fl49_n${n}_${a}_$rep.log | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernel_ms_per_step'];print(d['value'], d['ms_per_step'], d.get('per_rank',{}).get('ms_per_step'))")"
  done
done
done
