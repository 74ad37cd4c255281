# multi-GPU bench of the final tree (check 85): dist check, then N = 2, 4 on one 4-GPU box
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build85.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29851 scripts/dist_check.py > gpurun_out/dist_check85.log 2>&1; echo dist_check rc=$?
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2986$n bench.py --gpus $n > gpurun_out/bench85_n$n.log 2>&1
  echo "N=$n rc=$? $(grep '^{' gpurun_out/bench85_n$n.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'], d['ms_per_step'], d['e2e']['value'])")"
done
