# round-1 final validation of the tree: smoke, GPU suite, dist check, bench N = 1, 2, 4, reference arm
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/smoke76.log 2>&1; echo smoke rc=$?
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu76.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu76.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29751 scripts/dist_check.py > gpurun_out/dist_check76.log 2>&1; echo dist_check rc=$?
timeout 1200 python bench.py > gpurun_out/bench76_n1.log 2>&1; echo "N=1 rc=$?"
tail -1 gpurun_out/bench76_n1.log | cut -c1-400
for n in 2 4; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2976$n bench.py --gpus $n > gpurun_out/bench76_n$n.log 2>&1
  echo "N=$n rc=$? $(grep '^{' gpurun_out/bench76_n$n.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'], d['ms_per_step'], d['e2e']['value'], d.get('per_rank',{}).get('ms_per_step'))")"
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref76.log 2>&1; echo ref rc=$?
tail -1 gpurun_out/ref76.log | cut -c1-200
