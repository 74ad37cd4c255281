mkdir -p gpurun_out
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 scripts/dist_check.py > gpurun_out/dist_check2b.log 2>&1; echo dist_check rc=$?
grep rank0 gpurun_out/dist_check2b.log; tail -3 gpurun_out/dist_check2b.log
for a in nvlink nccl nvlink; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 2 --steps 20 --warmup 3 --no-e2e --assembly $a > gpurun_out/b2b.log 2>&1
  echo "[$a] rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/b2b.log').read().strip().splitlines()[-1]);k=d['kernel_ms_per_step'];print(d['value'], d['ms_per_step'], round(sum(k.values()),3))")"
done
