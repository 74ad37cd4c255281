mkdir -p gpurun_out
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521 scripts/dist_check.py > gpurun_out/dist_check4.log 2>&1; echo dist_check4 rc=$?
tail -2 gpurun_out/dist_check4.log
for n in 1 2 4; do
  if [ $n = 1 ]; then
    timeout 600 python bench.py --gpus 1 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/scale_n$n.log 2>&1
  else
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2953$n bench.py --gpus $n --steps 20 --warmup 3 > gpurun_out/scale_n$n.log 2>&1
  fi
  echo "N=$n rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/scale_n$n.log').read().strip().splitlines()[-1]);print(d['value'], d['ms_per_step'], d['kernel_ms_per_step']['scan_ms'], d['e2e']['value'])")"
done
