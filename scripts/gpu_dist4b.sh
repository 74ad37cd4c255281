mkdir -p gpurun_out
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29621 scripts/dist_check.py > gpurun_out/dist_check4b.log 2>&1; echo dist_check4 rc=$?
grep rank0 gpurun_out/dist_check4b.log
for n in 1 2 4; do
  if [ $n = 1 ]; then
    timeout 900 python bench.py --gpus 1 --steps 20 --warmup 3 > gpurun_out/scale_b_n$n.log 2>&1
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2963$n bench.py --gpus $n --steps 20 --warmup 3 > gpurun_out/scale_b_n$n.log 2>&1
  fi
  echo "N=$n rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/scale_b_n$n.log').read().strip().splitlines()[-1]);k=d['kernel_ms_per_step'];print(d['value'], d['ms_per_step'], round(sum(k.values()),3), d['e2e']['value'])")"
done
for n in 2 4; do
  timeout 300 python bench.py --impl reference --gpus $n --steps 3 --warmup 1 > gpurun_out/ref_n$n.log 2>&1; echo "ref N=$n rc=$?"
done
