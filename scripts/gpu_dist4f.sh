# LPT + record-granular NVLink assembly: correctness (dist_check, 4 ranks) and N = 2, 4
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build43.log 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29671 scripts/dist_check.py > gpurun_out/dist_check43.log 2>&1; echo dist_check4 rc=$?
grep rank0 gpurun_out/dist_check43.log
for n in 2 4; do
  for sh in lpt contiguous; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2967$n bench.py --gpus $n --steps 20 --warmup 3 --no-e2e --shard $sh > gpurun_out/scale_f_n${n}_$sh.log 2>&1
    echo "N=$n $sh rc=$? $(grep '^{' gpurun_out/scale_f_n${n}_$sh.log | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernel_ms_per_step'];print(d['value'], d['ms_per_step'], d.get('per_rank'), d['gpu_launches'])")"
  done
done
