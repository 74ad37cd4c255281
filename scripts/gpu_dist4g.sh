# LPT vs contiguous, N = 2, 4, two repetitions each (alternating)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build44.log 2>&1
for rep in 1 2; do
for n in 2 4; do
  for sh in lpt contiguous; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2968$n bench.py --gpus $n --steps 30 --warmup 3 --no-e2e --shard $sh > gpurun_out/scale_g_n${n}_${sh}_$rep.log 2>&1
    echo "rep $rep N=$n $sh rc=$? $(grep '^{' gpurun_out/scale_g_n${n}_${sh}_$rep.log | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernel_ms_per_step'];print(d['value'], d['ms_per_step'], d.get('host_synced',{}).get('ms_per_step'), d.get('per_rank'))")"
  done
done
done
