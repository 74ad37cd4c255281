# N = 1, 2, 4 with the host-pipelined timed loop (default) and the per-step-synced one
mkdir -p gpurun_out
for n in 1 2 4; do
  for hs in end step; do
    if [ $n = 1 ]; then
      timeout 900 python bench.py --gpus 1 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --host-sync $hs > gpurun_out/scale_c_n${n}_$hs.log 2>&1
    else
      timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2964$n bench.py --gpus $n --steps 20 --warmup 3 --no-e2e --host-sync $hs > gpurun_out/scale_c_n${n}_$hs.log 2>&1
    fi
    echo "N=$n $hs rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/scale_c_n${n}_$hs.log').read().strip().splitlines()[-1]);k=d['kernel_ms_per_step'];print(d['value'], d['ms_per_step'], round(sum(k.values()),3), d.get('host_synced'), {a: round(b,3) for a,b in k.items()})")"
  done
done
