# N = 4 step overhead: assembly on/off, comm stream priority
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build45.log 2>&1
for rep in 1 2; do
for v in "nvlink 0" "none 0" "nvlink -5"; do
  set -- $v
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29691 bench.py --gpus 4 --steps 30 --warmup 3 --no-e2e --assembly $1 --comm-priority $2 > gpurun_out/ov45_$1_$2_$rep.log 2>&1
  echo "rep $rep $1 prio $2 rc=$? $(grep '^{' gpurun_out/ov45_$1_$2_$rep.log | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernel_ms_per_step'];print(d['value'], d['ms_per_step'], round(sum(k.values()),3), d.get('per_rank'))")"
done
done
