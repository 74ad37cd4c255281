# N = 4: NVLink assembly kernel grid (SM slots taken from the overlapped kernels)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build47.log 2>&1
for rep in 1 2; do
for c in 296 64 16; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29692 bench.py --gpus 4 --steps 30 --warmup 3 --no-e2e --assemble-ctas $c > gpurun_out/ac47_${c}_$rep.log 2>&1
  echo "rep $rep ctas $c rc=$? $(grep '^{' gpurun_out/ac47_${c}_$rep.log | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernel_ms_per_step'];print(d['value'], d['ms_per_step'], round(sum(k.values()),3), d.get('per_rank'))")"
done
done
