# merge parity (merge path) + N = 1, 2, 4 with double-buffered NVLink assembly
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build36.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "merge" > gpurun_out/pytest_merge36.log 2>&1; echo merge rc=$?
tail -3 gpurun_out/pytest_merge36.log
timeout 600 python scripts/merge_bench.py > gpurun_out/merge36.log 2>&1; echo mb rc=$?; cat gpurun_out/merge36.log
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2965$n bench.py --gpus $n --steps 20 --warmup 3 --no-e2e > gpurun_out/scale_d_n${n}.log 2>&1
  echo "N=$n rc=$? $(grep '^{' gpurun_out/scale_d_n${n}.log | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernel_ms_per_step'];print(d['value'], d['ms_per_step'], round(sum(k.values()),3), d.get('host_synced'), {a: round(b,3) for a,b in k.items()})")"
done
