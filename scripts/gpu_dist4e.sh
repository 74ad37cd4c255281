# K1b (offsets up front) parity; N = 1, 2, 4 with per-rank times; ncu launch list (filtered)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build42.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu42.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu42.log
for n in 1 2 4; do
  if [ $n = 1 ]; then
    timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/scale_e_n$n.log 2>&1
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2966$n bench.py --gpus $n --steps 20 --warmup 3 --no-e2e > gpurun_out/scale_e_n$n.log 2>&1
  fi
  echo "N=$n rc=$? $(grep '^{' gpurun_out/scale_e_n$n.log | python -c "import json,sys;d=json.loads(sys.stdin.read());k=d['kernel_ms_per_step'];print(d['value'], d['ms_per_step'], round(sum(k.values()),3), d.get('host_synced'), d.get('per_rank'), {a: round(b,3) for a,b in k.items()})")"
done
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-clocks"
$CMD > gpurun_out/plain42.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv --log-file gpurun_out/launches42.csv \
    $CMD > gpurun_out/ncu_launch42.log 2>&1
echo launches rc=$?
