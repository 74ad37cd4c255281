mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu14.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu14.log
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/b14.log 2>&1
echo "rc=$? $(tail -1 gpurun_out/b14.log)"
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --steps 20 --warmup 3 --no-e2e > gpurun_out/b14_n2.log 2>&1
echo "N=2 rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/b14_n2.log').read().strip().splitlines()[-1]);k=d['kernel_ms_per_step'];print(d['value'], d['ms_per_step'], round(sum(k.values()),3))")"
