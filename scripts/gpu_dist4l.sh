# the other configs on the multi-GPU path: Qwen3-14B (configs[3], 8 GPUs in the paper's
# setup: here N = 2, 4), Qwen3-4B (configs[1]) at N = 2, 4, and fp32 Qwen3-8B at N = 1, 4
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build53.log 2>&1
for v in "4 M4 bf16" "2 M4 bf16" "4 M2 bf16" "2 M2 bf16" "4 M3 fp32"; do
  set -- $v
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 --master-port 2973$1 bench.py --gpus $1 --config $2 --dtype $3 --steps 20 --warmup 3 --no-e2e > gpurun_out/cfg53_n$1_$2_$3.log 2>&1
  echo "N=$1 $2 $3 rc=$? $(grep '^{' gpurun_out/cfg53_n$1_$2_$3.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'], d['ms_per_step'], d['payload']['ratio'], d['roofline']['achieved'], d.get('per_rank',{}).get('ms_per_step'))")"
done
timeout 900 python bench.py --config M3 --dtype fp32 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/cfg53_n1_M3_fp32.log 2>&1
echo "N=1 M3 fp32 rc=$? $(grep '^{' gpurun_out/cfg53_n1_M3_fp32.log | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'], d['ms_per_step'], d['payload']['ratio'], d['roofline']['achieved'], d['kernel_ms_per_step'])")"
