# fixed-width codec parity + full gpu suite + bench (LEB128 default, then fixed)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build29.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k fixed > gpurun_out/pytest_fixed29.log 2>&1; echo fixed rc=$?
tail -15 gpurun_out/pytest_fixed29.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu29.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu29.log
for codec in leb128 fixed; do
  timeout 600 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --index-codec $codec > gpurun_out/b29_$codec.log 2>&1
  echo "$codec rc=$? $(python -c "import json;d=json.loads(open('gpurun_out/b29_$codec.log').read().strip().splitlines()[-1]);k=d['kernel_ms_per_step'];print(d['value'], d['ms_per_step'], d['payload']['body_bytes'], d['payload']['naive_fixed_width_bytes'], {a: round(b,3) for a,b in k.items()})")"
done
