mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu22.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu22.log
python - <<'PY' > gpurun_out/digest_bench.log 2>&1
import time, torch, sys
sys.path.insert(0, ".")
import paper_2602_11456_b200 as sd
ctx = sd.DeltaContext("cuda:0")
for n in (268_586_518, 12_286_121_436 // 4):
    b = torch.randint(0, 255, (n,), dtype=torch.uint8, device="cuda")
    ctx.digest(b); torch.cuda.synchronize()
    t = time.perf_counter(); reps = 5
    for _ in range(reps): ctx.digest(b)
    dt = (time.perf_counter() - t) / reps
    print(f"digest {n} bytes: {dt*1e3:.3f} ms = {n/dt/1e9:.1f} GB/s")
PY
cat gpurun_out/digest_bench.log
