"""K2 (k_tiles_scan) device time on the M3 workload: delta_size (K1 + K2 + size readback) in a
loop with profiling on, printing K2's CUDA-event time of the last 10 calls (ms).
    python scripts/k2_time.py      (GPU box)"""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import __graft_entry__ as entry
entry.build()
import paper_2602_11456_b200 as sd
from workload import generate_pair, qwen3
dev = torch.device("cuda", 0)
specs = qwen3("8B")
ts = []
for k, sp in enumerate(specs):
    o, w = generate_pair(sp, k, 0, rho=0.01, pattern="uniform", device=dev)
    ts.append((sp.name, o, w))
tl = sd.TensorList(ts)
ctx = sd.DeltaContext(dev)
ctx.set_profiling(True)
v = []
for i in range(12):
    try:
        ctx.delta_size(tl)
    except Exception:  # noqa: BLE001 (timing only)
        pass
    v.append(ctx.last_timing()["lens_ms"])
print("k2_ms", [round(x, 4) for x in v[2:]])
