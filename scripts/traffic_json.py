"""profiles/ncu_traffic.json from one `scripts/gpu_run.sh TAG traffic` capture (ncu --metrics
dram__bytes_read.sum,dram__bytes_write.sum,... over bench.py --steps 1 --warmup 0, M3, N=1):
per kernel the DRAM bytes of its FIRST launch (cold, serialised) — what bench.py reports as the
roofline's `traffic` for K1.
    python scripts/traffic_json.py gpurun_out/TAG/traffic.csv TAG > profiles/ncu_traffic.json"""
import csv
import json
import sys
from collections import OrderedDict

path, tag = sys.argv[1], sys.argv[2]
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
h = rows[0]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = OrderedDict()
for r in rows[1:]:
    per.setdefault((int(r[ii]), r[ki].split("(")[0].replace("void ", "").split("<")[0].split("::")[-1]), {})[r[mi]] = \
        float(r[vi].replace(",", ""))
kernels = OrderedDict()
for (_, name), m in sorted(per.items()):
    if name in kernels:
        continue  # first launch of each kernel
    kernels[name] = {"dram_read_bytes": int(m.get("dram__bytes_read.sum", 0)),
                     "dram_write_bytes": int(m.get("dram__bytes_write.sum", 0)),
                     "ncu_ns": int(m.get("gpu__time_duration.sum", 0)),
                     "dram_active_pct": round(100 * m["dram__cycles_active.avg"] / m["dram__cycles_elapsed.avg"], 2)
                     if m.get("dram__cycles_elapsed.avg") else None}
print(json.dumps({
    "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,dram__cycles_active.avg,... --clock-control "
              f"none (first launch of each kernel, cold L2, serialised), bench.py --steps 1 --warmup 0, M3 Qwen3-8B "
              f"rho=0.01 uniform bf16, N=1; capture {tag} (profiles/r02/traffic_{tag}.csv), same tree as the bench",
    "config": {"config": "M3", "rho": 0.01, "pattern": "uniform", "dtype": "bf16", "n_gpus": 1},
    "kernels": kernels}, indent=1))
