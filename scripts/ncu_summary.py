"""Summarise ncu outputs: launch-list CSV (per-kernel share) and a --set full report."""
import csv
import subprocess
import sys
from collections import defaultdict


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    h, data = rows[hdr], rows[hdr + 1:]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(list)
    for r in data:
        agg[r[ki].split("(")[0].replace("void ", "")].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    out = ["kernel | launches | mean ms | share of our kernels' time", "---|---|---|---"]
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        out.append(f"{k} | {len(v)} | {sum(v) / len(v) / 1e6:.4f} | {sum(v) / tot:.3f}")
    return "\n".join(out)


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "launch__grid_size", "lts__t_sectors_op_read.sum", "lts__t_sectors_op_write.sum",
        "lts__t_sector_hit_rate.pct", "smsp__inst_executed.sum",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard",
        "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
        "smsp__warp_issue_stalled_lg_throttle_per_warp_active.pct",
        "smsp__warp_issue_stalled_barrier_per_warp_active.pct"]


def full(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, units, data = rows[0], rows[1], rows[2:]
    out = []
    for r in data:
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "")
        out.append(f"### {name}  grid {r[h.index('launch__grid_size')]}")
        for w in WANT:
            if w in h:
                i = h.index(w)
                out.append(f"- {w}: {r[i]} {units[i]}")
    return "\n".join(out)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(f"## {p}\n")
        print(launches(p) if p.endswith(".csv") else full(p))
        print()
