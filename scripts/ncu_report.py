"""Round summary of ncu captures: per-kernel section metrics of a --set full / --section report
and the executed warp-instructions per warp (source page), as markdown.
    python scripts/ncu_report.py LABEL REPORT.ncu-rep [LABEL REPORT ...]"""
import csv
import io
import subprocess
import sys

WANT = ("Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
        "Issued Warp Per Scheduler", "No Eligible", "Registers Per Thread", "Achieved Occupancy",
        "L2 Hit Rate", "Warp Cycles Per Issued Instruction")


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    res = {}
    for r in rows[1:]:
        k = r[ki].split("(")[0].replace("void ", "")
        if r[mi] in WANT and r[mi] not in res.setdefault(k, {}):
            res[k][r[mi]] = f"{r[vi]} {r[ui]}".strip()
    return res


def instr_per_warp(rep, kernel):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kernel}",
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    try:
        h = next(r for r in rows if "Address" in r)
    except StopIteration:
        return None
    if "Instructions Executed" not in h:  # a section-only capture has no source counters
        return None
    ai, ie = h.index("Address"), h.index("Instructions Executed")
    data = [r for r in rows if len(r) > ie and r[ai].startswith("0x")]
    if not data:
        return None
    first = min(data, key=lambda r: int(r[ai], 16))
    return sum(int(r[ie]) for r in data) / max(int(first[ie]), 1)


for label, rep in zip(sys.argv[1::2], sys.argv[2::2]):
    print(f"### {label} (`{rep}`)\n")
    d = details(rep)
    print("kernel | " + " | ".join(WANT) + " | warp-instr per warp")
    print("---|" + "---|" * len(WANT) + "---")
    for k, m in d.items():
        ipw = instr_per_warp(rep, k.split("<")[0].split("::")[-1])
        print(f"{k} | " + " | ".join(m.get(w, "") for w in WANT) + (f" | {ipw:.0f}" if ipw else " | "))
    print()
