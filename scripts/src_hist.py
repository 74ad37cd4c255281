"""ncu --page source --print-source cuda,sass --csv (file) -> executed warp-instructions and stall
samples per CUDA source line (top N), normalised per warp of the kernel's first instruction."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
h = next(r for r in rows if r and r[0] == "Line No")
ie, ws = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
cur, per, stall, src, first = None, defaultdict(int), defaultdict(int), {}, None
lowest = None
for r in rows[rows.index(h) + 1:]:
    if len(r) <= ie:
        continue
    if r[0]:
        if not r[0].isdigit():
            continue
        cur = int(r[0])
        src[cur] = r[1].strip()
        continue
    if not r[2].startswith("0x"):
        continue
    n = int(r[ie])
    a = int(r[2], 16)
    if lowest is None or a < lowest:  # the kernel's entry instruction: executed once per warp
        lowest, first = a, n
    per[cur] += n
    stall[cur] += int(r[ws])
tot = sum(per.values())
print(f"warps {first}  warp-instr per warp {tot / first:.1f}  stall samples {sum(stall.values())}")
for ln in sorted(per, key=lambda k: -per[k])[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]:
    print(f"{ln:5d} {per[ln] / first:7.1f}  stalls {stall[ln]:6d}  {src.get(ln, '')[:90]}")
