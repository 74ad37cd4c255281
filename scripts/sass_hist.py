"""ncu --page source --print-source sass --csv (file) -> per-opcode executed warp-instructions and
stall samples, normalised per warp of the first instruction (one kernel per file)."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
h = next(r for r in rows if "Address" in r)
ai, si, ie, ws = h.index("Address"), h.index("Source"), h.index("Instructions Executed"), \
    h.index("Warp Stall Sampling (All Samples)")
data = [r for r in rows if len(r) > ie and r[ai].startswith("0x")]
first = int(data[0][ie])
tot = sum(int(r[ie]) for r in data)
print(f"sass lines {len(data)}  warps {first}  warp-instr per warp {tot / first:.1f}  stall samples {sum(int(r[ws]) for r in data)}")
c, cs = Counter(), Counter()
for r in data:
    t = r[si].strip().split()
    op = (t[1] if t and t[0].startswith("@") else (t[0] if t else "?")).split(".")[0]
    c[op] += int(r[ie])
    cs[op] += int(r[ws])
for op, n in c.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 30):
    print(f"{op:10s} {n / first:8.1f} per warp   stall samples {cs[op]}")
