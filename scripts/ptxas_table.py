"""ptxas -v output (stdin) -> one line per kernel: registers, spill bytes, shared memory."""
import re
import subprocess
import sys

cur, rows = None, []
for ln in sys.stdin:
    m = re.search(r"Compiling entry function '(\w+)'", ln)
    if m:
        cur = {"name": m.group(1)}
        rows.append(cur)
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", ln)
    if m:
        cur["spill"] = f"{m.group(1)}/{m.group(2)}"
    m = re.search(r"Used (\d+) registers", ln)
    if m:
        cur["regs"] = m.group(1)
    m = re.search(r"(\d+) bytes smem", ln)
    if m:
        cur["smem"] = m.group(1)
names = subprocess.run(["cu++filt"], input="\n".join(r["name"] for r in rows), capture_output=True,
                       text=True).stdout.splitlines()
for r, n in zip(rows, names):
    n = n.split(">(")[0] + ">" if ">(" in n else n.split("(")[0]
    print(f"{r.get('regs', '?'):>4} regs  spill {r.get('spill', '?'):>8}  smem {r.get('smem', '0'):>6}  {n}")
