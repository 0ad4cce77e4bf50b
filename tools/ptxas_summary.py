"""Summarise `nvcc -Xptxas -v` output: kernel -> registers, stack, spills (reads stdin)."""
import re
import subprocess
import sys

txt = sys.stdin.read()
cur = None
rows = []
for line in txt.splitlines():
    m = re.search(r"Compiling entry function '([^']+)'", line)
    if m:
        cur = {"name": m.group(1)}
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        cur["stack"], cur["spill_st"], cur["spill_ld"] = map(int, m.groups())
    m = re.search(r"Used (\d+) registers", line)
    if m:
        cur["regs"] = int(m.group(1))
        rows.append(cur)
        cur = None
names = subprocess.run(["c++filt"], input="\n".join(r["name"] for r in rows), capture_output=True, text=True).stdout.split("\n")
for r, n in zip(rows, names):
    n = re.sub(r"\(.*", "", n).replace("odp::", "")
    if len(sys.argv) > 1 and not re.search(sys.argv[1], n):
        continue
    print(f"{r['regs']:4d} regs {r.get('stack', 0):4d} B stack {r.get('spill_st', 0):4d}/{r.get('spill_ld', 0):4d} spill  {n}")
