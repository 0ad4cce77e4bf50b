"""Summarise ptxas -v output (registers / spills) for one kernel family from a build log."""
import re, subprocess, sys
fam = sys.argv[2] if len(sys.argv) > 2 else "k_march"
cur = None
rows = {}
for l in open(sys.argv[1]):
    m = re.search(r"Compiling entry function '(\S+)'", l)
    if m:
        cur = m.group(1)
        continue
    if cur and fam in cur:
        if "spill" in l or "registers" in l:
            rows.setdefault(cur, []).append(l.strip())
for k, v in rows.items():
    dem = subprocess.run(["c++filt"], input=k, capture_output=True, text=True).stdout.strip()
    dem = re.sub(r"\(odp::MarchArgs.*", "", dem).replace("odp::", "")
    regs = re.search(r"Used (\d+) registers", " ".join(v))
    sp = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", " ".join(v))
    print(f"{dem:55s} regs={regs.group(1) if regs else '?':>4} spill st/ld={sp.group(1) + '/' + sp.group(2) if sp else '-'}")
