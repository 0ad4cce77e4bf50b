"""Mean per-kernel gpu__time_duration from an ncu --csv launch list."""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID") 
hdr = rows[start]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = defaultdict(list)
for r in rows[start + 1:]:
    if len(r) > vi:
        agg[r[ki][:70]].append(float(r[vi].replace(",", "")))
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{len(v):5d} x {sum(v)/len(v)/1e3:9.2f} us  {100*sum(v)/tot:5.1f}%  {k}")
