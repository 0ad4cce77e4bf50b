"""Turn gpurun_out/ captures into committed summaries under profiles/ (round tag argv[1])."""
import collections
import csv
import io
import json
import os
import re
import shutil
import subprocess
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
src = "gpurun_out"
os.makedirs("profiles", exist_ok=True)

# 1) launch list: share of device time per kernel (cold-cache, serialised; compare shares)
rows = []
with open(os.path.join(src, "launches.csv")) as fh:
    lines = [l for l in fh if l.startswith('"')]
rd = list(csv.reader(io.StringIO("".join(lines))))
hdr = rd[0]
ik, iv, im = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
tot = collections.defaultdict(float)
cnt = collections.Counter()
for r in rd[1:]:
    if r[im] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r[ik]).replace("odp::", "")
    v = float(r[iv].replace(",", ""))
    tot[name] += v
    cnt[name] += 1
unit = rd[1][hdr.index("Metric Unit")] if len(rd) > 1 else "?"
alltot = sum(tot.values())
summary = [f"# {tag} launch list (ncu --metrics gpu__time_duration.sum --clock-control none, c4 4 steps)",
           f"# unit: {unit}; shares of summed device time; cold-cache serialised launches", ""]
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    summary.append(f"{v / alltot:7.2%}  {cnt[k]:5d} launches  avg {v / cnt[k]:12.3f} {unit}  {k}")
open(f"profiles/{tag}_launch_shares.txt", "w").write("\n".join(summary) + "\n")
shutil.copy(os.path.join(src, "launches.csv"), f"profiles/{tag}_launches.csv")

# 2) full capture: per-kernel metrics + traffic per launch
rep = os.path.join(src, "prof_full.ncu-rep")
if os.path.exists(rep):
    out = subprocess.run([sys.executable, "tools/ncu_summary.py", rep], capture_output=True, text=True).stdout
    open(f"profiles/{tag}_ncu_full_summary.txt", "w").write(out)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    h = rr[0]
    traffic = {}
    for r in rr[2:]:
        d = dict(zip(h, r))
        targs = re.search(r"<([^>]*)>", d["Kernel Name"]).group(1).split(", ")
        kind = "pass2" if targs[4].strip() in ("1", "true", "(bool)1") else "pass1"
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
        rd_b = float(d["dram__bytes_read.sum"]) * scale[rr[1][h.index("dram__bytes_read.sum")]]
        wr_b = float(d["dram__bytes_write.sum"]) * scale[rr[1][h.index("dram__bytes_write.sum")]]
        traffic[f"c4:{kind}"] = rd_b + wr_b
        traffic[f"c4:{kind}:kernel"] = re.sub(r"\(.*", "", d["Kernel Name"])
    traffic["_source"] = f"profiles/{tag}_ncu_full_summary.txt (dram__bytes_read.sum + dram__bytes_write.sum, one launch each)"
    old = json.load(open("profiles/ncu_traffic.json")) if os.path.exists("profiles/ncu_traffic.json") else {}
    old.update(traffic)                     # keep the other workloads' entries (t1, v2)
    json.dump(old, open("profiles/ncu_traffic.json", "w"), indent=1)
if os.path.exists(os.path.join(src, "bench.json")):
    shutil.copy(os.path.join(src, "bench.json"), f"profiles/{tag}_bench.json")
print(open(f"profiles/{tag}_launch_shares.txt").read())
print(open("profiles/ncu_traffic.json").read())
