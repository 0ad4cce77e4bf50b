"""Per-launch figures of an `ncu --set full` capture of one HJ solve, written into
profiles/ncu_kernels.json for bench.py's roofline (DRAM traffic and issue roofline per kernel).

usage: python tools/ncu_kernels.py rep.ncu-rep|raw.csv WORKLOAD [ACCURACY]
The capture must hold the march launches of one time step in launch order: MEDIUM
[pass 1, pass 2 (RK stage 1), pass 1, pass 2 (RK stage 2)], LOW [pass 1, pass 2].  CPU only."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep, workload = sys.argv[1], sys.argv[2]
acc = sys.argv[3] if len(sys.argv) > 3 else "medium"
if rep.endswith(".csv"):                  # `ncu -i rep --page raw --csv --print-units base` output
    raw = open(rep).read()
else:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"], capture_output=True,
                         text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
col = {h: i for i, h in enumerate(hdr)}


def val(r, name):
    return float(r[col[name]].replace(",", "")) if r[col[name]] else 0.0


launches = []
for r in rows[2:]:
    name = r[col["Kernel Name"]]
    if "k_march" not in name:
        continue
    targs = name.split("k_march<", 1)[1].split(">", 1)[0].replace("(bool)", "").replace("(int)", "").split(",")
    pass2 = targs[4].strip() in ("1", "true")           # k_march<F, NDIM, R, NP, PASS2, ...>
    launches.append({
        "kernel": name[:160],
        "pass2": pass2,
        "duration_ms": val(r, "gpu__time_duration.sum") * 1e3 if val(r, "gpu__time_duration.sum") < 10 else val(r, "gpu__time_duration.sum") / 1e6,
        "dram_bytes": val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum"),
        "warp_inst": val(r, "smsp__inst_executed.sum"),
        "issue_active_pct": val(r, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
        # L2 traffic: every L2 sector access (32 B) -- the SM side (srcunit tex: TMA + LDG) and all
        "lts_bytes_sm": 32.0 * val(r, "lts__t_sectors_srcunit_tex.sum") if "lts__t_sectors_srcunit_tex.sum" in col else None,
        "lts_bytes": 32.0 * val(r, "lts__t_sectors.sum") if "lts__t_sectors.sum" in col else None,
    })
names = ["pass1", "pass2_rk1", "pass1", "pass2_rk2"] if acc == "medium" else ["pass1", "pass2"]
out = {}
for nm, l in zip(names, launches):
    assert l["pass2"] == nm.startswith("pass2"), (nm, l["kernel"])
    out.setdefault(nm, l)
path = os.path.join(ROOT, "profiles", "ncu_kernels.json")
allp = json.load(open(path)) if os.path.exists(path) else {}
allp[workload] = out
allp["_source"] = ("ncu --set full --clock-control none of tools/profile_run.py (one time step), per launch: "
                   "dram__bytes_read.sum + dram__bytes_write.sum, smsp__inst_executed.sum, "
                   "smsp__issue_active.avg.pct_of_peak_sustained_active, 32 x lts__t_sectors(_srcunit_tex).sum")
json.dump(allp, open(path, "w"), indent=1)
print(json.dumps(out, indent=1))
