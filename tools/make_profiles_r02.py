"""Round-2 profile summaries under profiles/ from the captures tools/profile_round2.sh leaves in
gpurun_out/ (launch list, ncu --set full raw metric pages and SASS source pages as CSV)."""
import collections
import csv
import gzip
import io
import json
import os
import re
import shutil
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
src = "gpurun_out"
out = []

# 1) launch list of the c4 bench command's solve: shares of device time per kernel
lines = [l for l in open(os.path.join(src, f"{tag}_launches.csv")) if l.startswith('"')]
rd = list(csv.reader(io.StringIO("".join(lines))))
hdr = rd[0]
ik, iv, im, iu = (hdr.index(h) for h in ("Kernel Name", "Metric Value", "Metric Name", "Metric Unit"))
tot, cnt = collections.defaultdict(float), collections.Counter()
durs = collections.defaultdict(list)
for r in rd[1:]:
    if r[im] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(odp::MarchArgs.*|\(.*", "", r[ik]).replace("odp::", "")
    tot[name] += float(r[iv].replace(",", ""))
    cnt[name] += 1
    durs[name].append(float(r[iv].replace(",", "")))
unit = rd[1][iu]
T = sum(tot.values())
sh = [f"# {tag} launch list: ncu --metrics gpu__time_duration.sum --clock-control none of tools/profile_run.py c4 0.05",
      f"# (c4 30^6 MEDIUM, tau in [0, 0.05]); unit {unit}; cold-cache serialised launches: compare SHARES",
      "# 'active' = mean over the launches that did work: the graph-batched step loop launches one step past",
      "# tau_target whose kernels exit at once on the device-resident state (~2.5 us each), which deflates 'avg'", ""]
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    act = [x for x in durs[k] if x > 0.01 * max(durs[k])]
    sh.append(f"{v / T:7.2%}  {cnt[k]:4d} launches  avg {v / cnt[k]:12.1f}  active {len(act):3d} x {sum(act) / len(act):12.1f} {unit}  {k}")
open(f"profiles/{tag}_launch_shares.txt", "w").write("\n".join(sh) + "\n")
shutil.copy(os.path.join(src, f"{tag}_launches.csv"), f"profiles/{tag}_launches.csv")

# 2) ncu --set full: per launch metrics, stall breakdown, SASS opcode mix per warp-step
def summarize(cap, workload, points, names, nodes_per_warp_step=64):
    rows = list(csv.reader(open(os.path.join(src, f"{cap}_raw.csv"))))
    h = rows[0]
    c = {k: i for i, k in enumerate(h)}
    ks = [r for r in rows[2:] if "k_march" in r[c["Kernel Name"]]]
    sass = gzip.open(os.path.join(src, f"{cap}_sass.csv.gz"), "rt").read().split('"Kernel Name",')[1:]
    res = [f"## {workload} ({points:.3g} nodes): one time step, ncu --set full --clock-control none"]
    for li, (nm, r) in enumerate(zip(names, ks)):
        f = lambda k: float(r[c[k]].replace(",", "") or 0) if k in c else float("nan")
        dur = f("gpu__time_duration.sum")
        dur_ms = dur * 1e3 if dur < 10 else dur / 1e6
        dram = f("dram__bytes_read.sum") + f("dram__bytes_write.sum")
        wi = f("smsp__inst_executed.sum")
        steps = points / nodes_per_warp_step
        st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): f(k) for k in h
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
        S = sum(st.values()) or 1
        top = ", ".join(f"{k} {v / S:.0%}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:7])
        res.append(f"### {nm}: {re.sub(r'[(].*', '', r[c['Kernel Name']])[:90]}")
        res.append(f"  duration {dur_ms:.3f} ms | DRAM {dram / 1e9:.2f} GB = {dram / points:.1f} B/node | "
                   f"L2 sectors x32 {32 * f('lts__t_sectors.sum') / 1e9:.1f} GB | warp inst {wi / 1e9:.3f} G = "
                   f"{wi / steps:.0f} per warp-step (32 node pairs) | issue active "
                   f"{f('smsp__issue_active.avg.pct_of_peak_sustained_active'):.1f} % | warps/SMSP "
                   f"{f('smsp__warps_active.avg.per_cycle_active'):.2f} | regs {f('launch__registers_per_thread'):.0f}")
        res.append(f"  stall samples: {top}")
        # SASS opcode mix (executions per warp-step), from the source page of the same launch
        blk = sass[2 * li] if 2 * li < len(sass) else None     # the source page lists each launch twice
        if blk:
            rr = list(csv.reader(io.StringIO(blk.split("\n", 1)[1])))
            hh = rr[0]
            isrc, iex = hh.index("Source"), hh.index("Instructions Executed")
            hist = collections.Counter()
            for x in rr[1:]:
                if len(x) == len(hh):
                    op = re.sub(r"^@!?U?P\w+\s+", "", x[isrc].strip()).split(" ")[0]
                    hist[op] += int(x[iex] or 0)
            res.append("  SASS per warp-step: " + ", ".join(f"{k} {v / steps:.1f}" for k, v in hist.most_common(24)))
    return res

out += summarize(f"{tag}_c4", "c4 30^6 MEDIUM", 30 ** 6, ["pass 1 (RK stage 1)", "pass 2 (RK stage 1)", "pass 1 (RK stage 2)", "pass 2 (RK stage 2)"])
out += [""]
out += summarize(f"{tag}_c5low", "c5-slab LOW 8x48^5", 8 * 48 ** 5, ["pass 1", "pass 2"])
open(f"profiles/{tag}_ncu_full_summary.txt", "w").write("\n".join(out) + "\n")
print("\n".join(sh[:12]))
print("\n".join(out))
