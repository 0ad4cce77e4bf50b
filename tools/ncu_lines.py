"""Per-source-line dynamic instruction counts (thread instr / point) of the first kernel in an ncu report."""
import csv, collections, io, subprocess, sys
rep, npts = sys.argv[1], float(sys.argv[2])
kre = sys.argv[3] if len(sys.argv) > 3 else "."
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass", "--kernel-name", f"regex:{kre}",
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
per_line = collections.defaultdict(lambda: [0, 0, ''])
cur = None; hdr = None; cur_file = None
for r in rows:
    if not r: continue
    if r[0] == 'File Path': cur_file = r[1].split('/')[-1]; continue
    if r[0] == 'Function Name': continue
    if r[0] == 'Line No': hdr = r; iT = hdr.index('Thread Instructions Executed'); iW = 4; continue
    if r[0]:
        cur = (cur_file, int(r[0])); per_line[cur][2] = r[1]; continue
    try: t = int(r[iT] or 0); w = int(r[iW] or 0)
    except Exception: continue
    per_line[cur][0] += t; per_line[cur][1] += w
tot = sum(v[0] for v in per_line.values()); totw = sum(v[1] for v in per_line.values()) or 1
print(f"total thread instr / point: {tot / npts:.1f}")
for k, v in sorted(per_line.items(), key=lambda x: -x[1][0])[:int(sys.argv[4]) if len(sys.argv) > 4 else 40]:
    print(f"{v[0] / npts:7.1f}/pt stall {v[1] / totw:5.1%}  {k[0]}:{k[1]}  {v[2].strip()[:90]}")
