"""Per-CUDA-source-line instruction counts of one kernel (ncu --print-source cuda,sass).
usage: python tools/ncu_cuda_lines.py rep.ncu-rep kernel-substr [top]"""
import csv, io, subprocess, sys, collections
rep, ksub = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 50
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
lines = raw.split("\n")
fname = fn = None
agg = collections.Counter()
src = {}
i = 0
hdr = None
for ln in lines:
    if ln.startswith('"File Path"'):
        fname = ln.split(",", 1)[1].strip('"').split("/")[-1]
        continue
    if ln.startswith('"Function Name"'):
        fn = ln.split(",", 1)[1]
        continue
    if ln.startswith('"Line No"'):
        hdr = next(csv.reader([ln]))
        continue
    if not hdr or not fn or ksub not in fn:
        continue
    r = next(csv.reader([ln])) if ln else None
    if not r or len(r) < len(hdr):
        continue
    iex = hdr.index("Instructions Executed")
    try:
        n = int(r[iex] or 0)
    except ValueError:
        continue
    key = (fname, r[0])
    agg[key] += n
    src[key] = r[1][:100]
tot = sum(agg.values()) or 1
print("total", tot)
for k, n in agg.most_common(top):
    print(f"{n / tot:6.1%} {k[0][:18]:18s}:{k[1]:>4}  {src[k]}")
