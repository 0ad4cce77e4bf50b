"""Top SASS instructions by warp-stall samples of one kernel block of an `ncu --page source --csv
--print-source sass` dump (gzip ok).  usage: python tools/ncu_stall_lines.py dump.csv[.gz] BLOCK [reason] [top]"""
import csv, gzip, io, sys, collections
path, blk = sys.argv[1], int(sys.argv[2])
reason = sys.argv[3] if len(sys.argv) > 3 else "Warp Stall Sampling (All Samples)"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
raw = (gzip.open(path, "rt") if path.endswith(".gz") else open(path)).read()
b = raw.split('"Kernel Name",')[blk]
name, body = b.split("\n", 1)
rows = list(csv.reader(io.StringIO(body)))
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
ins = [r for r in rows[1:] if len(r) == len(hdr)]
tot = collections.Counter()
for r in ins:
    for h in hdr:
        if h.startswith("stall_") and "Not Issued" not in h:
            tot[h] += int(r[ix[h]] or 0)
S = sum(tot.values())
print(name[:110]); print("samples", S, " ".join(f"{k[6:]}:{v / S:.1%}" for k, v in tot.most_common(10)))
key = ix[reason]
ins_sorted = sorted(range(len(ins)), key=lambda i: -int(ins[i][key] or 0))
for i in ins_sorted[:top]:
    r = ins[i]
    st = sorted(((h[6:], int(r[ix[h]] or 0)) for h in hdr if h.startswith("stall_") and "Not Issued" not in h), key=lambda x: -x[1])[:3]
    print(f"{i:5d} {int(r[key] or 0):6d} exec {int(r[ix['Instructions Executed']] or 0):10d}  {r[ix['Source']].strip()[:60]:60s} {st}")
