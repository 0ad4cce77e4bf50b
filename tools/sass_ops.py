"""Opcode histogram (executed warp instructions) of each kernel section in an
`ncu -i rep --page source --csv --print-source sass` dump.  usage: sass_ops.py dump.csv [nodes]"""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
nodes = float(sys.argv[2]) if len(sys.argv) > 2 else None
secs, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1][:90], "hdr": None, "rows": []}
        secs.append(cur)
    elif r and r[0] in ("Address", "# Address") and cur is not None:
        cur["hdr"] = r
    elif cur is not None and cur["hdr"] and len(r) == len(cur["hdr"]):
        cur["rows"].append(r)
for s in secs:
    h = s["hdr"]
    ie, si = h.index("Instructions Executed"), h.index("Source")
    ops, tot = collections.Counter(), 0
    for r in s["rows"]:
        try:
            n = int(r[ie] or 0)
        except ValueError:
            continue
        t = r[si].split()
        if not t:
            continue
        op = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
        ops[op.split(".")[0]] += n
        tot += n
    print("==", s["name"], f"total {tot:.3e}")
    for k, v in ops.most_common(22):
        extra = f"  per-node {v * 32 / nodes:6.1f}" if nodes else ""
        print(f"   {k:10s} {100 * v / tot:5.1f}%{extra}")
