"""Per-SASS-instruction execution counts of one kernel in an ncu report: the hottest region and an
opcode histogram weighted by executions.  usage: python tools/ncu_sass_hot.py rep.ncu-rep [kernel-substr] [top]"""
import csv, io, re, subprocess, sys, collections
rep = sys.argv[1]
ksub = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
blocks = raw.split('"Kernel Name",')
for b in blocks[1:]:
    name = b.split("\n", 1)[0]
    if ksub and ksub not in name:
        continue
    rows = list(csv.reader(io.StringIO(b.split("\n", 1)[1])))
    hdr = rows[0]
    ia, isrc, iex, ismp = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    ins = [(r[ia], r[isrc].strip(), int(r[iex] or 0), int(r[ismp] or 0)) for r in rows[1:] if len(r) > iex]
    tot = sum(x[2] for x in ins)
    print("==", name[:120], "total warp-inst", tot)
    hist = collections.Counter()
    for a, s, n, _ in ins:
        op = re.sub(r"^@!?U?P\w+\s+", "", s).split(" ")[0]
        hist[op.split(".")[0]] += n
    for op, n in hist.most_common(30):
        print(f"   {op:12s} {n / tot:6.1%}")
    mx = max(x[2] for x in ins)
    print("   -- instructions executed >= 50% of the max count (the steady-state loop):")
    hot = [x for x in ins if x[2] >= 0.5 * mx]
    print("   count", len(hot), "max", mx)
    if "--dump" in sys.argv:
        for a, s, n, smp in ins:
            if n >= 0.5 * mx:
                print(f"   {n:>10d} {smp:>6d}  {s}")
