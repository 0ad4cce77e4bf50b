"""Isolated vs sustained launch times of the c4 kernels (why ncu's launch list is ~25 % faster than
the bench's live per-launch events): one time step at a time with idle gaps, then a full solve,
with nvidia-smi power / clocks sampled every 50 ms.  usage: python tools/power_probe.py [gap_s]"""
import subprocess
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2204_05520_b200 as odp
from inputs import CONFIGS, make_v0

gap = float(sys.argv[1]) if len(sys.argv) > 1 else 0.5
w = CONFIGS["c4"]
V0 = torch.from_numpy(make_v0(w)).cuda()
g = odp.Grid(w.N, w.lo, w.hi, w.periodic_mask)
out = torch.empty((1,) + w.N, device="cuda")


def solve(t1):
    _, info = odp.hj_solve(g, w.dynamics, w.params, V0, (0.0, t1), w.accuracy, w.mode, out=out, cfl=w.cfl,
                           timing=True, raise_on_error=False)
    k, st = info["kernel_ms"], info["stages"]
    return st, k["pass1"] / st, k["pass2"] / st


smi = subprocess.Popen(["nvidia-smi", "--query-gpu=timestamp,clocks.sm,clocks.mem,power.draw,temperature.gpu,"
                        "clocks_throttle_reasons.active", "--format=csv,noheader", "-lms", "50"],
                       stdout=subprocess.PIPE, text=True)
solve(0.0125)
marks = []
for i in range(8):
    time.sleep(gap)
    marks.append(("isolated", time.time()))
    st, p1, p2 = solve(0.0125)
    marks.append(("end", time.time()))
    print(f"isolated step {i}: stages={st} pass1 {p1:.3f} ms pass2(mean) {p2:.3f} ms", flush=True)
time.sleep(gap)
for t1 in (0.1, 1.0, 1.0):
    marks.append((f"sustained {t1}", time.time()))
    st, p1, p2 = solve(t1)
    marks.append(("end", time.time()))
    print(f"sustained tau 0..{t1}: stages={st} pass1 {p1:.3f} ms pass2(mean) {p2:.3f} ms", flush=True)
time.sleep(0.3)
smi.terminate()
lines = smi.stdout.read().strip().splitlines()
print("nvidia-smi samples (timestamp, sm MHz, mem MHz, W, C, reasons):")
for ln in lines:
    print("  ", ln)
print("marks:", [(m, round(t, 3)) for m, t in marks])
