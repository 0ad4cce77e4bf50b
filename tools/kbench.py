"""Per-pass kernel timing of a few steps of a config (used to compare libodp.so variants).
usage: ODP_LIB_PATH=variants/x.so python tools/kbench.py c4 0.1 [kernel]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2204_05520_b200 as odp
from inputs import CONFIGS, make_v0

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
t1 = float(sys.argv[2]) if len(sys.argv) > 2 else 0.1
kernel = sys.argv[3] if len(sys.argv) > 3 else "auto"
w = CONFIGS[name]
w = w.__class__(**{**w.__dict__, "tau": (0.0, t1)})
V0 = torch.from_numpy(make_v0(w)).cuda()
g = odp.Grid(w.N, w.lo, w.hi, w.periodic_mask)
out = torch.empty((1,) + w.N, device="cuda")
odp.hj_solve(g, w.dynamics, w.params, V0, w.tau, w.accuracy, w.mode, out=out, cfl=w.cfl, kernel=kernel, raise_on_error=False)
best = None
for _ in range(3):
    _, info = odp.hj_solve(g, w.dynamics, w.params, V0, w.tau, w.accuracy, w.mode, out=out, cfl=w.cfl, kernel=kernel,
                           timing=True, raise_on_error=False)
    k = info["kernel_ms"]
    st = info["stages"]
    cur = (k["pass1"] / st, k["pass2"] / st)
    best = cur if best is None or sum(cur) < sum(best) else best
p1, p2 = best
rate = w.points / ((p1 + p2) / 1e3)
print(f"{name:6s} stages={st:4d} pass1 {p1:7.3f} ms  pass2 {p2:7.3f} ms  -> {rate:.3e} pt-stage/s "
      f"({rate * 16 / 6557.1e9:.1%} of HBM roofline @16 B/pt)")
