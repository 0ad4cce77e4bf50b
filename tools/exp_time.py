"""Experiment timing (not a bench): run c4 for a few steps with the current env knobs and print the
per-launch average of pass 1 / pass 2 from the library's CUDA events, ignoring the solve status (the
ODP_MARCH_DBG modes compute garbage on purpose)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2204_05520_b200 as odp
from inputs import CONFIGS, make_v0

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
w = CONFIGS[name]
w = w.__class__(**{**w.__dict__, "tau": (0.0, 0.1)})
V0 = torch.from_numpy(make_v0(w)).cuda()
g = odp.Grid(w.N, w.lo, w.hi, w.periodic_mask)
for rep in range(2):
    out, info = odp.hj_solve(g, w.dynamics, w.params, V0, w.tau, w.accuracy, w.mode, cfl=w.cfl, timing=True,
                             raise_on_error=False)
torch.cuda.synchronize()
st = max(1, info["stages"])
km = info["kernel_ms"]
print(f"{name} stages={info['stages']} status={info['status']} pass1 {km['pass1'] / st:.3f} ms  pass2 {km['pass2'] / st:.3f} ms")
