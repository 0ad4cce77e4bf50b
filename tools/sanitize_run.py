"""Small invocations of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck, one tool per run): march passes (6D MEDIUM and LOW, 3D Dubins with a periodic axis, a
ragged row block), the generic family, time-to-reach (3D, periodic theta with N <= 64: the tile
halo wrap) and value iteration."""
import math
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2204_05520_b200 as odp
from inputs import CONFIGS, TTR_CONFIGS, VI_CONFIGS, Workload, coarsened, make_reward, make_v0

torch.cuda.set_device(0)
cases = [
    coarsened(CONFIGS["c4"], (8, 7, 8, 7, 10, 8), tau=(0.0, 0.05)),                        # march MEDIUM 6D
    coarsened(CONFIGS["c5slab-low"], (6, 6, 7, 6, 12, 12), tau=(0.0, 0.05)),              # march LOW 6D
    coarsened(CONFIGS["c1"], (21, 19, 16), tau=(0.0, 0.2)),                               # march 3D, periodic columns
    coarsened(CONFIGS["c3"], (8, 7, 10, 9, 8), tau=(0.0, 0.05)),                           # periodic marching axis
    Workload("ragged", (9, 7, 11, 13), (-2.0, -1.0, -2.0, -1.0), (2.0, 1.0, 2.0, 1.0), (0, 0, 0, 0), "HOLONOMIC_BOX",
             (1.0, 0.2, -1.0), (0.0, 0.1), "medium", 0.5, "brt", ("random_smooth", 5)),     # generic family
]
for w in cases:
    V0 = torch.from_numpy(make_v0(w)).cuda()
    for kw in ({}, {"single_pass": True}):
        out, info = odp.solve_workload(w, V0, **kw)
        torch.cuda.synchronize()
        print(w.name, kw, info["steps"], float(out.abs().max()), flush=True)
w = coarsened(TTR_CONFIGS["t1"], (20, 18, 12))                                                 # periodic theta N = 12
g = odp.Grid(w.N, w.lo, w.hi, w.periodic_mask)
phi, tinfo = odp.ttr_solve(g, w.dynamics, w.params, torch.from_numpy(make_v0(w)).cuda(), eps=1e-5, max_iters=200)
torch.cuda.synchronize()
print("ttr", tinfo["iters"], float(phi.max()), flush=True)
g.close()
w = VI_CONFIGS["v0"]
g = odp.Grid(w.N, w.lo, w.hi, w.periodic_mask)
V, vinfo = odp.vi_solve(g, w.model, w.params, torch.from_numpy(make_reward(w)).cuda(), max_iters=20, fixed_iters=True)
torch.cuda.synchronize()
print("vi", vinfo["iters"], float(V.max()), flush=True)
g.close()
