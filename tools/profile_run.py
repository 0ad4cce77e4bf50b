"""Small fixed workload for ncu captures: a few steps of a config through odp_hj_solve."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2204_05520_b200 as odp
from inputs import CONFIGS, make_v0

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
t1 = float(sys.argv[2]) if len(sys.argv) > 2 else 0.02
kernel = sys.argv[3] if len(sys.argv) > 3 else "auto"
w = CONFIGS[name]
w = w.__class__(**{**w.__dict__, "tau": (0.0, t1)})
V0 = torch.from_numpy(make_v0(w)).cuda()
out, info = odp.solve_workload(w, V0, kernel=kernel)
torch.cuda.synchronize()
print(name, info, float(out.abs().max()))
