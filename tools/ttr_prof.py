"""One short odp_ttr_solve on a TTR workload (for ncu): max_iters iterations."""
import sys
import torch
sys.path.insert(0, '.')
from inputs import TTR_CONFIGS, make_v0
from paper_2204_05520_b200 import capi
w = TTR_CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "t1"]
it = int(sys.argv[2]) if len(sys.argv) > 2 else 16
g = capi.Grid(w.N, w.lo, w.hi, w.periodic_mask)
V0 = torch.from_numpy(make_v0(w)).cuda()
phi, info = capi.ttr_solve(g, w.dynamics, w.params, V0, max_iters=it, use_graph=False)
torch.cuda.synchronize()
print(info)
