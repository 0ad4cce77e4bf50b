"""Short value iteration on a VI workload (for ncu / timing): fixed iteration count, direct launches."""
import sys
import torch
sys.path.insert(0, '.')
from inputs import VI_CONFIGS, make_reward
from paper_2204_05520_b200 import capi
w = VI_CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "v2"]
it = int(sys.argv[2]) if len(sys.argv) > 2 else 8
g = capi.Grid(w.N, w.lo, w.hi, w.periodic_mask)
R = torch.from_numpy(make_reward(w)).cuda()
for rep in range(3):
    V, info = capi.vi_solve(g, w.model, w.params, R, max_iters=it, fixed_iters=True, use_graph=False)
    torch.cuda.synchronize()
    print(rep, it, "iter_ms", info["iter_ms"] / it, "loop ms/iter", info["kernel_ms"] / it)
V, info = capi.vi_solve(g, w.model, w.params, R, threshold=1e-6, use_graph=False)
print("converged", info["iters"], "iter_ms", info["iter_ms"] / info["iters"])
