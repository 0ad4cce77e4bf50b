"""Where does the end-to-end c4 time go?  pinned H2D / device solve / D2H vs odp_hj_solve_host."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
import paper_2204_05520_b200 as odp
from inputs import CONFIGS, make_v0
w = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
g = odp.Grid(w.N, w.lo, w.hi, w.periodic_mask)
V0h = make_v0(w)
V0p = torch.from_numpy(V0h).pin_memory()
outp = torch.empty((len(w.tau) - 1,) + w.N, dtype=torch.float32).pin_memory()
V0d = torch.empty(w.N, dtype=torch.float32, device="cuda")
outd = torch.empty((len(w.tau) - 1,) + w.N, dtype=torch.float32, device="cuda")
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    V0d.copy_(V0p, non_blocking=True); torch.cuda.synchronize(); t1 = time.perf_counter()
    odp.hj_solve(g, w.dynamics, w.params, V0d, w.tau, w.accuracy, w.mode, out=outd, cfl=w.cfl)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    outp.copy_(outd, non_blocking=True); torch.cuda.synchronize(); t3 = time.perf_counter()
    odp.hj_solve_host(g, w.dynamics, w.params, V0p, w.tau, w.accuracy, w.mode, out=outp, cfl=w.cfl)
    t4 = time.perf_counter()
    print(f"rep {rep}: H2D {t1-t0:.3f}s ({V0h.nbytes/(t1-t0)/1e9:.1f} GB/s)  solve {t2-t1:.3f}s  D2H {t3-t2:.3f}s  "
          f"sum {t3-t0:.3f}s  | hj_solve_host {t4-t3:.3f}s", flush=True)
