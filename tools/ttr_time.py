"""Time odp_ttr_solve on a TTR workload: iterations, device ms, ns per node-iteration, GB/s at 12 B/node."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
from inputs import TTR_CONFIGS, make_v0, coarsened
from paper_2204_05520_b200 import capi
name = sys.argv[1] if len(sys.argv) > 1 else "t1"
w = TTR_CONFIGS[name]
sizes = [tuple(int(s) for s in a.split("x")) for a in sys.argv[2:]] or [w.N]
for N in sizes:
    ww = coarsened(w, N)
    g = capi.Grid(ww.N, ww.lo, ww.hi, ww.periodic_mask)
    V0 = torch.from_numpy(make_v0(ww)).cuda()
    phi, info = capi.ttr_solve(g, ww.dynamics, ww.params, V0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    phi, info = capi.ttr_solve(g, ww.dynamics, ww.params, V0, phi=phi)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    P = ww.points
    it = info["iters"]
    print(f"{N}: iters {it} total {ms:.2f} ms, loop {info['kernel_ms']:.2f} ms, {1e3*ms/it:.2f} us/iter, "
          f"{12*P*it/(ms/1e3)/1e9:.0f} GB/s @12B, {P*it/(ms/1e3)/1e9:.1f} Gnode-it/s, launches {g.launch_count()}", flush=True)
    g.close()
