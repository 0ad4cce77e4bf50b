"""Debug: GPU TTR iterates vs the oracle-side Jacobi iterates, k = 1..K."""
import sys, math
import numpy as np
sys.path.insert(0, '.')
from tests.test_gpu_ttr import _gpu, _coords, CASES
from inputs import axis_nodes
from oracle import brute
sel = sys.argv[1] if len(sys.argv) > 1 else "DUBINS3D"
for dyn, prm, per, N in CASES:
    if dyn != sel:
        continue
    n = len(N)
    lo, hi = _coords(dyn, per, N)
    axes = [axis_nodes(N[d], lo[d], hi[d], bool(per[d])) for d in range(n)]
    X = np.meshgrid(*axes, indexing="ij")
    V0 = (np.sqrt(X[0] ** 2 + X[1] ** 2) - 1.0 + 0.05 * np.random.default_rng(7).uniform(-1, 1, N)).astype(np.float32)
    for k in (1, 2, 3, 5, 10):
        ref, _ = brute.ttr_jacobi(N, lo, hi, per, dyn, prm, V0, eps=1e-300, max_iter=k)
        out, info = _gpu(N, lo, hi, per, dyn, prm, V0, eps=1e-30, max_iters=k)
        d = np.abs(out - ref)
        i = np.unravel_index(np.argmax(d), d.shape)
        print(dyn, N, k, info["iters"], "maxdiff", d.max(), "at", i, out[i], ref[i], flush=True)
    break
