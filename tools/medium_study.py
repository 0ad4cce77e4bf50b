"""MEDIUM (ENO2 + TVD-RK2) parity study on the GPU box: one step at full size with the oracle's
ENO ambiguity mask, and full-horizon statistics on coarsened configs."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import oracle
from inputs import CONFIGS, coarsened, make_v0
from tests.parity_util import run_gpu


def dilate(mask, r):
    out = mask.copy()
    for ax in range(mask.ndim):
        for k in range(1, r + 1):
            sl_a = [slice(None)] * mask.ndim
            sl_b = [slice(None)] * mask.ndim
            sl_a[ax] = slice(k, None)
            sl_b[ax] = slice(None, -k)
            out[tuple(sl_a)] |= mask[tuple(sl_b)]
            out[tuple(sl_b)] |= mask[tuple(sl_a)]
    return out


def one_step(name, t1):
    w = CONFIGS[name]
    w = w.__class__(**{**w.__dict__, "tau": (0.0, t1)})
    V0 = make_v0(w)
    t = time.time()
    out, info = run_gpu(w, V0)
    tg = time.time() - t
    t = time.time()
    ref = oracle.solve_workload(w, V0=V0, ambiguity=True)
    to = time.time() - t
    d = np.abs(out[0].astype(np.float64) - ref.out[0])
    amb = ref.ambiguous.astype(bool)
    m = dilate(amb, 2)
    print(f"{name} one step (t1={t1}): steps {info['steps']}/{ref.steps}  gpu {tg:.1f}s oracle {to:.1f}s")
    print(f"   max|dV| all {d.max():.3e}  outside ambiguity mask {d[~m].max():.3e}  inside {d[m].max() if m.any() else 0:.3e}"
          f"  ambiguous nodes {amb.sum()} masked {m.sum()}  nodes>1e-4: {(d > 1e-4).sum()}")
    del out, ref, d, amb, m


def horizon(w0, N, tau):
    w = coarsened(w0, N, tau=tau)
    V0 = make_v0(w)
    out, info = run_gpu(w, V0)
    ref = oracle.solve_workload(w, V0=V0)
    f32 = oracle.solve_workload(w, V0=V0, store_f32=True)
    for k in range(out.shape[0]):
        d = np.abs(out[k] - ref.out[k])
        e = np.abs(f32.out[k] - ref.out[k])
        r = ref.out[k]
        memb = ((out[k] <= 0) != (r <= 0))
        print(f"{w.name} t={tau[k+1]}: gpu max {d.max():.2e} p99.9 {np.quantile(d, 0.999):.2e} p99 {np.quantile(d, 0.99):.2e} "
              f"frac>1e-4 {(d > 1e-4).mean():.2e} | f32s max {e.max():.2e} frac>1e-4 {(e > 1e-4).mean():.2e} | "
              f"memb mismatch |V|>=1e-4: {(memb & (np.abs(r) >= 1e-4)).sum()} |V|>=1e-3: {(memb & (np.abs(r) >= 1e-3)).sum()}"
              f" near-zero gpu max {d[np.abs(r) < 0.2].max():.2e}")


if __name__ == "__main__":
    what = sys.argv[1:] or ["horizon", "c4", "c3"]
    if "horizon" in what:
        horizon(CONFIGS["c4"], (12,) * 6, (0.0, 0.25, 0.5, 1.0))
        horizon(CONFIGS["c3"], (16,) * 5, (0.0, 0.5, 1.0, 2.0, 3.0))
        horizon(CONFIGS["c4"], (16,) * 6, (0.0, 0.5, 1.0))
    if "c4" in what:
        one_step("c4", 0.005)
    if "c3" in what:
        one_step("c3", 0.004)
