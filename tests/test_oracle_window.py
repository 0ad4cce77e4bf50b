"""Pins of two oracle modes the GPU parity tests rely on.

* Z12 -- windowed oracle: after s stages a node depends only on nodes within R s along each axis
  (Algorithm 2 is a radius-R star stencil per stage; the BRT min is pointwise) once
  alpha^max -- hence dt (l.164-167) -- is the full grid's.  A solve on a sub-box clipped at the real
  faces must therefore reproduce the full solve at the box centre.  Pinned against the full oracle
  solve itself (a different computation: one grid, no windows), with a negative control.
* Z4 -- float32-storage conditioning, the evidence behind reading A7 (CFL 0.8 LOW, 0.5 MEDIUM):
  the oracle with V rounded to float32 after every stage against itself in float64.  LOW meets
  Z4's 5e-5; MEDIUM does not at any tested CFL (ENO2 picks flip at float32 near-ties, reading A28:
  the gap barely moves when C is lowered, so A7 keeps 0.5 and the MEDIUM GPU bar is the oracle's
  own envelope, tests/parity_util.py::assert_parity_envelope).
"""
import numpy as np
import pytest

import oracle
from inputs import CONFIGS, coarsened, make_v0
from tests.parity_util import full_grid_amax, sample_nodes, windowed_oracle


def _with(w, **kw):
    return w.__class__(**{**w.__dict__, **kw})


@pytest.mark.parametrize("acc", ["low", "medium"])
def test_windowed_oracle_equals_the_full_solve(acc):
    w = coarsened(CONFIGS["c4"], (13, 11, 12, 10, 11, 12), tau=(0.0, 0.06))
    w = _with(w, accuracy=acc, cfl=0.8 if acc == "low" else 0.5)
    full = oracle.solve_workload(w, V0=make_v0(w))
    assert full.steps >= 2
    amax = full_grid_amax(w)
    np.testing.assert_allclose(amax, [2.0, 0.8, 2.0, 0.8, 2.0, 0.8], rtol=0, atol=1e-15)
    nodes = sample_nodes(w.N, 6, seed=5)
    vals = windowed_oracle(w, nodes, 1 if acc == "low" else 2, full.steps, amax)
    for node, (v, steps, _) in zip(nodes, vals):
        assert steps == full.steps
        assert abs(v - full.out[-1][node]) <= 1e-12, (node, v, full.out[-1][node])
    # negative control: without the full grid's alpha^max a box missing the velocity extremes takes
    # a different dt sequence and lands elsewhere
    mid = tuple(n // 2 for n in w.N)
    R = 1 if acc == "low" else 2
    hw = R * (1 if acc == "low" else 2) * full.steps
    box = [(max(0, i - hw), min(n, i + hw + 1) - max(0, i - hw)) for i, n in zip(mid, w.N)]
    if all(b > 0 or b + c < n for (b, c), n in zip(box[1::2], w.N[1::2])):
        from inputs import axis_nodes
        ax = [axis_nodes(n, l, h, False) for n, l, h in zip(w.N, w.lo, w.hi)]
        r = oracle.hj_solve(tuple(c for _, c in box), tuple(ax[d][b] for d, (b, c) in enumerate(box)),
                            tuple(ax[d][b + c - 1] for d, (b, c) in enumerate(box)), 0, w.dynamics, w.params,
                            make_v0(w, box=box), w.tau, w.accuracy, w.mode, cfl=w.cfl)
        loc = tuple(i - b for i, (b, _) in zip(mid, box))
        assert r.steps != full.steps or abs(r.out[-1][loc] - full.out[-1][mid]) > 1e-9


def test_z4_float32_storage_gap_fixes_reading_a7():
    w = coarsened(CONFIGS["c4"], (10,) * 6, tau=(0.0, 1.0))
    V0 = make_v0(w)
    gaps = {}
    for C in (0.5, 0.3):
        a = oracle.solve_workload(w, V0=V0, cfl=C)
        b = oracle.solve_workload(w, V0=V0, cfl=C, store_f32=True)
        d = np.abs(a.out - b.out)
        gaps[C] = (float(d.max()), float((d > 1e-4).mean()))
    # MEDIUM: Z4's 5e-5 fails at both CFLs and lowering C does not cure it (not a CFL effect) ...
    assert gaps[0.5][0] > 5e-5 and gaps[0.3][0] > 5e-5, gaps
    assert gaps[0.3][0] > 0.4 * gaps[0.5][0], gaps
    # ... and it is confined to isolated nodes (ENO2 decision flips, reading A28)
    assert gaps[0.5][1] < 1e-3, gaps
    # LOW (upwind + Euler) at C = 0.8 meets Z4 (reading A7)
    wl = _with(w, accuracy="low", cfl=0.8)
    a = oracle.solve_workload(wl, V0=V0)
    b = oracle.solve_workload(wl, V0=V0, store_f32=True)
    assert float(np.abs(a.out - b.out).max()) <= 5e-5
