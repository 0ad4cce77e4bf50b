"""GPU parity at the BASELINE.json sizes, in the launch configuration bench.py times (kernel="auto").

* c2 (60^4, LOW): the whole horizon [0, 4] against the full float64 oracle, strict 1e-4.
* c3 (40^5) and c4 (30^6) (MEDIUM): one and two full time steps on the full grid, strict 1e-4
  except within the stencil radius of an oracle-flagged ENO2 near-tie (reading A28).
* c5 slab (8 x 48^5, 2.0e9 points, LOW): one time step on the full slab, strict 1e-4.
* MEDIUM over the whole horizon on coarsened copies (c3 to tau = 1, c4 to tau = 1): the oracle-
  envelope bar (strict 1e-4 wherever the oracle's own float32 envelope is below 5e-5, reading A28).
  (c3 beyond tau ~ 1 is dominated by the unstable extrapolated inflow faces, reading A29.)
* MEDIUM at full size over the whole horizon: c4 (30^6, tau in [0, 1], 79 steps) and c3 (40^5, to
  tau = 1) against float64 oracle values at ~2e5 sampled nodes (uniform, face bands, whole in-plane
  tiles) written by tests/golden/make_full_size_oracle.py (a committed script calling only oracle/),
  with the oracle's float32-storage run as its envelope.
* c5 slab MEDIUM (8 x 48^5, 2.0e9 points), one and two time steps: the windowed oracle (pin Z12,
  tests/test_oracle_window.py) at sampled nodes, faces and slab ends included.
"""
import os

import numpy as np
import pytest

import oracle
from inputs import CONFIGS, coarsened, make_v0
from tests.parity_util import (TOL, assert_parity, assert_parity_envelope, assert_parity_one_step, full_grid_amax,
                                oracle_envelope, run_gpu, sample_nodes, windowed_oracle)

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

pytestmark = pytest.mark.gpu


def _with_tau(w, tau):
    return w.__class__(**{**w.__dict__, "tau": tuple(tau)})


def test_c2_full_size_full_horizon():
    w = CONFIGS["c2"]
    V0 = make_v0(w)
    out, info = run_gpu(w, V0)
    ref = oracle.solve_workload(w, V0=V0)
    assert info["steps"] == ref.steps == 410
    assert_parity(out, ref.out, what="c2 full")


@pytest.mark.parametrize("name,tau", [("c4", (0.0, 0.005)), ("c4", (0.0, 0.02)), ("c3", (0.0, 0.004)),
                                      ("c3", (0.0, 0.012))])
def test_medium_full_size_one_and_two_steps(name, tau):
    w = _with_tau(CONFIGS[name], tau)
    V0 = make_v0(w)
    out, info = run_gpu(w, V0)
    ref = oracle.solve_workload(w, V0=V0, ambiguity=True)
    assert info["steps"] == ref.steps and info["stages"] == ref.stages
    assert_parity_one_step(out, ref, R=2 * (ref.stages - 1), what=f"{name} {tau}")


def test_c5_slab_low_one_step():
    w = _with_tau(CONFIGS["c5slab-low"], (0.0, 0.01))
    V0 = make_v0(w)
    out, info = run_gpu(w, V0)
    ref = oracle.solve_workload(w, V0=V0)
    assert info["steps"] == ref.steps
    assert_parity(out, ref.out, what="c5 slab LOW")


@pytest.mark.parametrize("name,N,tau", [("c4", (12,) * 6, (0.0, 0.25, 0.5, 1.0)), ("c4", (16,) * 6, (0.0, 0.5, 1.0)),
                                        ("c3", (16,) * 5, (0.0, 0.5, 1.0))])
def test_medium_full_horizon_coarse(name, N, tau):
    w = coarsened(CONFIGS[name], N, tau=tau)
    V0 = make_v0(w)
    out, info = run_gpu(w, V0)
    ref, E = oracle_envelope(w, V0, nperturb=2)
    assert info["steps"] == ref.steps
    assert_parity_envelope(out, ref, E, what=f"{w.name} tau={tau[1:]}")


@pytest.mark.parametrize("name", ["c4", "c3"])
def test_medium_full_size_full_horizon_sampled(name):
    path = os.path.join(GOLDEN, f"{name}_full_horizon.npz")
    if not os.path.exists(path):
        pytest.skip(f"fixture {path} not generated (tests/golden/make_full_size_oracle.py)")
    fx = np.load(path)
    w = _with_tau(CONFIGS[name], tuple(fx["tau"]))
    assert tuple(fx["N"]) == w.N
    V0 = make_v0(w)
    out, info = run_gpu(w, V0)
    assert info["steps"] == int(fx["meta_f64"][0]) and info["stages"] == int(fx["meta_f64"][1])
    idx = fx["idx"]
    g = out[-1].reshape(-1)[idx].astype(np.float64)
    r = fx["V_f64"]
    E = np.abs(fx["V_f32store"] - r)
    d = np.abs(g - r)
    stable = E <= TOL / 2
    print(f"{name}: {len(idx)} nodes, max|dV| {d.max():.3e} (stable {d[stable].max():.3e}), max E {E.max():.3e}, "
          f"off {(d > TOL).sum()} vs oracle spread {(E > TOL).sum()}")

    class _Base:
        out = r
    assert_parity_envelope(g, _Base, E, what=f"{name} full size, {len(idx)} sampled nodes")


@pytest.mark.parametrize("steps", [1, 2])
def test_c5_slab_medium_windowed(steps):
    w0 = CONFIGS["c5slab-med"]
    amax = full_grid_amax(w0)
    # tau just below `steps` CFL steps (the last one clipped, reading A9; the GPU takes alpha^max in
    # float32, 0.8f = 0.8 (1 + 1.5e-8), so the margin is 1e-6)
    dt = 0.5 / float(np.sum(amax / np.array([(h - l) / (n - 1) for n, l, h in zip(w0.N, w0.lo, w0.hi)])))
    w = _with_tau(w0, (0.0, steps * dt * (1 - 1e-6)))
    V0 = make_v0(w)
    out, info = run_gpu(w, V0)
    nodes = sample_nodes(w.N, 40 if steps == 1 else 8, seed=11 + steps, faces=steps == 1)
    vals = windowed_oracle(w, nodes, 2, steps, amax)
    got = out[-1]
    errs = []
    for node, (v, st, _) in zip(nodes, vals):
        assert st == info["steps"] == steps
        errs.append(abs(float(got[node]) - v))
    assert max(errs) <= TOL, (max(errs), nodes[int(np.argmax(errs))])
