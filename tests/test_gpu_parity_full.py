"""GPU parity at the BASELINE.json sizes, in the launch configuration bench.py times (kernel="auto").

* c2 (60^4, LOW): the whole horizon [0, 4] against the full float64 oracle, strict 1e-4.
* c3 (40^5) and c4 (30^6) (MEDIUM): one and two full time steps on the full grid, strict 1e-4
  except within the stencil radius of an oracle-flagged ENO2 near-tie (reading A28).
* c5 slab (8 x 48^5, 2.0e9 points, LOW): one time step on the full slab, strict 1e-4.
* MEDIUM over the whole horizon on coarsened copies (c3 to tau = 1, c4 to tau = 1): quantile bar.
  (c3 beyond tau ~ 1 is dominated by the unstable extrapolated inflow faces, reading A29.)
"""
import numpy as np
import pytest

import oracle
from inputs import CONFIGS, coarsened, make_v0
from tests.parity_util import (assert_parity, assert_parity_multistep_medium, assert_parity_one_step, run_gpu)

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
    ref = oracle.solve_workload(w, V0=V0)
    assert info["steps"] == ref.steps
    for k in range(out.shape[0]):
        assert_parity_multistep_medium(out[k], ref.out[k], what=f"{w.name} tau={tau[k + 1]}")
