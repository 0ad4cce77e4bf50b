"""The resident kernel (ODP_KERNEL_RESIDENT, odp.cu k_resident): a whole solve in one cooperative
launch.  Its passes are the generic family's per-node bodies and its control steps the control
kernels' bodies run on a CTA-local state, so the result must be BITWISE the generic family's
(snapshots, steps, stages, tau) -- and therefore carries the generic family's oracle parity, which
test_gpu_parity.py checks for "resident" directly as well."""
import math

import numpy as np
import pytest

from inputs import CONFIGS, Workload, coarsened, holonomic, make_v0
from tests.parity_util import assert_parity, run_gpu, run_oracle

pytestmark = pytest.mark.gpu

CASES = [
    ("c1", None),                                      # 20 save intervals, LOW, periodic theta
    ("c2", (14, 12, 11, 13)),
    ("c3", (11, 10, 12, 9, 8)),
    ("c4", (8, 7, 8, 6, 7, 9)),
    ("f2", (14, 12, 11)),                              # Eq. 7: alpha^max over 3 coordinates (k_amax3 body)
]


def _case(name, N, acc):
    w = CONFIGS[name] if N is None else coarsened(CONFIGS[name], N, tau=(0.0, 0.05, 0.15, 0.2))
    return w.__class__(**{**w.__dict__, "accuracy": acc, "cfl": 0.8 if acc == "low" else 0.5})


@pytest.mark.parametrize("name,N", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("acc", ["low", "medium"])
@pytest.mark.parametrize("mode", ["brt", "brs"])
def test_resident_is_bitwise_the_generic_family(name, N, acc, mode):
    w = _case(name, N, acc)
    w = w.__class__(**{**w.__dict__, "mode": mode})
    for seed in (None, 1):
        V0 = make_v0(w, seed=seed)
        a, ia = run_gpu(w, V0, kernel="resident", write_initial=True)
        b, ib = run_gpu(w, V0, kernel="generic", write_initial=True)
        assert np.array_equal(a, b), (name, acc, mode, seed, float(np.abs(a - b).max()))
        assert (ia["steps"], ia["stages"], ia["tau_reached"]) == (ib["steps"], ib["stages"], ib["tau_reached"])


def test_resident_c1_against_the_oracle_and_one_launch():
    import torch
    import paper_2204_05520_b200 as odp
    w = CONFIGS["c1"]
    V0 = make_v0(w, seed=4)
    g = odp.Grid(w.N, w.lo, w.hi, w.periodic_mask)
    out, info = odp.hj_solve(g, w.dynamics, w.params, torch.from_numpy(V0).cuda(), w.tau, w.accuracy, w.mode,
                             cfl=w.cfl)                                   # AUTO picks resident here
    torch.cuda.synchronize()
    assert g.launch_count() == 2                       # k_init_state + the one cooperative launch
    ref = run_oracle(w, V0)
    assert_parity(out.cpu().numpy(), ref.out, what="c1 resident")
    assert info["steps"] == ref.steps and info["stages"] == ref.stages
    # the CTA count does not change the result (min/max partials are exact in any order)
    for ctas in ("1", "7", "64"):
        import os
        os.environ["ODP_RESIDENT_CTAS"] = ctas
        try:
            o2, _ = odp.hj_solve(g, w.dynamics, w.params, torch.from_numpy(V0).cuda(), w.tau, w.accuracy, w.mode,
                                 cfl=w.cfl, kernel="resident")
        finally:
            del os.environ["ODP_RESIDENT_CTAS"]
        assert torch.equal(o2, out), ctas


def test_resident_numeric_failure_matches_the_generic_family():
    import torch
    import paper_2204_05520_b200 as odp
    w = holonomic(2, 11, 1.0, "HOLONOMIC_BOX", (1.0, 0.0, -1.0), (0.0, 0.5), "low")
    V0 = make_v0(w)
    V0[3, 4] = np.nan
    _, info = odp.solve_workload(w, torch.from_numpy(V0).cuda(), kernel="resident", raise_on_error=False)
    assert info["status"] == odp.capi.ODP_ENUMERIC and "numerical" in odp.last_error()
    w2 = Workload("div", (21, 21), (-1.0, -1.0), (1.0, 1.0), (0, 0), "HOLONOMIC_BOX", (1.0, 0.0, -1.0),
                  (0.0, 10.0, 50.0), "low", 40.0, "brs", ("random_smooth", 1))
    V0 = make_v0(w2)
    _, ia = odp.solve_workload(w2, torch.from_numpy(V0).cuda(), kernel="resident", raise_on_error=False)
    _, ib = odp.solve_workload(w2, torch.from_numpy(V0).cuda(), kernel="generic", raise_on_error=False)
    assert ia["status"] == ib["status"] == 2
    assert (ia["steps"], ia["stages"], ia["tau_reached"]) == (ib["steps"], ib["stages"], ib["tau_reached"])


def test_resident_pair_dubins_against_the_oracle():
    # Eq. 7: alpha_d depends on (x, y, theta), so every step's alpha^max is the
    # grid-wide maximum k_amax3 takes -- inside the one launch, after one more grid barrier
    import torch
    import paper_2204_05520_b200 as odp
    w = Workload("pd", (12, 11, 10), (-6.0, -10.0, -math.pi), (20.0, 10.0, math.pi), (0, 0, 1), "PAIR_DUBINS3D",
                 (5.0, 5.0, 1.0, 1.0, 1.0), (0.0, 0.1, 0.4), "low", 0.8, "brt", ("cylinder", (0, 1), 5.0))
    V0 = make_v0(w)
    g = odp.Grid(w.N, w.lo, w.hi, w.periodic_mask)
    out, info = odp.hj_solve(g, w.dynamics, w.params, torch.from_numpy(V0).cuda(), w.tau, w.accuracy, w.mode,
                             cfl=w.cfl)                                   # AUTO picks resident here
    torch.cuda.synchronize()
    assert g.launch_count() == 2
    ref = run_oracle(w, V0)
    assert_parity(out.cpu().numpy(), ref.out, what="pair-dubins resident")
    assert info["steps"] == ref.steps and info["stages"] == ref.stages
    b, _ = odp.solve_workload(w, torch.from_numpy(V0).cuda(), kernel="generic")
    assert torch.equal(out, b)


def test_resident_refuses_where_it_does_not_apply():
    import torch
    import paper_2204_05520_b200 as odp
    w1 = _case("c2", (14, 12, 11, 13), "low")
    V1 = torch.from_numpy(make_v0(w1)).cuda()
    with pytest.raises(odp.OdpError, match="resident"):
        odp.solve_workload(w1, V1, kernel="resident", timing=True)
    # AUTO with kernel timing falls back to the launch-per-pass path (same result)
    a, _ = odp.solve_workload(w1, V1, kernel="auto", timing=True)
    b, _ = odp.solve_workload(w1, V1, kernel="resident")
    assert a.shape == b.shape
