"""The multi-GPU code path on one GPU: odp_grid_partition with a 1-rank NCCL communicator runs the
stage reduction as per-CTA partials -> range record -> ncclAllReduce(max) -> finalize (the path
every rank takes at 2/4/8 GPUs); the result must be bitwise the unpartitioned solve.  The halo
exchange itself needs >= 2 GPUs (a single gpurun box has one)."""
import numpy as np
import pytest

from inputs import CONFIGS, coarsened, make_v0

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,N,acc", [("c4", (12, 10, 12, 10, 12, 10), "medium"), ("c4", (12, 10, 12, 10, 12, 10), "low"),
                                        ("c1", (41, 41, 36), "low"), ("c3", (10, 9, 12, 9, 8), "medium")])
@pytest.mark.parametrize("kernel", ["march", "generic"])   # "auto" is the resident kernel on one rank
def test_one_rank_communicator_path_is_bitwise(name, N, acc, kernel):
    import torch
    import paper_2204_05520_b200 as odp
    from paper_2204_05520_b200 import dist as odist
    w = coarsened(CONFIGS[name], N, tau=(0.0, 0.05, 0.1))
    w = w.__class__(**{**w.__dict__, "accuracy": acc, "cfl": 0.8 if acc == "low" else 0.5})
    V0 = make_v0(w, seed=1)
    ref, rinfo = odp.solve_workload(w, torch.from_numpy(V0).cuda(), kernel=kernel)
    g = odist.partitioned_grid(w, 0, 1, torch.cuda.current_device(), force_comm=True)
    assert g.local_extent() == (0, w.N[0])
    out, info = odp.hj_solve(g, w.dynamics, w.params, torch.from_numpy(odist.local_v0(w, 0, 1, seed=1)).cuda(),
                             w.tau, w.accuracy, w.mode, cfl=w.cfl, kernel=kernel)
    torch.cuda.synchronize()
    assert info["steps"] == rinfo["steps"] and info["stages"] == rinfo["stages"]
    np.testing.assert_array_equal(out.cpu().numpy(), ref.cpu().numpy())
    g.close()


@pytest.mark.parametrize("name,N,acc", [("c4", (12, 10, 12, 10, 12, 10), "medium"), ("c4", (12, 10, 12, 10, 12, 10), "low"),
                                        ("c1", (41, 41, 36), "low"), ("c3", (10, 9, 12, 9, 8), "medium"),
                                        ("c2", (14, 12, 12, 16), "low")])
def test_single_pass_is_bitwise_the_two_pass_solve(name, N, acc):
    # for functors whose alpha does not depend on the derivative range the
    # single-pass path skips pass 1 after the first step; same alpha, same dt sequence, same arithmetic
    import torch
    import paper_2204_05520_b200 as odp
    w = coarsened(CONFIGS[name], N, tau=(0.0, 0.05, 0.1))
    w = w.__class__(**{**w.__dict__, "accuracy": acc, "cfl": 0.8 if acc == "low" else 0.5})
    V0 = torch.from_numpy(make_v0(w, seed=2)).cuda()
    ref, rinfo = odp.solve_workload(w, V0, kernel="march")      # AUTO would run k_resident here
    out, info = odp.solve_workload(w, V0, kernel="march", single_pass=True)
    assert info["single_pass"] == (name != "c2")      # CAR4D's alpha depends on the range's sign set
    assert info["steps"] == rinfo["steps"] and info["stages"] == rinfo["stages"]
    np.testing.assert_array_equal(out.cpu().numpy(), ref.cpu().numpy())


def test_single_pass_guard_reports_divergence():
    import torch
    import paper_2204_05520_b200 as odp
    from inputs import Workload
    import oracle
    w = Workload("div", (21, 21, 20), (-1.0, -1.0, -1.0), (1.0, 1.0, 1.0), (0, 0, 0), "HOLONOMIC_BOX",
                 (1.0, 0.0, -1.0), (0.0, 50.0), "low", 40.0, "brs", ("random_smooth", 3))
    V0 = make_v0(w)
    ref = oracle.solve_workload(w, V0=V0, raise_on_error=False)
    out, info = odp.solve_workload(w, torch.from_numpy(V0).cuda(), raise_on_error=False, single_pass=True)
    two, tinfo = odp.solve_workload(w, torch.from_numpy(V0).cuda(), raise_on_error=False)
    assert ref.status == 2 and info["status"] == 2 and tinfo["status"] == 2
    assert info["single_pass"]
    assert info["steps"] == tinfo["steps"] == ref.steps and info["stages"] == tinfo["stages"]
    assert info["tau_reached"] == tinfo["tau_reached"]


@pytest.mark.parametrize("name,N,acc", [("c4", (12, 10, 12, 10, 12, 10), "medium"), ("c4", (9, 10, 8, 10, 12, 10), "low"),
                                        ("c3", (10, 9, 12, 9, 8), "medium"), ("c2", (14, 12, 12, 16), "low")])
@pytest.mark.parametrize("comm", [False, True])
def test_split_pass1_overlap_path_is_bitwise(name, N, acc, comm, monkeypatch):
    # with >1 rank, pass 1 runs on the interior axis-0 planes while the halo exchange is
    # in flight on a side stream, then on the boundary planes; ODP_SPLIT_PASS1=1 forces that path on
    # one rank (without and with the 1-rank communicator) -- same result bit for bit
    import torch
    import paper_2204_05520_b200 as odp
    from paper_2204_05520_b200 import dist as odist
    w = coarsened(CONFIGS[name], N, tau=(0.0, 0.05, 0.1))
    w = w.__class__(**{**w.__dict__, "accuracy": acc, "cfl": 0.8 if acc == "low" else 0.5})
    V0 = torch.from_numpy(make_v0(w, seed=3)).cuda()
    ref, rinfo = odp.solve_workload(w, V0, kernel="march")
    monkeypatch.setenv("ODP_SPLIT_PASS1", "1")
    if comm:
        g = odist.partitioned_grid(w, 0, 1, torch.cuda.current_device(), force_comm=True)
        out, info = odp.hj_solve(g, w.dynamics, w.params, V0, w.tau, w.accuracy, w.mode, cfl=w.cfl, kernel="march")
        n_split = g.launch_count()
        monkeypatch.setenv("ODP_SPLIT_PASS1", "0")
        odp.hj_solve(g, w.dynamics, w.params, V0, w.tau, w.accuracy, w.mode, cfl=w.cfl, kernel="march")
        assert n_split > g.launch_count()          # the split path ran (one extra pass-1 launch per stage)
        monkeypatch.setenv("ODP_SPLIT_PASS1", "1")
        g.close()
    else:
        out, info = odp.solve_workload(w, V0, kernel="march")
    torch.cuda.synchronize()
    assert info["steps"] == rinfo["steps"] and info["stages"] == rinfo["stages"]
    np.testing.assert_array_equal(out.cpu().numpy(), ref.cpu().numpy())
    # and with per-launch timing (direct launches, both pass-1 launches inside one timed region)
    out2, info2 = odp.solve_workload(w, V0, kernel="march", timing=True)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out2.cpu().numpy(), ref.cpu().numpy())
    assert info2["kernel_ms"]["pass1"] > 0


@pytest.mark.parametrize("name,N,acc", [("c4", (12, 10, 12, 10, 12, 10), "medium"), ("c4", (12, 10, 12, 10, 12, 10), "low"),
                                        ("c1", (41, 41, 36), "low"), ("c3", (12, 11, 12, 10, 8), "medium")])
def test_single_pass_matches_the_oracle(name, N, acc):
    # SURVEY.md §8(f1) against the float64 oracle directly (not only against the two-pass GPU solve):
    # LOW strict 1e-4, MEDIUM the oracle-envelope bar (reading A28)
    import torch
    import paper_2204_05520_b200 as odp
    from tests.parity_util import assert_parity, assert_parity_envelope, oracle_envelope, run_oracle
    w = coarsened(CONFIGS[name], N, tau=(0.0, 0.2, 0.5))
    w = w.__class__(**{**w.__dict__, "accuracy": acc, "cfl": 0.8 if acc == "low" else 0.5})
    V0 = make_v0(w, seed=3)
    out, info = odp.solve_workload(w, torch.from_numpy(V0).cuda(), single_pass=True)
    assert info["single_pass"]
    out = out.cpu().numpy()
    if acc == "low":
        ref = run_oracle(w, V0)
        assert_parity(out, ref.out, what=f"single pass {name}")
    else:
        ref, E = oracle_envelope(w, V0)
        assert_parity_envelope(out, ref, E, what=f"single pass {name}")
    assert info["steps"] == ref.steps
