"""continuous-MDP value iteration (Algorithm 1; readings A36-A38)
through the C-ABI (odp_vi_solve) against the float64 oracle.

* fixed iteration counts: every GPU iterate equals the oracle's Jacobi iterate node by node (the
  successors are integers decided in float32 on both sides, so any wrong successor shows up as an
  O(gamma p) difference, far above the float32 tolerance);
* convergence: the GPU result is within the contraction bound of the exact fixed point (policy
  iteration) and of the holonomic closed form gamma^d / (1 - gamma);
* full size (v2, 384x384x128): one GPU Bellman step at 400 sampled nodes equals the float64 step
  the oracle computes there from the GPU's previous iterate.
"""
import math

import numpy as np
import pytest

import oracle
from inputs import VI_CONFIGS, axis_nodes, make_reward
from oracle import brute

pytestmark = pytest.mark.gpu


def _gpu(N, lo, hi, per, model, prm, R, **kw):
    import torch
    from paper_2204_05520_b200 import capi
    g = capi.Grid(N, lo, hi, sum(1 << d for d in range(len(N)) if per[d]))
    try:
        Rt = torch.from_numpy(np.ascontiguousarray(R, dtype=np.float32)).cuda()
        V, info = capi.vi_solve(g, model, prm, Rt, **kw)
        torch.cuda.synchronize()
        return V.cpu().numpy().astype(np.float64), info
    finally:
        g.close()


def _tol(ref):
    return 4e-6 * max(1.0, float(np.abs(ref).max()))


DUB = (1.0, 1.0, 0.25, 0.1, 0.1, 0.95)
CASES = [("DUBINS3D", DUB, (25, 25, 9), (0, 0, 1)),
         ("DUBINS3D", (1.3, 0.7, 0.37, 0.17, 0.2, 0.9), (19, 23, 17), (0, 0, 1)),
         ("DUBINS3D", (1.0, 1.0, 0.25, 0.1, 0.1, 0.95), (300, 7, 5), (0, 0, 1)),
         ("HOLONOMIC", (1.0, 0.3, 0.9), (37,), (0,)),
         ("HOLONOMIC", (1.0, 0.3, 0.9), (29, 33), (1, 0)),
         ("HOLONOMIC", (2.0, 0.25, 0.8), (9, 10, 11, 7), (0, 1, 0, 1)),
         ("HOLONOMIC", (1.0, 0.5, 0.7), (5, 6, 5, 4, 6, 5), (0,) * 6)]


def _bounds(N, per):
    lo = tuple(-math.pi if per[d] else -5.0 + d for d in range(len(N)))
    hi = tuple(math.pi if per[d] else 5.0 + 0.5 * d for d in range(len(N)))
    return lo, hi


def _reward(N, seed):
    rng = np.random.default_rng(seed)
    R = np.where(rng.uniform(size=N) < 0.05, 1.0, 0.0) - np.where(rng.uniform(size=N) < 0.05, 1.0, 0.0)
    return (R + 0.01 * rng.uniform(-1, 1, N)).astype(np.float32)


@pytest.mark.parametrize("model,prm,N,per", CASES, ids=[f"{c[0]}-{'x'.join(map(str, c[2]))}" for c in CASES])
def test_vi_iterates_match_oracle(model, prm, N, per):
    lo, hi = _bounds(N, per)
    R = _reward(N, 1)
    pm = sum(1 << d for d in range(len(N)) if per[d])
    for t in (1, 2, 7, 30):
        ref, it, _ = oracle.vi_solve(N, lo, hi, pm, model, prm, R, threshold=0.0, max_iters=t)
        out, info = _gpu(N, lo, hi, per, model, prm, R, max_iters=t, fixed_iters=True)
        assert info["iters"] == t
        np.testing.assert_allclose(out, ref, atol=_tol(ref), rtol=0, err_msg=f"t={t}")


def test_vi_dubins_converges_to_exact_fixed_point():
    w = VI_CONFIGS["v0"]
    R = make_reward(w, seed=2)
    Vstar = brute.vi_policy_iteration(w.N, w.lo, w.hi, w.periodic, w.model, w.params, R)
    out, info = _gpu(w.N, w.lo, w.hi, w.periodic, w.model, w.params, R, threshold=1e-6)
    gamma = w.params[-1]
    assert info["last_change"] < 1e-6
    bound = gamma / (1 - gamma) * 1e-6 + 2e-6 * np.abs(Vstar).max() / (1 - gamma)
    assert np.abs(out - Vstar).max() <= bound, (np.abs(out - Vstar).max(), bound)
    # (iteration counts are not compared: a 1e-6 threshold is at float32 resolution for |V| ~ 10, so
    # the float32 change crosses it later than the float64 one -- 285 vs 271 iterations here)
    ref, it, _ = oracle.vi_solve(w.N, w.lo, w.hi, w.periodic_mask, w.model, w.params, R, threshold=1e-6)
    assert info["iters"] >= it - 2


@pytest.mark.parametrize("N,per,goal", [((41, 37), (0, 1), (30, 5)), ((12, 11, 10), (1, 0, 0), (0, 10, 4))])
def test_vi_holonomic_closed_form(N, per, goal):
    n = len(N)
    lo, hi = (0.0,) * n, tuple(float(N[d] if per[d] else N[d] - 1) for d in range(n))      # dx = 1
    gamma = 0.9
    R = np.zeros(N, np.float32)
    R[goal] = 1.0
    out, info = _gpu(N, lo, hi, per, "HOLONOMIC", (1.0, 1.0, gamma), R, threshold=1e-7)
    I = np.meshgrid(*[np.arange(N[d]) for d in range(n)], indexing="ij")
    dist = sum((np.minimum(np.abs(I[d] - goal[d]), N[d] - np.abs(I[d] - goal[d])) if per[d]
                else np.abs(I[d] - goal[d])) for d in range(n))
    np.testing.assert_allclose(out, gamma ** dist / (1 - gamma), atol=2e-5)


def test_vi_graph_direct_and_host_entries_agree():
    from paper_2204_05520_b200 import capi
    w = VI_CONFIGS["v1"]
    R = make_reward(w)
    a, ia = _gpu(w.N, w.lo, w.hi, w.periodic, w.model, w.params, R, use_graph=True)
    b, ib = _gpu(w.N, w.lo, w.hi, w.periodic, w.model, w.params, R, use_graph=False)
    np.testing.assert_array_equal(a, b)
    assert ia["iters"] == ib["iters"]
    g = capi.Grid(w.N, w.lo, w.hi, w.periodic_mask)
    c, ic = capi.vi_solve_host(g, w.model, w.params, R)
    g.close()
    np.testing.assert_array_equal(a, c.astype(np.float64))


def test_vi_v2_full_size_sampled_bellman_step():
    import torch
    from paper_2204_05520_b200 import capi
    w = VI_CONFIGS["v2"]
    R = make_reward(w, seed=5)
    g = capi.Grid(w.N, w.lo, w.hi, w.periodic_mask)
    Rt = torch.from_numpy(R).cuda()
    t = 25
    Vt, _ = capi.vi_solve(g, w.model, w.params, Rt, max_iters=t, fixed_iters=True)
    Vt = Vt.cpu().numpy().astype(np.float64)
    Vt1, _ = capi.vi_solve(g, w.model, w.params, Rt, max_iters=t + 1, fixed_iters=True)
    Vt1 = Vt1.cpu().numpy().astype(np.float64)
    g.close()
    acts, p, gamma = brute.vi_model(w.model, w.params, 3)
    rng = np.random.default_rng(9)
    idxs = [tuple(int(rng.integers(0, w.N[d])) for d in range(3)) for _ in range(300)]
    idxs += [(0, 5, 3), (w.N[0] - 1, w.N[1] - 1, 0), (7, 0, w.N[2] - 1)]          # faces and the seam
    for idx in idxs:
        best = -np.inf
        for a in range(len(acts)):
            ev = sum(p[k] * Vt.ravel()[oracle.vi_successor(w.N, w.lo, w.hi, w.periodic_mask, w.model, w.params,
                                                           idx, a, k)] for k in range(len(p)))
            best = max(best, float(R[idx]) + gamma * ev)
        assert abs(Vt1[idx] - best) <= 4e-6 * max(1.0, abs(best)), (idx, Vt1[idx], best)
