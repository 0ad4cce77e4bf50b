"""Pins of the value-iteration oracle (Alg. 1; readings A36-A38).

* uniform reward r: V_t = r (1 - gamma^t) / (1 - gamma) after t iterations, and the stop test of
  l.8-10 fires at the first t with r gamma^(t-1) < threshold (geometric series, exact);
* holonomic one-cell moves, reward 1 on a goal node: V* = gamma^d / (1 - gamma), d the grid (L1,
  wrapped on periodic axes) distance to the goal (shortest path with discount);
* nearest-node successors: hand-computed shifts (ties toward the larger index), the SPEC
  nearest_index golden example, and the NumPy successor tables;
* Dubins MDP with slip: Jacobi and in-place orders reach the exact Bellman fixed point computed by
  policy iteration (sparse linear solves) in oracle/brute.py; Jacobi iterates equal NumPy's.
"""
import math

import numpy as np
import pytest

import oracle
from oracle import brute


def _grid(N, per, half=(2.0, 1.5, math.pi)):
    lo = tuple(-math.pi if per[d] else -half[d % 2] for d in range(len(N)))
    hi = tuple(math.pi if per[d] else half[d % 2] for d in range(len(N)))
    return lo, hi


@pytest.mark.parametrize("model,params,N,per", [("HOLONOMIC", (1.0, 0.1, 0.9), (7, 6), (0, 0)),
                                                ("DUBINS3D", (1.0, 1.0, 0.2, 0.05, 0.1, 0.8), (6, 5, 8), (0, 0, 1))])
def test_vi_uniform_reward_geometric_series(model, params, N, per):
    lo, hi = _grid(N, per)
    r, gamma, thr = 0.7, params[-1], 1e-5
    R = np.full(N, r, np.float32)
    for t in (1, 2, 5, 17):
        V, it, _ = oracle.vi_solve(N, lo, hi, sum(1 << d for d in range(len(N)) if per[d]), model, params, R,
                                   threshold=0.0, max_iters=t)
        assert it == t
        np.testing.assert_allclose(V, float(np.float32(r)) * (1 - gamma ** t) / (1 - gamma), rtol=1e-13)
    V, it, ch = oracle.vi_solve(N, lo, hi, sum(1 << d for d in range(len(N)) if per[d]), model, params, R,
                                threshold=thr)
    t_expect = next(t for t in range(1, 10000) if float(np.float32(r)) * gamma ** (t - 1) < thr)
    assert it == t_expect
    np.testing.assert_allclose(ch, float(np.float32(r)) * gamma ** (it - 1), rtol=1e-9)


@pytest.mark.parametrize("N,per,goal", [((9, 7), (0, 0), (6, 2)), ((8, 6, 5), (0, 1, 0), (1, 5, 2)),
                                        ((11,), (1,), (3,))])
@pytest.mark.parametrize("order", ["jacobi", "gauss_seidel"])
def test_vi_holonomic_discounted_shortest_path(N, per, goal, order):
    n = len(N)
    lo, hi = (0.0,) * n, tuple(float(N[d] if per[d] else N[d] - 1) for d in range(n))   # dx = 1
    gamma = 0.9
    R = np.zeros(N, np.float32)
    R[goal] = 1.0
    V, it, _ = oracle.vi_solve(N, lo, hi, sum(1 << d for d in range(n) if per[d]), "HOLONOMIC", (1.0, 1.0, gamma), R,
                               threshold=1e-12, order=order)
    I = np.meshgrid(*[np.arange(N[d]) for d in range(n)], indexing="ij")
    dist = 0
    for d in range(n):
        e = np.abs(I[d] - goal[d])
        dist = dist + (np.minimum(e, N[d] - e) if per[d] else e)
    np.testing.assert_allclose(V, gamma ** dist / (1 - gamma), atol=1e-10)


def test_vi_successor_rounding_and_faces():
    # x axis: dx = 0.5; dt v = 0.75 -> 1.5 cells -> tie, toward the larger index -> 2; v/2 -> 0.75 cells -> 1
    N, lo, hi = (9, 5, 8), (0.0, 0.0, -math.pi), (4.0, 2.0, math.pi)
    prm = (0.75, 1.0, 1.0, 0.0, 0.0, 0.9)          # vbar 0.75, wbar 1, dt 1, no slip
    st = [5 * 8, 8, 1]
    th0 = 4                                           # th = 0
    for a, shift in ((3, 2), (4, 2), (0, 1), (1, 1)):
        f = oracle.vi_successor(N, lo, hi, 4, "DUBINS3D", prm, (2, 2, th0), a, 0)
        i0 = f // st[0]
        assert i0 == 2 + shift
    # clamp at the x face (th = 0, +2 cells from the last node); w = +1 rad per step = 1.27 cells of
    # pi/4 -> +1 (th index 4 -> 5), and from th index 7 it wraps to 0
    f = oracle.vi_successor(N, lo, hi, 4, "DUBINS3D", prm, (8, 2, 4), 5, 0)
    assert f // st[0] == 8 and f % 8 == 5
    f = oracle.vi_successor(N, lo, hi, 4, "DUBINS3D", prm, (4, 2, 7), 5, 0)
    assert f % 8 == 0
    # NumPy tables agree everywhere
    prm = (1.3, 0.9, 0.37, 0.11, 0.1, 0.9)
    succ = brute.vi_successors(N, lo, hi, (0, 0, 1), "DUBINS3D", prm)
    rng = np.random.default_rng(0)
    for _ in range(200):
        idx = tuple(int(rng.integers(0, N[d])) for d in range(3))
        a, k = int(rng.integers(0, 6)), int(rng.integers(0, 3))
        flat = int(np.ravel_multi_index(idx, N))
        assert oracle.vi_successor(N, lo, hi, 4, "DUBINS3D", prm, idx, a, k) == succ[a][k][flat]


def _dubins_case(N, seed=0):
    lo, hi = (-2.0, -1.5, -math.pi), (2.0, 1.5, math.pi)
    rng = np.random.default_rng(seed)
    R = np.zeros(N, np.float32)
    I = np.meshgrid(*[np.linspace(lo[d], hi[d] if d < 2 else hi[d] - 2 * math.pi / N[d], N[d]) for d in range(3)],
                    indexing="ij")
    R[(I[0] - 1.0) ** 2 + (I[1] - 0.5) ** 2 < 0.5] = 1.0
    R[(I[0] + 0.5) ** 2 + I[1] ** 2 < 0.3] = -1.0
    R += rng.uniform(-0.01, 0.01, N).astype(np.float32)
    return lo, hi, R


@pytest.mark.parametrize("order", ["jacobi", "gauss_seidel"])
def test_vi_dubins_reaches_policy_iteration_fixed_point(order):
    N = (9, 8, 10)
    prm = (1.0, 1.2, 0.5, 0.2, 0.1, 0.85)
    lo, hi, R = _dubins_case(N)
    Vstar = brute.vi_policy_iteration(N, lo, hi, (0, 0, 1), "DUBINS3D", prm, R)
    V, it, ch = oracle.vi_solve(N, lo, hi, 4, "DUBINS3D", prm, R, threshold=1e-11, order=order)
    assert ch < 1e-11
    # contraction: |V - V*| <= gamma / (1 - gamma) * last change
    np.testing.assert_allclose(V, Vstar, atol=1e-9)


def test_vi_jacobi_iterates_equal_numpy():
    N = (7, 6, 8)
    prm = (1.1, 0.8, 0.4, 0.15, 0.2, 0.9)
    lo, hi, R = _dubins_case(N, seed=3)
    for t in (1, 3, 8):
        V, it, _ = oracle.vi_solve(N, lo, hi, 4, "DUBINS3D", prm, R, threshold=0.0, max_iters=t)
        np.testing.assert_allclose(V, brute.vi_jacobi(N, lo, hi, (0, 0, 1), "DUBINS3D", prm, R, t), atol=1e-13)


@pytest.mark.parametrize("N,per", [((5, 6, 5, 4, 6, 5), (0,) * 6), ((9, 10, 11, 7), (0, 1, 0, 1)), ((13,), (1,))])
def test_vi_holonomic_jacobi_iterates_equal_numpy(N, per):
    n = len(N)
    lo = tuple(-5.0 + d for d in range(n))
    hi = tuple(5.0 + 0.5 * d for d in range(n))
    R = np.random.default_rng(1).uniform(-1, 1, N).astype(np.float32)
    prm = (2.0, 0.9, 0.8)       # step 1.8: shifts of 0..2 cells depending on the axis spacing
    pm = sum(1 << d for d in range(n) if per[d])
    for t in (1, 4):
        V, _, _ = oracle.vi_solve(N, lo, hi, pm, "HOLONOMIC", prm, R, threshold=0.0, max_iters=t)
        np.testing.assert_allclose(V, brute.vi_jacobi(N, lo, hi, per, "HOLONOMIC", prm, R, t), atol=1e-13)


def test_vi_successor_ties_round_half_up():
    """SPEC nearest_index ("ties round toward the larger index"; example S:69-70: on the 1D grid
    [0, 0.25, 0.5, 0.75, 1] the midpoint 0.375 snaps to index 2).  Holonomic moves of exactly half a
    cell: +e from node 1 lands on 0.375 -> node 2; -e lands on 0.125 -> node 1 (the larger index),
    where round-half-to-even would pick node 0."""
    N, lo, hi = (5,), (0.0,), (1.0,)
    prm = (0.125, 1.0, 0.9)                       # speed * dt = 0.125 = half of dx = 0.25
    # actions: 0 stay, 1 +e0, 2 -e0
    assert oracle.vi_successor(N, lo, hi, 0, "HOLONOMIC", prm, (1,), 1, 0) == 2
    assert oracle.vi_successor(N, lo, hi, 0, "HOLONOMIC", prm, (1,), 2, 0) == 1
    assert oracle.vi_successor(N, lo, hi, 0, "HOLONOMIC", prm, (0,), 1, 0) == 1
    assert oracle.vi_successor(N, lo, hi, 0, "HOLONOMIC", prm, (2,), 2, 0) == 2
    # 2.5 cells -> 3 (half-to-even would give 2), -1.5 cells -> -1 (half-to-even: -2)
    N, lo, hi = (16,), (0.0,), (15.0,)
    prm = (2.5, 1.0, 0.9)
    assert oracle.vi_successor(N, lo, hi, 0, "HOLONOMIC", prm, (5,), 1, 0) == 8
    assert oracle.vi_successor(N, lo, hi, 0, "HOLONOMIC", prm, (5,), 2, 0) == 3
    prm = (1.5, 1.0, 0.9)
    assert oracle.vi_successor(N, lo, hi, 0, "HOLONOMIC", prm, (5,), 2, 0) == 4
    # the NumPy tables follow the same rule
    succ = brute.vi_successors(N, lo, hi, (0,), "HOLONOMIC", (2.5, 1.0, 0.9))
    assert succ[1][0][5] == 8 and succ[2][0][5] == 3
