"""time-to-reach by Lax-Friedrichs iteration (Algorithm 3; readings
A31-A35) through the C-ABI (odp_ttr_solve) against the float64 oracle.

* holonomic dynamics: the fixed point is unique, so the GPU (Jacobi order, reading A35) must match
  the oracle's Gauss-Seidel sweeps (Algorithm 3 as printed) node by node;
* every dynamics: the GPU matches the oracle-side Jacobi iteration (oracle/brute.py, same order as
  the GPU) node by node, including the faces whose values depend on the iteration path;
* full size (t1, 256^3): every sampled reached node is a fixed point of the float64 update map,
  target nodes are 0, the faces obey l.14-15.
"""
import math

import numpy as np
import pytest

import oracle
from inputs import TTR_CONFIGS, axis_nodes, make_v0
from oracle import brute

pytestmark = pytest.mark.gpu


def _gpu(N, lo, hi, per, dyn, prm, V0, **kw):
    import torch
    from paper_2204_05520_b200 import capi
    g = capi.Grid(N, lo, hi, sum(1 << d for d in range(len(N)) if per[d]))
    try:
        V = torch.from_numpy(np.ascontiguousarray(V0, dtype=np.float32)).cuda()
        phi, info = capi.ttr_solve(g, dyn, prm, V, **kw)
        torch.cuda.synchronize()
        return phi.cpu().numpy().astype(np.float64), info
    finally:
        g.close()


def _case(n, N, per, r=1.0, seed=None, half=(3.0, 2.5)):
    lo = tuple(-half[d % 2] if not per[d] else -math.pi for d in range(n))
    hi = tuple(half[d % 2] if not per[d] else math.pi for d in range(n))
    axes = [axis_nodes(N[d], lo[d], hi[d], bool(per[d])) for d in range(n)]
    X = np.meshgrid(*axes, indexing="ij")
    v = np.sqrt(X[0] ** 2 + X[1] ** 2) - r
    if seed is not None:
        v = v + 0.05 * np.random.default_rng(seed).uniform(-1, 1, N)
    return lo, hi, v.astype(np.float32)


def _tol(ref):
    return 2e-5 * max(1.0, float(np.abs(ref[ref < 99]).max()))


@pytest.mark.parametrize("dyn,prm", [("HOLONOMIC_BALL", (1.0, -1.0)), ("HOLONOMIC_BOX", (1.0, 0.25, 1.0))])
@pytest.mark.parametrize("n,N", [(1, (61,)), (2, (41, 37)), (3, (17, 19, 16))])
def test_ttr_holonomic_matches_gauss_seidel_oracle(dyn, prm, n, N):
    per = (0,) * n
    if n == 1:
        lo, hi = (-3.0,), (3.0,)
        V0 = (np.abs(axis_nodes(N[0], -3.0, 3.0, False)) - 0.5).astype(np.float32)
    else:
        lo, hi, V0 = _case(n, N, per, seed=3)
    ref, _, ch = oracle.ttr_solve(N, lo, hi, 0, dyn, prm, V0, eps=1e-12, max_sweeps=20000)
    out, info = _gpu(N, lo, hi, per, dyn, prm, V0, eps=1e-7)
    assert info["iters"] < 100000
    np.testing.assert_allclose(out, ref, atol=_tol(ref), rtol=0)
    assert np.all(out[V0 <= 0] == 0.0)


CASES = [("HOLONOMIC_BALL", (1.3, -1.0), (0, 0), (23, 20)),
         ("HOLONOMIC_BOX", (1.0, 0.25, -1.0), (0, 1), (21, 24)),
         ("DUBINS3D", (1.0, 1.0, -1.0), (0, 0, 1), (13, 11, 12)),
         ("DUBINS3D", (1.0, 1.0, -1.0), (0, 0, 1), (16, 17, 18)),
         ("PAIR_DUBINS3D", (1.0, 1.0, 1.0, 0.5, -1.0), (0, 0, 1), (13, 11, 12)),
         ("CAR4D", (1.0, 1.0, 0.1, 0.1, -1.0), (0, 0, 0, 1), (11, 10, 7, 10)),
         ("CAR5D", (1.0, 1.0, -1.0), (0, 0, 1, 0, 0), (8, 9, 8, 5, 5)),
         ("DOUBLEINT6D", (1.0, 0.2, -1.0), (0,) * 6, (6, 5, 6, 5, 5, 6))]


def _coords(dyn, per, N):
    n = len(N)
    if dyn == "CAR4D":
        return (-3.0, -2.5, 0.2, -math.pi), (3.0, 2.5, 1.4, math.pi)
    if dyn == "CAR5D":
        return (-3.0, -2.5, -math.pi, 0.2, -1.0), (3.0, 2.5, math.pi, 1.4, 1.0)
    if dyn == "DOUBLEINT6D":
        return (-2.0, -1.0) * 3, (2.0, 1.0) * 3
    lo = tuple(-math.pi if per[d] else (-3.0, -2.5)[d % 2] for d in range(n))
    hi = tuple(math.pi if per[d] else (3.0, 2.5)[d % 2] for d in range(n))
    return lo, hi


@pytest.mark.parametrize("dyn,prm,per,N", CASES, ids=[f"{c[0]}-{'x'.join(map(str, c[3]))}" for c in CASES])
def test_ttr_matches_jacobi_oracle(dyn, prm, per, N):
    n = len(N)
    lo, hi = _coords(dyn, per, N)
    axes = [axis_nodes(N[d], lo[d], hi[d], bool(per[d])) for d in range(n)]
    X = np.meshgrid(*axes, indexing="ij")
    V0 = (np.sqrt(X[0] ** 2 + X[1] ** 2) - 1.0 + 0.05 * np.random.default_rng(7).uniform(-1, 1, N)).astype(np.float32)
    ref, iters = brute.ttr_jacobi(N, lo, hi, per, dyn, prm, V0, eps=1e-12)
    out, info = _gpu(N, lo, hi, per, dyn, prm, V0, eps=1e-7)
    np.testing.assert_allclose(out, ref, atol=_tol(ref), rtol=0)
    assert np.all(out[V0 <= 0] == 0.0) and np.all(out >= 0)
    assert info["last_change"] <= 1e-7 and iters < 200000


def test_ttr_unreachable_nodes_keep_big_and_graph_matches_direct():
    # zero control authority off axis 1: HOLONOMIC_BOX with ubar = dbar never moves -> H = -1,
    # sigma = 0 -> den = 0 keeps phi (l.10-11 undefined, A33): every non-target node stays `big`
    N, per = (12, 13), (0, 0)
    lo, hi, V0 = _case(2, N, per)
    out, info = _gpu(N, lo, hi, per, "HOLONOMIC_BOX", (0.5, 0.5, -1.0), V0, eps=1e-7, big=55.0)
    np.testing.assert_array_equal(out[V0 <= 0], 0.0)
    interior = np.zeros(N, bool)
    interior[1:-1, 1:-1] = True
    assert np.all(out[(V0 > 0) & interior] == 55.0)
    lo, hi, V0 = _case(2, (30, 31), per, seed=1)
    a, ia = _gpu((30, 31), lo, hi, per, "HOLONOMIC_BALL", (1.0, -1.0), V0, use_graph=True)
    b, ib = _gpu((30, 31), lo, hi, per, "HOLONOMIC_BALL", (1.0, -1.0), V0, use_graph=False)
    np.testing.assert_array_equal(a, b)
    assert ia["iters"] == ib["iters"]


def test_ttr_max_iters_cap():
    N, per = (40, 40), (0, 0)
    lo, hi, V0 = _case(2, N, per)
    out, info = _gpu(N, lo, hi, per, "HOLONOMIC_BALL", (1.0, -1.0), V0, max_iters=5)
    assert info["iters"] == 5 and info["last_change"] > 1e-6


def test_ttr_host_entry_matches_device_entry():
    from paper_2204_05520_b200 import capi
    N, per = (20, 22, 16), (0, 0, 1)
    lo, hi, V0 = _case(3, N, per, seed=2)
    a, _ = _gpu(N, lo, hi, per, "DUBINS3D", (1.0, 1.0, -1.0), V0)
    g = capi.Grid(N, lo, hi, 4)
    b, info = capi.ttr_solve_host(g, "DUBINS3D", (1.0, 1.0, -1.0), V0)
    g.close()
    np.testing.assert_array_equal(a, b.astype(np.float64))


def _sampled_fixed_point_residual(w, V0, phi, samples):
    """max over sampled reached interior nodes of |update(phi) - phi| (float64 map of brute.py on the
    3^n neighbourhood of each node), and of the face rule."""
    n = len(w.N)
    axes = [axis_nodes(w.N[d], w.lo[d], w.hi[d], bool(w.periodic[d])) for d in range(n)]
    dx = [axes[d][1] - axes[d][0] for d in range(n)]
    worst = 0.0
    for idx in samples:
        sl = []
        for d in range(n):
            sl.append(np.arange(idx[d] - 1, idx[d] + 2) % w.N[d])
        sub = phi[np.ix_(*sl)].astype(np.float64)
        lo = tuple(axes[d][idx[d]] - dx[d] for d in range(n))
        hi = tuple(axes[d][idx[d]] + dx[d] for d in range(n))
        new = brute.ttr_update_map((3,) * n, lo, hi, (0,) * n, w.dynamics, w.params, sub)
        c = (1,) * n
        worst = max(worst, abs(new[c] - sub[c]) / max(1.0, abs(sub[c])))
    return worst


def test_ttr_t1_full_size_fixed_point():
    w = TTR_CONFIGS["t1"]
    V0 = make_v0(w)
    out, info = _gpu(w.N, w.lo, w.hi, w.periodic, w.dynamics, w.params, V0, eps=1e-6)
    assert info["last_change"] <= 1e-6 and info["iters"] < 100000
    assert np.all(out[V0 <= 0] == 0.0) and np.all(out >= 0)
    rng = np.random.default_rng(11)
    reached = (out < 99) & (V0 > 0)
    reached[0], reached[-1], reached[:, 0], reached[:, -1] = False, False, False, False
    cand = np.argwhere(reached)
    samples = cand[rng.choice(len(cand), 400, replace=False)]
    assert _sampled_fixed_point_residual(w, V0, out, samples) < 2e-5
    # faces: l.14-15 idempotent
    a = brute.ttr_boundary_rule(w.N, w.periodic, out.copy())
    np.testing.assert_allclose(a, out, atol=1e-5, rtol=0)
    # the continuum TTR is at least the Euclidean distance to the disc (speed 1)
    X, Y = np.meshgrid(axis_nodes(w.N[0], w.lo[0], w.hi[0], False), axis_nodes(w.N[1], w.lo[1], w.hi[1], False),
                       indexing="ij")
    dist = np.maximum(np.sqrt(X ** 2 + Y ** 2) - 1.0, 0.0)[:, :, None]
    assert np.all(out[1:-1, 1:-1] >= dist[1:-1, 1:-1] - 0.1)


@pytest.mark.parametrize("N", [(24, 20), (12, 10, 14)])
def test_ttr_all_periodic_axes(N):
    # no faces at all: the interior launch is the iteration's last launch and runs the stop test
    n = len(N)
    per = (1,) * n
    lo, hi = (-2.0,) * n, (2.0,) * n
    axes = [axis_nodes(N[d], lo[d], hi[d], True) for d in range(n)]
    X = np.meshgrid(*axes, indexing="ij")
    V0 = (np.sqrt(sum(x ** 2 for x in X)) - 0.6).astype(np.float32)
    ref, _, _ = oracle.ttr_solve(N, lo, hi, (1 << n) - 1, "HOLONOMIC_BALL", (1.0, -1.0), V0, eps=1e-12,
                                 max_sweeps=20000)
    out, info = _gpu(N, lo, hi, per, "HOLONOMIC_BALL", (1.0, -1.0), V0, eps=1e-7)
    np.testing.assert_allclose(out, ref, atol=_tol(ref), rtol=0)
    assert info["last_change"] <= 1e-7


@pytest.mark.parametrize("fill", [1.0, -1.0])
def test_ttr_degenerate_targets(fill):
    # no target node: nothing is ever reached (phi stays `big`); every node a target: phi = 0
    N, per = (14, 13, 12), (0, 0, 1)
    lo, hi = (-2.0, -2.0, -math.pi), (2.0, 2.0, math.pi)
    V0 = np.full(N, fill, np.float32)
    out, info = _gpu(N, lo, hi, per, "DUBINS3D", (1.0, 1.0, -1.0), V0, big=77.0)
    np.testing.assert_array_equal(out, 77.0 if fill > 0 else 0.0)
    assert info["iters"] == 1 and info["last_change"] == 0.0
    ref, sweeps, _ = oracle.ttr_solve(N, lo, hi, 4, "DUBINS3D", (1.0, 1.0, -1.0), V0, big=77.0)
    np.testing.assert_array_equal(ref, out)


@pytest.mark.parametrize("dyn,prm,per,N", [c for c in CASES if len(c[3]) >= 3][:4])
def test_ttr_column_march_fallback_matches(dyn, prm, per, N, monkeypatch):
    # ODP_TTR_TILE=0: the column-marching kernel (the NDIM = 2 path) on the 3D+ cases
    monkeypatch.setenv("ODP_TTR_TILE", "0")
    n = len(N)
    lo, hi = _coords(dyn, per, N)
    axes = [axis_nodes(N[d], lo[d], hi[d], bool(per[d])) for d in range(n)]
    X = np.meshgrid(*axes, indexing="ij")
    V0 = (np.sqrt(X[0] ** 2 + X[1] ** 2) - 1.0 + 0.05 * np.random.default_rng(7).uniform(-1, 1, N)).astype(np.float32)
    ref, _ = brute.ttr_jacobi(N, lo, hi, per, dyn, prm, V0, eps=1e-12)
    out, info = _gpu(N, lo, hi, per, dyn, prm, V0, eps=1e-7)
    np.testing.assert_allclose(out, ref, atol=_tol(ref), rtol=0)
