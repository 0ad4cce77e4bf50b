"""Whole-solve pins of the float64 oracle against closed forms, invariants and brute force (no GPU).

Z1  Hopf-Lax ball (the north-star closed form V = |x| - r - t), LOW order 1 / MEDIUM order 2 (Z3)
Z2  Hopf-Lax box with disturbance; periodic wrap through the -pi/pi seam (Dubins, v = 0)
Z5  linear fields are advanced exactly (ghosts, derivatives, costate, Euler / RK2)
Z6  BRT monotone non-increase (LOW) and containment of the target
Z7  holonomic avoid BRT keeps V0
Z10 mirror symmetry of c1
Z11 agreement with the NumPy brute force on tiny grids, all functors, both accuracies and modes
errors: EINVAL / ENUMERIC classes
"""
import math
import zlib

import numpy as np
import pytest

import oracle
from oracle import brute
from inputs import CONFIGS, Workload, axis_nodes, coarsened, holonomic, make_v0


def _mesh(w):
    ax = [axis_nodes(n, l, h, bool(p)) for n, l, h, p in zip(w.N, w.lo, w.hi, w.periodic)]
    return np.meshgrid(*ax, indexing="ij")


# ---- Z1 / Z3 ------------------------------------------------------------------------------------
@pytest.mark.parametrize("acc,order,first", [("low", 1.0, 2.2e-2), ("medium", 2.0, 1.4e-3)])
def test_hopf_lax_ball_convergence(acc, order, first):
    errs = []
    for N in (41, 81, 161):
        w = holonomic(2, N, 2.0, "HOLONOMIC_BALL", (1.0, -1.0), (0.0, 0.5), acc, target=("norm_ball", 0.5))
        r = oracle.solve_workload(w)
        X = _mesh(w)
        R = np.sqrt(sum(x * x for x in X))
        exact = np.maximum(R - 0.5, 0.0) - 0.5        # = |x| - r - t where |x| >= t (north_star)
        band = (R >= 1.5) & (R <= 1.8)
        errs.append(np.abs(r.out[-1] - exact)[band].max())
    rates = [math.log2(errs[i] / errs[i + 1]) for i in range(2)]
    assert errs[0] < first
    assert min(rates) > order - 0.15, (errs, rates)


def test_hopf_lax_ball_3d():
    w = holonomic(3, 41, 2.0, "HOLONOMIC_BALL", (1.0, -1.0), (0.0, 0.3), "low", target=("norm_ball", 0.6))
    V0 = make_v0(w)
    a = oracle.solve_workload(w, V0=V0).out[-1]
    b = oracle.solve_workload(w.__class__(**{**w.__dict__, "mode": "brs"}), V0=V0).out[-1]
    X = _mesh(w)
    R = np.sqrt(sum(x * x for x in X))
    exact = np.maximum(R - 0.3, 0.0) - 0.6
    band = (R > 1.0) & (R < 1.5)          # smooth band, away from the origin kink layer and the faces
    assert np.abs(a - exact)[band].max() < 0.05     # O(h) with h = 0.1 (first order, Z1)
    assert np.abs(b - exact)[band].max() < 0.05
    assert np.all(a <= b + 1e-12)          # the BRT min can only lower V


# ---- Z2 -------------------------------------------------------------------------------------------
def test_hopf_lax_box_with_disturbance():
    errs = []
    for N in (41, 81, 161):
        w = holonomic(2, N, 2.0, "HOLONOMIC_BOX", (1.0, 0.25, -1.0), (0.0, 0.6), "low", target=("norm_ball", 0.5))
        r = oracle.solve_workload(w)
        X = _mesh(w)
        c = (1.0 - 0.25) * 0.6
        exact = np.sqrt(sum(np.maximum(np.abs(x) - c, 0.0) ** 2 for x in X)) - 0.5
        near = np.abs(exact) < 0.2
        errs.append(np.abs(r.out[-1] - exact)[near].max())
    assert errs[0] < 0.07 and errs[1] < 0.65 * errs[0] and errs[2] < 0.65 * errs[1], errs


def test_periodic_seam_dubins_rotation():
    # DUBINS3D with v = 0, minimising turn, BRS, V0 = cos(theta): V = cos(|theta| + w t) (or -1)
    errs = []
    for Nt in (36, 72, 144):
        w = Workload("seam", (3, 3, Nt), (-1.0, -1.0, -math.pi), (1.0, 1.0, math.pi), (0, 0, 1), "DUBINS3D",
                     (0.0, 1.0, -1.0), (0.0, 0.7), "low", 0.8, "brs", ("cos", 2))
        r = oracle.solve_workload(w)
        th = axis_nodes(Nt, -math.pi, math.pi, True)
        s = np.abs(th) + 0.7
        exact = np.where(s <= math.pi, np.cos(np.minimum(s, math.pi)), -1.0)
        errs.append(np.abs(r.out[-1][1, 1] - exact).max())
    assert errs[0] < 0.08 and errs[2] < 0.4 * errs[0], errs


# ---- Z5 -------------------------------------------------------------------------------------------
@pytest.mark.parametrize("acc", ["low", "medium"])
@pytest.mark.parametrize("dyn,prm,speed", [("HOLONOMIC_BALL", (1.3, -1.0), 1.3), ("HOLONOMIC_BOX", (1.0, 0.3, -1.0), 0.7)])
@pytest.mark.parametrize("mode", ["brs", "brt"])
def test_linear_field_exact(acc, dyn, prm, speed, mode):
    n = 3
    w = Workload("lin", (9, 7, 8), (-2.0, -1.0, -1.5), (2.0, 1.0, 1.5), (0, 0, 0), dyn, prm, (0.0, 0.25, 0.5),
                 acc, 0.8 if acc == "low" else 0.5, mode, ("plane", 0, 1.0, 0.0))
    r = oracle.solve_workload(w)
    X = _mesh(w)
    for k, t in enumerate((0.25, 0.5)):
        np.testing.assert_allclose(r.out[k], X[0] - speed * t, atol=1e-12)


@pytest.mark.parametrize("acc", ["low", "medium"])
def test_linear_field_dubins_drift_exact(acc):
    # w = 0: V0 = x advances as V = x + t v cos(theta) exactly (alpha_theta = 0)
    w = Workload("lin-dub", (9, 5, 12), (-4.0, -1.0, -math.pi), (4.0, 1.0, math.pi), (0, 0, 1), "DUBINS3D",
                 (0.8, 0.0, 1.0), (0.0, 0.3), acc, 0.8, "brs", ("plane", 0, 1.0, 0.0))
    r = oracle.solve_workload(w)
    X = _mesh(w)
    np.testing.assert_allclose(r.out[-1], X[0] + 0.3 * 0.8 * np.cos(X[2]), atol=1e-12)


@pytest.mark.parametrize("acc", ["low", "medium"])
def test_linear_field_pairwise_dubins_drift_exact(acc):
    # Eq. 7 with abar = bbar = 0: f = (-va + vb cos th, va sin th, 0); V0 = x advances as
    # V = x + t (-va + vb cos th) exactly (p = (1, 0, *), alpha_th = 0)
    w = Workload("lin-pd", (9, 5, 12), (-4.0, -1.0, -math.pi), (4.0, 1.0, math.pi), (0, 0, 1), "PAIR_DUBINS3D",
                 (0.8, 1.1, 0.0, 0.0, 1.0), (0.0, 0.3), acc, 0.8, "brs", ("plane", 0, 1.0, 0.0))
    r = oracle.solve_workload(w)
    X = _mesh(w)
    np.testing.assert_allclose(r.out[-1], X[0] + 0.3 * (-0.8 + 1.1 * np.cos(X[2])), atol=1e-12)


def test_linear_solve_spec_example():
    # 1D, f = 1, phi0 = x on [-2, 2], horizon 0.5 -> x + 0.5 within 1e-9 (max with u in [-1,1])
    w = Workload("lin1d", (41,), (-2.0,), (2.0,), (0,), "HOLONOMIC_BOX", (1.0, 0.0, 1.0), (0.0, 0.5), "low", 0.8,
                 "brs", ("plane", 0, 1.0, 0.0))
    r = oracle.solve_workload(w)
    np.testing.assert_allclose(r.out[-1], axis_nodes(41, -2, 2, False) + 0.5, atol=1e-9)


def test_frozen_dynamics_keep_v0():
    # u_max = 0 -> H = 0, alpha = 0, dt = remaining time (A20): one step per save, V unchanged
    w = holonomic(2, 11, 1.0, "HOLONOMIC_BOX", (0.0, 0.0, -1.0), (0.0, 0.5, 1.0), "low", mode="brs")
    V0 = make_v0(w)
    r = oracle.solve_workload(w, V0=V0)
    assert r.steps == 2
    np.testing.assert_array_equal(r.out[-1], V0.astype(np.float64))


def test_cfl_step_count():
    # alpha = (1, 1), dx = (0.1, 0.1), C = 1 -> dt = 0.05: horizon 0.5 in exactly 10 steps
    w = holonomic(2, 21, 1.0, "HOLONOMIC_BOX", (1.0, 0.0, -1.0), (0.0, 0.5), "low", cfl=1.0)
    r = oracle.solve_workload(w)
    assert r.steps == 10 and r.tau_reached == pytest.approx(0.5, abs=1e-12)
    w = holonomic(2, 21, 1.0, "HOLONOMIC_BOX", (1.0, 0.0, -1.0), (0.0, 0.5), "medium", cfl=0.5)
    r = oracle.solve_workload(w)
    assert r.steps == 20 and r.stages == 40


# ---- Z6 / Z7 --------------------------------------------------------------------------------------
def test_brt_monotone_and_contains_target_c1():
    w = CONFIGS["c1"]
    V0 = make_v0(w)
    r = oracle.solve_workload(w, V0=V0, write_initial=True)
    assert r.out.shape[0] == 21 and r.steps == 40
    diffs = np.diff(r.out, axis=0)
    # V^{k+1} <= V^k (LOW, Z6) exactly on nodes outside the domain of dependence of the x/y faces:
    # the extrapolated ghosts (A12) are not order-preserving, so increases start at face nodes and
    # travel inward one node per stage (2 stages per save interval here)
    for k in range(diffs.shape[0]):
        s = 2 * (k + 1) + 1
        if 41 - 2 * s <= 0:
            break
        assert diffs[k][s:41 - s, s:41 - s].max() <= 0.0, k
    assert np.all(r.out[-1][V0 <= 0] <= 0)                         # {V0 <= 0} subset {V <= 0}
    assert np.all(r.out[-1] <= V0.astype(np.float64) + 1e-15)


def test_brt_monotone_car4d_coarse():
    w = coarsened(CONFIGS["c2"], (40, 40, 12, 12), tau=(0.0, 0.1, 0.2))
    V0 = make_v0(w)
    r = oracle.solve_workload(w, V0=V0, write_initial=True)
    s = r.steps + 1      # x/y faces only (v-axis controls push away; theta is periodic)
    d = np.diff(r.out, axis=0)[:, s:40 - s, s:40 - s, 3:-3]
    assert d.max() <= 0.0
    assert (r.out[-1] <= 0).sum() > (V0 <= 0).sum()              # the tube grows


@pytest.mark.parametrize("acc", ["low", "medium"])
def test_holonomic_avoid_keeps_target(acc):
    w = holonomic(2, 41, 2.0, "HOLONOMIC_BALL", (1.0, 1.0), (0.0, 0.5), acc, target=("norm_ball", 0.5))
    V0 = make_v0(w)
    r = oracle.solve_workload(w, V0=V0)
    np.testing.assert_array_equal(r.out[-1], V0.astype(np.float64))


# ---- Z10 ------------------------------------------------------------------------------------------
def test_c1_mirror_symmetry():
    # c1: V(x, -y, -theta) = V(x, y, theta); theta nodes -pi + k d map to node (36 - k) mod 36
    w = CONFIGS["c1"]
    r = oracle.solve_workload(w)
    V = r.out[-1]
    k = (36 - np.arange(36)) % 36
    Vm = V[:, ::-1, :][:, :, k]
    assert np.abs(V - Vm).max() < 1e-12


def test_c4_pair_symmetries_coarse():
    w = coarsened(CONFIGS["c4"], (8,) * 6, tau=(0.0, 0.3))
    V = oracle.solve_workload(w).out[-1]
    # (p_i, v_i) -> (-p_i, -v_i) per pair and the permutation of pairs (x,y,z)
    np.testing.assert_allclose(V, V[::-1, ::-1], atol=1e-5)
    np.testing.assert_allclose(V, V.transpose(2, 3, 0, 1, 4, 5), atol=1e-12)


# ---- Z11 ------------------------------------------------------------------------------------------
TINY = [
    ("HOLONOMIC_BALL", (1.0, -1.0), 1, ()),
    ("HOLONOMIC_BALL", (1.0, 1.0), 2, ()),
    ("HOLONOMIC_BOX", (1.0, 0.3, -1.0), 3, (1,)),
    ("HOLONOMIC_BOX", (1.0, 0.3, 1.0), 4, ()),
    ("DUBINS3D", (1.0, 1.0, 1.0), 3, (2,)),
    ("DUBINS3D", (1.0, 0.5, -1.0), 3, (2,)),
    ("CAR4D", (1.5, 1.0, 0.25, 0.25, -1.0), 4, (3,)),
    ("CAR5D", (1.0, 2.0, -1.0), 5, (2,)),
    ("DOUBLEINT6D", (1.0, 0.2, -1.0), 6, ()),
    ("PAIR_DUBINS3D", (1.0, 1.2, 1.0, 0.8, 1.0), 3, (2,)),
    ("PAIR_DUBINS3D", (0.8, 1.0, 0.5, 0.7, -1.0), 3, (2,)),
]


@pytest.mark.parametrize("dyn,prm,n,per", TINY, ids=[f"{t[0]}-{t[2]}d-{t[1][-1]:+.0f}" for t in TINY])
@pytest.mark.parametrize("acc", ["low", "medium"])
def test_brute_force_agreement(dyn, prm, n, per, acc):
    rng = np.random.default_rng(zlib.crc32(f"{dyn}{n}{acc}{prm}".encode()))
    for seed in range(10 if n <= 4 else 3):
        N = tuple(int(v) for v in rng.integers(3, 8 if n <= 4 else 5, size=n))
        lo = tuple(float(v) for v in rng.uniform(-3, -1, n))
        hi = tuple(float(v) for v in rng.uniform(1, 3, n))
        periodic = tuple(1 if d in per else 0 for d in range(n))
        mode = "brt" if seed % 2 == 0 else "brs"
        w = Workload("tiny", N, lo, hi, periodic, dyn, prm, (0.0, 0.05, 0.12), acc, 0.8 if acc == "low" else 0.5,
                     mode, ("random_smooth", seed))
        V0 = make_v0(w)
        rb, steps = brute.solve(w, V0)
        ro = oracle.solve_workload(w, V0=V0)
        assert ro.steps == steps
        np.testing.assert_allclose(ro.out, rb, atol=1e-12, rtol=0)


# ---- errors ---------------------------------------------------------------------------------------
def test_error_classes():
    w = holonomic(2, 11, 1.0, "HOLONOMIC_BOX", (1.0, 0.0, -1.0), (0.0, 0.5), "low")
    V0 = make_v0(w)
    bad = [
        dict(tau=(0.1, 0.5)), dict(tau=(0.0, 0.5, 0.5)), dict(tau=(0.0,)), dict(params=(1.0, -1.0)),
        dict(dynamics="DUBINS3D", params=(1.0, 1.0, 1.0)), dict(params=(1.0, 0.0, 0.5)),
    ]
    for b in bad:
        ww = w.__class__(**{**w.__dict__, **b})
        r = oracle.solve_workload(ww, V0=V0, raise_on_error=False)
        assert r.status == oracle.EINVAL, b
    V0n = V0.copy()
    V0n[3, 4] = np.nan
    assert oracle.solve_workload(w, V0=V0n, raise_on_error=False).status == oracle.ENUMERIC
    r = oracle.solve_workload(w, V0=V0, cfl=25.0, raise_on_error=False)   # violates CFL -> diverges
    w2 = w.__class__(**{**w.__dict__, "tau": (0.0, 50.0), "mode": "brs", "target": ("random_smooth", 1)})
    r = oracle.solve_workload(w2, cfl=40.0, raise_on_error=False)
    assert r.status == oracle.ENUMERIC and 0 < r.tau_reached < 50.0
