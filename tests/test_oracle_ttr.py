"""Pins of the time-to-reach oracle (Alg. 3, Lax-Friedrichs sweeping; readings A31-A34).

* 1D: the exact TTR |x| - r (holonomic, unit speed) and (|x| - r)/(ubar - dbar) (box with
  disturbance) are fixed points of the scheme (linear between the target and the far boundary,
  which the boundary rule l.14-15 extrapolates exactly);
* 2D ball: TTR = |x| - r, first-order convergence away from the target;
* the Gauss-Seidel sweeps of the oracle and an independent NumPy Jacobi formulation (H by vertex
  enumeration) reach the same fixed point.
"""
import math

import numpy as np
import pytest

import oracle
from oracle import brute


@pytest.mark.parametrize("dyn,prm,speed", [("HOLONOMIC_BALL", (1.0, -1.0), 1.0), ("HOLONOMIC_BALL", (1.7, 1.0), 1.7),
                                           ("HOLONOMIC_BOX", (1.0, 0.3, -1.0), 0.7)])
def test_ttr_1d_exact(dyn, prm, speed):
    N = 61
    x = np.linspace(-3.0, 3.0, N)
    V0 = (np.abs(x) - 0.5).astype(np.float32)
    phi, sweeps, change = oracle.ttr_solve((N,), (-3.0,), (3.0,), 0, dyn, prm, V0, eps=1e-13)
    exact = np.maximum(np.abs(x) - 0.5, 0.0) / speed
    exact[V0 <= 0] = 0.0
    np.testing.assert_allclose(phi, exact, atol=1e-11)
    assert change <= 1e-13 and sweeps < 20


def test_ttr_2d_ball_first_order():
    errs = []
    for N in (41, 81, 161):
        x = np.linspace(-2.0, 2.0, N)
        X, Y = np.meshgrid(x, x, indexing="ij")
        R = np.sqrt(X ** 2 + Y ** 2)
        phi, _, change = oracle.ttr_solve((N, N), (-2.0, -2.0), (2.0, 2.0), 0, "HOLONOMIC_BALL", (1.0, -1.0),
                                          (R - 0.5).astype(np.float32), eps=1e-10)
        band = (R > 0.7) & (R < 1.8)
        errs.append(float(np.abs(phi - (R - 0.5))[band].max()))
        assert change <= 1e-10
    assert errs[0] > errs[1] > errs[2]
    orders = [math.log2(errs[k] / errs[k + 1]) for k in range(2)]
    assert min(orders) >= 0.9, (errs, orders)


def _case(dyn, n, per, seed=5):
    rng = np.random.default_rng(seed)
    N = (13, 11, 12, 9)[:n] if n < 4 else (11, 10, 7, 10)
    lo = (-3.0, -2.5, -math.pi)[:n] if n < 4 else (-3.0, -2.5, 0.2, -math.pi)
    hi = (3.0, 2.5, math.pi)[:n] if n < 4 else (3.0, 2.5, 1.4, math.pi)
    axes = [lo[d] + np.arange(N[d]) * ((hi[d] - lo[d]) / (N[d] if per[d] else N[d] - 1)) for d in range(n)]
    X = np.meshgrid(*axes, indexing="ij")
    V0 = (np.sqrt(X[0] ** 2 + X[1] ** 2) - 1.0 + 0.05 * rng.uniform(-1, 1, N)).astype(np.float32)
    return N, lo, hi, V0


@pytest.mark.parametrize("dyn,prm,per", [("HOLONOMIC_BALL", (1.0, -1.0), (0, 0)),
                                         ("HOLONOMIC_BOX", (1.0, 0.25, -1.0), (0, 1))])
def test_ttr_gauss_seidel_and_jacobi_share_the_fixed_point(dyn, prm, per):
    N, lo, hi, V0 = _case(dyn, 2, per)
    pmask = sum(1 << d for d in range(2) if per[d])
    phi, sweeps, change = oracle.ttr_solve(N, lo, hi, pmask, dyn, prm, V0, eps=1e-13, max_sweeps=20000)
    ref, iters = brute.ttr_jacobi(N, lo, hi, per, dyn, prm, V0, eps=1e-13)
    assert change <= 1e-13 and sweeps < 20000 and iters < 200000
    np.testing.assert_allclose(phi, ref, atol=1e-9)
    assert np.all(phi[V0 <= 0] == 0.0) and np.all(phi >= 0.0)
    rb, iters_rb = brute.ttr_jacobi(N, lo, hi, per, dyn, prm, V0, eps=1e-13, order="red_black")
    np.testing.assert_allclose(rb, ref, atol=1e-9)         # red-black ordering: same fixed point
    assert iters_rb < iters


@pytest.mark.parametrize("dyn,prm,n,per", [("HOLONOMIC_BALL", (1.0, -1.0), 2, (0, 0)),
                                           ("HOLONOMIC_BOX", (1.0, 0.25, -1.0), 2, (0, 1)),
                                           ("DUBINS3D", (1.0, 1.0, -1.0), 3, (0, 0, 1)),
                                           ("PAIR_DUBINS3D", (1.0, 1.0, 1.0, 0.5, -1.0), 3, (0, 0, 1)),
                                           ("CAR4D", (1.0, 1.0, 0.1, 0.1, -1.0), 4, (0, 0, 0, 1))])
def test_ttr_converged_phi_is_a_fixed_point_of_the_update(dyn, prm, n, per):
    """Every interior non-target node the sweep reached satisfies phi = LF-update(phi) (l.10-12) with
    H and sigma from the independent NumPy formulation, the rest have phi <= update, target nodes are
    0 and the boundary rule (l.14-15) is idempotent.  (With the min in l.14-15 the boundary values
    depend on the iteration path, so Gauss-Seidel and Jacobi fixed points differ near the faces for
    non-holonomic dynamics; this is the path-independent check.)"""
    N, lo, hi, V0 = _case(dyn, n, per)
    pmask = sum(1 << d for d in range(n) if per[d])
    phi, sweeps, change = oracle.ttr_solve(N, lo, hi, pmask, dyn, prm, V0, eps=1e-13, max_sweeps=20000)
    assert change <= 1e-13 and sweeps < 20000
    new = brute.ttr_update_map(N, lo, hi, per, dyn, prm, phi)
    _, _, _, _, _, interior = brute._ttr_setup(N, lo, hi, per, dyn, prm)
    upd = interior & (V0 > 0)
    reached = upd & (phi < 100.0)
    assert reached.sum() > 0.5 * upd.sum()
    np.testing.assert_allclose(new[reached], phi[reached], atol=1e-9, rtol=0)
    assert np.all(new[upd] >= phi[upd] - 1e-9)
    assert np.all(phi[V0 <= 0] == 0.0) and np.all(phi >= 0.0)
    again = brute.ttr_boundary_rule(N, per, phi.copy())
    np.testing.assert_allclose(again, phi, atol=1e-12, rtol=0)


def test_ttr_2d_box_linf_target_rates():
    # xdot_i = u_i + d_i, |u_i| <= ubar, |d_i| <= dbar: the minimum time to the square
    # {max|x_i| <= r} is (max_i |x_i| - r) / (ubar - dbar) (each axis closes independently).  It has
    # kinks on the diagonals, where a monotone scheme converges at the Crandall-Lions rate h^(1/2) in
    # the max norm; away from them the rate is >= 1
    ubar, dbar, r = 1.0, 0.25, 0.5
    e_all, e_off = [], []
    for N in (41, 81, 161):
        x = np.linspace(-2.0, 2.0, N)
        X, Y = np.meshgrid(x, x, indexing="ij")
        M = np.maximum(np.abs(X), np.abs(Y))
        phi, _, change = oracle.ttr_solve((N, N), (-2.0, -2.0), (2.0, 2.0), 0, "HOLONOMIC_BOX", (ubar, dbar, -1.0),
                                          (M - r).astype(np.float32), eps=1e-10)
        err = np.abs(phi - np.maximum(M - r, 0.0) / (ubar - dbar))
        band = (M > 0.7) & (M < 1.8)
        e_all.append(float(err[band].max()))
        e_off.append(float(err[band & (np.abs(np.abs(X) - np.abs(Y)) > 0.3)].max()))
        assert change <= 1e-10
    r_all = [math.log2(e_all[k] / e_all[k + 1]) for k in range(2)]
    r_off = [math.log2(e_off[k] / e_off[k + 1]) for k in range(2)]
    assert all(0.4 <= q <= 0.7 for q in r_all), (e_all, r_all)
    assert min(r_off) >= 1.0, (e_off, r_off)
