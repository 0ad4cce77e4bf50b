"""Unit pins of the float64 oracle (no GPU): grid, ghosts, derivatives, functors, alpha, CFL.

Each test pins an oracle function to something other than itself: a worked example
(tests/golden/spec_examples.json, cited), a closed form, or a brute-force enumeration.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle
from oracle import brute

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


# ---- a1: grid ------------------------------------------------------------------
@pytest.mark.parametrize("ex", GOLD["grid"], ids=lambda e: e["cite"][:5])
def test_grid_examples(ex):
    mask = sum(1 << d for d, p in enumerate(ex["periodic"]) if p)
    dx, coords = oracle.grid_axes(ex["N"], ex["lo"], ex["hi"], mask)
    np.testing.assert_allclose(dx, ex["spacing"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(coords[0], ex["coords"], rtol=0, atol=1e-15)


@pytest.mark.parametrize("ex", GOLD["grid_errors"], ids=lambda e: e["cite"][:5])
def test_grid_errors(ex):
    n = len(ex["N"])
    lo = ex.get("lo", [0.0] * n)
    hi = ex.get("hi", [1.0] * n)
    with pytest.raises(oracle.OracleError) as e:
        oracle.grid_axes(ex["N"], lo, hi, 0)
    assert e.value.status == oracle.EINVAL


# ---- a2: ghosts (P:237 addGhostExtrapolate; reading A12) --------------------------------
@pytest.mark.parametrize("ex", GOLD["ghosts"], ids=lambda e: e["cite"][:5])
def test_ghost_examples(ex):
    assert oracle.line_value(ex["line"], bool(ex["periodic"]), ex["j"]) == ex["value"]


def test_ghost_second_layer_and_low_face():
    # k = 2 beyond the high face: 2 + 2*|2-1| = 4; low face of [5, 3, ...]: 5 + k*2
    assert oracle.line_value([0.0, 1.0, 2.0], False, 4) == 4.0
    assert oracle.line_value([5.0, 3.0, 0.0], False, -1) == 7.0
    assert oracle.line_value([5.0, 3.0, 0.0], False, -2) == 9.0
    # sgn(0) = +1 at a zero edge value
    assert oracle.line_value([0.0, 1.0, 2.0], False, -1) == 1.0
    # negative edge extrapolates away from zero: never crosses the zero level set
    assert oracle.line_value([-1.0, -3.0, 0.0], False, -2) == -5.0
    # periodic wrap on both sides
    assert oracle.line_value([10.0, 11.0, 12.0, 13.0], True, -1) == 13.0
    assert oracle.line_value([10.0, 11.0, 12.0, 13.0], True, -2) == 12.0
    assert oracle.line_value([10.0, 11.0, 12.0, 13.0], True, 5) == 11.0


def test_ghosts_continue_linear_fields_exactly():
    # a linear field whose magnitude grows toward both faces (zero crossing inside) is continued
    # exactly by the sign-adjusted rule; one whose magnitude shrinks outward is not (it bends away
    # from the zero level set instead)
    line = -1.5 + 0.5 * np.arange(7)
    for j in (-2, -1, 7, 8):
        assert oracle.line_value(line, False, j) == pytest.approx(-1.5 + 0.5 * j, abs=1e-14)
    line = 2.0 + 0.5 * np.arange(7)
    assert oracle.line_value(line, False, -1) == 2.5


# ---- a3: derivatives (reading A13) ---------------------------------------------
@pytest.mark.parametrize("ex", GOLD["upwind"], ids=lambda e: e["cite"][:5])
def test_upwind_examples(ex):
    W = np.array(ex["line"])
    Dm, Dp = oracle.derivs(W, [0.0], [float(len(W) - 1)], 0, "low")
    assert Dm[0, ex["node"]] == ex["left"] and Dp[0, ex["node"]] == ex["right"]


def test_eno2_quadratic_vertex_is_exact():
    # x^2 on dz = 1 at x = 0: both one-sided ENO2 derivatives are exactly 0 (corrected)
    x = np.arange(-4.0, 5.0)
    Dm, Dp = oracle.derivs(x ** 2, [-4.0], [4.0], 0, "medium")
    assert Dm[0, 4] == 0.0 and Dp[0, 4] == 0.0
    # and away from the vertex ENO2 is exact for quadratics: d/dx x^2 = 2x
    np.testing.assert_allclose(Dm[0, 2:7], 2 * x[2:7], atol=1e-12)
    np.testing.assert_allclose(Dp[0, 2:7], 2 * x[2:7], atol=1e-12)


@pytest.mark.parametrize("acc", ["low", "medium"])
def test_derivatives_exact_on_linear_fields_nd(acc):
    # W = c x_a - b (zero crossing inside, constant along the other axes): exact D+- = c on axis a
    N = (5, 6, 7)
    lo, hi = [-1.0, -2.0, 0.5], [1.0, 1.0, 3.0]
    axes = [np.linspace(l, h, n) for l, h, n in zip(lo, hi, N)]
    X = np.meshgrid(*axes, indexing="ij")
    for a, (c, b) in enumerate([(1.5, 0.1), (-0.7, 0.3), (2.0, 3.5)]):
        W = c * X[a] - b
        Dm, Dp = oracle.derivs(W, lo, hi, 0, acc)
        for d in range(3):
            want = c if d == a else 0.0
            np.testing.assert_allclose(Dm[d], want, atol=1e-12)
            np.testing.assert_allclose(Dp[d], want, atol=1e-12)


@pytest.mark.parametrize("acc,order", [("low", 1.0), ("medium", 2.0)])
def test_derivative_convergence_order_on_sin(acc, order):
    # periodic sin on [0, 2pi): error of D+- against cos drops by 2^order per refinement
    errs = []
    for N in (40, 80, 160, 320):
        x = 2 * np.pi * np.arange(N) / N
        Dm, Dp = oracle.derivs(np.sin(x), [0.0], [2 * np.pi], 1, acc)
        errs.append(max(np.abs(Dm[0] - np.cos(x)).max(), np.abs(Dp[0] - np.cos(x)).max()))
    rates = [math.log2(errs[i] / errs[i + 1]) for i in range(3)]
    assert min(rates) > order - 0.1 and max(rates) < order + 0.2, (errs, rates)


def test_eno2_picks_smoother_stencil_at_a_kink():
    # |x| around the kink: D- on the left side must not see the kink when a smoother stencil exists
    x = np.arange(-5.0, 6.0)
    Dm, Dp = oracle.derivs(np.abs(x), [-5.0], [5.0], 0, "medium")
    # at x = -2 both stencils for D+ ... the one avoiding x=0 gives exactly -1
    assert Dm[0, 3] == -1.0 and Dp[0, 3] == -1.0  # x = -2
    assert Dm[0, 7] == 1.0 and Dp[0, 7] == 1.0    # x = +2


# ---- a5: CFL dt (Alg. 2 l.167) --------------------------------------------------------
@pytest.mark.parametrize("ex", GOLD["cfl"], ids=lambda e: e["cite"][:5])
def test_cfl_examples(ex):
    assert oracle.cfl_dt(ex["alpha"], ex["dx"], ex["factor"]) == pytest.approx(ex["dt"], rel=1e-15)


def test_cfl_degenerate_and_clip():
    assert oracle.cfl_dt([0.0, 0.0], [0.1, 0.1], 0.8, remaining=0.37) == 0.37   # A20
    assert oracle.cfl_dt([1.0, 1.0], [0.1, 0.1], 1.0, remaining=0.01) == 0.01   # A9
    # homogeneous: scaling alpha by c scales dt by 1/c
    assert oracle.cfl_dt([3.0, 1.5], [0.2, 0.1], 0.8) == pytest.approx(oracle.cfl_dt([1.0, 0.5], [0.2, 0.1], 0.8) / 3)


# ---- a6: optimal control / Hamiltonian (Eq. 4; Alg. 2 l.154-156) -- pin Z9 ------------------------
FUNCTORS = [
    ("HOLONOMIC_BOX", (1.0, 0.3, -1.0), 3, None),
    ("HOLONOMIC_BOX", (0.7, 0.2, 1.0), 2, None),
    ("DUBINS3D", (1.0, 1.0, 1.0), 3, None),
    ("DUBINS3D", (1.3, 0.7, -1.0), 3, None),
    ("CAR4D", (1.5, 1.0, 0.25, 0.25, -1.0), 4, None),
    ("CAR4D", (1.5, 1.0, 0.25, 0.4, 1.0), 4, None),
    ("CAR5D", (1.0, 2.0, -1.0), 5, None),
    ("DOUBLEINT6D", (1.0, 0.2, -1.0), 6, None),
    ("DOUBLEINT6D", (1.0, 0.2, 1.0), 6, None),
    ("PAIR_DUBINS3D", (5.0, 5.0, 1.0, 1.0, 1.0), 3, None),     # Eq. 7, air3D-like speeds
    ("PAIR_DUBINS3D", (1.0, 1.5, 0.7, 0.4, -1.0), 3, None),
]
ALPHA_FUNCTORS = [f for f in FUNCTORS if f[0] != "PAIR_DUBINS3D"]


@pytest.mark.parametrize("dyn,prm,n,_", FUNCTORS)
def test_hamiltonian_matches_vertex_enumeration(dyn, prm, n, _):
    rng = np.random.default_rng(7)
    for trial in range(300):
        x = rng.uniform(-3, 3, n)
        p = rng.normal(size=n)
        if trial % 10 == 0:
            p[rng.integers(n)] = 0.0      # ties: H must not depend on the tie-break
        H, u, d, f = oracle.hamiltonian(dyn, prm, x, p)
        Hb = brute.hamiltonian(dyn, prm, [np.array(v) for v in x], [np.array(v) for v in p])
        assert H == pytest.approx(float(Hb), abs=1e-12)
        # the returned u*, d* are admissible and produce H = p.f (Alg. 2 l.155-156)
        assert float(np.dot(p, f)) == pytest.approx(H, abs=1e-12)


@pytest.mark.parametrize("dyn,prm,n,_", FUNCTORS)
def test_optimal_control_is_a_saddle(dyn, prm, n, _):
    # for random admissible (u, d): goal -1 -> p.f(u*, d) <= H <= p.f(u, d*) ... (min over u, max over d)
    rng = np.random.default_rng(11)
    f_, U, D, goal, _ball = brute.model(dyn, prm, n)
    for trial in range(100):
        x = rng.uniform(-3, 3, n)
        p = rng.normal(size=n)
        H, us, ds, f = oracle.hamiltonian(dyn, prm, x, p)
        nu, nd = len(U[0]), len(D[0])
        for _ in range(10):
            u = np.array(U[0]) * 0 + rng.uniform(-1, 1, nu) * np.abs(U[0])
            d = rng.uniform(-1, 1, nd) * np.abs(D[0]) if nd else np.zeros(0)
            fu = oracle.rate(dyn, prm, x, u, ds[:nd])     # deviate the control, keep d*
            fd = oracle.rate(dyn, prm, x, us[:nu], d)     # deviate the disturbance, keep u*
            if goal < 0:
                assert np.dot(p, fu) >= H - 1e-12 and np.dot(p, fd) <= H + 1e-12
            else:
                assert np.dot(p, fu) <= H + 1e-12 and np.dot(p, fd) >= H - 1e-12


def test_ball_hamiltonian_closed_form():
    rng = np.random.default_rng(3)
    for n in (1, 2, 3, 6):
        for _ in range(50):
            p = rng.normal(size=n)
            x = rng.normal(size=n)
            H, u, _, f = oracle.hamiltonian("HOLONOMIC_BALL", (1.7, -1.0), x, p)
            assert H == pytest.approx(-1.7 * np.linalg.norm(p), rel=1e-14)
            assert np.linalg.norm(u[:n]) == pytest.approx(1.7, rel=1e-14)
    H, u, _, _ = oracle.hamiltonian("HOLONOMIC_BALL", (1.0, 1.0), [0.0, 0.0], [0.0, 0.0])
    assert H == 0.0 and not u.any()


# ---- a5/a7: alpha (Alg. 2 l.162; reading A5) ------------------------------------------------------
@pytest.mark.parametrize("dyn,prm,n,_", ALPHA_FUNCTORS)
def test_alpha_dominates_and_is_attained(dyn, prm, n, _):
    rng = np.random.default_rng(5)
    for trial in range(60):
        x = rng.uniform(-3, 3, n)
        a = rng.normal(size=n)
        b = rng.normal(size=n)
        if trial % 3 == 0:
            b = a + np.abs(rng.normal(size=n))      # some ranges of one sign only
        minD, maxD = np.minimum(a, b), np.maximum(a, b)
        al = oracle.alpha(dyn, prm, x, minD, maxD)
        Ab = brute.alpha(dyn, prm, [np.array(v) for v in x], minD, maxD)
        np.testing.assert_allclose(al, [float(v) for v in Ab], atol=1e-12)
        best = np.zeros(n)
        for _ in range(200):   # dominance over random costates in the box
            p = rng.uniform(minD, maxD)
            _, _, _, f = oracle.hamiltonian(dyn, prm, x, p)
            assert np.all(np.abs(f) <= al + 1e-12)
            best = np.maximum(best, np.abs(f))
        for corner in range(1 << n):   # attained at a corner of the box (bang-bang: sign patterns)
            p = np.where([(corner >> k) & 1 for k in range(n)], maxD, minD)
            _, _, _, f = oracle.hamiltonian(dyn, prm, x, p)
            best = np.maximum(best, np.abs(f))
        np.testing.assert_allclose(best, al, atol=1e-12)


def test_alpha_ball_exact_maximum():
    # ball: |dH/dp_d| = ubar |p_d|/|p| over the box; attained at |p_d| max and |p_e| min
    al = oracle.alpha("HOLONOMIC_BALL", (2.0, -1.0), [0, 0, 0], [-1.0, 0.5, -0.2], [3.0, 2.0, 0.4])
    assert al[0] == pytest.approx(2.0 * 3 / math.sqrt(9 + 0.25), rel=1e-14)
    assert al[1] == pytest.approx(2.0 * 2 / math.sqrt(4), rel=1e-14)
    assert al[2] == pytest.approx(2.0 * 0.4 / math.sqrt(0.16 + 0.25), rel=1e-14)
    rng = np.random.default_rng(1)
    lo, hi = np.array([-1.0, 0.5, -0.2]), np.array([3.0, 2.0, 0.4])
    for _ in range(5000):
        p = rng.uniform(lo, hi)
        assert np.all(2.0 * np.abs(p) / np.linalg.norm(p) <= al + 1e-12)


def test_alpha_config_values_table_c2():
    # SURVEY.md table C-2 alpha^max on the config grids: c2 (4.25, 4.25, 1.5, 1), c4 (2, 0.8, ...)
    from inputs import CONFIGS, axis_nodes
    w = CONFIGS["c2"]
    ax = [axis_nodes(n, l, h, bool(p)) for n, l, h, p in zip(w.N, w.lo, w.hi, w.periodic)]
    best = np.zeros(4)
    for v in ax[2]:
        for th in ax[3]:
            best = np.maximum(best, oracle.alpha("CAR4D", w.params, [0, 0, v, th], [-1] * 4, [1] * 4))
    np.testing.assert_allclose(best, [4.25, 4.25, 1.5, 1.0], atol=1e-12)
    w = CONFIGS["c4"]
    al = oracle.alpha("DOUBLEINT6D", w.params, [0, 2.0, 0, -2.0, 0, 1.0], [-1] * 6, [1] * 6)
    np.testing.assert_allclose(al, [2.0, 0.8, 2.0, 0.8, 1.0, 0.8], atol=1e-12)


@pytest.mark.parametrize("prm", [(5.0, 5.0, 1.0, 1.0, 1.0), (1.0, 1.5, 0.7, 0.4, -1.0)])
def test_alpha_pairwise_dubins_eq7(prm):
    # A30: alpha over the sign set of q = p_x y - p_y x - p_th (exact range over the box, linear in p)
    # and, for th, the sign set of p_th taken independently.  x, y: exact maximum (attained at a box
    # corner); th: an upper bound of |dH/dp_th| (dominance), equal to abar + bbar when q and p_th
    # can take both signs.
    rng = np.random.default_rng(17)
    for trial in range(80):
        x = rng.uniform(-6, 6, 3)
        a, b = rng.normal(size=3), rng.normal(size=3)
        if trial % 3 == 0:
            b = a + np.abs(rng.normal(size=3))
        minD, maxD = np.minimum(a, b), np.maximum(a, b)
        al = oracle.alpha("PAIR_DUBINS3D", prm, x, minD, maxD)
        Ab = brute.alpha("PAIR_DUBINS3D", prm, [np.array(v) for v in x], minD, maxD)
        np.testing.assert_allclose(al, [float(v) for v in Ab], atol=1e-12)
        best = np.zeros(3)
        for _ in range(300):
            p = rng.uniform(minD, maxD)
            _, _, _, f = oracle.hamiltonian("PAIR_DUBINS3D", prm, x, p)
            assert np.all(np.abs(f) <= al + 1e-12)
            best = np.maximum(best, np.abs(f))
        for corner in range(8):
            p = np.where([(corner >> k) & 1 for k in range(3)], maxD, minD)
            _, _, _, f = oracle.hamiltonian("PAIR_DUBINS3D", prm, x, p)
            best = np.maximum(best, np.abs(f))
        np.testing.assert_allclose(best[:2], al[:2], atol=1e-12)
    # both sign sets full -> alpha_th = abar + bbar
    al = oracle.alpha("PAIR_DUBINS3D", prm, [1.0, 2.0, 0.3], [-1.0, -1.0, -1.0], [1.0, 1.0, 1.0])
    assert al[2] == pytest.approx(prm[2] + prm[3], rel=1e-15)
