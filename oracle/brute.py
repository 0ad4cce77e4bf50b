"""NumPy "full temporaries" brute force of the time-dependent HJ step (pin Z11).

TEST INFRASTRUCTURE (see oracle/__init__.py).  A second, independently written formulation of
PAPER.md Algorithm 2 in the MATLAB style the paper contrasts itself with (Fig. 3,
P:174-179): every temporary (ghost-padded copies, D-/D+ per axis, H, alpha) is a full N-D array.
Differences from oracle/odp_oracle.c, on purpose:
  * ghosts are materialised by padding the whole array per axis instead of per-node lookups;
  * H = ext_u ext_d p.f(x,u,d) by ENUMERATING the vertices of the control and disturbance boxes
    (Eq. 4) instead of the closed-form bang-bang choice (ball control: closed form);
  * alpha_d = max over the achievable sign patterns of the costate (box [minD, maxD]) of
    |f_d(x, u*, d*)|, with u*, d* again found by vertex enumeration.
Only for tiny grids (3..7 nodes per axis).
"""
from __future__ import annotations

import itertools
import math

import numpy as np

from inputs import axis_nodes


def _sgn(v):
    return np.where(v >= 0, 1.0, -1.0)


def pad(W, d, r, periodic):
    """Return W padded with r ghost layers on both sides of axis d (readings A12, A15)."""
    N = W.shape[d]
    take = lambda i: np.take(W, [i], axis=d)
    if periodic:
        lo = np.take(W, list(range(N - r, N)), axis=d)
        hi = np.take(W, list(range(0, r)), axis=d)
        return np.concatenate([lo, W, hi], axis=d)
    e0, i0 = take(0), take(1)
    e1, i1 = take(N - 1), take(N - 2)
    s0 = np.abs(e0 - i0) * _sgn(e0)
    s1 = np.abs(e1 - i1) * _sgn(e1)
    lows = [e0 + k * s0 for k in range(r, 0, -1)]     # ghost -r .. -1
    highs = [e1 + k * s1 for k in range(1, r + 1)]    # ghost N .. N+r-1
    return np.concatenate(lows + [W] + highs, axis=d)


def _sl(d, ndim, a, b):
    s = [slice(None)] * ndim
    s[d] = slice(a, b)
    return tuple(s)


def derivatives(W, dx, periodic, accuracy):
    """Full arrays D-[d], D+[d] (§3.4.4; ENO2 per reading A13)."""
    n = W.ndim
    Dm, Dp = [], []
    r = 1 if accuracy == "low" else 2
    for d in range(n):
        Pd = pad(W, d, r, bool(periodic[d]))
        N = W.shape[d]
        v = {k: Pd[_sl(d, n, r + k, r + k + N)] for k in range(-r, r + 1)}
        h = dx[d]
        if accuracy == "low":
            Dm.append((v[0] - v[-1]) / h)
            Dp.append((v[1] - v[0]) / h)
        else:
            d2 = {j: v[j + 1] - 2.0 * v[j] + v[j - 1] for j in (-1, 0, 1)}
            pick = lambda a, b: np.where(np.abs(a) <= np.abs(b), a, b)
            Dm.append((v[0] - v[-1]) / h + pick(d2[-1], d2[0]) / (2.0 * h))
            Dp.append((v[1] - v[0]) / h - pick(d2[0], d2[1]) / (2.0 * h))
    return Dm, Dp


# ---- dynamics as plain f(x, u, d) with explicit control/disturbance boxes ------------------------
def model(dyn, params, n):
    """Returns (f(X, u, d) -> list of n arrays, U vertices, D vertices, goal, ball)."""
    p = list(params)
    goal = p[-1]
    if dyn == "HOLONOMIC_BALL":
        return (lambda X, u, d: [u[k] + 0.0 * X[k] for k in range(n)]), None, [()], goal, p[0]
    if dyn == "HOLONOMIC_BOX":
        U = list(itertools.product(*[(-p[0], p[0])] * n))
        D = list(itertools.product(*[(-p[1], p[1])] * n))
        return (lambda X, u, d: [u[k] + d[k] + 0.0 * X[k] for k in range(n)]), U, D, goal, None
    if dyn == "DUBINS3D":
        v, wb = p[0], p[1]
        f = lambda X, u, d: [v * np.cos(X[2]), v * np.sin(X[2]), u[0] + 0.0 * X[2]]
        return f, [(-wb,), (wb,)], [()], goal, None
    if dyn == "CAR4D":
        ab, wb, dxb, dyb = p[:4]
        f = lambda X, u, d: [X[2] * np.cos(X[3]) + d[0], X[2] * np.sin(X[3]) + d[1], u[0] + 0.0 * X[0], u[1] + 0.0 * X[0]]
        U = list(itertools.product((-ab, ab), (-wb, wb)))
        D = list(itertools.product((-dxb, dxb), (-dyb, dyb)))
        return f, U, D, goal, None
    if dyn == "CAR5D":
        ab, alb = p[:2]
        f = lambda X, u, d: [X[3] * np.cos(X[2]), X[3] * np.sin(X[2]), X[4] + 0.0 * X[0], u[0] + 0.0 * X[0], u[1] + 0.0 * X[0]]
        return f, list(itertools.product((-ab, ab), (-alb, alb))), [()], goal, None
    if dyn == "DOUBLEINT6D":
        ub, db = p[:2]
        f = lambda X, u, d: [X[1], u[0] + d[0] + 0.0 * X[0], X[3], u[1] + d[1] + 0.0 * X[0], X[5], u[2] + d[2] + 0.0 * X[0]]
        return f, list(itertools.product(*[(-ub, ub)] * 3)), list(itertools.product(*[(-db, db)] * 3)), goal, None
    if dyn == "PAIR_DUBINS3D":      # Eq. 7: u = a (evader), d = b (pursuer)
        va, vb, ab, bb = p[:4]
        f = lambda X, u, d: [-va + vb * np.cos(X[2]) + u[0] * X[1], va * np.sin(X[2]) - u[0] * X[0],
                             d[0] - u[0] + 0.0 * X[0]]
        return f, [(-ab,), (ab,)], [(-bb,), (bb,)], goal, None
    raise ValueError(dyn)


def hamiltonian(dyn, params, X, Pc):
    """H = ext_u ext_d p.f by vertex enumeration; goal -1: min_u max_d, +1: max_u min_d (A1)."""
    n = len(X)
    f, U, D, goal, ball = model(dyn, params, n)
    if ball is not None:
        nrm = np.sqrt(sum(q * q for q in Pc))
        return goal * ball * nrm
    ext_u = np.minimum if goal < 0 else np.maximum
    ext_d = np.maximum if goal < 0 else np.minimum
    H = None
    for u in U:
        inner = None
        for d in D:
            fx = f(X, u, d)
            val = sum(Pc[k] * fx[k] for k in range(n))
            inner = val if inner is None else ext_d(inner, val)
        H = inner if H is None else ext_u(H, inner)
    return H


def alpha(dyn, params, X, minD, maxD):
    """alpha_d(x) = max over achievable costate sign patterns of |f_d(x, u*, d*)| (A5)."""
    n = len(X)
    f, U, D, goal, ball = model(dyn, params, n)
    shape = np.broadcast(*X).shape
    if ball is not None:
        out = []
        for d in range(n):
            Md = max(abs(minD[d]), abs(maxD[d]))
            if Md == 0:
                out.append(np.zeros(shape))
                continue
            den = Md * Md
            for e in range(n):
                if e != d and not (minD[e] <= 0 <= maxD[e]):
                    den += min(abs(minD[e]), abs(maxD[e])) ** 2
            out.append(np.full(shape, ball * Md / math.sqrt(den)))
        return out
    if dyn == "PAIR_DUBINS3D":
        # the switching function q = p_x y - p_y x - p_th is linear in p: its range over the costate
        # box is attained at the box corners (enumerated here); b* follows sgn(p_th)   (A30)
        va, vb, ab, bb = list(params)[:4]
        corners = list(itertools.product((minD[0], maxD[0]), (minD[1], maxD[1]), (minD[2], maxD[2])))
        qs = [c[0] * X[1] - c[1] * X[0] - c[2] for c in corners]
        qlo = np.minimum.reduce([np.broadcast_to(q, shape) for q in qs])
        qhi = np.maximum.reduce([np.broadcast_to(q, shape) for q in qs])
        out = [np.zeros(shape) for _ in range(n)]
        st = ([1.0] if maxD[2] >= 0 else []) + ([-1.0] if minD[2] < 0 else [])
        for sq, mask in ((1.0, qhi >= 0), (-1.0, qlo < 0)):
            a = goal * ab * sq
            for sb in st:
                b = -goal * bb * sb
                fx = f(X, (a,), (b,))
                for k in range(n):
                    out[k] = np.where(mask, np.maximum(out[k], np.abs(np.broadcast_to(fx[k], shape))), out[k])
        return out
    signsets = []
    for d in range(n):
        s = []
        if maxD[d] >= 0:
            s.append(1.0)
        if minD[d] < 0:
            s.append(-1.0)
        signsets.append(s)
    best = [np.zeros(shape) for _ in range(n)]
    zero = [0.0] * 3
    for sv in itertools.product(*signsets):
        # u* = argext_u sv.f(x,u,d) (the d-part is additive and separable), then d* likewise
        def score(u, d):
            fx = f(X, u, d)
            return sum(sv[k] * fx[k] for k in range(n))
        d_any = D[0]
        cand = [(u, score(u, d_any)) for u in U]
        # pointwise arg-ext over vertices
        ustar_score = cand[0][1]
        ustar_idx = np.zeros(shape, dtype=int)
        for i, (u, sc) in enumerate(cand[1:], start=1):
            better = sc > ustar_score if goal > 0 else sc < ustar_score
            ustar_idx = np.where(better, i, ustar_idx)
            ustar_score = np.where(better, sc, ustar_score)
        u_any = U[0]
        candd = [(d, score(u_any, d)) for d in D]
        dstar_score = candd[0][1]
        dstar_idx = np.zeros(shape, dtype=int)
        for i, (d, sc) in enumerate(candd[1:], start=1):
            better = sc < dstar_score if goal > 0 else sc > dstar_score
            dstar_idx = np.where(better, i, dstar_idx)
            dstar_score = np.where(better, sc, dstar_score)
        for iu, u in enumerate(U):
            for idd, d in enumerate(D):
                mask = (ustar_idx == iu) & (dstar_idx == idd)
                if not mask.any():
                    continue
                fx = f(X, u, d)
                for k in range(n):
                    best[k] = np.where(mask, np.maximum(best[k], np.abs(np.broadcast_to(fx[k], shape))), best[k])
    return best


def solve(w, V0, cfl=None, store_initial=False):
    """Whole solve in full-temporaries style; returns (snapshots at tau[1:], steps)."""
    n = w.dims
    dx = [(h - l) / (N if p else N - 1) for N, l, h, p in zip(w.N, w.lo, w.hi, w.periodic)]
    axes = [axis_nodes(N, l, h, bool(p)) for N, l, h, p in zip(w.N, w.lo, w.hi, w.periodic)]
    X = np.meshgrid(*axes, indexing="ij")
    C = cfl if cfl is not None else w.cfl
    V = V0.astype(np.float64).copy()
    T = V0.astype(np.float64)

    def L_of(W):
        Dm, Dp = derivatives(W, dx, w.periodic, w.accuracy)
        minD = [min(Dm[d].min(), Dp[d].min()) for d in range(n)]
        maxD = [max(Dm[d].max(), Dp[d].max()) for d in range(n)]
        Pc = [(Dm[d] + Dp[d]) / 2.0 for d in range(n)]
        H = hamiltonian(w.dynamics, w.params, X, Pc)
        A = alpha(w.dynamics, w.params, X, minD, maxD)
        L = H + sum(A[d] * (Dp[d] - Dm[d]) / 2.0 for d in range(n))
        amax = [float(A[d].max()) for d in range(n)]
        return L, amax

    t, steps, outs = 0.0, 0, []
    eps = 1e-12 * max(1.0, w.tau[-1])
    for k in range(1, len(w.tau)):
        while w.tau[k] - t > eps:
            L, amax = L_of(V)
            s = sum(a / h for a, h in zip(amax, dx))
            dt = C / s if s > 0 else w.tau[k] - t
            dt = min(dt, w.tau[k] - t)
            if w.accuracy == "low":
                Vn = V + dt * L
            else:
                V1 = V + dt * L
                L1, _ = L_of(V1)
                Vn = 0.5 * (V + (V1 + dt * L1))
            if w.mode == "brt":
                Vn = np.minimum(Vn, T)
            V = Vn
            t += dt
            steps += 1
        outs.append(V.copy())
    return np.stack(outs), steps



def _ttr_setup(N, lo, hi, periodic, dyn, params):
    n = len(N)
    prm = list(params)
    prm[-1] = -1.0
    dx = [(hi[d] - lo[d]) / (N[d] if periodic[d] else N[d] - 1) for d in range(n)]
    axes = [lo[d] + np.arange(N[d]) * dx[d] for d in range(n)]
    X = np.meshgrid(*axes, indexing="ij")
    sig = [np.broadcast_to(s, tuple(N)) for s in alpha(dyn, prm, X, [-1.0] * n, [1.0] * n)]
    interior = np.ones(tuple(N), dtype=bool)
    for d in range(n):
        if not periodic[d]:
            sl = [slice(None)] * n
            sl[d] = 0
            interior[tuple(sl)] = False
            sl[d] = N[d] - 1
            interior[tuple(sl)] = False
    return n, prm, dx, X, sig, interior


def ttr_update_map(N, lo, hi, periodic, dyn, params, phi, setup=None):
    """The Lax-Friedrichs update of Alg. 3 l.5-11 (readings A32-A33) evaluated at every node from
    the iterate phi, H by vertex enumeration (hamiltonian() with goal -1), sigma from alpha() on
    the box [-1, 1]^n.  Values on non-periodic faces are meaningless (rolls wrap there)."""
    n, prm, dx, X, sig, _ = setup or _ttr_setup(N, lo, hi, periodic, dyn, params)
    P, num = [], 0.0
    for d in range(n):
        vp, vm = np.roll(phi, -1, axis=d), np.roll(phi, 1, axis=d)
        P.append((vp - vm) / (2 * dx[d]))
        num = num + sig[d] * (vp + vm) / (2 * dx[d])
    den = sum(sig[d] / dx[d] for d in range(n))
    H = -hamiltonian(dyn, prm, X, P) - 1.0
    return np.where(den > 0, (num - H) / np.where(den > 0, den, 1.0), phi)


def ttr_boundary_rule(N, periodic, phi):
    """Alg. 3 l.14-15 along each non-periodic axis in order (reading A34), in place."""
    n = len(N)
    for d in range(n):
        if periodic[d]:
            continue

        def sl(i):
            s = [slice(None)] * n
            s[d] = i
            return tuple(s)
        for e, a, b in ((0, 1, 2), (N[d] - 1, N[d] - 2, N[d] - 3)):
            phi[sl(e)] = np.minimum(np.maximum(2 * phi[sl(a)] - phi[sl(b)], phi[sl(b)]), phi[sl(e)])
    return phi


def ttr_jacobi(N, lo, hi, periodic, dyn, params, V0, eps=1e-12, max_iter=200000, big=100.0, order="jacobi"):
    """Independent NumPy formulation of the time-to-reach iteration (Alg. 3, readings A31-A35):
    order "jacobi": every node from the previous iterate; order "red_black": the nodes with an even
    index sum first (from the previous iterate), then the odd ones from the updated values (an
    in-place Gauss-Seidel ordering, reading A35); then the boundary rule.  Its fixed point equals
    the oracle's Gauss-Seidel one where the boundary rule's min never binds on a non-monotone path
    (holonomic cases); see test_oracle_ttr."""
    setup = _ttr_setup(N, lo, hi, periodic, dyn, params)
    interior = setup[5]
    target = np.asarray(V0, dtype=np.float32) <= 0
    phi = np.where(target, 0.0, big)
    upd = interior & ~target
    colour = np.indices(tuple(N)).sum(axis=0) % 2
    for it in range(max_iter):
        old = phi.copy()
        if order == "jacobi":
            phi = np.where(upd, np.minimum(ttr_update_map(N, lo, hi, periodic, dyn, params, phi, setup), phi), phi)
        else:
            for c in (0, 1):
                m = upd & (colour == c)
                phi = np.where(m, np.minimum(ttr_update_map(N, lo, hi, periodic, dyn, params, phi, setup), phi), phi)
        ttr_boundary_rule(N, periodic, phi)
        if np.abs(phi - old).max() <= eps:
            return phi, it + 1
    return phi, max_iter


# ------------------------------------------------------------------------------------------------
# Value iteration (Alg. 1, readings A36-A38): an independent NumPy formulation -- successor tables
# for every (action, outcome) at once, Jacobi iteration, and the exact Bellman fixed point by policy
# iteration (sparse linear solves), which Alg. 1 does not use at all.
# ------------------------------------------------------------------------------------------------
def vi_model(model, params, n):
    """(actions as float32 parameter rows, outcome probabilities, gamma)."""
    f32 = np.float32
    if model == "HOLONOMIC":
        speed, dt, gamma = params
        step = f32(dt) * f32(speed)
        acts = [np.zeros(n, f32)]
        for d in range(n):
            for sgn in (1, -1):
                a = np.zeros(n, f32)
                a[d] = step if sgn > 0 else -step
                acts.append(a)
        return acts, np.array([1.0]), float(gamma)
    if model == "DUBINS3D":
        vbar, wbar, dt, slip, pslip, gamma = params
        acts = []
        for v in (f32(0.5) * f32(vbar), f32(vbar)):
            for w in (-f32(wbar), f32(0.0), f32(wbar)):
                acts.append(np.array([v, w], f32))
        return acts, np.array([1.0 - 2.0 * pslip, pslip, pslip]), float(gamma)
    raise ValueError(model)


def vi_successors(N, lo, hi, periodic, model, params):
    """succ[a][k] = flat successor index of every node (float32 arithmetic, nearest node, wrap/clamp)."""
    f32 = np.float32
    n = len(N)
    dx = [(hi[d] - lo[d]) / (N[d] if periodic[d] else N[d] - 1) for d in range(n)]
    inv_dx = [f32(1.0 / dx[d]) for d in range(n)]
    I = np.meshgrid(*[np.arange(N[d]) for d in range(n)], indexing="ij")
    acts, p, _ = vi_model(model, params, n)
    K = len(p)
    strides = [int(np.prod(N[d + 1:])) for d in range(n)]
    out = []
    for a in acts:
        row = []
        for k in range(K):
            if model == "HOLONOMIC":
                delta = [np.full(tuple(N), a[d], f32) for d in range(n)]
            else:
                th = lo[2] + I[2] * dx[2]
                c, s = np.cos(th).astype(f32), np.sin(th).astype(f32)
                dt = f32(params[2])
                sig = f32(0.0) if k == 0 else (f32(params[3]) if k == 1 else -f32(params[3]))
                dtv = dt * a[0]
                delta = [(dtv * c) - (sig * s), (dtv * s) + (sig * c), np.full(tuple(N), dt * a[1], f32)]
            flat = np.zeros(tuple(N), np.int64)
            for d in range(n):
                q = (delta[d] * inv_dx[d]).astype(f32)
                fl = np.floor(q)                       # nearest node, ties toward the larger index
                j = I[d] + (fl + ((q - fl) >= f32(0.5))).astype(np.int64)
                j = np.mod(j, N[d]) if periodic[d] else np.clip(j, 0, N[d] - 1)
                flat = flat + j * strides[d]
            row.append(flat.ravel())
        out.append(row)
    return out


def vi_jacobi(N, lo, hi, periodic, model, params, R, iters):
    """`iters` Jacobi iterations V_{t+1} = max_a (R + gamma sum_k p_k V_t(s'_k)) from V_0 = 0."""
    succ = vi_successors(N, lo, hi, periodic, model, params)
    _, p, gamma = vi_model(model, params, len(N))
    Rf = np.asarray(R, np.float32).astype(np.float64).ravel()
    V = np.zeros_like(Rf)
    for _ in range(iters):
        V = np.max([Rf + gamma * sum(p[k] * V[sa[k]] for k in range(len(p))) for sa in succ], axis=0)
    return V.reshape(tuple(N))


def vi_policy_iteration(N, lo, hi, periodic, model, params, R, max_rounds=200):
    """Exact fixed point of the Bellman operator by policy iteration: evaluate the greedy policy with a
    sparse solve of (I - gamma P_pi) V = R, improve, repeat until the policy is stable."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as spla
    succ = vi_successors(N, lo, hi, periodic, model, params)
    _, p, gamma = vi_model(model, params, len(N))
    Rf = np.asarray(R, np.float32).astype(np.float64).ravel()
    P = Rf.size
    rows = np.arange(P)
    pol = np.zeros(P, np.int64)
    V = np.zeros(P)
    for _ in range(max_rounds):
        M = sp.identity(P, format="csr")
        for k in range(len(p)):
            cols = np.choose(pol, [succ[a][k] for a in range(len(succ))]) if len(succ) > 1 else succ[0][k]
            M = M - gamma * p[k] * sp.csr_matrix((np.ones(P), (rows, cols)), shape=(P, P))
        V = spla.spsolve(M.tocsc(), Rf)
        Q = np.array([Rf + gamma * sum(p[k] * V[sa[k]] for k in range(len(p))) for sa in succ])
        best = Q.max(axis=0)
        # keep the current action unless another is strictly better (ties: no change)
        cur = Q[pol, rows]
        new = np.where(best > cur + 1e-12 * (1 + np.abs(best)), Q.argmax(axis=0), pol)
        if np.array_equal(new, pol):
            return V.reshape(tuple(N))
        pol = new
    raise RuntimeError("policy iteration did not converge")
