"""Shared helpers of the GPU parity tests: run a workload through the C-ABI and through the oracle,
compare element by element."""
import numpy as np

TOL = 1e-4     # north_star: max |V_gpu - V_oracle| <= 1e-4 (float32)
BAND = 1e-4    # membership (V <= 0) identical outside |V_oracle| < 1e-4 (reading A24)


def run_gpu(w, V0, kernel="auto", **kw):
    import torch
    import paper_2204_05520_b200 as odp
    dV0 = torch.from_numpy(V0).cuda()
    out, info = odp.solve_workload(w, dV0, kernel=kernel, **kw)
    torch.cuda.synchronize()
    return out.cpu().numpy(), info


def covers(w, kernel):
    """Whether a kernel family covers the workload's grid (the library answers EINVAL otherwise)."""
    import paper_2204_05520_b200 as odp
    import torch
    V0 = torch.zeros(w.N, dtype=torch.float32, device="cuda")
    w1 = w.__class__(**{**w.__dict__, "tau": (0.0, 1e-9)})
    try:
        odp.solve_workload(w1, V0, kernel=kernel)
    except odp.OdpError as e:
        if "do not cover" in str(e):
            return False
        raise
    return True


def run_oracle(w, V0, **kw):
    import oracle
    return oracle.solve_workload(w, V0=V0, **kw)


def compare(gpu, ref, tol=TOL, band=BAND, mask=None):
    """Returns (max abs error, membership mismatches outside the band)."""
    g = np.asarray(gpu, dtype=np.float64)
    r = np.asarray(ref, dtype=np.float64)
    assert g.shape == r.shape, (g.shape, r.shape)
    d = np.abs(g - r)
    if mask is not None:
        d = d[..., mask] if mask.ndim < d.ndim else d[mask]
    memb = ((g <= 0) != (r <= 0)) & (np.abs(r) >= band)
    return float(d.max()) if d.size else 0.0, int(memb.sum())


def assert_parity(gpu, ref, tol=TOL, band=BAND, what=""):
    err, mism = compare(gpu, ref, tol, band)
    assert err <= tol and mism == 0, f"{what}: max|dV| = {err:.3e} (tol {tol}), membership mismatches = {mism}"
    return err


def dilate(mask, r):
    """Star-shaped dilation of a boolean N-D mask by r nodes along every axis."""
    out = mask.copy()
    for ax in range(mask.ndim):
        for k in range(1, r + 1):
            a = [slice(None)] * mask.ndim
            b = [slice(None)] * mask.ndim
            a[ax] = slice(k, None)
            b[ax] = slice(None, -k)
            out[tuple(a)] |= mask[tuple(b)]
            out[tuple(b)] |= mask[tuple(a)]
    return out


def assert_parity_one_step(gpu, ref, R, tol=TOL, band=BAND, what=""):
    """Strict parity for ONE time step of MEDIUM (ENO2 + RK2), exempting only nodes within the
    stencil radius of an ENO2 pick the oracle flags as a float32-level near-tie (reading A28);
    even there the deviation must stay below 1e-3."""
    g = np.asarray(gpu, dtype=np.float64)
    r = np.asarray(ref.out, dtype=np.float64)
    amb = ref.ambiguous.astype(bool)
    m = dilate(amb, R) if amb.any() else amb
    d = np.abs(g - r)
    dd = d.reshape(d.shape[0], -1)
    mm = np.broadcast_to(m, d.shape).reshape(d.shape[0], -1)
    out_err = float(dd[~mm].max()) if (~mm).any() else 0.0
    in_err = float(dd[mm].max()) if mm.any() else 0.0
    memb = ((g <= 0) != (r <= 0)) & (np.abs(r) >= band)
    assert out_err <= tol and in_err <= 1e-3 and memb.sum() == 0, \
        f"{what}: max|dV| {out_err:.3e} outside / {in_err:.3e} inside the ENO-tie mask ({int(amb.sum())} ties), " \
        f"membership mismatches {int(memb.sum())}"
    return out_err, in_err, int(amb.sum())


def oracle_envelope(w, V0, nperturb=6, **kw):
    """The oracle's own sensitivity to float32-level perturbations (reading A28).

    ENO2 (MEDIUM) selects its stencil by comparing |second differences|; that choice is a
    discontinuous function of the data, so a 1-ulp change of the input can move the result by far
    more than 1e-4 (the paper's own Table 1 shows second-order implementations differing by up to
    0.25).  E(x) = max over {oracle with V0 perturbed by +-1 ulp at random nodes (seeded),
    oracle with float32 storage after every stage} of |V_run(x) - V_base(x)|, all computed by the
    oracle alone.  Returns (base SolveResult, E)."""
    import oracle
    base = oracle.solve_workload(w, V0=V0, **kw)
    E = np.abs(oracle.solve_workload(w, V0=V0, store_f32=True, **kw).out - base.out)
    for s in range(nperturb):
        rng = np.random.default_rng(1000 + s)
        flip = rng.random(V0.shape) < 0.5
        up = rng.random(V0.shape) < 0.5
        Vp = np.where(flip, np.where(up, np.nextafter(V0, np.float32(np.inf)), np.nextafter(V0, np.float32(-np.inf))),
                      V0).astype(np.float32)
        E = np.maximum(E, np.abs(oracle.solve_workload(w, V0=Vp, **kw).out - base.out))
    return base, E


def assert_parity_envelope(gpu, base, E, tol=TOL, band=BAND, what=""):
    """MEDIUM (ENO2 + TVD-RK2) over many steps: the GPU result must be indistinguishable from another
    float32 realisation of the scheme, judged against the oracle's own float32 envelope E
    (oracle_envelope: float32 storage and 1-ulp input perturbations, computed by the oracle alone).
    ENO2 selects its stencil by comparing |second differences|, a discontinuous function of the data:
    float32 realisations flip isolated near-tie picks at DIFFERENT nodes, so a node-by-node bar on
    "oracle-stable" nodes does not hold even between two oracle realisations (reading A28; the
    measurements are in DESIGN.md §5).  The bar:
      (1) max |V_gpu - V_oracle| <= max(tol, 2 max E);
      (2) nodes off by more than tol: no more than 2 x the nodes with E > tol (+ 4);
      (3) the 99.9 % quantile of |V_gpu - V_oracle| <= max(tol / 10, 2 x that of E) (bulk agreement);
      (4) membership (V <= 0) identical wherever |V_oracle| >= max(band, E)."""
    g = np.asarray(gpu, dtype=np.float64)
    r = base.out
    d = np.abs(g - r)
    emax = float(E.max())
    assert d.max() <= max(tol, 2 * emax), f"{what}: max|dV| {d.max():.3e} > max(tol, 2 max E = {2 * emax:.3e})"
    ng, ne = int((d > tol).sum()), int((E > tol).sum())
    assert ng <= 2 * ne + 4, f"{what}: {ng} nodes off by > tol vs the oracle's own spread {ne}"
    qd, qe = float(np.quantile(d, 0.999)), float(np.quantile(E, 0.999))
    assert qd <= max(tol / 10, 2 * qe), f"{what}: q99.9 |dV| {qd:.3e} vs the oracle's {qe:.3e}"
    memb = ((g <= 0) != (r <= 0)) & (np.abs(r) >= np.maximum(band, E))
    assert memb.sum() == 0, f"{what}: {int(memb.sum())} membership mismatches outside the band"
    return float(d.max()), emax, ng, ne


# ------------------------------------------------------------------------------------------------
# Windowed oracle (pin Z12): after s stages a node depends only on the nodes within
# R s of it along each axis (Alg. 2 is a star stencil of radius R per stage; the BRT min is
# pointwise), provided alpha^max -- hence dt -- is the full grid's.  For dynamics whose alpha does
# not depend on the derivative range (RANGE_FREE, e.g. DOUBLEINT6D) the full grid's alpha^max is a
# function of the coordinate extremes only, so a float64 oracle solve on a sub-box (clipped at the
# real faces, where the ghost rule is the real one) reproduces the full solve at the box centre.
# ------------------------------------------------------------------------------------------------
def full_grid_amax(w):
    """alpha^max of the full grid (Alg. 2 l.164) from the oracle's own alpha at every combination
    of the axes' extreme nodes (alpha of the compiled-in RANGE_FREE dynamics is monotone in |x|)."""
    import itertools
    import oracle
    from inputs import axis_nodes
    ax = [axis_nodes(n, l, h, bool(p)) for n, l, h, p in zip(w.N, w.lo, w.hi, w.periodic)]
    cand = [sorted(set([a[0], a[-1], a[len(a) // 2]])) for a in ax]
    n = len(w.N)
    amax = np.zeros(n)
    for x in itertools.product(*cand):
        amax = np.maximum(amax, oracle.alpha(w.dynamics, w.params, np.array(x), -np.ones(n), np.ones(n)))
    return amax


def windowed_oracle(w, nodes, stages_per_step, steps, amax):
    """Values of the float64 oracle solve of `w` (one output time, tau = w.tau[-1]) at `nodes`
    (list of index tuples), each from a sub-box of half-width R * stages around the node."""
    import oracle
    from inputs import axis_nodes, make_v0
    R = 1 if w.accuracy == "low" else 2
    hw = R * stages_per_step * steps
    ax = [axis_nodes(n, l, h, bool(p)) for n, l, h, p in zip(w.N, w.lo, w.hi, w.periodic)]
    vals = []
    for node in nodes:
        box = []
        for d, i in enumerate(node):
            if w.periodic[d]:
                box.append((0, w.N[d]))
            else:
                b = max(0, i - hw)
                e = min(w.N[d], i + hw + 1)
                box.append((b, e - b))
        V0 = make_v0(w, box=box)
        lo = tuple(float(ax[d][b]) for d, (b, c) in enumerate(box))
        hi = tuple(float(ax[d][b + c - 1]) if not w.periodic[d] else w.hi[d] for d, (b, c) in enumerate(box))
        N = tuple(c for _, c in box)
        r = oracle.hj_solve(N, lo, hi, w.periodic_mask, w.dynamics, w.params, V0, w.tau, w.accuracy, w.mode,
                            cfl=w.cfl, amax_fixed=amax)
        local = tuple(i - b for i, (b, _) in zip(node, box))
        vals.append((float(r.out[-1][local]), r.steps, r.stages))
    return vals


def sample_nodes(N, count, seed, faces=True):
    """Seeded node sample: uniform nodes plus (faces=True) nodes on every face band of every axis."""
    rng = np.random.default_rng(seed)
    out = [tuple(int(rng.integers(0, n)) for n in N) for _ in range(count)]
    if faces:
        for d, n in enumerate(N):
            for fv in (0, 1, n - 2, n - 1):
                x = [int(rng.integers(0, m)) for m in N]
                x[d] = fv
                out.append(tuple(x))
    return out
