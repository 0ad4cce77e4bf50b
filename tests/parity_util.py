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


def assert_parity_multistep_medium(gpu, ref, tol=TOL, what="", q=0.999, max_tol=2e-3):
    """Parity over MANY steps of MEDIUM (ENO2 + RK2).

    ENO2 picks its stencil by comparing |second differences|; that choice is a discontinuous
    function of the data, so two float evaluations of the same scheme (float32 GPU, float64
    oracle -- or the oracle against itself with a 1-ulp perturbed input) occasionally pick
    differently at a near-tie and then differ at that node by a few 1e-4 (reading A28; the paper's
    own Table 1 shows second-order implementations disagreeing by up to 0.25).  Bar:
      * the q-quantile (99.9 %) of |V_gpu - V_oracle| <= 1e-4 (the north_star tolerance),
      * max |V_gpu - V_oracle| <= 2e-3 (isolated tie events only),
      * membership identical wherever |V_oracle| >= 1e-3, and outside |V_oracle| < 1e-4 on all
        but 1e-5 of the nodes.
    """
    g = np.asarray(gpu, dtype=np.float64)
    r = np.asarray(ref.out if hasattr(ref, "out") else ref, dtype=np.float64)
    d = np.abs(g - r)
    qv = float(np.quantile(d, q))
    mx = float(d.max())
    memb = (g <= 0) != (r <= 0)
    hard = int((memb & (np.abs(r) >= 1e-3)).sum())
    soft = float((memb & (np.abs(r) >= BAND)).mean())
    assert qv <= tol and mx <= max_tol and hard == 0 and soft <= 1e-5, \
        f"{what}: q{q} {qv:.3e}, max {mx:.3e}, membership mismatches |V|>=1e-3: {hard}, band fraction {soft:.2e}"
    return qv, mx


def oracle_envelope(w, V0, nperturb=2, **kw):
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
    """Strict 1e-4 parity where the oracle itself is stable, the oracle's own spread elsewhere.

      (1) max |V_gpu - V_oracle| <= max(tol, 2 max E)
      (2) nodes with |dV| > tol are no more frequent than 2x the nodes with E > tol (+0.1 % slack)
      (3) membership identical wherever |V_oracle| >= max(band, E)
    """
    g = np.asarray(gpu, dtype=np.float64)
    r = base.out
    d = np.abs(g - r)
    emax = float(E.max())
    assert d.max() <= max(tol, 2 * emax), f"{what}: max|dV| {d.max():.3e} > max(tol, 2 max E = {2 * emax:.3e})"
    frac_g = float((d > tol).mean())
    frac_e = float((E > tol).mean())
    assert frac_g <= 2 * frac_e + 1e-3, f"{what}: {frac_g:.4%} of nodes off by > tol vs oracle spread {frac_e:.4%}"
    memb = ((g <= 0) != (r <= 0)) & (np.abs(r) >= np.maximum(band, E))
    assert memb.sum() == 0, f"{what}: {int(memb.sum())} membership mismatches outside the band"
    return float(d.max()), emax, frac_g, frac_e
