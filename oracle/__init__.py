"""float64 CPU ORACLE of the OptimizedDP time-dependent HJ step (§3.2, Alg. 2).

TEST INFRASTRUCTURE.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
`--impl reference` legs may import this package.  It shares no code with the CUDA path
(paper_2204_05520_b200/) and never calls it; the product path never imports it.

`odp_oracle.c` is the oracle proper (plain per-node loops, fp64, OpenMP).  `brute.py` is a
second, independently written NumPy "full temporaries" formulation (the MATLAB style of
P:174-179) used to cross-check it on tiny grids (pin Z11).

Every function here is pinned by tests/test_oracle_*.py; see DESIGN.md §4 for the pin table.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "odp_oracle.c")
_LIB = os.path.join(_HERE, "libodp_oracle.so")

DYN_IDS = {"HOLONOMIC_BALL": 0, "HOLONOMIC_BOX": 1, "DUBINS3D": 2, "CAR4D": 3, "CAR5D": 4, "DOUBLEINT6D": 5,
           "PAIR_DUBINS3D": 6}
ACC_IDS = {"low": 1, "medium": 2}
MODE_IDS = {"brs": 0, "brt": 1}
OK, EINVAL, ENUMERIC, ENOMEM = 0, 1, 2, 5


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2, OpenMP, no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
                               "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        D = ctypes.POINTER(ctypes.c_double)
        I64 = ctypes.POINTER(ctypes.c_int64)
        F = ctypes.POINTER(ctypes.c_float)
        c_int, c_u32, c_dbl = ctypes.c_int, ctypes.c_uint32, ctypes.c_double
        _lib.oracle_grid_axes.argtypes = [c_int, I64, D, D, c_u32, D, D]
        _lib.oracle_line_value.argtypes = [D, ctypes.c_int64, c_int, ctypes.c_int64]
        _lib.oracle_line_value.restype = c_dbl
        _lib.oracle_derivs.argtypes = [c_int, I64, D, D, c_u32, D, c_int, D, D]
        _lib.oracle_hamiltonian.argtypes = [c_int, D, c_int, c_int, D, D, D, D, D, D]
        _lib.oracle_rate.argtypes = [c_int, D, c_int, c_int, D, D, D, D]
        _lib.oracle_alpha.argtypes = [c_int, D, c_int, c_int, D, D, D, D]
        _lib.oracle_stage.argtypes = [c_int, I64, D, D, c_u32, c_int, D, c_int, D, c_int, D, D, c_int]
        _lib.oracle_hj_solve.argtypes = [c_int, I64, D, D, c_u32, c_int, D, c_int, F, F, D, c_int, c_int,
                                         c_int, c_dbl, c_int, c_int, D, D, D, I64, I64, c_int,
                                         ctypes.c_void_p]
        _lib.oracle_ttr_solve.argtypes = [c_int, I64, D, D, c_u32, c_int, D, c_int, F, c_dbl, c_dbl,
                                          ctypes.c_int64, D, I64, D]
        _lib.oracle_vi_solve.argtypes = [c_int, I64, D, D, c_u32, c_int, D, c_int, F, c_dbl, ctypes.c_int64,
                                         c_int, D, I64, D]
        _lib.oracle_vi_successor.argtypes = [c_int, I64, D, D, c_u32, c_int, D, c_int, I64, c_int, c_int, I64]
        _lib.oracle_max_threads.restype = c_int
        _lib.oracle_cfl_dt.argtypes = [c_int, D, D, c_dbl, c_dbl]
        _lib.oracle_cfl_dt.restype = c_dbl
    return _lib


def _d(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _i64(a):
    a = np.ascontiguousarray(a, dtype=np.int64)
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


class OracleError(RuntimeError):
    def __init__(self, status, msg=""):
        super().__init__(f"oracle status {status} {msg}")
        self.status = status


def max_threads() -> int:
    return int(lib().oracle_max_threads())


def cfl_dt(amax, dx, cfl: float, remaining: float = float("inf")) -> float:
    aa, ap = _d(amax)
    xa, xp = _d(dx)
    return float(lib().oracle_cfl_dt(len(aa), ap, xp, float(cfl), float(remaining)))


def grid_axes(N, lo, hi, periodic_mask: int):
    n = len(N)
    Na, Np = _i64(N)
    loa, lop = _d(lo)
    hia, hip = _d(hi)
    dx = np.zeros(n)
    coords = np.zeros(int(np.sum(Na)))
    st = lib().oracle_grid_axes(n, Np, lop, hip, periodic_mask, dx.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                coords.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    if st:
        raise OracleError(st)
    out, off = [], 0
    for d in range(n):
        out.append(coords[off:off + Na[d]].copy())
        off += Na[d]
    return dx, out


def line_value(W, periodic: bool, j: int) -> float:
    Wa, Wp = _d(W)
    return float(lib().oracle_line_value(Wp, len(Wa), int(periodic), int(j)))


def derivs(W, lo, hi, periodic_mask: int, accuracy: str):
    W = np.ascontiguousarray(W, dtype=np.float64)
    n = W.ndim
    Na, Np = _i64(W.shape)
    loa, lop = _d(lo)
    hia, hip = _d(hi)
    Dm = np.zeros((n,) + W.shape)
    Dp = np.zeros((n,) + W.shape)
    st = lib().oracle_derivs(n, Np, lop, hip, periodic_mask, W.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                             ACC_IDS[accuracy], Dm.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                             Dp.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    if st:
        raise OracleError(st)
    return Dm, Dp


def hamiltonian(dyn: str, params, x, p):
    n = len(x)
    pa, pp = _d(params)
    xa, xp = _d(x)
    qa, qp = _d(p)
    H = ctypes.c_double()
    u, dd, f = np.zeros(6), np.zeros(6), np.zeros(6)
    st = lib().oracle_hamiltonian(DYN_IDS[dyn], pp, len(pa), n, xp, qp, ctypes.byref(H),
                                  u.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                  dd.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                  f.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    if st:
        raise OracleError(st)
    return H.value, u, dd, f[:n]


def rate(dyn: str, params, x, u, d):
    n = len(x)
    pa, pp = _d(params)
    xa, xp = _d(x)
    ua, up = _d(np.resize(np.asarray(u, dtype=np.float64), 6) if len(u) else np.zeros(6))
    da, dp_ = _d(np.resize(np.asarray(d, dtype=np.float64), 6) if len(d) else np.zeros(6))
    f = np.zeros(6)
    st = lib().oracle_rate(DYN_IDS[dyn], pp, len(pa), n, xp, up, dp_, f.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    if st:
        raise OracleError(st)
    return f[:n]


def alpha(dyn: str, params, x, minD, maxD):
    n = len(x)
    pa, pp = _d(params)
    xa, xp = _d(x)
    mna, mnp = _d(minD)
    mxa, mxp = _d(maxD)
    out = np.zeros(n)
    st = lib().oracle_alpha(DYN_IDS[dyn], pp, len(pa), n, xp, mnp, mxp, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    if st:
        raise OracleError(st)
    return out


def stage(W, lo, hi, periodic_mask: int, dyn: str, params, accuracy: str, nthreads: int = 0):
    """One L(W) evaluation; returns (L, minD, maxD, alpha_max, maxabs, nan)."""
    W = np.ascontiguousarray(W, dtype=np.float64)
    n = W.ndim
    Na, Np = _i64(W.shape)
    loa, lop = _d(lo)
    hia, hip = _d(hi)
    pa, pp = _d(params)
    L = np.zeros(W.shape)
    rng = np.zeros(3 * n + 2)
    st = lib().oracle_stage(n, Np, lop, hip, periodic_mask, DYN_IDS[dyn], pp, len(pa),
                            W.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ACC_IDS[accuracy],
                            L.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                            rng.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), nthreads)
    if st:
        raise OracleError(st)
    return L, rng[:n], rng[n:2 * n], rng[2 * n:3 * n], rng[3 * n], bool(rng[3 * n + 1])


class SolveResult:
    def __init__(self, out, tau_reached, steps, stages, status):
        self.out, self.tau_reached, self.steps, self.stages, self.status = out, tau_reached, steps, stages, status


def hj_solve(N, lo, hi, periodic_mask: int, dyn: str, params, V0, tau: Sequence[float], accuracy: str,
             mode: str, cfl: float = 0.0, target=None, write_initial: bool = False, store_f32: bool = False,
             amax_fixed=None, nthreads: int = 0, raise_on_error: bool = True, ambiguity: bool = False) -> SolveResult:
    """Full oracle solve (O0-O9). V0/target float32 arrays of shape N; returns float64 snapshots."""
    N = tuple(int(v) for v in N)
    n = len(N)
    V0 = np.ascontiguousarray(V0, dtype=np.float32).reshape(N)
    Na, Np = _i64(N)
    loa, lop = _d(lo)
    hia, hip = _d(hi)
    pa, pp = _d(params)
    ta, tp = _d(tau)
    nout = len(ta) if write_initial else len(ta) - 1
    out = np.zeros((nout,) + N, dtype=np.float64)
    tgt = None
    if target is not None:
        tgt = np.ascontiguousarray(target, dtype=np.float32).reshape(N)
    amf = None
    if amax_fixed is not None:
        amf = np.ascontiguousarray(amax_fixed, dtype=np.float64)
    amb = np.zeros(N, dtype=np.uint8) if ambiguity else None
    tr = ctypes.c_double()
    steps = ctypes.c_int64()
    stages = ctypes.c_int64()
    Fp = ctypes.POINTER(ctypes.c_float)
    Dp = ctypes.POINTER(ctypes.c_double)
    st = lib().oracle_hj_solve(n, Np, lop, hip, periodic_mask, DYN_IDS[dyn], pp, len(pa), V0.ctypes.data_as(Fp),
                               tgt.ctypes.data_as(Fp) if tgt is not None else None, tp, len(ta),
                               ACC_IDS[accuracy], MODE_IDS[mode], float(cfl), int(write_initial), int(store_f32),
                               amf.ctypes.data_as(Dp) if amf is not None else None, out.ctypes.data_as(Dp),
                               ctypes.byref(tr), ctypes.byref(steps), ctypes.byref(stages), int(nthreads),
                               amb.ctypes.data if amb is not None else None)
    if st and raise_on_error:
        raise OracleError(st)
    r = SolveResult(out, tr.value, steps.value, stages.value, st)
    r.ambiguous = amb
    return r


def ttr_solve(N, lo, hi, periodic_mask: int, dyn: str, params, V0, eps: float = 1e-6, max_sweeps: int = 10000,
              big: float = 100.0):
    """Time-to-reach by Lax-Friedrichs sweeping (Alg. 3, readings A31-A34).  Target = {V0 <= 0}.
    Returns (phi float64 array of shape N, sweeps, last max |phi - phi_old|)."""
    N = tuple(int(v) for v in N)
    n = len(N)
    V0 = np.ascontiguousarray(V0, dtype=np.float32).reshape(N)
    Na, Np = _i64(N)
    loa, lop = _d(lo)
    hia, hip = _d(hi)
    pa, pp = _d(params)
    out = np.zeros(N, dtype=np.float64)
    sw = ctypes.c_int64()
    ch = ctypes.c_double()
    st = lib().oracle_ttr_solve(n, Np, lop, hip, periodic_mask, DYN_IDS[dyn], pp, len(pa),
                                V0.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), float(big), float(eps),
                                int(max_sweeps), out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                ctypes.byref(sw), ctypes.byref(ch))
    if st:
        raise OracleError(st)
    return out, sw.value, ch.value


MDP_IDS = {"HOLONOMIC": 0, "DUBINS3D": 1}


def vi_solve(N, lo, hi, periodic_mask: int, model: str, params, R, threshold: float = 1e-6,
             max_iters: int = 100000, order: str = "jacobi"):
    """Value iteration (Alg. 1, readings A36-A38).  R: float32 reward per node.  order "jacobi" or
    "gauss_seidel" (in place, 8 orderings, §4.3).  Returns (V float64 of shape N, iterations, last change)."""
    N = tuple(int(v) for v in N)
    R = np.ascontiguousarray(R, dtype=np.float32).reshape(N)
    Na, Np = _i64(N)
    loa, lop = _d(lo)
    hia, hip = _d(hi)
    pa, pp = _d(params)
    out = np.zeros(N, dtype=np.float64)
    it = ctypes.c_int64()
    ch = ctypes.c_double()
    st = lib().oracle_vi_solve(len(N), Np, lop, hip, periodic_mask, MDP_IDS[model], pp, len(pa),
                               R.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), float(threshold), int(max_iters),
                               {"jacobi": 0, "gauss_seidel": 1}[order],
                               out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ctypes.byref(it), ctypes.byref(ch))
    if st:
        raise OracleError(st)
    return out, it.value, ch.value


def vi_successor(N, lo, hi, periodic_mask: int, model: str, params, idx, a: int, k: int) -> int:
    """Flat index of the nearest-node successor of node idx under action a, outcome k (A36)."""
    N = tuple(int(v) for v in N)
    Na, Np = _i64(N)
    loa, lop = _d(lo)
    hia, hip = _d(hi)
    pa, pp = _d(params)
    ia, ip = _i64(idx)
    out = ctypes.c_int64()
    st = lib().oracle_vi_successor(len(N), Np, lop, hip, periodic_mask, MDP_IDS[model], pp, len(pa), ip, int(a),
                                   int(k), ctypes.byref(out))
    if st:
        raise OracleError(st)
    return out.value


def solve_workload(w, V0=None, seed=None, **kw) -> SolveResult:
    """Oracle solve of an inputs.Workload."""
    from inputs import make_v0
    if V0 is None:
        V0 = make_v0(w, seed=seed)
    kw.setdefault("cfl", w.cfl)
    return hj_solve(w.N, w.lo, w.hi, w.periodic_mask, w.dynamics, w.params, V0, w.tau, w.accuracy, w.mode, **kw)
