"""B200-native time-dependent Hamilton-Jacobi level-set step of OptimizedDP (arXiv 2204.05520).

The hot path (§3.2 Algorithm 2) runs in hand-written sm_100a CUDA kernels behind the C-ABI
in include/odp.h (libodp.so, built in-tree).  This package is the thin Python binding: argument
marshalling only, torch for device memory and streams.  There is no CPU fallback: importing the
package fails loudly if libodp.so has not been built.
"""
from .capi import (ACCURACY, DYNAMICS, MODE, Grid, Loopback, OdpError, comm_unique_id, hj_solve,  # noqa: F401
                   hj_solve_host, last_error, partition_extent, ttr_solve, ttr_solve_host, version, vi_solve, vi_solve_host)


def solve_workload(w, V0, **kw):
    """Convenience: run an inputs.Workload-like object (N, lo, hi, periodic_mask, dynamics, params,
    tau, accuracy, mode, cfl) through odp_hj_solve on the current CUDA device."""
    g = Grid(w.N, w.lo, w.hi, w.periodic_mask)
    try:
        kw.setdefault("cfl", w.cfl)
        return hj_solve(g, w.dynamics, w.params, V0, w.tau, w.accuracy, w.mode, **kw)
    finally:
        g.close()
