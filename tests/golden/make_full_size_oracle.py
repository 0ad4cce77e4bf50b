"""Writes the full-size, full-horizon oracle fixtures of tests/test_gpu_parity_full.py.

Calls ONLY oracle/ and inputs/ (never the CUDA path): the float64 oracle solves c4 (30^6,
DOUBLEINT6D, ENO2 + TVD-RK2, BRT, CFL 0.5, tau in [0, 1]; BASELINE.json configs[3]) over the whole
horizon -- once as written (float64 storage) and once with float32 storage after every stage (the
oracle's own float32 envelope, reading A28 / pin Z4) -- and stores the values at a seeded sample of
nodes: uniform random nodes, random nodes on the face bands (one coordinate in {0, 1, N-2, N-1}) and
every node of a few whole in-plane tiles.  Algorithm 2 is the authority; the
oracle follows it step by step (oracle/odp_oracle.c).

usage:  python tests/golden/make_full_size_oracle.py c4 [c3]    (hours on 8 cores; ~40 min per run on 16)
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from inputs import CONFIGS, make_v0  # noqa: E402

# c3 is compared to tau = 1 only: beyond that the extrapolated inflow faces dominate (reading A29)
CASES = {"c4": (0.0, 1.0), "c3": (0.0, 1.0)}


def sample_nodes(N, seed=20204, n_uniform=200_000, n_face=20_000):
    rng = np.random.default_rng(seed)
    P = int(np.prod(N))
    uni = np.unique(rng.integers(0, P, size=n_uniform, dtype=np.int64))
    idx = np.stack([rng.integers(0, n, size=n_face) for n in N], axis=1)
    ax = rng.integers(0, len(N), size=n_face)
    face_vals = np.array([0, 1, -2, -1])
    fv = face_vals[rng.integers(0, 4, size=n_face)]
    for k in range(n_face):
        idx[k, ax[k]] = fv[k] % N[ax[k]]
    face = np.ravel_multi_index(tuple(idx.T), N)
    # whole in-plane tiles (the two innermost axes) at the centre, at a face corner, at a mixed spot
    tiles = []
    outer = [tuple(n // 2 for n in N[:-2]), tuple(0 for _ in N[:-2]), tuple(n - 1 for n in N[:-2]),
             tuple((1 if d % 2 else n - 2) for d, n in enumerate(N[:-2]))]
    M = N[-2] * N[-1]
    for o in outer:
        base = np.ravel_multi_index(o + (0, 0), N)
        tiles.append(base + np.arange(M, dtype=np.int64))
    return np.unique(np.concatenate([uni, face] + tiles))


def main(names):
    for name in names:
        tau = CASES[name]
        w0 = CONFIGS[name]
        w = w0.__class__(**{**w0.__dict__, "tau": tau})
        V0 = make_v0(w)
        idx = sample_nodes(w.N)
        path = os.path.join(HERE, f"{name}_full_horizon.npz")
        res = {}
        for store_f32 in (False, True):
            t = time.time()
            r = oracle.solve_workload(w, V0=V0, store_f32=store_f32)
            key = "f32" if store_f32 else "f64"
            res[key] = r.out[-1].reshape(-1)[idx].copy()
            res[key + "_meta"] = np.array([r.steps, r.stages, r.tau_reached])
            print(f"{name} store_f32={store_f32}: steps {r.steps} stages {r.stages} ({time.time() - t:.0f} s)",
                  flush=True)
            del r
        np.savez_compressed(path, idx=idx, V_f64=res["f64"], V_f32store=res["f32"], meta_f64=res["f64_meta"],
                            meta_f32store=res["f32_meta"], N=np.array(w.N), tau=np.array(tau),
                            threads=np.array(oracle.max_threads()))
        print("wrote", path, len(idx), "nodes", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c4"])
