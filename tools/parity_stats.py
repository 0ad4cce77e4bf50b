"""Diagnostic (GPU): GPU-vs-oracle difference statistics against the oracle's own float32 envelope
for the MEDIUM parity cases (designing the envelope bar; tests/parity_util.py)."""
import math
import sys

import numpy as np

sys.path.insert(0, ".")
from inputs import CONFIGS, Workload, coarsened, make_v0
from tests.parity_util import oracle_envelope, run_gpu

cases = [
    ("car4d-small-brs", Workload("small", (15, 14, 13, 12), (-5.0, -5.0, 0.0, -math.pi), (5.0, 5.0, 4.0, math.pi), (0, 0, 0, 1),
                                 "CAR4D", (1.5, 1.0, 0.25, 0.25, -1.0), (0.0, 0.1, 0.25), "medium", 0.5, "brs",
                                 ("random_smooth", 4)), 0),
    ("c4@12", coarsened(CONFIGS["c4"], (12,) * 6, tau=(0.0, 0.25, 0.5, 1.0)), None),
    ("c4@16", coarsened(CONFIGS["c4"], (16,) * 6, tau=(0.0, 0.5, 1.0)), None),
    ("c3@16", coarsened(CONFIGS["c3"], (16,) * 5, tau=(0.0, 0.5, 1.0)), None),
]
for name, w, seed in cases:
    V0 = make_v0(w, seed=seed)
    for extra in ({}, {"single_pass": True}):
        out, info = run_gpu(w, V0, **extra)
        for npert in (2, 6):
            ref, E = oracle_envelope(w, V0, nperturb=npert)
            d = np.abs(out.astype(np.float64) - ref.out)
            stable = E <= 5e-5
            print(f"{name} {extra} npert={npert}: n={d.size} max d {d.max():.2e} max E {E.max():.2e} "
                  f"off(d>1e-4) {(d > 1e-4).sum()} E>1e-4 {(E > 1e-4).sum()} | stable-violations "
                  f"{((d > 1e-4) & stable).sum()} (max {d[stable].max():.2e}) | q99.9 d {np.quantile(d, 0.999):.2e} E {np.quantile(E, 0.999):.2e}",
                  flush=True)
