"""Debug helper: GPU vs oracle on one small case, per-axis error profile and per-step growth."""
import math
import sys

import numpy as np

sys.path.insert(0, ".")
from inputs import Workload, make_v0
from tests.parity_util import run_gpu, run_oracle

np.set_printoptions(precision=1, linewidth=200)
cases = {
    "car4d": ("CAR4D", (1.5, 1.0, 0.25, 0.25, -1.0), (15, 14, 13, 12), (-5.0, -5.0, 0.0, -math.pi), (5.0, 5.0, 4.0, math.pi), (0, 0, 0, 1)),
    "car5d": ("CAR5D", (1.0, 2.0, -1.0), (11, 10, 12, 9, 8), (-5.0, -5.0, -math.pi, 0.0, -2.0), (5.0, 5.0, math.pi, 3.0, 2.0), (0, 0, 1, 0, 0)),
}
for name in sys.argv[1:] or ["car4d"]:
    dyn, prm, N, lo, hi, per = cases[name]
    for acc in ("medium", "low"):
        for seed in (None, 0):
            taus = tuple(0.025 * k for k in range(11))
            w = Workload("dbg", N, lo, hi, per, dyn, prm, taus, acc, 0.5 if acc == "medium" else 0.8, "brs", ("random_smooth", len(N)))
            V0 = make_v0(w, seed=seed)
            ref = run_oracle(w, V0)
            f32 = run_oracle(w, V0, store_f32=True)
            for kernel in ("generic", "auto"):
                out, info = run_gpu(w, V0, kernel=kernel)
                d = np.abs(out - ref.out)
                print(f"{name} {acc} seed={seed} {kernel}: steps {info['steps']}/{ref.steps} per-save max|dV|",
                      " ".join(f"{x:.1e}" for x in d.reshape(d.shape[0], -1).max(1)))
            e = np.abs(f32.out - ref.out)
            print("   oracle f32-storage gap      ", " ".join(f"{x:.1e}" for x in e.reshape(e.shape[0], -1).max(1)))
            dl = d[-1]
            for ax in range(len(N)):
                print("   axis", ax, np.log10(dl.max(axis=tuple(i for i in range(len(N)) if i != ax)) + 1e-30))
