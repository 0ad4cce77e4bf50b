import sys; sys.path.insert(0, ".")
import numpy as np
from inputs import CONFIGS, make_v0
from tests.parity_util import run_gpu, run_oracle
import oracle
w = CONFIGS["f2"]
V0 = make_v0(w)
out, info = run_gpu(w, V0)
ref = run_oracle(w, V0)
d = np.abs(out[-1] - ref.out[-1])
i = np.unravel_index(np.argmax(d), d.shape)
print("max", d.max(), "at", i, "V", ref.out[-1][i], "V0", V0[i], "q99.9", np.quantile(d, 0.999), "q99", np.quantile(d, 0.99))
f32 = oracle.solve_workload(w, V0=V0, store_f32=True)
e = np.abs(f32.out[-1] - ref.out[-1])
print("oracle f32-storage vs f64: max", e.max(), "q99.9", np.quantile(e, 0.999))
near = np.abs(ref.out[-1]) < 0.5
print("near zero level: gpu max", d[near].max(), "f32 max", e[near].max())
