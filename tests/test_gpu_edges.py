"""Edge cases of the HJ path (SURVEY.md §8(d) parity list): the smallest grids the C-ABI accepts,
degenerate dynamics (alpha = 0: reading A20), save intervals far below the CFL step (reading A9's
clipping), many snapshots, a ragged innermost extent on every kernel family."""
import math

import numpy as np
import pytest

from inputs import Workload, make_v0
from tests.parity_util import assert_parity, assert_parity_envelope, covers, oracle_envelope, run_gpu, run_oracle

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("N", [(3,), (3, 3), (3, 4, 3), (5, 5, 5)])
@pytest.mark.parametrize("acc", ["low", "medium"])
def test_smallest_grids(N, acc):
    n = len(N)
    w = Workload("tiny", N, (-1.0,) * n, (1.0,) * n, (0,) * n, "HOLONOMIC_BOX", (1.0, 0.3, -1.0), (0.0, 0.2, 0.5),
                 acc, 0.8 if acc == "low" else 0.5, "brt", ("random_smooth", 3))
    V0 = make_v0(w, seed=1)
    out, info = run_gpu(w, V0)
    if acc == "low":
        ref = run_oracle(w, V0)
        assert_parity(out, ref.out, what=f"tiny {N} {acc}")
    else:
        ref, E = oracle_envelope(w, V0)
        assert_parity_envelope(out, ref, E, what=f"tiny {N} {acc}")
    assert info["steps"] == ref.steps


@pytest.mark.parametrize("mode", ["brs", "brt"])
def test_zero_dynamics_keeps_v0_and_takes_one_step_per_interval(mode):
    # ubar = dbar: H = 0 and alpha = 0 everywhere, so dt = tau_k - tau (A20) and V never changes
    w = Workload("still", (12, 11, 10), (-1.0,) * 3, (1.0,) * 3, (0, 0, 1), "HOLONOMIC_BOX", (0.5, 0.5, 1.0),
                 (0.0, 0.3, 0.7, 1.0), "medium", 0.5, mode, ("random_smooth", 2))
    V0 = make_v0(w, seed=2)
    out, info = run_gpu(w, V0)
    for k in range(3):
        np.testing.assert_array_equal(out[k], V0)
    assert info["steps"] == 3
    ref = run_oracle(w, V0)
    assert ref.steps == 3


def test_save_intervals_below_the_cfl_step():
    w = Workload("clip", (21, 19, 16), (-4.0, -4.0, -math.pi), (4.0, 4.0, math.pi), (0, 0, 1), "DUBINS3D",
                 (1.0, 1.0, -1.0), (0.0, 1e-9, 2e-9, 1e-3, 0.0500001, 0.1), "low", 0.8, "brt",
                 ("cylinder", (0, 1), 1.0))
    V0 = make_v0(w, seed=3)
    out, info = run_gpu(w, V0)
    ref = run_oracle(w, V0)
    assert_parity(out, ref.out, what="clipped save times")
    assert info["steps"] == ref.steps and abs(info["tau_reached"] - 0.1) < 1e-12


def test_many_snapshots():
    tau = tuple(0.01 * k for k in range(51))
    w = Workload("snaps", (17, 15, 12), (-2.0, -2.0, -math.pi), (2.0, 2.0, math.pi), (0, 0, 1), "DUBINS3D",
                 (1.0, 0.7, 1.0), tau, "low", 0.8, "brt", ("cylinder", (0, 1), 0.8))
    V0 = make_v0(w, seed=4)
    out, info = run_gpu(w, V0)
    ref = run_oracle(w, V0)
    assert out.shape[0] == 50
    assert_parity(out, ref.out, what="50 snapshots")
    assert info["steps"] == ref.steps


@pytest.mark.parametrize("kernel", ["generic", "tiled", "stream", "march"])
def test_ragged_innermost_extent(kernel):
    # odd innermost extents exercise the partial tiles / half-filled vector lanes of each family
    w = Workload("ragged", (9, 7, 11, 13), (-2.0, -1.0, -2.0, -1.0), (2.0, 1.0, 2.0, 1.0), (0, 0, 0, 0),
                 "HOLONOMIC_BOX", (1.0, 0.2, -1.0), (0.0, 0.15), "medium", 0.5, "brt", ("random_smooth", 5))
    if kernel in ("stream", "march") and not covers(w, kernel):
        pytest.skip(f"{kernel} family does not cover odd innermost extents")
    if kernel == "tiled" and (w.N[-1] * w.N[-2]) % 4:
        pytest.skip("tiled family needs a tile of 4k floats")
    V0 = make_v0(w, seed=5)
    out, info = run_gpu(w, V0, kernel=kernel)
    ref, E = oracle_envelope(w, V0)
    assert_parity_envelope(out, ref, E, what=f"ragged {kernel}")
