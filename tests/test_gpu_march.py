"""GPU parity of the march kernel family's special paths against the float64 oracle.

The march family (kernels_march.cuh) changes how the stencil is evaluated, not what: edge-shared
ENO2 picks carried along the marching axis, an edge-assigned pass 1 (each node contributes its
upper edge; face nodes add the face edges), in-plane ghosts formed in registers, periodic wraps
written into the shared tile by their owners, packed float2 arithmetic.  These cases aim at every
branch of that code: periodic rows / columns / marching axis, both vector widths, marching
segments that start and end inside the column, tiny extents where the faces of an axis overlap,
and derivative ranges (pass 1) that feed alpha and dt directly (the holonomic ball, whose alpha
depends on the range magnitudes, so a missed or spurious D+-value changes the result).
"""
import math
import os

import numpy as np
import pytest

from inputs import Workload
from tests.parity_util import assert_parity, assert_parity_one_step, covers, run_gpu, run_oracle

pytestmark = pytest.mark.gpu

CASES = [
    # name, dynamics, params, N, lo, hi, periodic
    ("ball3-percol", "HOLONOMIC_BALL", (1.0, -1.0), (7, 9, 12), (-1.0, -1.2, -1.4), (1.0, 1.2, 1.4), (0, 0, 1)),
    ("ball4-perrow", "HOLONOMIC_BALL", (1.0, -1.0), (6, 5, 9, 10), (-1.0,) * 4, (1.0,) * 4, (0, 0, 1, 0)),
    ("ball4-perboth", "HOLONOMIC_BALL", (0.8, 1.0), (5, 7, 6, 8), (-1.0,) * 4, (1.0,) * 4, (0, 0, 1, 1)),
    ("box5-permarch", "HOLONOMIC_BOX", (1.0, 0.3, -1.0), (5, 6, 7, 6, 8), (-1.0,) * 5, (1.0,) * 5, (0, 0, 1, 0, 0)),
    ("ball6-tiny", "HOLONOMIC_BALL", (1.0, -1.0), (3, 4, 3, 5, 5, 4), (-1.0,) * 6, (1.0,) * 6, (0,) * 6),
    ("ball6-perside", "HOLONOMIC_BALL", (1.0, -1.0), (5, 6, 4, 7, 6, 8), (-1.0,) * 6, (1.0,) * 6, (1, 0, 1, 0, 0, 0)),
    ("dubins-c1like", "DUBINS3D", (1.0, 1.0, 1.0), (13, 11, 16), (-4.0, -4.0, -math.pi), (4.0, 4.0, math.pi), (0, 0, 1)),
    ("car5", "CAR5D", (1.0, 2.0, -1.0), (7, 6, 8, 9, 8), (-5.0, -5.0, -math.pi, 0.0, -2.0), (5.0, 5.0, math.pi, 3.0, 2.0),
     (0, 0, 1, 0, 0)),
    ("dint6", "DOUBLEINT6D", (1.0, 0.2, -1.0), (6, 5, 7, 6, 6, 8), (-4.0, -2.0) * 3, (4.0, 2.0) * 3, (0,) * 6),
]


def noise_v0(N, seed, amp=0.1):
    """A rough field: the extremes of D+- fall anywhere, faces included (pass-1 coverage)."""
    rng = np.random.default_rng(seed)
    base = np.zeros(N)
    for ax, n in enumerate(N):
        sh = [1] * len(N)
        sh[ax] = n
        base = base + 0.3 * np.cos(np.linspace(0.0, 2.5 + ax, n)).reshape(sh)
    return (base + amp * rng.uniform(-1.0, 1.0, N)).astype(np.float32)


@pytest.fixture(params=[None, "2", "4"], ids=["vec-auto", "vec2", "vec4"])
def march_env(request):
    old_v, old_k = os.environ.get("ODP_MARCH_VEC"), os.environ.get("ODP_MARCH_K")
    if request.param:
        os.environ["ODP_MARCH_VEC"] = request.param
    yield request.param
    for k, v in (("ODP_MARCH_VEC", old_v), ("ODP_MARCH_K", old_k)):
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("acc", ["low", "medium"])
@pytest.mark.parametrize("seg", [None, "2", "3"], ids=["whole", "K2", "K3"])
def test_march_paths(case, acc, seg, march_env):
    name, dyn, prm, N, lo, hi, per = case
    if march_env == "4" and N[-1] % 4:
        pytest.skip("VEC=4 needs N1 % 4 == 0")
    if march_env == "2" and N[-1] % 2:
        pytest.skip("VEC=2 needs an even N1")
    if seg:
        os.environ["ODP_MARCH_K"] = seg
    else:
        os.environ.pop("ODP_MARCH_K", None)
    w = Workload(name, N, lo, hi, per, dyn, prm, (0.0, 0.02, 0.05), acc, 0.8 if acc == "low" else 0.5, "brt",
                 ("random_smooth", len(N)))
    if not covers(w, "march"):
        pytest.skip("march family does not cover this grid")
    for seed in (0, 1):
        V0 = noise_v0(N, seed)
        out, info = run_gpu(w, V0, kernel="march")
        if acc == "low":
            ref = run_oracle(w, V0)
            assert_parity(out, ref.out, what=f"{name} {acc} seed={seed}")
        else:
            ref = run_oracle(w, V0, ambiguity=True)
            assert_parity_one_step(out, ref, R=2 * ref.stages, what=f"{name} {acc} seed={seed}")
        assert info["steps"] == ref.steps and info["stages"] == ref.stages
        assert abs(info["tau_reached"] - ref.tau_reached) < 1e-12


@pytest.mark.parametrize("acc", ["low", "medium"])
def test_march_matches_stream_bits_of_range(acc):
    # The derivative range of pass 1 is evaluated with the same float32 operations by both families,
    # so on a functor whose alpha depends on the range magnitudes (the ball) the step counts and dt
    # sequence coincide and the results agree to rounding of the Hamiltonian assembly.
    N = (8, 7, 9, 12)
    w = Workload("ball4", N, (-1.0,) * 4, (1.0,) * 4, (0, 0, 0, 0), "HOLONOMIC_BALL", (1.0, -1.0), (0.0, 0.03, 0.06),
                 acc, 0.8 if acc == "low" else 0.5, "brs", ("random_smooth", 4))
    V0 = noise_v0(N, 7)
    a, ia = run_gpu(w, V0, kernel="march")
    b, ib = run_gpu(w, V0, kernel="stream")
    assert ia["steps"] == ib["steps"] and ia["tau_reached"] == ib["tau_reached"]
    assert np.abs(a - b).max() <= 2e-6


@pytest.mark.parametrize("mode", ["brt", "brs"])
@pytest.mark.parametrize("N", [(6, 5, 7, 6, 6, 8), (3, 4, 3, 5, 48, 48), (5, 6, 74, 14)],
                         ids=["dint6-generic", "dint6-c5-instance", "car4-ragged-rows"])
def test_low_target_staging_is_bitwise(N, mode):
    # LOW pass 2 stages the target by TMA with the step's tiles (MarchArgs::xs); with
    # ODP_MARCH_XS=0 it reads it per thread one step ahead.  Same float32 operations: identical bits.
    # (3, 4, 3, 5, 48, 48) runs the shape-specialised c5 instance; 74 rows in blocks of 16 leave a
    # ragged last row block (10 rows: a shorter target copy).
    if len(N) == 6:
        w = Workload("dint6", N, (-4.0, -2.0) * 3, (4.0, 2.0) * 3, (0,) * 6, "DOUBLEINT6D", (1.0, 0.2, -1.0),
                     (0.0, 0.03, 0.06), "low", 0.8, mode, ("random_smooth", 6))
    else:
        w = Workload("car4", N, (-5.0, -5.0, 0.0, -math.pi), (5.0, 5.0, 4.0, math.pi), (0, 0, 0, 1), "CAR4D",
                     (1.5, 1.0, 0.25, 0.25, -1.0), (0.0, 0.05, 0.1), "low", 0.8, mode, ("random_smooth", 4))
    V0 = noise_v0(N, 3)
    old, old_b = os.environ.get("ODP_MARCH_XS"), os.environ.get("ODP_MARCH_B")
    try:
        if len(N) == 4:
            os.environ["ODP_MARCH_B"] = "16"
        os.environ.pop("ODP_MARCH_XS", None)
        a, ia = run_gpu(w, V0, kernel="march")
        os.environ["ODP_MARCH_XS"] = "0"
        b, ib = run_gpu(w, V0, kernel="march")
    finally:
        for k, v in (("ODP_MARCH_XS", old), ("ODP_MARCH_B", old_b)):
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    assert ia["steps"] == ib["steps"] and ia["stages"] == ib["stages"]
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
    ref = run_oracle(w, V0)
    assert_parity(a, ref.out, what=f"{w.name} {mode} staged target")
