"""Seeded, synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no derivatives, Hamiltonians,
dissipation, time stepping).  It only states the five BASELINE.json workloads
 as plain data and builds their initial value function
V0 on the grid nodes, in float64, rounded once to float32 (reading A18: both
sides start from bit-identical float32 values).

Node positions follow the problem statement of PAPER.md §3.4.1 ("number
of grid nodes, upper bound, and lower bound for each dimension, and periodic
dimension"), with the periodic upper endpoint excluded (reading A15).  The
target shapes are the signed-distance cylinders/spheres of PAPER.md §3.4.2
(P:239-240).

Dynamics are named by string; the oracle (oracle/) and the C-ABI binding
(paper_2204_05520_b200/) each map the name to their own identifier.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace
from typing import Optional, Sequence, Tuple

import numpy as np

PI = math.pi


@dataclass(frozen=True)
class Workload:
    name: str
    N: Tuple[int, ...]
    lo: Tuple[float, ...]
    hi: Tuple[float, ...]
    periodic: Tuple[int, ...]
    dynamics: str            # HOLONOMIC_BALL | HOLONOMIC_BOX | DUBINS3D | CAR4D | CAR5D | DOUBLEINT6D
    params: Tuple[float, ...]
    tau: Tuple[float, ...]
    accuracy: str            # "low" (upwind1 + Euler) | "medium" (ENO2 + TVD-RK2)
    cfl: float
    mode: str                # "brt" | "brs"
    target: Tuple            # ("cylinder"|"sphere", axes, radius) | ("plane", axis, sign, offset) | ("cos", axis)
    note: str = ""

    @property
    def dims(self) -> int:
        return len(self.N)

    @property
    def points(self) -> int:
        return int(np.prod(self.N, dtype=np.int64))

    @property
    def periodic_mask(self) -> int:
        m = 0
        for d, p in enumerate(self.periodic):
            if p:
                m |= 1 << d
        return m


def _uniform_tau(T: float, k: int) -> Tuple[float, ...]:
    return tuple(T * i / k for i in range(k + 1))


# --- The five BASELINE.json configs; params layouts follow SURVEY.md table C-2:
#     DUBINS3D [v, wbar, goal]; CAR4D [abar, wbar, dxbar, dybar, goal]; CAR5D [abar, alphabar, goal];
#     DOUBLEINT6D [ubar, dbar, goal]; goal = -1 minimise (reach), +1 maximise (avoid).
C1 = Workload(
    name="c1", N=(41, 41, 36), lo=(-4.0, -4.0, -PI), hi=(4.0, 4.0, PI), periodic=(0, 0, 1),
    dynamics="DUBINS3D", params=(1.0, 1.0, +1.0), tau=tuple(round(0.1 * k, 12) for k in range(21)),
    accuracy="low", cfl=0.8, mode="brt", target=("cylinder", (0, 1), 1.0),
    note="3D Dubins car, avoid, BRT over [0,2], 20 saves (reading A17)")
C2 = Workload(
    name="c2", N=(60, 60, 60, 60), lo=(-5.0, -5.0, 0.0, -PI), hi=(5.0, 5.0, 4.0, PI), periodic=(0, 0, 0, 1),
    dynamics="CAR4D", params=(1.5, 1.0, 0.25, 0.25, -1.0), tau=(0.0, 4.0),
    accuracy="low", cfl=0.8, mode="brt", target=("cylinder", (0, 1), 1.0),
    note="4D car with acceleration, reach with disturbance")
C3 = Workload(
    name="c3", N=(40, 40, 40, 40, 40), lo=(-5.0, -5.0, -PI, 0.0, -2.0), hi=(5.0, 5.0, PI, 3.0, 2.0),
    periodic=(0, 0, 1, 0, 0), dynamics="CAR5D", params=(1.0, 2.0, -1.0), tau=(0.0, 3.0),
    accuracy="medium", cfl=0.5, mode="brt", target=("cylinder", (0, 1), 1.5),
    note="5D car, reach (reading A16), ENO2 + TVD-RK2 at CFL 0.5 (reading A7)")
C4 = Workload(
    name="c4", N=(30,) * 6, lo=(-4.0, -2.0, -4.0, -2.0, -4.0, -2.0), hi=(4.0, 2.0, 4.0, 2.0, 4.0, 2.0),
    periodic=(0,) * 6, dynamics="DOUBLEINT6D", params=(1.0, 0.2, -1.0), tau=(0.0, 1.0),
    accuracy="medium", cfl=0.5, mode="brt", target=("sphere", (0, 2, 4), 1.0),
    note="6D double integrator, 7.29e8 points, ENO2 + TVD-RK2 at CFL 0.5")
C5_LOW = Workload(
    name="c5-low", N=(64, 48, 48, 48, 48, 48), lo=C4.lo, hi=C4.hi, periodic=(0,) * 6,
    dynamics="DOUBLEINT6D", params=(1.0, 0.2, -1.0), tau=(0.0, 0.5),
    accuracy="low", cfl=0.8, mode="brt", target=("sphere", (0, 2, 4), 1.0),
    note="6D at scale (65 GB per array): 2/4/8 GPUs only")
C5_MED = replace(C5_LOW, name="c5-med", accuracy="medium", cfl=0.5)
# the paper's own 3D example, Eq. 7, at Table 1's 3D shape 100^3.
# The paper gives neither speeds, input bounds, domain nor target; reading A30 takes the classic
# pursuit-evasion setting of that system: va = vb = 5, |a|, |b| <= 1, capture radius 5,
# x in [-6, 20], y in [-10, 10], th in [-pi, pi) periodic, horizon 2.8; the evader (a) avoids
# (goal +1, maximise), the pursuer (b) does the opposite.  First order (Table 1's "1st order ENO").
F2 = Workload(
    name="f2", N=(100, 100, 100), lo=(-6.0, -10.0, -PI), hi=(20.0, 10.0, PI), periodic=(0, 0, 1),
    dynamics="PAIR_DUBINS3D", params=(5.0, 5.0, 1.0, 1.0, +1.0), tau=(0.0, 2.8),
    accuracy="low", cfl=0.8, mode="brt", target=("cylinder", (0, 1), 5.0),
    note="Eq. 7 pairwise Dubins capture (reading A30), 100^3, upwind + Euler")

CONFIGS = {w.name: w for w in (C1, C2, C3, C4, C5_LOW, C5_MED, F2)}


# time-to-reach (Algorithm 3) workloads.  The paper benchmarks no TTR
# problem, so the bench case is the classic Dubins-car TTR to a disc (reading A35): v = 1, |w| <= 1,
# x, y in [-5, 5], th in [-pi, pi) periodic, target disc of radius 1 at the origin, 256^3 nodes
# (3 float32 arrays = 200 MB, above L2).  tau / accuracy / cfl / mode are unused by the TTR path.
T1 = Workload(
    name="t1", N=(256, 256, 256), lo=(-5.0, -5.0, -PI), hi=(5.0, 5.0, PI), periodic=(0, 0, 1),
    dynamics="DUBINS3D", params=(1.0, 1.0, -1.0), tau=(0.0, 1.0), accuracy="low", cfl=0.8, mode="brt",
    target=("cylinder", (0, 1), 1.0), note="Dubins-car time-to-reach a unit disc, 256^3")
TTR_CONFIGS = {T1.name: T1}


# value iteration (Algorithm 1) workloads.  Table 3 times
# value iteration on 3D grids 25x25x9, 40x40x20, 50x50x30 without stating the MDP; reading A36's
# Dubins-car MDP stands in: x, y in [-5, 5], th in [-pi, pi) periodic, v in {0.5, 1}, |w| <= 1,
# dt = 0.25, lateral slip 0.1 with probability 0.1 each side, gamma = 0.95; reward +1 on a goal disc
# (centre (3, 2), radius 1), -1 on an obstacle disc (centre (-1, 0), radius 1.5), 0 elsewhere.
@dataclass(frozen=True)
class MdpWorkload:
    name: str
    N: Tuple[int, ...]
    lo: Tuple[float, ...]
    hi: Tuple[float, ...]
    periodic: Tuple[int, ...]
    model: str
    params: Tuple[float, ...]
    goal: Tuple[float, float, float]
    obstacle: Tuple[float, float, float]
    note: str = ""

    @property
    def points(self) -> int:
        return int(np.prod(self.N, dtype=np.int64))

    @property
    def periodic_mask(self) -> int:
        return sum(1 << d for d, p in enumerate(self.periodic) if p)


def _vi(name, N, note=""):
    return MdpWorkload(name=name, N=N, lo=(-5.0, -5.0, -PI), hi=(5.0, 5.0, PI), periodic=(0, 0, 1),
                       model="DUBINS3D", params=(1.0, 1.0, 0.25, 0.1, 0.1, 0.95), goal=(3.0, 2.0, 1.0),
                       obstacle=(-1.0, 0.0, 1.5), note=note)


VI_CONFIGS = {w.name: w for w in (
    _vi("v0", (25, 25, 9), "Table 3 smallest shape"),
    _vi("v1", (50, 50, 30), "Table 3 largest shape"),
    _vi("v2", (384, 384, 128), "the same MDP at 1.9e7 nodes (3 float32 arrays = 226 MB, above L2)"),
)}


def make_reward(w: MdpWorkload, seed: Optional[int] = None, noise: float = 1e-3) -> np.ndarray:
    """Reward per node (float32): +1 on the goal disc, -1 on the obstacle disc (x, y only), 0 else;
    seed adds noise * U(-1, 1)."""
    ax = [axis_nodes(n, l, h, bool(p)) for n, l, h, p in zip(w.N, w.lo, w.hi, w.periodic)]
    X, Y = np.meshgrid(ax[0], ax[1], indexing="ij")
    R2 = np.zeros(X.shape)
    gx, gy, gr = w.goal
    ox, oy, orad = w.obstacle
    R2[(X - gx) ** 2 + (Y - gy) ** 2 <= gr ** 2] = 1.0
    R2[(X - ox) ** 2 + (Y - oy) ** 2 <= orad ** 2] = -1.0
    R = np.broadcast_to(R2[..., None], w.N).astype(np.float64)
    if seed is not None:
        R = R + noise * np.random.default_rng(seed).uniform(-1.0, 1.0, w.N)
    return np.ascontiguousarray(R.astype(np.float32))


def axis_nodes(N: int, lo: float, hi: float, periodic: bool) -> np.ndarray:
    """Node positions of one axis (problem statement; reading A15)."""
    h = (hi - lo) / (N if periodic else (N - 1))
    return lo + h * np.arange(N, dtype=np.float64)


def sub_box(w: Workload, axis0_range: Tuple[int, int], name: Optional[str] = None) -> Workload:
    """The planes [a, b) of axis 0 of `w` as their own grid with identical spacing (c5-slab, reading A27)."""
    a, b = axis0_range
    assert not w.periodic[0]
    x0 = axis_nodes(w.N[0], w.lo[0], w.hi[0], False)
    N = (b - a,) + tuple(w.N[1:])
    lo = (float(x0[a]),) + tuple(w.lo[1:])
    hi = (float(x0[b - 1]),) + tuple(w.hi[1:])
    return replace(w, name=name or f"{w.name}[{a}:{b}]", N=N, lo=lo, hi=hi)


C5_SLAB_LOW = sub_box(C5_LOW, (28, 36), name="c5slab-low")
C5_SLAB_MED = sub_box(C5_MED, (28, 36), name="c5slab-med")
CONFIGS[C5_SLAB_LOW.name] = C5_SLAB_LOW
CONFIGS[C5_SLAB_MED.name] = C5_SLAB_MED


def coarsened(w: Workload, N: Sequence[int], name: Optional[str] = None, tau=None) -> Workload:
    """Same dynamics, bounds and target on a different node count (test-sized copies)."""
    return replace(w, name=name or f"{w.name}@{'x'.join(map(str, N))}", N=tuple(int(n) for n in N),
                   tau=tuple(tau) if tau is not None else w.tau)


def make_v0(w: Workload, seed: Optional[int] = None, noise: float = 1e-3, i0=None, box=None) -> np.ndarray:
    """Initial value V0 = target signed distance on the nodes, float64 -> float32 (reading A18).

    seed=None gives the plain workload; an integer seed adds noise*U(-1,1) from
    numpy.random.default_rng(seed) (the seeded parity variants of SURVEY.md §8(d)).
    i0 = (begin, count) returns only the axis-0 slab [begin, begin + count) -- bitwise the same
    values as slicing the whole array (a multi-GPU rank builds just its own slab).
    box = [(begin, count) per axis] returns the sub-box -- bitwise the same values as slicing the
    whole array (the windowed checks of pin Z12 build only the boxes they need; unseeded only).
    """
    if seed is None and box is None:
        # large requests (a c5 rank slab is up to 8e9 points): build the float32 result an axis-0
        # plane at a time, so the float64 intermediate stays one plane (bitwise the same values)
        b0, c0 = (0, w.N[0]) if i0 is None else (int(i0[0]), int(i0[1]))
        plane = int(np.prod(w.N[1:], dtype=np.int64))
        if c0 * plane > (1 << 26) and c0 > 1:
            out = np.empty((c0,) + tuple(w.N[1:]), dtype=np.float32)
            for k in range(c0):
                out[k] = make_v0(w, box=[(b0 + k, 1)] + [(0, n) for n in w.N[1:]])[0]
            return out
    axes = [axis_nodes(n, l, h, bool(p)) for n, l, h, p in zip(w.N, w.lo, w.hi, w.periodic)]
    kind = w.target[0]
    shape = w.N
    if i0 is not None:
        b, c = int(i0[0]), int(i0[1])
        axes[0] = axes[0][b:b + c]
        shape = (c,) + tuple(w.N[1:])
    if box is not None:
        assert i0 is None and seed is None
        axes = [ax[int(b):int(b) + int(c)] for ax, (b, c) in zip(axes, box)]
        shape = tuple(int(c) for _, c in box)
    if kind in ("cylinder", "sphere"):
        _, taxes, radius = w.target
        acc = np.zeros((1,) * len(shape), dtype=np.float64)
        for a in taxes:
            s = [1] * len(shape)
            s[a] = shape[a]
            acc = acc + axes[a].reshape(s) ** 2
        v = np.sqrt(acc) - radius
    elif kind == "plane":           # signed distance to {x_axis = offset} times sign
        _, a, sign, offset = w.target
        s = [1] * len(shape)
        s[a] = shape[a]
        v = sign * (axes[a].reshape(s) - offset)
    elif kind == "cos":
        _, a = w.target
        s = [1] * len(shape)
        s[a] = shape[a]
        v = np.cos(axes[a].reshape(s))
    elif kind == "norm_ball":      # |x| - r over all axes (holonomic closed forms)
        radius = w.target[1]
        acc = np.zeros((1,) * len(shape), dtype=np.float64)
        for a in range(len(shape)):
            s = [1] * len(shape)
            s[a] = shape[a]
            acc = acc + axes[a].reshape(s) ** 2
        v = np.sqrt(acc) - radius
    elif kind == "random_smooth":  # sum of random low-frequency cosines (brute-force tiny grids)
        _, rseed = w.target
        rng = np.random.default_rng(rseed)
        v = np.zeros((1,) * len(shape), dtype=np.float64)
        for a in range(len(shape)):
            s = [1] * len(shape)
            s[a] = shape[a]
            c = rng.uniform(0.3, 1.2)
            ph = rng.uniform(-PI, PI)
            v = v + rng.uniform(-1, 1) * np.cos(c * axes[a] + ph).reshape(s)
        v = v + rng.uniform(-0.5, 0.5)
    else:
        raise ValueError(f"unknown target {kind}")
    v = np.broadcast_to(v, shape).astype(np.float64)
    if seed is not None:
        rng = np.random.default_rng(seed)
        nz = rng.uniform(-1.0, 1.0, size=w.N)
        if i0 is not None:
            nz = nz[int(i0[0]):int(i0[0]) + int(i0[1])]
        v = v + noise * nz
    return np.ascontiguousarray(v.astype(np.float32))


def holonomic(n: int, N: int, half: float, dyn: str, params, tau, accuracy: str, mode: str = "brt",
              target=("norm_ball", 0.5), cfl: Optional[float] = None, name: str = "holo") -> Workload:
    """Holonomic test problems on [-half, half]^n (closed forms Z1/Z2/Z5)."""
    return Workload(name=name, N=(N,) * n, lo=(-half,) * n, hi=(half,) * n, periodic=(0,) * n,
                    dynamics=dyn, params=tuple(params), tau=tuple(tau), accuracy=accuracy,
                    cfl=(0.8 if accuracy == "low" else 0.5) if cfl is None else cfl, mode=mode,
                    target=target)
