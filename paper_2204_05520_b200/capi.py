"""Thin ctypes binding of include/odp.h (argument marshalling only; every step runs in libodp.so).

The product path never falls back to anything else: if libodp.so is missing, importing this
module raises.  Torch supplies device memory and streams only.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ODP_LIB_PATH") or os.path.join(HERE, "libodp.so")

ODP_OK, ODP_EINVAL, ODP_ENUMERIC, ODP_ECUDA, ODP_ENCCL, ODP_ENOMEM = 0, 1, 2, 3, 4, 5
ACCURACY = {"low": 1, "medium": 2}
MODE = {"brs": 0, "brt": 1}
KERNEL = {"auto": 0, "generic": 1, "tiled": 2, "stream": 3, "march": 4, "resident": 5}
DYNAMICS = {"HOLONOMIC_BALL": 0, "HOLONOMIC_BOX": 1, "DUBINS3D": 2, "CAR4D": 3, "CAR5D": 4, "DOUBLEINT6D": 5,
            "PAIR_DUBINS3D": 6}

# every symbol include/odp.h declares (checked by tests/test_capi_host.py)
EXPORTS = ("odp_grid_create", "odp_grid_destroy", "odp_grid_info", "odp_hj_solve", "odp_hj_solve_host",
           "odp_partition_extent", "odp_comm_unique_id", "odp_grid_partition", "odp_grid_local_extent",
           "odp_last_launch_count", "odp_last_error", "odp_version", "odp_ttr_solve", "odp_ttr_solve_host",
           "odp_vi_solve", "odp_vi_solve_host", "odp_loopback_create", "odp_grid_partition_loopback",
           "odp_loopback_destroy")
MDP_MODELS = {"HOLONOMIC": 0, "DUBINS3D": 1}


class odp_solve_opts(ctypes.Structure):
    _fields_ = [("cfl", ctypes.c_double),
                ("target", ctypes.c_void_p),
                ("stream", ctypes.c_void_p),
                ("write_initial", ctypes.c_int),
                ("kernel", ctypes.c_int),
                ("use_graph", ctypes.c_int),
                ("tau_reached", ctypes.POINTER(ctypes.c_double)),
                ("steps_taken", ctypes.POINTER(ctypes.c_longlong)),
                ("stages_taken", ctypes.POINTER(ctypes.c_longlong)),
                ("kernel_ms", ctypes.POINTER(ctypes.c_double)),
                ("single_pass", ctypes.c_int),
                ("single_pass_used", ctypes.POINTER(ctypes.c_int))]


class odp_ttr_opts(ctypes.Structure):
    _fields_ = [("eps", ctypes.c_double),
                ("max_iters", ctypes.c_longlong),
                ("big", ctypes.c_double),
                ("stream", ctypes.c_void_p),
                ("use_graph", ctypes.c_int),
                ("iters_taken", ctypes.POINTER(ctypes.c_longlong)),
                ("last_change", ctypes.POINTER(ctypes.c_double)),
                ("kernel_ms", ctypes.POINTER(ctypes.c_double))]


class odp_vi_opts(ctypes.Structure):
    _fields_ = [("threshold", ctypes.c_double),
                ("max_iters", ctypes.c_longlong),
                ("fixed_iters", ctypes.c_int),
                ("stream", ctypes.c_void_p),
                ("use_graph", ctypes.c_int),
                ("iters_taken", ctypes.POINTER(ctypes.c_longlong)),
                ("last_change", ctypes.POINTER(ctypes.c_double)),
                ("kernel_ms", ctypes.POINTER(ctypes.c_double))]


class OdpError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"odp status {status}: {msg}")
        self.status = status


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2204_05520_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    D = ctypes.POINTER(ctypes.c_double)
    I64 = ctypes.POINTER(ctypes.c_int64)
    vp = ctypes.c_void_p
    lib.odp_grid_create.argtypes = [ctypes.c_int, D, D, I64, ctypes.c_uint32, ctypes.POINTER(vp)]
    lib.odp_grid_create.restype = ctypes.c_int
    lib.odp_grid_destroy.argtypes = [vp]
    lib.odp_grid_destroy.restype = None
    lib.odp_grid_info.argtypes = [vp, ctypes.POINTER(ctypes.c_int), I64, D, I64]
    lib.odp_grid_info.restype = ctypes.c_int
    for name in ("odp_hj_solve", "odp_hj_solve_host"):
        f = getattr(lib, name)
        f.argtypes = [vp, ctypes.c_int, D, ctypes.c_int, vp, D, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp,
                      ctypes.POINTER(odp_solve_opts)]
        f.restype = ctypes.c_int
    for name in ("odp_ttr_solve", "odp_ttr_solve_host"):
        f = getattr(lib, name)
        f.argtypes = [vp, ctypes.c_int, D, ctypes.c_int, vp, vp, ctypes.POINTER(odp_ttr_opts)]
        f.restype = ctypes.c_int
    for name in ("odp_vi_solve", "odp_vi_solve_host"):
        f = getattr(lib, name)
        f.argtypes = [vp, ctypes.c_int, D, ctypes.c_int, vp, vp, ctypes.POINTER(odp_vi_opts)]
        f.restype = ctypes.c_int
    lib.odp_partition_extent.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.c_int, I64, I64]
    lib.odp_partition_extent.restype = ctypes.c_int
    lib.odp_comm_unique_id.argtypes = [vp]
    lib.odp_comm_unique_id.restype = ctypes.c_int
    lib.odp_grid_partition.argtypes = [vp, ctypes.c_int, ctypes.c_int, vp, ctypes.c_int]
    lib.odp_grid_partition.restype = ctypes.c_int
    lib.odp_loopback_create.argtypes = [ctypes.c_int, ctypes.POINTER(vp)]
    lib.odp_loopback_create.restype = ctypes.c_int
    lib.odp_grid_partition_loopback.argtypes = [vp, ctypes.c_int, vp]
    lib.odp_grid_partition_loopback.restype = ctypes.c_int
    lib.odp_loopback_destroy.argtypes = [vp]
    lib.odp_loopback_destroy.restype = None
    lib.odp_grid_local_extent.argtypes = [vp, I64, I64]
    lib.odp_grid_local_extent.restype = ctypes.c_int
    lib.odp_last_launch_count.argtypes = [vp]
    lib.odp_last_launch_count.restype = ctypes.c_longlong
    lib.odp_last_error.argtypes = []
    lib.odp_last_error.restype = ctypes.c_char_p
    lib.odp_version.argtypes = []
    lib.odp_version.restype = ctypes.c_char_p
    return lib


_lib = _load()


def lib():
    return _lib


def last_error() -> str:
    return _lib.odp_last_error().decode()


def version() -> str:
    return _lib.odp_version().decode()


def _check(status: int):
    if status != ODP_OK:
        raise OdpError(status, last_error())


def _dp(a):
    a = np.ascontiguousarray(a, dtype=np.float64)
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def partition_extent(N0: int, nranks: int, rank: int):
    """odp_partition_extent: (first axis-0 plane, plane count) of `rank`'s slab."""
    b, c = ctypes.c_int64(), ctypes.c_int64()
    _check(_lib.odp_partition_extent(int(N0), int(nranks), int(rank), ctypes.byref(b), ctypes.byref(c)))
    return b.value, c.value


def comm_unique_id() -> bytes:
    """odp_comm_unique_id: a 128-byte NCCL unique id (rank 0; broadcast it to the other ranks)."""
    buf = ctypes.create_string_buffer(128)
    _check(_lib.odp_comm_unique_id(ctypes.cast(buf, ctypes.c_void_p)))
    return buf.raw


class Grid:
    """odp_grid_create / odp_grid_destroy."""

    def __init__(self, N: Sequence[int], lo: Sequence[float], hi: Sequence[float], periodic_mask: int = 0):
        self.N = tuple(int(v) for v in N)
        Na = np.ascontiguousarray(self.N, dtype=np.int64)
        loa, lop = _dp(lo)
        hia, hip = _dp(hi)
        h = ctypes.c_void_p()
        _check(_lib.odp_grid_create(len(self.N), lop, hip, Na.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                    ctypes.c_uint32(periodic_mask), ctypes.byref(h)))
        self.handle = h
        self.local_N = self.N

    @property
    def points(self) -> int:
        return int(np.prod(self.local_N, dtype=np.int64))

    def info(self):
        dims = ctypes.c_int()
        N = np.zeros(6, dtype=np.int64)
        dx = np.zeros(6)
        P = ctypes.c_int64()
        _check(_lib.odp_grid_info(self.handle, ctypes.byref(dims), N.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                  dx.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), ctypes.byref(P)))
        n = dims.value
        return dict(dims=n, N=tuple(N[:n]), dx=tuple(dx[:n]), points=P.value)

    def partition(self, rank: int, nranks: int, uid: Optional[bytes], device: int):
        """odp_grid_partition: this handle becomes rank `rank`'s axis-0 slab (collective over ranks)."""
        buf = ctypes.create_string_buffer(uid, 128) if uid is not None else None
        _check(_lib.odp_grid_partition(self.handle, int(rank), int(nranks),
                                       ctypes.cast(buf, ctypes.c_void_p) if buf is not None else None, int(device)))
        b, c = self.local_extent()
        self.local_N = (c,) + self.N[1:]

    def partition_loopback(self, rank: int, lb: "Loopback"):
        """odp_grid_partition_loopback: rank `rank`'s slab on a one-GPU loopback transport (tests)."""
        _check(_lib.odp_grid_partition_loopback(self.handle, int(rank), lb.handle))
        b, c = self.local_extent()
        self.local_N = (c,) + self.N[1:]

    def local_extent(self):
        b, c = ctypes.c_int64(), ctypes.c_int64()
        _check(_lib.odp_grid_local_extent(self.handle, ctypes.byref(b), ctypes.byref(c)))
        return b.value, c.value

    def launch_count(self) -> int:
        return int(_lib.odp_last_launch_count(self.handle))

    def close(self):
        if getattr(self, "handle", None):
            _lib.odp_grid_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Loopback:
    """odp_loopback_create / odp_loopback_destroy: the one-GPU test transport of nranks slab handles."""

    def __init__(self, nranks: int):
        h = ctypes.c_void_p()
        _check(_lib.odp_loopback_create(int(nranks), ctypes.byref(h)))
        self.handle = h
        self.nranks = int(nranks)

    def close(self):
        if getattr(self, "handle", None):
            _lib.odp_loopback_destroy(self.handle)
            self.handle = None


class SolveInfo(dict):
    pass


def _opts(cfl, target_ptr, stream_ptr, write_initial, kernel, timing, single_pass=False):
    o = odp_solve_opts()
    o.cfl = float(cfl or 0.0)
    o.target = target_ptr
    o.stream = stream_ptr
    o.write_initial = int(bool(write_initial))
    o.kernel = KERNEL[kernel]
    o.use_graph = 0
    tr = ctypes.c_double()
    st = ctypes.c_longlong()
    sg = ctypes.c_longlong()
    km = (ctypes.c_double * 4)()
    o.tau_reached = ctypes.pointer(tr)
    o.steps_taken = ctypes.pointer(st)
    o.stages_taken = ctypes.pointer(sg)
    o.kernel_ms = ctypes.cast(km, ctypes.POINTER(ctypes.c_double)) if timing else None
    o.single_pass = int(bool(single_pass))
    spu = ctypes.c_int()
    o.single_pass_used = ctypes.pointer(spu)
    return o, (tr, st, sg, km, spu)


def _info(keep, timing, status):
    tr, st, sg, km, spu = keep
    info = SolveInfo(tau_reached=tr.value, steps=st.value, stages=sg.value, status=status,
                     single_pass=bool(spu.value))
    if timing:
        info["kernel_ms"] = dict(pass1=km[0], pass2=km[1], control=km[2], pass2_rk2=km[3])
    return info


def hj_solve(grid: Grid, dynamics: str, params, V0, tau, accuracy: str, mode: str, out=None, cfl: float = 0.0,
             target=None, write_initial: bool = False, kernel: str = "auto", stream=None, timing: bool = False,
             raise_on_error: bool = True, single_pass: bool = False):
    """odp_hj_solve on torch CUDA tensors (device pointers).  Returns (out, info)."""
    import torch
    assert V0.is_cuda and V0.dtype == torch.float32 and V0.is_contiguous()
    ntau = len(tau)
    nout = ntau if write_initial else ntau - 1
    if out is None:
        out = torch.empty((nout,) + tuple(grid.local_N), dtype=torch.float32, device=V0.device)
    assert out.is_cuda and out.dtype == torch.float32 and out.is_contiguous() and out.numel() == nout * grid.points
    if target is not None:
        assert target.is_cuda and target.dtype == torch.float32 and target.is_contiguous()
    if stream is None:
        stream = torch.cuda.current_stream(V0.device)
    pa, pp = _dp(params)
    ta, tp = _dp(tau)
    o, keep = _opts(cfl, target.data_ptr() if target is not None else None, stream.cuda_stream, write_initial,
                    kernel, timing, single_pass)
    status = _lib.odp_hj_solve(grid.handle, DYNAMICS[dynamics], pp, len(pa), V0.data_ptr(), tp, len(ta),
                               ACCURACY[accuracy], MODE[mode], out.data_ptr(), ctypes.byref(o))
    if status != ODP_OK and raise_on_error:
        raise OdpError(status, last_error())
    return out, _info(keep, timing, status)


def hj_solve_host(grid: Grid, dynamics: str, params, V0: np.ndarray, tau, accuracy: str, mode: str, out=None,
                  cfl: float = 0.0, target=None, write_initial: bool = False, kernel: str = "auto", stream=None,
                  timing: bool = False, raise_on_error: bool = True, single_pass: bool = False):
    """odp_hj_solve_host: V0/out/target are host arrays (numpy or pinned torch CPU tensors)."""
    def host_ptr(a):
        if hasattr(a, "data_ptr"):
            return a.data_ptr()
        assert a.dtype == np.float32 and a.flags["C_CONTIGUOUS"]
        return a.ctypes.data
    ntau = len(tau)
    nout = ntau if write_initial else ntau - 1
    if out is None:
        out = np.empty((nout,) + tuple(grid.local_N), dtype=np.float32)
    pa, pp = _dp(params)
    ta, tp = _dp(tau)
    o, keep = _opts(cfl, host_ptr(target) if target is not None else None,
                    stream.cuda_stream if stream is not None else None, write_initial, kernel, timing, single_pass)
    status = _lib.odp_hj_solve_host(grid.handle, DYNAMICS[dynamics], pp, len(pa), host_ptr(V0), tp, len(ta),
                                    ACCURACY[accuracy], MODE[mode], host_ptr(out), ctypes.byref(o))
    if status != ODP_OK and raise_on_error:
        raise OdpError(status, last_error())
    return out, _info(keep, timing, status)


def _ttr_opts(eps, max_iters, big, stream_ptr, use_graph):
    o = odp_ttr_opts()
    o.eps = float(eps)
    o.max_iters = int(max_iters)
    o.big = float(big)
    o.stream = stream_ptr
    o.use_graph = int(bool(use_graph))
    it, ch, km = ctypes.c_longlong(), ctypes.c_double(), (ctypes.c_double * 3)()
    o.iters_taken = ctypes.pointer(it)
    o.last_change = ctypes.pointer(ch)
    o.kernel_ms = ctypes.cast(km, ctypes.POINTER(ctypes.c_double))
    return o, (it, ch, km)


def _ttr_info(it, ch, km):
    return dict(iters=it.value, last_change=ch.value, kernel_ms=km[0],
                interior_ms=km[1] if km[1] >= 0 else None, faces_ms=km[2] if km[2] >= 0 else None)


def ttr_solve(grid: Grid, dynamics: str, params, V0, phi=None, eps: float = 1e-6, max_iters: int = 100000,
              big: float = 100.0, stream=None, use_graph: bool = True):
    """odp_ttr_solve (Algorithm 3) on torch CUDA tensors.  Returns (phi, info) with
    info = {iters, last_change, kernel_ms}."""
    import torch
    assert V0.is_cuda and V0.dtype == torch.float32 and V0.is_contiguous() and V0.numel() == grid.points
    if phi is None:
        phi = torch.empty(tuple(grid.local_N), dtype=torch.float32, device=V0.device)
    assert phi.is_cuda and phi.dtype == torch.float32 and phi.is_contiguous() and phi.numel() == grid.points
    if stream is None:
        stream = torch.cuda.current_stream(V0.device)
    pa, pp = _dp(params)
    o, (it, ch, km) = _ttr_opts(eps, max_iters, big, stream.cuda_stream, use_graph)
    _check(_lib.odp_ttr_solve(grid.handle, DYNAMICS[dynamics], pp, len(pa), V0.data_ptr(), phi.data_ptr(),
                              ctypes.byref(o)))
    return phi, _ttr_info(it, ch, km)


def ttr_solve_host(grid: Grid, dynamics: str, params, V0: np.ndarray, phi=None, eps: float = 1e-6,
                   max_iters: int = 100000, big: float = 100.0, use_graph: bool = True):
    """odp_ttr_solve_host: V0 / phi are host float32 arrays (copies inside the call)."""
    V0 = np.ascontiguousarray(V0, dtype=np.float32)
    assert V0.size == grid.points
    if phi is None:
        phi = np.empty(tuple(grid.local_N), dtype=np.float32)
    assert phi.dtype == np.float32 and phi.flags["C_CONTIGUOUS"] and phi.size == grid.points
    pa, pp = _dp(params)
    o, (it, ch, km) = _ttr_opts(eps, max_iters, big, None, use_graph)
    _check(_lib.odp_ttr_solve_host(grid.handle, DYNAMICS[dynamics], pp, len(pa), V0.ctypes.data, phi.ctypes.data,
                                   ctypes.byref(o)))
    return phi, _ttr_info(it, ch, km)


def _vi_opts(threshold, max_iters, fixed_iters, stream_ptr, use_graph):
    o = odp_vi_opts()
    o.threshold = float(threshold)
    o.max_iters = int(max_iters)
    o.fixed_iters = int(bool(fixed_iters))
    o.stream = stream_ptr
    o.use_graph = int(bool(use_graph))
    it, ch, km = ctypes.c_longlong(), ctypes.c_double(), (ctypes.c_double * 2)()
    o.iters_taken = ctypes.pointer(it)
    o.last_change = ctypes.pointer(ch)
    o.kernel_ms = ctypes.cast(km, ctypes.POINTER(ctypes.c_double))
    return o, (it, ch, km)


def _vi_info(it, ch, km):
    return dict(iters=it.value, last_change=ch.value, kernel_ms=km[0], iter_ms=km[1] if km[1] >= 0 else None)


def vi_solve(grid: Grid, model: str, params, R, V=None, threshold: float = 1e-6, max_iters: int = 100000,
             fixed_iters: bool = False, stream=None, use_graph: bool = True):
    """odp_vi_solve (Algorithm 1) on torch CUDA tensors.  Returns (V, info)."""
    import torch
    assert R.is_cuda and R.dtype == torch.float32 and R.is_contiguous() and R.numel() == grid.points
    if V is None:
        V = torch.empty(tuple(grid.local_N), dtype=torch.float32, device=R.device)
    assert V.is_cuda and V.dtype == torch.float32 and V.is_contiguous() and V.numel() == grid.points
    if stream is None:
        stream = torch.cuda.current_stream(R.device)
    pa, pp = _dp(params)
    o, keep = _vi_opts(threshold, max_iters, fixed_iters, stream.cuda_stream, use_graph)
    _check(_lib.odp_vi_solve(grid.handle, MDP_MODELS[model], pp, len(pa), R.data_ptr(), V.data_ptr(), ctypes.byref(o)))
    return V, _vi_info(*keep)


def vi_solve_host(grid: Grid, model: str, params, R: np.ndarray, V=None, threshold: float = 1e-6,
                  max_iters: int = 100000, fixed_iters: bool = False, use_graph: bool = True):
    """odp_vi_solve_host: R / V are host float32 arrays (copies inside the call)."""
    R = np.ascontiguousarray(R, dtype=np.float32)
    assert R.size == grid.points
    if V is None:
        V = np.empty(tuple(grid.local_N), dtype=np.float32)
    assert V.dtype == np.float32 and V.flags["C_CONTIGUOUS"] and V.size == grid.points
    pa, pp = _dp(params)
    o, keep = _vi_opts(threshold, max_iters, fixed_iters, None, use_graph)
    _check(_lib.odp_vi_solve_host(grid.handle, MDP_MODELS[model], pp, len(pa), R.ctypes.data, V.ctypes.data,
                                  ctypes.byref(o)))
    return V, _vi_info(*keep)
