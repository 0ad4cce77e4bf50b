"""Host-side checks of the C-ABI (no GPU): the library loads, exports every symbol of
include/odp.h, and validates arguments before any device work."""
import ctypes
import re
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def capi():
    from paper_2204_05520_b200 import build
    build.build()
    from paper_2204_05520_b200 import capi as c
    return c


def test_header_symbols_exported(capi):
    hdr = open(os.path.join(ROOT, "include", "odp.h")).read()
    declared = set(re.findall(r"\b(odp_[a-z_0-9]+)\s*\(", hdr))
    assert declared == set(capi.EXPORTS), declared ^ set(capi.EXPORTS)
    lib = ctypes.CDLL(capi.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name


def test_version(capi):
    assert "sm_100a" in capi.version()


def test_grid_create_and_info(capi):
    g = capi.Grid((41, 41, 36), (-4, -4, -np.pi), (4, 4, np.pi), 0b100)
    info = g.info()
    assert info["dims"] == 3 and info["N"] == (41, 41, 36) and info["points"] == 41 * 41 * 36
    np.testing.assert_allclose(info["dx"], (0.2, 0.2, 2 * np.pi / 36), rtol=1e-15)
    g.close()


@pytest.mark.parametrize("N,lo,hi", [((3,) * 7, (0,) * 7, (1,) * 7), ((2, 5), (0, 0), (1, 1)), ((5, 5), (0, 1), (1, 1))])
def test_grid_errors(capi, N, lo, hi):
    with pytest.raises(capi.OdpError) as e:
        capi.Grid(N, lo, hi, 0)
    assert e.value.status == capi.ODP_EINVAL and capi.last_error()


@pytest.mark.parametrize("kw,msg", [
    (dict(dynamics="DUBINS3D", params=(1, 1, 1)), "needs dims"),
    (dict(params=(1.0, 0.2)), "params"),
    (dict(params=(1.0, 0.2, 0.5)), "goal"),
    (dict(tau=(0.1, 1.0)), "tau[0]"),
    (dict(tau=(0.0, 1.0, 1.0)), "strictly"),
    (dict(tau=(0.0,)), "ntau"),
    (dict(accuracy=3), "accuracy"),
    (dict(mode=7), "mode"),
])
def test_solve_validation_before_device_work(capi, kw, msg):
    g = capi.Grid((5, 5), (-1, -1), (1, 1), 0)
    a = dict(dynamics="HOLONOMIC_BOX", params=(1.0, 0.2, -1.0), tau=(0.0, 0.5), accuracy=1, mode=1)
    a.update(kw)
    pa = np.ascontiguousarray(a["params"], dtype=np.float64)
    ta = np.ascontiguousarray(a["tau"], dtype=np.float64)
    D = ctypes.POINTER(ctypes.c_double)
    st = capi.lib().odp_hj_solve(g.handle, capi.DYNAMICS[a["dynamics"]], pa.ctypes.data_as(D), len(pa),
                                 ctypes.c_void_p(16), ta.ctypes.data_as(D), len(ta), a["accuracy"], a["mode"],
                                 ctypes.c_void_p(32), None)
    assert st == capi.ODP_EINVAL
    assert msg in capi.last_error()
    g.close()


def test_unknown_dynamics(capi):
    g = capi.Grid((5, 5), (-1, -1), (1, 1), 0)
    p = np.zeros(3)
    t = np.array([0.0, 1.0])
    D = ctypes.POINTER(ctypes.c_double)
    st = capi.lib().odp_hj_solve(g.handle, 9, p.ctypes.data_as(D), 3, ctypes.c_void_p(16), t.ctypes.data_as(D), 2,
                                 1, 1, ctypes.c_void_p(32), None)
    assert st == capi.ODP_EINVAL and "unknown dynamics" in capi.last_error()
    g.close()


@pytest.mark.parametrize("N,per,kw,msg", [
    ((5, 5), 0, dict(dynamics="DUBINS3D", params=(1, 1, -1)), "needs dims"),
    ((5, 5), 0, dict(params=(1.0, 0.2)), "params"),
    ((5, 5), 0, dict(params=(1.0, 0.2, 0.0)), "goal"),
    ((5, 3), 0, {}, "N[1]=3 < 4"),
    ((5, 5), 0, dict(alias=True), "aliases"),
])
def test_ttr_validation_before_device_work(capi, N, per, kw, msg):
    g = capi.Grid(N, (-1, -1), (1, 1), per)
    a = dict(dynamics="HOLONOMIC_BOX", params=(1.0, 0.2, -1.0))
    a.update(kw)
    pa = np.ascontiguousarray(a["params"], dtype=np.float64)
    out = ctypes.c_void_p(16 if a.get("alias") else 32)
    st = capi.lib().odp_ttr_solve(g.handle, capi.DYNAMICS[a["dynamics"]], pa.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                  len(pa), ctypes.c_void_p(16), out, None)
    assert st == capi.ODP_EINVAL
    assert msg in capi.last_error()
    g.close()
