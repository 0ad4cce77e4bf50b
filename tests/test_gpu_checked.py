"""The march, generic, time-to-reach and value-iteration kernels under device-side bounds checks
(libodp_check.so, built with -DODP_CHECK): every shared-memory read of the march kernels, every TMA
bulk copy (source range in the halo-padded buffer, 16-B alignment, destination inside the dynamic
shared memory) and the global window / Vn / target / output accesses, and the time-to-reach tile
loader's sources, are checked; a failed check prints its code and traps.  compute-sanitizer is
closed on this pool (its runs left GPUs needing a reset), so this is the memcheck substitute.  The
checks change no arithmetic: the printed results must equal the production library's exactly."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(lib):
    env = dict(os.environ)
    if lib:
        env["ODP_LIB_PATH"] = lib
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_run.py")], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=900)
    return r.returncode, r.stdout, r.stderr


def test_kernels_pass_device_bounds_checks():
    from paper_2204_05520_b200 import build
    lib = build.build(check=True)
    assert b"odp check" in open(lib, "rb").read()          # the checks are compiled in
    rc, out_chk, err = _run(lib)
    assert rc == 0 and "odp check" not in out_chk + err, (out_chk[-2000:], err[-2000:])
    rc2, out, err2 = _run(None)
    assert rc2 == 0, err2[-2000:]
    assert out_chk == out
    assert len(out.strip().splitlines()) >= 12
