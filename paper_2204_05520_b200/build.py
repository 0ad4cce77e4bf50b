"""Build libodp.so in-tree with nvcc for sm_100a (no JIT cache, no CPU fallback)."""
from __future__ import annotations

import glob
import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libodp.so")
LIB_CHECK = os.path.join(HERE, "libodp_check.so")   # -DODP_CHECK: device bounds checks (tests/test_gpu_checked.py)
SRC = os.path.join(HERE, "csrc", "odp.cu")

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared", "--expt-relaxed-constexpr"]


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*")) + [os.path.join(ROOT, "include", "odp.h")])


def source_hash(check: bool = False) -> str:
    """sha256 over the sources, the nvcc flags and the variant: the build is redone when it changes
    (file contents, not mtimes: a checkout or a copy to the GPU box does not trigger a rebuild)."""
    h = hashlib.sha256()
    h.update(" ".join(NVCC_FLAGS + (["-DODP_CHECK"] if check else [])).encode())
    for p in sources():
        h.update(os.path.relpath(p, ROOT).encode())
        with open(p, "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()


def needs_build(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    stamp = lib + ".sha256"
    if not os.path.exists(stamp):
        return True
    with open(stamp) as fh:
        return fh.read().strip() != source_hash(check=lib == LIB_CHECK)


def build(force: bool = False, verbose: bool = False, check: bool = False) -> str:
    """nvcc -> libodp.so (or, check=True, libodp_check.so with the ODP_CHECK device checks)."""
    lib = LIB_CHECK if check else LIB
    if not force and not needs_build(lib):
        return lib
    nvcc = os.environ.get("NVCC", "nvcc")
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [nvcc, *NVCC_FLAGS, *(["-DODP_CHECK"] if check else []), "-o", tmp, SRC]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(tmp, lib)
    with open(lib + ".sha256", "w") as fh:
        fh.write(source_hash(check=check) + "\n")
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, check="--check" in sys.argv))
