"""Build libvem.so (sm_100a) in-tree with nvcc.

    nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false ...

--fmad=false is load-bearing: it forbids the compiler from contracting a*b+c
into DFMA/FFMA, so the only fused operations are the explicit fma() calls that
the CPU oracle performs too (bit-identity, SURVEY.md §7 hard part (c)).  No
fast-math: IEEE division, sqrt and denormals stay on.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libvem.so")
SOURCES = ["vem_kernels.cu", "vem_host.cu", "vem_probe.cu"]
# bench/test infrastructure (config-input generator, chunk checksums): a
# separate library, so the product libvem.so carries only the math path
AUX_LIB = os.path.join(HERE, "libvem_aux.so")
AUX_SOURCES = ["vem_aux.cu"]
# every header under csrc/ (vem_math.cuh, vem_stream.cuh, the generated
# tables, ...) plus the public C header: any of them newer than the library
# makes it stale
HEADERS = sorted(f for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))) + ["../../include/vem.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "--fmad=false", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _stale(lib: str = LIB, sources=SOURCES) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    for f in sources + HEADERS + ["../build.py"]:
        p = os.path.join(CSRC, f)
        if os.path.exists(p) and os.path.getmtime(p) > t:
            return True
    return False


CHECK_LIB = os.path.join(HERE, "libvem_check.so")


def _link(lib: str, sources, verbose: bool, extra=()):
    objs = []
    bdir = os.path.join(HERE, "_build")
    os.makedirs(bdir, exist_ok=True)
    for s in sources:
        o = os.path.join(bdir, s.replace(".cu", ".o"))
        if extra:
            o = o.replace(".o", "_check.o")
        cmd = [nvcc(), *NVCC_FLAGS, *extra, "-c", os.path.join(CSRC, s), "-o", o]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
        objs.append(o)
    tmp = lib + ".tmp"
    # static cudart: the library carries its own 12.9 runtime (torch bundles an
    # older libcudart.so.12); both share the device's primary context, so
    # torch-allocated pointers and torch streams are valid here.
    cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static",
           *objs, "-o", tmp]
    subprocess.run(cmd, check=True)
    os.replace(tmp, lib)


def build(force: bool = False, verbose: bool = False) -> str:
    if force or _stale():
        _link(LIB, SOURCES, verbose)
    if force or _stale(AUX_LIB, AUX_SOURCES):
        _link(AUX_LIB, AUX_SOURCES, verbose)
    return LIB


def build_check(force: bool = False, verbose: bool = False) -> str:
    """The bounds-checked variant (-DVEM_CHECK) for the guard tests; load it
    with VEM_LIB=<path> (paper_2001_09258_b200/_lib.py)."""
    if force or _stale(CHECK_LIB, SOURCES):
        _link(CHECK_LIB, SOURCES, verbose, extra=("-DVEM_CHECK",))
    return CHECK_LIB


if __name__ == "__main__":
    if "--check" in sys.argv:
        print(build_check(force="--force" in sys.argv, verbose=True))
    else:
        print(build(force="--force" in sys.argv, verbose=True))
