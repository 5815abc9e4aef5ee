"""ctypes binding of oracle/_build/libvem_sleef.so: upstream SLEEF 3.8 (the
paper's library, AVX-512 entry points inside torch's libtorch_cpu.so) -- the
<= 1 ulp cross-check of north_star.  Test infrastructure only."""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PATH = os.path.join(ROOT, "oracle", "_build", "libvem_sleef.so")
_L = None


def available() -> str | None:
    """None if usable, else why not."""
    try:
        flags = open("/proc/cpuinfo").read()
    except OSError:
        return "no /proc/cpuinfo"
    if " avx512f" not in flags:
        return "host CPU has no AVX-512F (SLEEF's avx512f entry points)"
    if not os.path.exists(PATH):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=False)
    if not os.path.exists(PATH):
        return "libvem_sleef.so not built"
    return None


def lib():
    global _L
    if _L is None:
        _L = ctypes.CDLL(PATH)
        _L.sleef_run.restype = ctypes.c_double
        _L.sleef_run.argtypes = [ctypes.c_char_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                 ctypes.c_size_t, ctypes.c_int]
    return _L


def sleef_eval(name: str, x: np.ndarray, y: np.ndarray | None = None, threads: int = 8):
    """SLEEF's function for vem entry `name` over x (and y); None if SLEEF has
    no such entry.  Pads to a multiple of 16 lanes."""
    n = x.size
    m = (n + 15) // 16 * 16
    xp = np.zeros(m, dtype=x.dtype)
    xp[:n] = x
    yp = None
    if y is not None:
        yp = np.ones(m, dtype=y.dtype)
        yp[:n] = y
    out = np.empty(m, dtype=x.dtype)
    t = lib().sleef_run(name.encode(), xp.ctypes.data, None if yp is None else yp.ctypes.data, out.ctypes.data, m,
                        threads)
    if t < 0:
        return None
    return out[:n]


def ulp_distance(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Distance in units in the last place between same-format arrays, on the
    ordered line of representable values (+0 == -0); both NaN -> 0, exactly
    one NaN -> inf.  Returned as float64."""
    if a.dtype == np.float64:
        ia, ib, mask = a.view(np.int64), b.view(np.int64), np.int64(0x7FFFFFFFFFFFFFFF)
    else:
        ia, ib, mask = a.view(np.int32).astype(np.int64), b.view(np.int32).astype(np.int64), np.int64(0x7FFFFFFF)
    oa = np.where(ia < 0, -(ia & mask), ia & mask)
    ob = np.where(ib < 0, -(ib & mask), ib & mask)
    same = (oa >= 0) == (ob >= 0)
    with np.errstate(over="ignore"):
        d_same = np.abs(oa - ob).astype(np.float64)  # exact in int64 when the signs agree
    d_cross = np.abs(oa).astype(np.float64) + np.abs(ob).astype(np.float64)
    d = np.where(same, d_same, d_cross)
    na, nb = np.isnan(a), np.isnan(b)
    d = np.where(na & nb, 0.0, d)
    return np.where(na ^ nb, np.inf, d)
