"""ctypes bindings to the TEST-ONLY libraries under oracle/ (the checker).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg import
this module.  It builds oracle/_build with `make` when the shared objects are
missing (gcc only; no GPU needed).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
BUILD = os.path.join(ORACLE_DIR, "_build")
REF = os.path.join(ORACLE_DIR, "_ref")

FN_ID = {"sin": 0, "cos": 1, "tan": 2, "atan": 3, "exp": 4, "log": 5, "pow": 6, "fmod": 7, "asin": 8, "acos": 9,
         "atan2": 10, "fdim": 11}

_P = ctypes.c_void_p
_N = ctypes.c_size_t


def build_oracle():
    subprocess.run(["make", "-s", "-C", ORACLE_DIR], check=True)


def _load(name):
    path = os.path.join(BUILD, name)
    if not os.path.exists(path):
        build_oracle()
    return ctypes.CDLL(path)


_oracle = None
_mpfr = None


def oracle():
    global _oracle
    if _oracle is None:
        _oracle = _load("libvem_oracle.so")
    return _oracle


def mpfr():
    global _mpfr
    if _mpfr is None:
        _mpfr = _load("libvem_mpfr.so")
    return _mpfr


def ptr(a: np.ndarray):
    return a.ctypes.data_as(_P)


def oracle_eval(name: str, *args: np.ndarray) -> np.ndarray:
    """Evaluate vo_<name>_arr over numpy arrays (all threads)."""
    L = oracle()
    f = getattr(L, f"vo_{name}_arr")
    x = np.ascontiguousarray(args[0])
    out = np.empty_like(x)
    if len(args) == 1:
        f.argtypes = [_P, _P, _N]
        f(ptr(x), ptr(out), x.size)
    else:
        y = np.ascontiguousarray(args[1])
        f.argtypes = [_P, _P, _P, _N]
        f(ptr(x), ptr(y), ptr(out), x.size)
    return out


def ulp_errors(fn: str, x: np.ndarray, act: np.ndarray, y: np.ndarray | None = None) -> np.ndarray:
    L = mpfr()
    out = np.empty(x.size, dtype=np.float64)
    if x.dtype == np.float64:
        f = L.mp_ulp_d
    else:
        f = L.mp_ulp_f
    f.argtypes = [ctypes.c_int, _P, _P, _P, _P, _N]
    f(FN_ID[fn], ptr(x), ptr(y) if y is not None else None, ptr(act), ptr(out), x.size)
    return out


def reduce_oracle(kind: str, x: np.ndarray, level: int = 1):
    L = oracle()
    n = x.size
    hi = np.empty(n); lo = np.empty(n); q = np.empty(n, dtype=np.int32)
    if kind == "trig":
        f = L.vo_trig_reduce_d; f.argtypes = [_P, _P, _P, _P, _N]; f(ptr(x), ptr(hi), ptr(lo), ptr(q), n)
    elif kind == "ph":
        f = L.vo_ph_reduce_d; f.argtypes = [_P, _P, _P, _P, _N]; f(ptr(x), ptr(hi), ptr(lo), ptr(q), n)
    elif kind == "ph_int":
        f = L.vo_ph_int_reduce_d; f.argtypes = [_P, _P, _P, _P, _N]; f(ptr(x), ptr(hi), ptr(lo), ptr(q), n)
    elif kind == "cw":
        f = L.vo_cw_reduce_d; f.argtypes = [_P, _P, _P, _P, _N, ctypes.c_int]
        f(ptr(x), ptr(hi), ptr(lo), ptr(q), n, level)
    return hi, lo, q


def ref_lib(variant: str):
    path = os.path.join(REF, f"libvemref_{variant}.so")
    if not os.path.exists(path):
        if os.path.isdir("/root/reference/proj/core"):
            subprocess.run(["python", os.path.join(ORACLE_DIR, "ref_build.py")], check=True)
        else:
            return None
    return ctypes.CDLL(path)


def reduce_ref(variant: str, kind: str, x: np.ndarray, level: int = 1, table: bytes | None = None):
    L = ref_lib(variant)
    n = x.size
    hi = np.empty(n); lo = np.empty(n); q = np.empty(n, dtype=np.int64)
    if kind == "cw":
        f = L.ref_cw_reduce; f.argtypes = [_P, _P, _P, _P, _N, ctypes.c_int]
        f(ptr(x), ptr(hi), ptr(lo), ptr(q), n, level)
    elif kind == "ph":
        f = L.ref_ph_reduce; f.argtypes = [_P, _P, _P, _P, _N]; f(ptr(x), ptr(hi), ptr(lo), ptr(q), n)
    elif kind == "ph_table":
        L.ref_set_table.argtypes = [ctypes.c_char_p, _N]
        assert L.ref_set_table(table, len(table)) == 0
        f = L.ref_ph_reduce_table; f.argtypes = [_P, _P, _P, _P, _N]; f(ptr(x), ptr(hi), ptr(lo), ptr(q), n)
    elif kind == "trig":
        f = L.ref_trig_reduce; f.argtypes = [_P, _P, _P, _P, _N]; f(ptr(x), ptr(hi), ptr(lo), ptr(q), n)
    return hi, lo, q


def ph_table_bytes(prec: str = "d") -> bytes:
    L = oracle()
    f = L.vo_ph_table_d if prec == "d" else L.vo_ph_table_f
    f.restype = ctypes.POINTER(ctypes.c_double)
    n = 4096 if prec == "d" else 4 * 104
    p = f()
    return np.ctypeslib.as_array(p, shape=(n,)).copy().tobytes()


# ------------------------------------------------ config inputs (host twin)
_gen = None


def gen():
    global _gen
    if _gen is None:
        L = _load("libvem_gen.so")
        L.vg_fill.argtypes = [_P, _P, _N, ctypes.c_uint64]
        L.vg_checksum.argtypes = [_P, _N, ctypes.c_int, ctypes.c_uint64, ctypes.c_int, _P]
        _gen = L
    return _gen


def gen_fill(recipe: dict, n: int, offset: int = 0) -> np.ndarray:
    """oracle/vem_gen_host.c: elements [offset, offset+n) of a recipe."""
    from paper_2001_09258_b200 import inputs as I
    out = np.empty(n, dtype=np.float32 if recipe["f32"] else np.float64)
    r = I.recipe_struct(recipe)
    gen().vg_fill(ctypes.byref(r), ptr(out), n, offset)
    return out


def gen_checksum(a: np.ndarray, offset: int = 0, log2chunk: int = 24) -> dict:
    n = a.size
    if n == 0:
        return {}
    c0 = offset >> log2chunk
    c1 = (offset + n - 1) >> log2chunk
    sums = np.zeros(c1 - c0 + 1, dtype=np.uint64)
    gen().vg_checksum(ptr(np.ascontiguousarray(a)), n, a.dtype.itemsize, offset, log2chunk, ptr(sums))
    return {c0 + k: int(v) for k, v in enumerate(sums)}
