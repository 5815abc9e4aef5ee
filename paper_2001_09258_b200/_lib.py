"""ctypes binding of libvem.so (the C ABI in include/vem.h).

Fails loudly when the shared object is missing or cannot be loaded: there is
no CPU fallback anywhere in the product path.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# VEM_LIB: an alternative build of the same library (A/B timing of two builds)
LIB_PATH = os.environ.get("VEM_LIB") or os.path.join(HERE, "libvem.so")

_P = ctypes.c_void_p
_N = ctypes.c_size_t

UNARY = {
    "sin_d_u10": "d", "cos_d_u10": "d", "tan_d_u10": "d",
    "sin_d_u10_ph": "d", "cos_d_u10_ph": "d", "tan_d_u10_ph": "d",
    "atan_d_u10": "d", "exp_d_u10": "d", "exp_d_u35": "d", "log_d_u10": "d", "log_d_u35": "d",
    "sin_f_u10": "f", "cos_f_u10": "f", "tan_f_u10": "f",
    "sin_f_u10_ph": "f", "cos_f_u10_ph": "f", "tan_f_u10_ph": "f",
    "exp_f_u10": "f", "exp_f_u35": "f", "log_f_u10": "f", "log_f_u35": "f",
    # u35 trig/atan, asin/acos, f32 atan
    "sin_d_u35": "d", "cos_d_u35": "d", "tan_d_u35": "d", "atan_d_u35": "d",
    "asin_d_u10": "d", "asin_d_u35": "d", "acos_d_u10": "d", "acos_d_u35": "d",
    "sin_f_u35": "f", "cos_f_u35": "f", "tan_f_u35": "f", "atan_f_u10": "f", "atan_f_u35": "f",
    "asin_f_u10": "f", "asin_f_u35": "f", "acos_f_u10": "f", "acos_f_u35": "f",
}
BINARY = {
    "pow_d_u10": "d", "pow_d_u35": "d", "fmod_d": "d",
    "pow_f_u10": "f", "pow_f_u35": "f", "fmod_f": "f",
    # atan2 (first operand y), fdim
    "atan2_d_u10": "d", "atan2_d_u35": "d", "fdim_d": "d",
    "atan2_f_u10": "f", "atan2_f_u35": "f", "fdim_f": "f",
}
ALL = {**UNARY, **BINARY}

_lib = None


class VemError(RuntimeError):
    pass


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise VemError(f"libvem.so not built ({LIB_PATH}); run __graft_entry__.build() "
                       "or python paper_2001_09258_b200/build.py -- there is no CPU fallback")
    L = ctypes.CDLL(LIB_PATH)
    for name in UNARY:
        f = getattr(L, "vem_" + name)
        f.argtypes = [_P, _P, _N, _P]
        f.restype = ctypes.c_int
    for name in BINARY:
        f = getattr(L, "vem_" + name)
        f.argtypes = [_P, _P, _P, _N, _P]
        f.restype = ctypes.c_int
    for name in ("vem_trig_reduce_d", "vem_ph_reduce_d"):
        f = getattr(L, name)
        f.argtypes = [_P, _P, _P, _P, _N, _P]
        f.restype = ctypes.c_int
    L.vem_cw_reduce_d.argtypes = [_P, _P, _P, _P, _N, ctypes.c_int, _P]
    L.vem_cw_reduce_d.restype = ctypes.c_int
    L.vem_ph_reduce_f.argtypes = [_P, _P, _P, _N, _P]
    L.vem_ph_reduce_f.restype = ctypes.c_int
    L.vem_ph_table_d.argtypes = [ctypes.c_char_p]
    L.vem_ph_table_d.restype = ctypes.c_int
    L.vem_launch_count.argtypes = []
    L.vem_launch_count.restype = ctypes.c_uint64
    L.vem_version.restype = ctypes.c_char_p
    L.vem_run_sharded.argtypes = [ctypes.c_char_p, _P, _P, _P, _N, ctypes.c_int,
                                  ctypes.POINTER(ctypes.c_double)]
    L.vem_run_sharded.restype = ctypes.c_int
    L.vem_run_sharded_on.argtypes = [ctypes.c_char_p, _P, _P, _P, _N, ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                                     ctypes.POINTER(ctypes.c_double)]
    L.vem_run_sharded_on.restype = ctypes.c_int
    L.vem_probe_peak.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
    L.vem_probe_peak.restype = ctypes.c_int
    _lib = L
    return L


def check(rc: int, what: str):
    if rc != 0:
        raise VemError(f"{what} failed with cudaError {rc}")


def launch_count() -> int:
    return int(lib().vem_launch_count())


def probe_peak(kind: str = "fp64", iters: int = 4096) -> float:
    """Measured FMA throughput in Gop/s (one FMA = one op) on the current device."""
    v = ctypes.c_double(0.0)
    check(lib().vem_probe_peak(0 if kind == "fp64" else 1, iters, ctypes.byref(v)), "vem_probe_peak")
    return v.value


def ph_table_bytes() -> bytes:
    buf = ctypes.create_string_buffer(32768)
    check(lib().vem_ph_table_d(buf), "vem_ph_table_d")
    return buf.raw
