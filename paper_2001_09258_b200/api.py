"""Host-side mirror of the reference's function interface over device arrays.

The reference exposes each function as `name`, `name_u35`, `name_det`
 on one lane vector (backend.hpp:294-305).  Here each name
takes a CUDA tensor (torch is only the device-memory/stream plumbing) and
calls the matching C-ABI entry point (include/vem.h) on the current torch
stream.  The u10 kernels ARE the deterministic variants (bit-identical to the
CPU oracle), so `name_det` aliases `name`.  Errors are in-band (NaN/Inf), as
in the reference; misuse (CPU tensor, wrong dtype, non-contiguous, mismatched
device or size) raises.

Note on `name_det`: the reference's deterministic variants are Estrin-ordered
and meant to be bit-identical across its backends.
Here the `_det` names alias the u10 kernels, which are bit-identical to vem's
own CPU oracle (oracle/vem_oracle.c) on every input -- deterministic across
GPUs, shard counts and launch shapes -- but use Horner evaluation and vem's
integer Payne-Hanek, so their digests are NOT the reference's _det digests.
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib

_SUFFIX = {torch.float64: "d", torch.float32: "f"}


def _entry(fn: str, acc: str, x: torch.Tensor, ph: bool = False) -> str:
    if not isinstance(x, torch.Tensor) or not x.is_cuda:
        raise TypeError(f"vem.{fn}: expected a CUDA tensor (no CPU fallback)")
    if x.dtype not in _SUFFIX:
        raise TypeError(f"vem.{fn}: dtype {x.dtype} unsupported (float32/float64)")
    p = _SUFFIX[x.dtype]
    name = f"{fn}_{p}" if fn in ("fmod", "fdim") else f"{fn}_{p}_{acc}"
    if ph:
        name += "_ph"
    if name not in _lib.ALL:
        raise TypeError(f"vem: no entry point {name}")
    return name


def _check_operand(what: str, name: str, t: torch.Tensor, ref: torch.Tensor, n: int):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"vem.{name}: {what} must be a CUDA tensor (no CPU fallback)")
    if t.device != ref.device:
        raise ValueError(f"vem.{name}: {what} is on {t.device}, x is on {ref.device}")
    if t.dtype != ref.dtype:
        raise TypeError(f"vem.{name}: {what} dtype {t.dtype} != x dtype {ref.dtype}")
    if t.numel() != n:
        raise ValueError(f"vem.{name}: {what} has {t.numel()} elements, x has {n}")
    if not t.is_contiguous():
        raise ValueError(f"vem.{name}: {what} must be contiguous")


def call(name: str, x: torch.Tensor, y: torch.Tensor | None = None, out: torch.Tensor | None = None):
    """Launch vem_<name> on tensors, asynchronous on x.device's current stream.

    Every operand must be a contiguous CUDA tensor on x's device with x's
    dtype and element count; misuse raises before anything is launched (an
    out-of-bounds launch would leave a sticky device error instead)."""
    if name not in _lib.ALL:
        raise TypeError(f"vem: no entry point {name}")
    if not isinstance(x, torch.Tensor) or not x.is_cuda:
        raise TypeError(f"vem.{name}: expected a CUDA tensor (no CPU fallback)")
    want = torch.float64 if _lib.ALL[name] == "d" else torch.float32
    if x.dtype != want:
        raise TypeError(f"vem.{name}: dtype {x.dtype}, expected {want}")
    n = x.numel()
    _check_operand("x", name, x, x, n)
    if name in _lib.BINARY:
        if y is None:
            raise ValueError(f"vem.{name}: second operand missing")
        _check_operand("second operand", name, y, x, n)
    elif y is not None:
        raise ValueError(f"vem.{name}: unary entry point takes one operand")
    L = _lib.lib()
    with torch.cuda.device(x.device):
        if out is None:
            out = torch.empty_like(x)
        _check_operand("out", name, out, x, n)
        s = torch.cuda.current_stream(x.device).cuda_stream
        if name in _lib.BINARY:
            rc = getattr(L, "vem_" + name)(x.data_ptr(), y.data_ptr(), out.data_ptr(), n, s)
        else:
            rc = getattr(L, "vem_" + name)(x.data_ptr(), out.data_ptr(), n, s)
    _lib.check(rc, "vem_" + name)
    return out


def _u(fn, acc="u10", ph=False):
    def f(x, out=None):
        return call(_entry(fn, acc, x, ph), x, out=out)
    f.__name__ = fn if acc == "u10" else f"{fn}_{acc}"
    return f


def _b(fn, acc="u10"):
    def f(x, y, out=None):
        return call(_entry(fn, acc, x), x, y, out=out)
    f.__name__ = fn if acc == "u10" else f"{fn}_{acc}"
    return f


sin = sin_det = _u("sin")
cos = cos_det = _u("cos")
tan = tan_det = _u("tan")
sin_ph = _u("sin", ph=True)
cos_ph = _u("cos", ph=True)
tan_ph = _u("tan", ph=True)
atan = atan_det = _u("atan")
exp = exp_det = _u("exp")
exp_u35 = _u("exp", "u35")
log = log_det = _u("log")
log_u35 = _u("log", "u35")
pow = pow_det = _b("pow")  # noqa: A001
pow_u35 = _b("pow", "u35")
fmod = fmod_det = _b("fmod")
# SURVEY.md §8(f).1
sin_u35 = _u("sin", "u35")
cos_u35 = _u("cos", "u35")
tan_u35 = _u("tan", "u35")
atan_u35 = _u("atan", "u35")
asin = asin_det = _u("asin")
asin_u35 = _u("asin", "u35")
acos = acos_det = _u("acos")
acos_u35 = _u("acos", "u35")
atan2 = atan2_det = _b("atan2")  # atan2(y, x)
atan2_u35 = _b("atan2", "u35")
fdim = fdim_det = _b("fdim")


def trig_reduce(x: torch.Tensor, kind: str = "trig", level: int = 1):
    """Device trig_reduce / cody_waite_reduce / payne_hanek_reduce -> (hi, lo, q)."""
    L = _lib.lib()
    if not isinstance(x, torch.Tensor) or not x.is_cuda or not x.is_contiguous():
        raise TypeError("vem.trig_reduce: expected a contiguous CUDA tensor")
    if x.dtype not in _SUFFIX:
        raise TypeError(f"vem.trig_reduce: dtype {x.dtype} unsupported (float32/float64)")
    with torch.cuda.device(x.device):
        return _trig_reduce(L, x, kind, level)


def _trig_reduce(L, x, kind, level):
    def _stream_ptr():
        return torch.cuda.current_stream(x.device).cuda_stream

    if x.dtype == torch.float32:
        r = torch.empty(x.shape, dtype=torch.float64, device=x.device)
        q = torch.empty(x.shape, dtype=torch.int32, device=x.device)
        _lib.check(L.vem_ph_reduce_f(x.data_ptr(), r.data_ptr(), q.data_ptr(), x.numel(), _stream_ptr()),
                   "vem_ph_reduce_f")
        return r, q
    hi = torch.empty_like(x)
    lo = torch.empty_like(x)
    q = torch.empty(x.shape, dtype=torch.int32, device=x.device)
    if kind == "trig":
        rc = L.vem_trig_reduce_d(x.data_ptr(), hi.data_ptr(), lo.data_ptr(), q.data_ptr(), x.numel(), _stream_ptr())
    elif kind == "ph":
        rc = L.vem_ph_reduce_d(x.data_ptr(), hi.data_ptr(), lo.data_ptr(), q.data_ptr(), x.numel(), _stream_ptr())
    else:
        rc = L.vem_cw_reduce_d(x.data_ptr(), hi.data_ptr(), lo.data_ptr(), q.data_ptr(), x.numel(), level,
                               _stream_ptr())
    _lib.check(rc, "vem reduce")
    return hi, lo, q


def run_sharded(name: str, x: np.ndarray, y: np.ndarray | None = None, ngpu: int = 1, devices=None):
    """Host arrays in, host array out, sharded contiguously over `ngpu`
    devices (or over the explicit `devices` list, repeats allowed) by the C++
    driver (vem_run_sharded[_on]).  Returns (out, max-over-shards kernel ms)."""
    L = _lib.lib()
    x = np.ascontiguousarray(x)
    out = np.empty_like(x)
    ms = ctypes.c_double(0.0)
    yp = None
    if y is not None:
        y = np.ascontiguousarray(y)
        if y.shape != x.shape or y.dtype != x.dtype:
            raise ValueError("vem.run_sharded: second operand must match the first")
        yp = y.ctypes.data
    if devices is None:
        rc = L.vem_run_sharded(name.encode(), x.ctypes.data, yp, out.ctypes.data, x.size, ngpu, ctypes.byref(ms))
    else:
        devs = (ctypes.c_int * len(devices))(*devices)
        rc = L.vem_run_sharded_on(name.encode(), x.ctypes.data, yp, out.ctypes.data, x.size, len(devices), devs,
                                  ctypes.byref(ms))
    _lib.check(rc, "vem_run_sharded")
    return out, ms.value
