"""vem-b200: batched elementwise C99 math (SLEEF-class, arXiv 2001.09258) on B200.

Product path: CUDA sm_100a kernels in libvem.so behind the C ABI of
include/vem.h; this package is the thin host mirror (ctypes) over it.
"""
from . import _lib  # noqa: F401
from ._lib import ALL, BINARY, UNARY, VemError, launch_count  # noqa: F401

__all__ = ["ALL", "BINARY", "UNARY", "VemError", "launch_count", "api"]


def __getattr__(name):
    if name == "api":
        from . import api
        return api
    raise AttributeError(name)
