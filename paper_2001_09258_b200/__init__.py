"""vem-b200: batched elementwise C99 math (SLEEF-class, arXiv 2001.09258) on B200.

Product path: CUDA sm_100a kernels in libvem.so behind the C ABI of
include/vem.h; this package is the thin host mirror (ctypes) over it.
"""
from . import _lib  # noqa: F401
from ._lib import ALL, BINARY, UNARY, VemError, launch_count  # noqa: F401

__all__ = ["ALL", "BINARY", "UNARY", "VemError", "launch_count"]
# the torch-facing mirror lives in paper_2001_09258_b200.api (imports torch)
