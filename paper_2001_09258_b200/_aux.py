"""ctypes binding of libvem_aux.so (csrc/vem_aux.h): the device twin of the
config-input generator (inputs.py) and the chunk checksums.  Bench and test
infrastructure only -- the math path is libvem.so (_lib.py)."""
from __future__ import annotations

import ctypes
import os

from . import inputs as I

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libvem_aux.so")
_lib = None


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} not built; run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        L.vem_aux_fill.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint64,
                                   ctypes.c_void_p]
        L.vem_aux_fill.restype = ctypes.c_int
        L.vem_aux_checksum.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_uint64,
                                       ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
        L.vem_aux_checksum.restype = ctypes.c_int
        _lib = L
    return _lib


def fill(recipe: dict, out, offset: int = 0):
    """Write elements [offset, offset + out.numel()) of `recipe` into the CUDA
    tensor `out` (float64 / float32 per the recipe), on its current stream."""
    import torch
    want = torch.float32 if recipe["f32"] else torch.float64
    assert out.is_cuda and out.is_contiguous() and out.dtype == want
    r = I.recipe_struct(recipe)
    with torch.cuda.device(out.device):
        rc = lib().vem_aux_fill(ctypes.byref(r), out.data_ptr(), out.numel(), offset,
                                torch.cuda.current_stream(out.device).cuda_stream)
    if rc:
        raise RuntimeError(f"vem_aux_fill failed: cudaError {rc}")
    return out


def checksum(t, offset: int = 0, log2chunk: int = 24):
    """{global chunk id: checksum contribution of t} (vem_aux.h definition),
    computed on the device; the one host sync is the readback of the sums."""
    import torch
    assert t.is_cuda and t.is_contiguous() and t.element_size() in (4, 8)
    n = t.numel()
    if n == 0:
        return {}
    c0 = offset >> log2chunk
    c1 = (offset + n - 1) >> log2chunk
    sums = torch.zeros(c1 - c0 + 1, dtype=torch.int64, device=t.device)
    with torch.cuda.device(t.device):
        rc = lib().vem_aux_checksum(t.data_ptr(), n, t.element_size(), offset, log2chunk, sums.data_ptr(),
                                    torch.cuda.current_stream(t.device).cuda_stream)
    if rc:
        raise RuntimeError(f"vem_aux_checksum failed: cudaError {rc}")
    return {c0 + k: int(v) & I.M64 for k, v in enumerate(sums.cpu().tolist())}
