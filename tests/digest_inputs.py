"""Inputs of the GPU bit-identity digests (SPEC.md:517-525 MD5 digests,
SURVEY.md 8(f).2): random bit patterns -- every class of binary64/binary32
value including NaNs, infinities, subnormals and huge trig arguments -- from
a per-entry-point SplitMix64 stream, so the GPU side can regenerate them
without the oracle."""
from __future__ import annotations

import zlib

import numpy as np

from paper_2001_09258_b200 import _lib
from paper_2001_09258_b200 import inputs as I

N_DIGEST = 1 << 24


def digest_inputs(name: str, n: int = N_DIGEST):
    seed = zlib.crc32(name.encode())
    f32 = _lib.ALL[name] == "f"
    arrs = []
    for k in range(2 if name in _lib.BINARY else 1):
        b = I.splitmix64(seed + 7919 * k, n)
        arrs.append((b & np.uint64(0xFFFFFFFF)).astype(np.uint32).view(np.float32) if f32 else b.view(np.float64))
    return arrs
