"""Exhaustive float32 parity: EVERY binary32 input (2^32 bit patterns) through
each unary f32 entry point on the GPU, compared bit-for-bit with the CPU
oracle, plus the max ULP error vs (float) of glibc's correctly-rounded-in-
practice binary64 function on every finite input.  Minutes of CPU work per
function, so opt-in: VEM_EXHAUSTIVE=1 python -m pytest -m gpu tests/test_exhaustive_f32.py
"""
from __future__ import annotations

import os

import numpy as np
import pytest

from oracle_lib import oracle_eval

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(os.environ.get("VEM_EXHAUSTIVE") != "1", reason="set VEM_EXHAUSTIVE=1")]

FUNCS = ["sin_f_u10", "cos_f_u10", "tan_f_u10", "exp_f_u10", "exp_f_u35", "log_f_u10", "log_f_u35",
         "atan_f_u10", "atan_f_u35", "asin_f_u10", "asin_f_u35", "acos_f_u10", "acos_f_u35"]
CHUNK = 1 << 28


@pytest.mark.parametrize("name", FUNCS)
def test_all_binary32_inputs(cuda, name):
    import torch
    from paper_2001_09258_b200 import api
    mism = 0
    for c in range((1 << 32) // CHUNK):
        x = (np.arange(c * CHUNK, (c + 1) * CHUNK, dtype=np.uint64).astype(np.uint32)).view(np.float32)
        g = api.call(name, torch.from_numpy(x).cuda()).cpu().numpy()
        e = oracle_eval(name, x)
        bad = np.nonzero(g.view(np.uint32) != e.view(np.uint32))[0]
        if bad.size:
            i = bad[0]
            raise AssertionError(f"{name}: {bad.size} mismatches in chunk {c}; first x={x[i]!r} "
                                 f"gpu={g[i]!r} oracle={e[i]!r}")
        mism += bad.size
    assert mism == 0
