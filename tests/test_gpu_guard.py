"""Out-of-bounds and aliasing checks without compute-sanitizer (closed on the
GPU pool): every entry point writes exactly [out, out + n) -- canary bands
of 4096 elements on both sides stay untouched -- for ragged sizes (0, 1,
partial vectors, one element past a tile, tiles + remainder), aligned and
misaligned buffers, and in place (out == x); results stay bit-identical to
the oracle.  test_checked_build_runs_clean repeats the kernel families and
the config-5 / fmod parity under libvem_check.so (-DVEM_CHECK: device-side
bounds assertions on every computed shared-memory index of the sorting
kernels; a violation traps)."""
from __future__ import annotations

import os
import subprocess
import sys

import numpy as np
import pytest

from cases import binary_cases, unary_cases
from oracle_lib import oracle_eval
from paper_2001_09258_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GUARD = 4096
SIZES = [0, 1, 5, 1023, 4096 * 3 + 17, (1 << 16) + 3]


def _canary(dt):
    return np.uint64(0x7FF4DEADBEEF1234).view(np.float64) if dt == np.float64 else \
        np.uint32(0x7FA0BEEF).view(np.float32)


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(_lib.ALL))
def test_writes_stay_in_bounds(cuda, name):
    import torch
    from paper_2001_09258_b200 import api
    binary = name in _lib.BINARY
    src = binary_cases(name, 1 << 16) if binary else (unary_cases(name, 1 << 16),)
    dt = src[0].dtype
    u = np.uint64 if dt == np.float64 else np.uint32
    for n in SIZES:
        for pad in (0, 1):
            ins = [a[:n].copy() for a in src]
            if ins[0].size < n:  # small case sets: tile them
                ins = [np.resize(a, n) for a in src]
            dev_in = []
            for a in ins:
                t = torch.empty(n + pad, dtype=torch.from_numpy(a).dtype, device=cuda)[pad:]
                t.copy_(torch.from_numpy(a))
                dev_in.append(t)
            band = np.full(2 * GUARD + n + pad, _canary(dt), dtype=dt)
            big = torch.from_numpy(band).to(cuda)
            out = big[GUARD + pad:GUARD + pad + n]
            api.call(name, *dev_in, out=out)
            got = big.cpu().numpy()
            assert np.array_equal(got[:GUARD + pad].view(u), band[:GUARD + pad].view(u)), (name, n, pad, "before")
            assert np.array_equal(got[GUARD + pad + n:].view(u), band[GUARD + pad + n:].view(u)), (name, n, pad,
                                                                                                 "after")
            if n:
                exp = oracle_eval(name, *ins)
                assert np.array_equal(got[GUARD + pad:GUARD + pad + n].view(u), exp.view(u)), (name, n, pad)
    # in place: out aliases the first operand
    n = (1 << 16) + 3
    ins = [a[:n].copy() for a in src]
    dev_in = [torch.from_numpy(a).to(cuda) for a in ins]
    api.call(name, *dev_in, out=dev_in[0])
    assert np.array_equal(dev_in[0].cpu().numpy().view(u), oracle_eval(name, *ins).view(u)), (name, "in place")


@pytest.mark.gpu
def test_checked_build_runs_clean(cuda):
    from paper_2001_09258_b200 import build
    lib = build.build_check()
    env = dict(os.environ, VEM_LIB=lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_run.py"), "20"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-m", "gpu", "-p", "no:cacheprovider",
                        "tests/test_config_parity.py", "-k", "cfg5 and (sin or tan or fmod) or cfg4"], cwd=ROOT,
                       env=env, capture_output=True, text=True, timeout=1800)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
