"""The trivial-result classes of the kernels (vem_math.cuh triv_*: exp, log,
pow, atan) against the oracle's FULL functions, on the CPU: wherever a rule
declares an argument trivial, its closed-form result must equal the full
function's bit for bit (k_stream skips the computation for those elements).
The rules are restated here in numpy from the CUDA source; the GPU side is
covered by the config-5 parity tests (where 50-97 % of the elements take
these paths)."""
from __future__ import annotations

import numpy as np
import pytest

from cases import rnd_bits
from oracle_lib import gen_fill, oracle_eval
from paper_2001_09258_b200 import inputs as I

CANON = np.uint64(0x7FF8000000000000).view(np.float64)
EXP_OVF = float.fromhex("0x1.62e42fefa39efp+9")
EXP_UNF = -float.fromhex("0x1.74910d52d3051p+9")
PIO2 = float.fromhex("0x1.921fb54442d18p+0")


def hi(x):
    return (x.view(np.uint64) >> np.uint64(32)).astype(np.uint32)


def triv_exp(x):
    h = hi(x) & np.uint32(0x7FFFFFFF)
    with np.errstate(invalid="ignore"):
        t = (h < 0x3C900000) | (x > EXP_OVF) | (x < EXP_UNF) | np.isnan(x)
        r = np.where(h < 0x3C900000, 1.0, np.where(x > EXP_OVF, np.inf, np.where(x < EXP_UNF, 0.0, CANON)))
    return t, r


def triv_log(x):
    ix = x.view(np.uint64)
    with np.errstate(over="ignore"):
        t = (ix - np.uint64(1)) >= np.uint64(0x7FEFFFFFFFFFFFFF)
    r = np.where((ix << np.uint64(1)) == 0, -np.inf, np.where(ix == np.uint64(0x7FF0000000000000), np.inf, CANON))
    return t, r


def triv_pow(x, y):
    hx = hi(x)
    hy, ly = hi(y) & np.uint32(0x7FFFFFFF), (y.view(np.uint64) & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    fx = ((hx & np.uint32(0x7FFFFFFF)) - np.uint32(0x00100000)) < np.uint32(0x7FE00000)
    fy = (hy < 0x7FF00000) & ((hy | ly) != 0)
    e = ((hx >> np.uint32(20)) & np.uint32(0x7FF)).astype(np.int64) - 1023
    with np.errstate(invalid="ignore", over="ignore"):
        p = y * np.where(e >= 0, e, e + 1).astype(np.float64)
        neg = (hx >> np.uint32(31)) == 1
        nanr = neg & (np.trunc(y) != y)
        t = fx & fy & (nanr | (~neg & ((p > 1025.0) | (p < -1077.0))))
    r = np.where(nanr, CANON, np.where(p > 1025.0, np.inf, 0.0))
    return t, r


def triv_atan(x):
    h = hi(x) & np.uint32(0x7FFFFFFF)
    t = (h >= 0x43500000) | (h < 0x3E400000)
    r = np.where(np.isnan(x), CANON, np.where(h < 0x3E400000, x, np.copysign(PIO2, x)))
    return t, r


def _edges(n):
    ex = np.array([EXP_OVF, EXP_UNF, 709.0, -745.0, 2.0 ** -54, 2.0 ** -55, 2.0 ** 54, 2.0 ** -27, 2.0 ** 60,
                   np.inf, -np.inf, np.nan, 0.0, -0.0, 5e-324, 1e308, -1e308])
    ex = np.concatenate([ex, -ex, np.nextafter(ex, np.inf), np.nextafter(ex, -np.inf)])
    wide = I.log_uniform(77, n, 1e-300, 1e300, signed=True)
    return np.concatenate([ex, wide, rnd_bits(78, n, np.float64), gen_fill(I.config_recipes(5, "sin", "d")[0], n)])


def _same(a, b):
    return np.array_equal(a.view(np.uint64), b.view(np.uint64))


@pytest.mark.parametrize("name,rule", [("exp_d_u10", triv_exp), ("exp_d_u35", triv_exp), ("log_d_u10", triv_log),
                                       ("log_d_u35", triv_log), ("atan_d_u10", triv_atan),
                                       ("atan_d_u35", triv_atan)])
def test_unary_trivial_results_equal_full_function(name, rule):
    x = _edges(200000)
    t, r = rule(x)
    full = oracle_eval(name, x)
    assert t.sum() > 1000
    assert _same(r[t], full[t]), name


@pytest.mark.parametrize("name", ["pow_d_u10", "pow_d_u35"])
def test_pow_trivial_results_equal_full_function(name):
    n = 200000
    x = np.concatenate([_edges(n), I.log_uniform(81, n, 1e-300, 1e300, signed=True)])
    y = np.concatenate([I.uniform(82, x.size - n, -30.0, 30.0), I.uniform(83, n, -2000.0, 2000.0)])
    y[:64] = np.array([1025.0, -1077.0, 31.0, -31.0] * 16)  # integer y with negative x -> full path
    t, r = triv_pow(x, y)
    full = oracle_eval(name, x, y)
    assert t.sum() > 10000
    assert _same(r[t], full[t]), name
    # config 2's domain never takes the trivial path, nor its maybe() hint
    # (the headline pays one test per lane and tile)
    x2, y2 = I.config_inputs(2, "pow", "d", 100000)
    assert not triv_pow(x2, y2)[0].any()
    assert not ((hi(x2) - np.uint32(0x3DD00000)) >= np.uint32(0x04400000)).any()


# ------------------------------------------------------------- GPU: carry-over
def _mixed_wide(seed, n, share_dense):
    """Wide-range arguments (mostly trivial results) with dense stretches:
    segments of 5000-70000 elements alternate between log-uniform magnitudes
    over the whole binary64 range and moderate ones, so warps enter and leave
    the compaction mode and the per-warp stacks carry pending elements across
    tiles with very different non-trivial shares."""
    rng = np.random.default_rng(seed)
    x = I.log_uniform(seed, n, 1e-300, 1e300, signed=True)
    pos = 0
    while pos < n:
        m = int(rng.integers(5000, 70000))
        if rng.random() < share_dense:
            x[pos:pos + m] = np.exp(rng.uniform(-12, 12, min(m, n - pos))) * rng.choice([-1.0, 1.0], min(m, n - pos))
        pos += m
    x[rng.integers(0, n, 64)] = np.array([np.inf, -np.inf, np.nan, 0.0] * 16)
    return x


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["pow_d_u10", "atan_d_u10", "atan_d_u35"])
def test_gpu_compaction_carry_over(cuda, name):
    """k_stream's trivial-class compaction with the per-warp carry-over stack
    (vem_kernels.cu): mixed trivial / dense inputs, ragged sizes (partial last
    tile, pending elements flushed at the end), misaligned buffers take the
    plain kernel, and in place -- all bit-identical to the oracle."""
    import torch
    from paper_2001_09258_b200 import api
    for n, seed, dense in ((1 << 21, 3, 0.25), ((1 << 20) + 12345, 4, 0.6), (300001, 5, 0.0), (4099, 6, 0.0)):
        x = _mixed_wide(seed, n, dense)
        args = [x]
        if name.startswith("pow"):
            y = I.uniform(seed + 100, n, -30.0, 30.0)
            y[::97] = np.round(y[::97])  # integer exponents: negative bases are not NaN
            args.append(y)
        want = oracle_eval(name, *args)
        dev = [torch.from_numpy(a).to(cuda) for a in args]
        out = torch.empty_like(dev[0])
        api.call(name, *dev, out=out)
        assert _same(out.cpu().numpy(), want), (name, n, "out of place")
        api.call(name, *dev, out=dev[0])  # in place: the stack holds its own copy of the arguments
        assert _same(dev[0].cpu().numpy(), want), (name, n, "in place")
