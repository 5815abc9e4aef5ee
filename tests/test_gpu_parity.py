"""GPU parity: every C-ABI entry point vs the CPU oracle, BIT-EXACT.

Inputs: special values (singletons / all pairs), random bit patterns
("random bits ... reinterprets"), and the BASELINE.json
config domains, at sizes the oracle finishes in seconds.  Comparison is on
raw bit patterns (NaNs are canonical on both sides), reporting the first
mismatching index.  Calls go through the C ABI (ctypes) on device buffers.
"""
from __future__ import annotations

import numpy as np
import pytest

from cases import binary_cases, unary_cases
from oracle_lib import oracle_eval, reduce_oracle

pytestmark = pytest.mark.gpu

from paper_2001_09258_b200 import _lib  # noqa: E402

N = 1 << 16


def _bits(a):
    return a.view(np.uint64 if a.dtype == np.float64 else np.uint32)


def _assert_bit_exact(name, got, exp, *inputs):
    g, e = _bits(got), _bits(exp)
    bad = np.nonzero(g != e)[0]
    if bad.size:
        i = bad[0]
        args = ", ".join(repr(a[i]) for a in inputs)
        raise AssertionError(f"{name}: {bad.size}/{g.size} mismatches; first at {i}: f({args}) "
                             f"gpu={got[i]!r} ({g[i]:#x}) oracle={exp[i]!r} ({e[i]:#x})")


def _gpu(name, *arrs):
    import torch
    from paper_2001_09258_b200 import api
    ts = [torch.from_numpy(a).cuda() for a in arrs]
    out = api.call(name, *ts)
    torch.cuda.synchronize()
    return out.cpu().numpy()


@pytest.mark.parametrize("name", sorted(_lib.UNARY))
def test_unary_bit_exact(cuda, name):
    x = unary_cases(name, N)
    got = _gpu(name, x)
    exp = oracle_eval(name, x)
    _assert_bit_exact(name, got, exp, x)


@pytest.mark.parametrize("name", sorted(_lib.BINARY))
def test_binary_bit_exact(cuda, name):
    x, y = binary_cases(name, N)
    got = _gpu(name, x, y)
    exp = oracle_eval(name, x, y)
    _assert_bit_exact(name, got, exp, x, y)


@pytest.mark.parametrize("name", ["sin_d_u10", "exp_f_u10", "pow_d_u10"])
def test_unaligned_and_ragged(cuda, name):
    """Scalar (unaligned) kernel path and ragged tails give identical bits."""
    import torch
    from paper_2001_09258_b200 import api
    n = 1000 + 3
    if name in _lib.BINARY:
        x, y = binary_cases(name, n)
        x, y = x[:n], y[:n]
        tx = torch.from_numpy(np.concatenate([[0.0], x]).astype(x.dtype)).cuda()[1:]
        ty = torch.from_numpy(np.concatenate([[0.0], y]).astype(y.dtype)).cuda()[1:]
        got = api.call(name, tx, ty).cpu().numpy()
        _assert_bit_exact(name, got, oracle_eval(name, x, y), x, y)
    else:
        x = unary_cases(name, n)[:n]
        tx = torch.from_numpy(np.concatenate([[0.0], x]).astype(x.dtype)).cuda()[1:]
        got = api.call(name, tx).cpu().numpy()
        _assert_bit_exact(name, got, oracle_eval(name, x), x)
    for m in (0, 1, 2, 3, 5, 7):
        xs = unary_cases("sin_d_u10", 64)[:m] if name not in _lib.BINARY else None
        if xs is not None and name == "sin_d_u10":
            got = _gpu(name, xs) if m else np.empty(0)
            _assert_bit_exact(name, got, oracle_eval(name, xs), xs)


@pytest.mark.parametrize("kind,level", [("trig", 0), ("cw", 1), ("cw", 2), ("ph", 0)])
def test_reduction_bit_exact(cuda, kind, level):
    import torch
    from paper_2001_09258_b200 import api, inputs as I
    if kind == "cw" and level == 1:
        x = I.uniform(31, N, -15, 15)
    elif kind == "cw":
        x = I.log_uniform(32, N, 1e-3, 1e14, signed=True)
    else:
        x = np.concatenate([unary_cases("sin_d_u10", N), I.log_uniform(33, N, 1e-300, 1e300, signed=True)])
    hi, lo, q = api.trig_reduce(torch.from_numpy(x).cuda(), kind, level)
    torch.cuda.synchronize()
    ehi, elo, eq = reduce_oracle(kind, x, level)
    _assert_bit_exact(f"{kind}{level}.hi", hi.cpu().numpy(), ehi, x)
    _assert_bit_exact(f"{kind}{level}.lo", lo.cpu().numpy(), elo, x)
    assert np.array_equal(q.cpu().numpy(), eq)


def test_round_ta_matches_reference_rule(cuda):
    """CUDA round() == backend.hpp:47-52 round_ta on ties and neighbours
    (exercised through cw1 quadrants at k.5 boundaries of 2x/pi)."""
    import torch
    from paper_2001_09258_b200 import api
    ks = np.arange(-9, 10, dtype=np.float64) + 0.5
    t = np.concatenate([ks, np.nextafter(ks, np.inf), np.nextafter(ks, -np.inf)])
    x = t / float.fromhex("0x1.45f306dc9c883p-1")
    x = x[np.abs(x) <= 15]
    hi, lo, q = api.trig_reduce(torch.from_numpy(x).cuda(), "cw", 1)
    ehi, elo, eq = reduce_oracle("cw", x, 1)
    assert np.array_equal(q.cpu().numpy(), eq)
    _assert_bit_exact("cw1", hi.cpu().numpy(), ehi, x)


def test_launch_counter_and_version(cuda):
    before = _lib.launch_count()
    _gpu("exp_d_u10", np.linspace(-1, 1, 100))
    assert _lib.launch_count() == before + 1
    assert b"sm_100a" in _lib.lib().vem_version()


@pytest.mark.parametrize("name", ["exp_f_u35", "sin_d_u10", "pow_d_u10", "fmod_d"])
def test_repeat_launches_are_deterministic(cuda, name):
    """Ten back-to-back launches over 2^22 elements give identical bits."""
    import torch
    from paper_2001_09258_b200 import api
    n = 1 << 22
    if name in _lib.BINARY:
        x, y = binary_cases(name, n)
        ts = [torch.from_numpy(x[:n]).cuda(), torch.from_numpy(y[:n]).cuda()]
    else:
        ts = [torch.from_numpy(unary_cases(name, n)[:n]).cuda()]
    ref = api.call(name, *ts).clone()
    for _ in range(10):
        out = api.call(name, *ts)
        assert torch.equal(out.view(torch.int64 if out.dtype == torch.float64 else torch.int32),
                           ref.view(torch.int64 if ref.dtype == torch.float64 else torch.int32))


@pytest.mark.parametrize("name", ["log_f_u35", "exp_f_u35", "exp_d_u10", "pow_f_u10", "sin_f_u10", "cos_d_u10"])
def test_tma_pipeline_vs_plain_kernel(cuda, name):
    """Regression for the cross-proxy WAR race (fence.proxy.async before a
    stage refill, vem_stream.cuh): the TMA-pipelined kernel over 2^28
    monotone inputs (a stale or early-refilled stage shows up as a result
    computed from another tile's input) must equal, bit for bit, the plain
    grid-stride kernel the library uses for misaligned pointers (same math,
    no shared-memory staging).  Several launches, since the race was rare."""
    import torch
    from paper_2001_09258_b200 import api
    n = 1 << 28 if name.endswith("_f_u35") or name.endswith("_f_u10") else 1 << 27
    dt = torch.float32 if "_f_" in name else torch.float64
    it = torch.int32 if dt == torch.float32 else torch.int64
    lo, hi = {"log": (1e-30, 1e30), "exp": (-80.0, 80.0), "pow": (0.01, 100.0), "sin": (-1e4, 1e4),
              "cos": (-14.0, 14.0)}[name.split("_")[0]]
    base = torch.empty(n + 1, dtype=dt, device="cuda")
    if name.startswith("log") or name.startswith("pow"):
        base.copy_(torch.logspace(np.log10(lo), np.log10(hi), n + 1, dtype=torch.float64, device="cuda").to(dt))
    else:
        base.copy_(torch.linspace(lo, hi, n + 1, dtype=torch.float64, device="cuda").to(dt))
    args_al = [base[:n]]
    args_un = [base[1:]]  # 4/8-byte offset -> unaligned -> plain kernel
    if name.startswith("pow"):
        y = torch.linspace(-3.0, 3.0, n + 1, dtype=torch.float64, device="cuda").to(dt)
        args_al.append(y[:n])
        args_un.append(y[1:])
    ref = api.call(name, *args_un)  # elements 1..n
    for _ in range(3):
        got = api.call(name, *[a for a in args_al])  # elements 0..n-1
        assert torch.equal(got[1:].view(it), ref[:-1].view(it)), name
        del got
    del ref, base
    torch.cuda.empty_cache()


@pytest.mark.parametrize("name", ["sin_d_u10", "cos_d_u10", "tan_d_u10"])
def test_cw1_boundary_in_small_warps(cuda, name):
    """Warps whose elements are all |x| < 15 take the branch-free CW1 body;
    |x| == 15 (still CW1 per reduction.hpp:189) and the next doubles above
    (CW2) must fall back to the selector without changing any result."""
    from paper_2001_09258_b200 import inputs as I
    n = 1 << 16
    x = I.uniform(77, n, -14.9, 14.9, np.float64)
    edge = np.array([15.0, -15.0, np.nextafter(15.0, 0.0), np.nextafter(15.0, 16.0), -np.nextafter(15.0, 16.0),
                     14.999999999999998], dtype=np.float64)
    idx = np.arange(0, n, 997)
    x[idx] = edge[np.arange(idx.size) % edge.size]
    _assert_bit_exact(name, _gpu(name, x), oracle_eval(name, x), x)


def test_chained_launches_in_place(cuda):
    """Programmatic dependent launch (tma::griddep_wait): a grid may start while
    the previous one in the stream drains, so every read of an input written
    by the previous grid must wait for it.  A chain of dependent, in-place
    calls on one stream (each reads the previous call's output) must equal
    the oracle composed the same way, over 2^24 elements (many tiles per CTA,
    back-to-back launches with no host synchronisation in between)."""
    import torch
    from paper_2001_09258_b200 import api
    n = 1 << 24
    x = unary_cases("sin_d_u10", n)[:n].copy()
    x = np.where(np.isfinite(x), np.clip(x, -700.0, 700.0), 0.5)
    buf = torch.from_numpy(x).cuda()
    chain = ["sin_d_u10", "exp_d_u10", "log_d_u35", "cos_d_u10", "exp_d_u35", "tan_d_u10"]
    for name in chain:
        api.call(name, buf, out=buf)  # in place: reads what the previous grid wrote
    sub = np.arange(0, n, 61)  # the oracle on a sample of the lanes
    exp = x[sub]
    for name in chain:
        exp = oracle_eval(name, exp)
    got = buf.cpu().numpy()[sub]
    _assert_bit_exact("chain", got, exp, x[sub])


def test_chained_launches_mixed_kernels(cuda):
    """Dependent calls across the kernel families (TMA stream,
    CTA work queue, straight-line fmodf) on one stream."""
    import torch
    from paper_2001_09258_b200 import api
    n = (1 << 22) + 77
    x, y = binary_cases("fmod_d", n)
    x, y = x[:n].copy(), y[:n].copy()
    tx, ty = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    t1 = api.call("fmod_d", tx, ty)            # CTA work queue
    t2 = api.call("exp_d_u10", t1)             # TMA stream, reads t1
    t3 = api.call("fmod_d", t2, ty)            # reads t2
    f1 = api.call("fmod_f", t3.float(), ty.float())  # straight-line streaming body
    f2 = api.call("log_f_u10", f1)
    sub = np.arange(0, n, 7)
    e1 = oracle_eval("fmod_d", x[sub], y[sub])
    e2 = oracle_eval("exp_d_u10", e1)
    e3 = oracle_eval("fmod_d", e2, y[sub])
    g1 = oracle_eval("fmod_f", e3.astype(np.float32), y[sub].astype(np.float32))
    g2 = oracle_eval("log_f_u10", g1)
    _assert_bit_exact("chain_d", t3.cpu().numpy()[sub], e3, x[sub])
    _assert_bit_exact("chain_f", f2.cpu().numpy()[sub], g2, x[sub])


@pytest.mark.parametrize("name", ["sin_d_u10", "cos_d_u10", "tan_d_u10", "sin_d_u35", "cos_d_u35", "tan_d_u35"])
def test_trig_trivial_elements_in_mixed_warps(cuda, name):
    """The class regrouping keeps |x| < 2^-27, zeros, subnormals and Inf/NaN
    out of the sorted rows and writes their closed-form result (x, 1.0 or the
    canonical NaN).  Warps mixing them with Payne-Hanek, CW2 and CW1 lanes,
    and values straddling 2^-27, must still equal the oracle bit for bit."""
    from paper_2001_09258_b200 import inputs as I
    n = 1 << 18
    rng = np.random.default_rng(2027)
    t = 2.0 ** -27
    pool = np.array([t, -t, np.nextafter(t, 0.0), -np.nextafter(t, 0.0), np.nextafter(t, 1.0), 0.0, -0.0,
                     5e-324, -5e-324, 2.2250738585072014e-308, np.inf, -np.inf, np.nan, 1e-300, 3e-9, 7.4e-9,
                     7.5e-9, 1e100, -1e300, 123456.789, 1e13, 2.0, -14.9, 15.0], dtype=np.float64)
    x = I.log_uniform(91, n, 1e-300, 1e300, np.float64, signed=True)
    sel = rng.random(n) < 0.3
    x[sel] = pool[rng.integers(0, pool.size, int(sel.sum()))]
    _assert_bit_exact(name, _gpu(name, x), oracle_eval(name, x), x)


def test_cuda_graph_capture_and_replay(cuda):
    """A chain of vem calls captured in a CUDA graph (the launches carry the
    programmatic-serialization attribute) and replayed must reproduce the
    eager results bit for bit, across replays with new input data."""
    import torch
    from paper_2001_09258_b200 import api
    n = (1 << 20) + 3
    x = torch.from_numpy(unary_cases("exp_d_u10", n)[:n].copy()).cuda()
    y = torch.from_numpy(binary_cases("pow_d_u10", n)[1][:n].copy()).cuda()
    o1, o2, o3 = torch.empty_like(x), torch.empty_like(x), torch.empty_like(x)

    def chain():
        api.call("exp_d_u10", x, out=o1)
        api.call("pow_d_u10", o1, y, out=o2)
        api.call("fmod_d", o2, y, out=o3)

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        chain()  # warm-up (occupancy queries, attributes) outside the capture
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        chain()
    for seed in range(3):
        with np.errstate(over="ignore"):
            x.copy_(torch.from_numpy(unary_cases("exp_d_u10", n)[:n].copy() * (1.0 + seed)).cuda())
        g.replay()
        torch.cuda.synchronize()
        got = o3.clone()
        chain()
        torch.cuda.synchronize()
        assert torch.equal(got.view(torch.int64), o3.view(torch.int64)), seed


@pytest.mark.gpu
def test_fmod_f_every_exponent_pair(cuda):
    """fmod_f (one straight-line streaming body, fmod_f_flat) on every
    (exponent of x, exponent of y) pair of binary32, subnormals included,
    random mantissas and signs, plus |x| == |y| and mantissa-equal pairs:
    bit-identical to the oracle (== glibc fmodf)."""
    rng = np.random.default_rng(0x5EEF)
    ex, ey = np.meshgrid(np.arange(0, 255, dtype=np.uint32), np.arange(0, 255, dtype=np.uint32))
    ex, ey = np.repeat(ex.ravel(), 4), np.repeat(ey.ravel(), 4)
    k = ex.size
    mx = rng.integers(0, 1 << 23, size=k, dtype=np.uint32)
    my = rng.integers(0, 1 << 23, size=k, dtype=np.uint32)
    my[::4] = mx[::4]  # same mantissa: E-bit shifts of one value
    sx = rng.integers(0, 2, size=k, dtype=np.uint32) << 31
    sy = rng.integers(0, 2, size=k, dtype=np.uint32) << 31
    x = (sx | (ex << 23) | mx).view(np.float32)
    y = (sy | (ey << 23) | my).view(np.float32)
    x = np.concatenate([x, x[: k // 4]])
    y = np.concatenate([y, -x[: k // 4]])  # |x| == |y|
    got = _gpu("fmod_f", x, y)
    _assert_bit_exact("fmod_f", got, oracle_eval("fmod_f", x, y), x, y)
