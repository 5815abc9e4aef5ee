"""fmod exactness (SPEC.md:604 criterion 2): the oracle's staged-divisor long
division is bit-identical to glibc fmod / fmodf (which are exact), including
|x/y| > DBL_MAX where SLEEF/the paper return NaN, and its
iteration count obeys the Appendix C bound adapted to 50 bits per step."""
from __future__ import annotations

import ctypes
import math
import os

import numpy as np

from cases import rnd_bits
from oracle_lib import BUILD, oracle_eval
from paper_2001_09258_b200 import inputs as I

D, F = np.float64, np.float32


def _eq(a, b):
    return np.array_equal(np.asarray(a).view(np.uint64 if a.dtype == D else np.uint32),
                          np.asarray(b).view(np.uint64 if b.dtype == D else np.uint32))


def _glibc(x, y):
    with np.errstate(all="ignore"):
        r = np.fmod(x, y)
    nan = np.isnan(r)
    r = r.copy()
    r[nan] = np.array([np.nan], dtype=r.dtype)[0]
    if r.dtype == D:
        r.view(np.uint64)[nan] = 0x7FF8000000000000
    else:
        r.view(np.uint32)[nan] = 0x7FC00000
    return r


def test_fmod_d_config4_bit_exact():
    x, y = I.config_inputs(4, "fmod", "d", 200000)
    assert _eq(oracle_eval("fmod_d", x, y), _glibc(x, y))


def test_fmod_f_config4_bit_exact():
    x, y = I.config_inputs(4, "fmod", "f", 200000)
    assert _eq(oracle_eval("fmod_f", x, y), _glibc(x, y))


def test_fmod_random_bits_and_subnormals():
    for dt in (D, F):
        x, y = rnd_bits(41, 200000, dt), rnd_bits(42, 200000, dt)
        assert _eq(oracle_eval("fmod_d" if dt == D else "fmod_f", x, y), _glibc(x, y))
    sub = np.array([5e-324, 1e-310, 2.2250738585072014e-308, 1.7976931348623157e308, 1e300, 3e-300, 0.75, 1e40])
    xs, ys = np.meshgrid(sub, sub, indexing="ij")
    xs, ys = xs.ravel(), ys.ravel()
    assert _eq(oracle_eval("fmod_d", xs, ys), _glibc(xs, ys))
    assert _eq(oracle_eval("fmod_d", -xs, ys), _glibc(-xs, ys))


def test_fmod_ratio_sweep_and_iteration_bound():
    """PAPER.md §7.1 generation law: d ~ U[1,100], n ~ U[0.95 r d, 1.05 r d],
    r = 1..1e25; exact vs glibc; iterations <= ceil(log2(n/d)/50) + 1."""
    L = ctypes.CDLL(os.path.join(BUILD, "libvem_oracle.so"))
    L.vo_fmod_d_iters.argtypes = [ctypes.c_double, ctypes.c_double]
    L.vo_fmod_d_iters.restype = ctypes.c_int
    rng = np.random.default_rng(3)
    for r in [1, 10, 1e5, 1e10, 1e15, 1e20, 1e25]:
        d = rng.uniform(1, 100, 5000)
        n = rng.uniform(0.95 * r * d, 1.05 * r * d)
        assert _eq(oracle_eval("fmod_d", n, d), _glibc(n, d))
        for a, b in zip(n[:200], d[:200]):
            it = L.vo_fmod_d_iters(a, b)
            bound = math.ceil(max(0.0, math.log2(a / b)) / 50) + 1
            assert it <= bound, (a, b, it, bound)


def test_fmod_spec_examples():
    x = np.array([1e40, 5.5, 7.0, -7.0, 0.0, -0.0, np.inf, 1.0, 1.0, np.nan, 1.0])
    y = np.array([0.75, 2.0, 7.0, 7.0, 3.0, 3.0, 1.0, np.inf, 0.0, 1.0, np.nan])
    assert _eq(oracle_eval("fmod_d", x, y), _glibc(x, y))


def test_fmod_first_step_matches_paper_example_value():
    """Fig. 2: 1e40 mod 0.75 = 0.25 (final value pinned;
    the printed intermediate depends on the quotient rule)."""
    assert oracle_eval("fmod_d", np.array([1e40]), np.array([0.75]))[0] == 0.25


def test_fmod_signed_step_schedule_model(tmp_path):
    """The device step (vem_math.cuh fmod_stepn_rs: signed remainders,
    Q = rint(rs RN(1/md)), one fix-up at the end) restated in C: every step
    exact (binary128 check) with |V| <= md, and 10^6 pending pairs (random
    bits, config-4-like, extreme divisor mantissas, subnormals) equal to
    glibc fmod bit for bit."""
    import subprocess
    src = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cpp", "fmod_signed_step.c")
    exe = str(tmp_path / "fss")
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", src, "-o", exe, "-lm", "-lquadmath"], check=True)
    out = subprocess.run([exe, "1600000"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "mismatches=0 bad_steps=0" in out.stdout
