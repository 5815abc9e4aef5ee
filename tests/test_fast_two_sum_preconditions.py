"""Preconditions behind the kernels' magnitude-ordered fast two-sums.

The oracle (oracle/vem_oracle.c) uses the 6-add two_sum (ddarith.hpp:27-35)
where the kernels use the 3-add fast two-sum (ddarith.hpp:37-44).  Both give
the same exact pair whenever the fast form is exact, so GPU == oracle bit for
bit; these tests pin the conditions that make the fast form exact:

- log_fast_d (vem_math.cuh): H.hi = E ln2 + log c is 0 or has an exponent
  >= that of L.hi ~ r for every table entry c (E = 0 case; |E| >= 1 gives
  |H.hi| >= 0.28).
- atan_d_u10 / atan2_d_u10: the -+1 and -+den pairs, sampled.
"""
import math
import os
import re

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TAB = os.path.join(ROOT, "paper_2001_09258_b200", "csrc", "vem_log_tables.h")


def _table(name):
    src = open(TAB).read()
    m = re.search(r"#define %s \\\n((?:.*\\\n)*.*)" % name, src)
    return [float.fromhex(t) for t in re.findall(r"-?0x[0-9a-fA-F.]+p[-+]?\d+", m.group(1))]


def _from_bits(u):
    return float(np.array([u], dtype=np.uint64).view(np.float64)[0])


def test_log_table_orders_the_final_two_sum():
    invc, hi = _table("VEM_LOGT_INVC_INIT"), _table("VEM_LOGT_HI_INIT")
    ln2h = float.fromhex("0x1.62e42fefa3800p-1")
    assert len(invc) == len(hi) == 256
    rmax_all = 0.0
    for i in range(256):
        rmax = 0.0
        for tmp in (i << 44, ((i + 1) << 44) - 1):  # subinterval ends (r is monotone in m)
            k = tmp >> 52
            m = _from_bits(tmp + 0x3FE8000000000000 - (k << 52))
            rmax = max(rmax, abs(m * invc[i] - 1.0))
        # L.hi = RN(r - r^2/2) in the u10 path: |L.hi| <= |r| + r^2/2,
        # rounded up by at most one ulp (a factor 1 + 2^-52)
        rmax = (rmax + rmax * rmax / 2) * (1 + 2.0 ** -52)
        rmax_all = max(rmax_all, rmax)
        if hi[i] != 0.0:
            assert math.frexp(hi[i])[1] >= math.frexp(rmax)[1], i
    for i in range(256):  # |E| >= 1
        for e in (-1.0, 1.0):
            assert abs(e * ln2h + hi[i]) > 0.28 > rmax_all


def _two_sum(a, b):
    s = a + b
    v = s - a
    return s, (a - (s - v)) + (b - v)


def _fast(a, b):
    s = a + b
    return s, b - (s - a)


def _same(p, q):
    return all(np.array_equal(x.view(np.int64), y.view(np.int64)) for x, y in zip(p, q))


def test_atan_and_atan2_pairs_match_two_sum():
    rng = np.random.default_rng(7)
    lo, hi = 0.41421356237309503, 2.414213562373095
    edges = np.array([0.5, 1.0, 2.0, lo, hi])
    a = np.concatenate([rng.uniform(lo, hi, 1 << 20), edges, np.nextafter(edges, 0), np.nextafter(edges, 9)])
    for c in (-1.0, 1.0):
        assert _same(_two_sum(a, np.full_like(a, c)), _fast(np.full_like(a, c), a))
    den = np.exp(rng.uniform(-700, 700, 1 << 20))
    # atan2_split pre-scales huge / tiny denominators by 2^-100 / 2^100: cover
    # the scaled ranges near 2^1000 and 2^-900, and subnormal numerators
    scaled = np.concatenate([np.ldexp(rng.uniform(1, 2, 1 << 16), rng.integers(995, 1024, 1 << 16)) * 2.0 ** -100,
                             np.ldexp(rng.uniform(1, 2, 1 << 16), rng.integers(-1022, -900, 1 << 16)) * 2.0 ** 100])
    den = np.concatenate([den, scaled])
    num = den * rng.uniform(lo, 1.0, den.size)
    sub_den = np.ldexp(rng.uniform(1, 2, 1 << 16), rng.integers(-1074, -1022, 1 << 16))
    sub_num = sub_den * rng.uniform(lo, 1.0, sub_den.size)  # subnormal numerators (and denominators)
    den = np.concatenate([den, sub_den])
    num = np.concatenate([num, sub_num])
    assert np.all(np.abs(den) >= np.abs(num))  # Fast2Sum's precondition
    for sg in (-1.0, 1.0):
        assert _same(_two_sum(num, sg * den), _fast(sg * den, num))
