"""Shared input sets for parity tests (seeded, deterministic)."""
from __future__ import annotations

import numpy as np

from paper_2001_09258_b200 import inputs as I

D, F = np.float64, np.float32

SPECIAL_D = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, -5e-324, 2.2250738585072014e-308,
                      1.7976931348623157e308, -1.7976931348623157e308, 1.0, -1.0, 0.5, 2.0, 15.0, -15.0,
                      1e14, -1e14, 1e14 * (1 + 2 ** -52), 1.5707963267948966, 3.141592653589793, 709.782712893384,
                      -745.1332191019411, 710.0, -746.0, 1e-310, 3.0, -3.0, 0.75, 1.5], dtype=D)
SPECIAL_F = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1e-45, -1e-45, 1.1754944e-38, 3.4028235e38,
                      -3.4028235e38, 1.0, -1.0, 0.5, 2.0, 88.72283, -103.97208, 89.0, -104.0, 1.5707964,
                      3.1415927, 3.0, -3.0, 0.75, 1.5], dtype=F)


def rnd_bits(seed, n, dt):
    b = I.splitmix64(seed, n)
    if dt == F:
        return (b & np.uint64(0xFFFFFFFF)).astype(np.uint32).view(np.float32)
    return b.view(np.float64)


def _pairs(sp):
    a, b = np.meshgrid(sp, sp, indexing="ij")
    return a.ravel(), b.ravel()


def unary_cases(name: str, n: int):
    """Inputs for unary entry point `name` (e.g. 'sin_d_u10')."""
    fn, p = name.split("_")[0], name.split("_")[1]
    dt = D if p == "d" else F
    parts = [SPECIAL_D if dt == D else SPECIAL_F, rnd_bits(11, n, dt)]
    if fn in ("asin", "acos"):  # domain [-1, 1], both fold regions and the endpoints
        edge = np.array([1.0, -1.0, 0.5, -0.5, np.nextafter(0.5, 1.0), np.nextafter(1.0, 0.0)], dtype=dt)
        parts += [edge, I.uniform(13, n, -1.0, 1.0, dt), I.uniform(14, n, 0.49, 1.0, dt),
                  I.log_uniform(15, n, 1e-300 if dt == D else 1e-37, 1.0, dt, signed=True)]
        return np.concatenate(parts).astype(dt)
    cfg = {"sin": [1, 3, 5], "cos": [1, 3, 5], "tan": [3, 5], "atan": [5], "exp": [2, 5], "log": [2, 5]}[fn]
    for c in cfg:
        if c == 5 and dt == F:
            continue
        if c == 1 and dt == F:
            continue
        parts.append(I.config_inputs(c, fn, p, n)[0])
    if dt == D:
        parts.append(I.log_uniform(12, n, 1e-320, 1e14, D, signed=True))
    return np.concatenate(parts).astype(dt)


def binary_cases(name: str, n: int):
    fn, p = name.split("_")[0], name.split("_")[1]
    dt = D if p == "d" else F
    sp = SPECIAL_D if dt == D else SPECIAL_F
    a, b = _pairs(sp)
    xs, ys = [a, rnd_bits(21, n, dt)], [b, rnd_bits(22, n, dt)]
    if fn in ("atan2", "fdim"):  # wide magnitudes, both signs, equal pairs
        lo, hi = (1e-300, 1e300) if dt == D else (1e-37, 3e38)
        for seed in (31, 33):
            xs.append(I.log_uniform(seed, n, lo, hi, dt, signed=True))
            ys.append(I.log_uniform(seed + 1, n, lo, hi, dt, signed=True))
        u = I.uniform(35, n, -3, 3, dt)
        xs += [u, I.uniform(36, n, -3, 3, dt)]
        ys += [u, I.uniform(37, n, -3, 3, dt)]
        return np.concatenate(xs).astype(dt), np.concatenate(ys).astype(dt)
    cfgs = {"pow": [2, 5], "fmod": [4, 5]}[fn]
    for c in cfgs:
        if c == 5 and dt == F:
            continue
        x, y = I.config_inputs(c, fn, p, n)
        xs.append(x)
        ys.append(y)
    if fn == "pow":
        # integer exponents with negative bases exercise the odd/even rules
        xs.append(I.uniform(23, n, -30, 30, dt))
        ys.append(np.round(I.uniform(24, n, -40, 40, dt)).astype(dt))
    return np.concatenate(xs).astype(dt), np.concatenate(ys).astype(dt)
