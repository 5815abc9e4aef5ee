"""Deterministic synthetic inputs for the BASELINE.json configurations.

There is no public dataset: the paper times uniform arguments on fixed
intervals; BASELINE.json's five configs name
the domains used here.  Generation follows SURVEY.md §8(d): a counter-based
SplitMix64 stream per (config, function), u = (bits >> 11) * 2^-53, uniform
a + (b-a)u, log-uniform 10^(lg a + (lg b - lg a) u) computed on the host and
uploaded (never regenerated on the device), an independent bit for random
signs, and for config 5 a 1% special-value overlay chosen by a separate
seeded stream.
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)


def splitmix64(seed: int, n: int, offset: int = 0) -> np.ndarray:
    with np.errstate(over="ignore"):
        i = np.arange(offset + 1, offset + n + 1, dtype=np.uint64)
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + i * GOLDEN
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def unit(seed: int, n: int) -> np.ndarray:
    return (splitmix64(seed, n) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def uniform(seed, n, a, b, dtype=np.float64):
    u = unit(seed, n)
    return (a + (b - a) * u).astype(dtype)


def log_uniform(seed, n, a, b, dtype=np.float64, signed=False):
    u = unit(seed, n)
    la, lb = np.log10(a), np.log10(b)
    v = np.power(10.0, la + (lb - la) * u)
    if dtype == np.float32:
        v = np.clip(v, np.float64(np.finfo(np.float32).tiny), np.float64(np.finfo(np.float32).max))
    v = v.astype(dtype)
    if signed:
        s = (splitmix64(seed ^ 0x5151, n) >> np.uint64(63)).astype(bool)
        v = np.where(s, -v, v)
    return v


def seed_for(cfg: int, fn_idx: int) -> int:
    return 0x5EEF0000 + cfg * 16 + fn_idx


SPECIALS_D = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, 0.0, 1.7976931348623157e308,
                       -1.7976931348623157e308], dtype=np.float64)


def overlay_specials(v: np.ndarray, seed: int, frac: float = 0.01) -> np.ndarray:
    """Replace ~frac of the entries by the 9 config-5 specials (uniformly)."""
    n = v.size
    u = unit(seed ^ 0xC0FFEE, n)
    pick = u < frac
    which = (splitmix64(seed ^ 0xBEEF, n) % np.uint64(9)).astype(np.int64)
    out = v.copy()
    sp = SPECIALS_D[which].astype(v.dtype)
    # entry 6: random subnormal
    sub = (splitmix64(seed ^ 0xD00D, n) & np.uint64((1 << 52) - 1)) | np.uint64(1)
    sub = sub.view(np.float64).astype(v.dtype)
    sp = np.where(which == 6, sub, sp)
    out[pick] = sp[pick]
    return out


# --------------------------------------------------------------- configs
FN_IDX = {"sin": 0, "cos": 1, "tan": 2, "atan": 3, "exp": 4, "log": 5, "pow": 6, "fmod": 7, "asin": 8, "acos": 9,
          "atan2": 10, "fdim": 11}


def config_inputs(cfg: int, fn: str, prec: str, n: int):
    """Return (x,) or (x, y) for BASELINE.json config `cfg` (1-based)."""
    dt = np.float64 if prec == "d" else np.float32
    s = seed_for(cfg, FN_IDX[fn] + (8 if prec == "f" else 0))
    if cfg == 1:
        return (uniform(s, n, -np.pi, np.pi, dt),)
    if cfg == 2:
        if prec == "d":
            if fn == "exp":
                return (uniform(s, n, -700.0, 700.0, dt),)
            if fn == "log":
                return (log_uniform(s, n, 1e-300, 1e300, dt),)
            if fn == "pow":
                return (log_uniform(s, n, 1e-10, 1e10, dt), uniform(s ^ 0xABCD, n, -30.0, 30.0, dt))
        else:
            if fn == "exp":
                return (uniform(s, n, -87.0, 88.0, dt),)
            if fn == "log":
                return (log_uniform(s, n, 1e-37, 3e38, dt),)
            if fn == "pow":
                return (log_uniform(s, n, 1e-3, 1e3, dt), uniform(s ^ 0xABCD, n, -10.0, 10.0, dt))
    if cfg == 3:
        hi = 1e300 if prec == "d" else 3e38
        return (log_uniform(s, n, 1.0, hi, dt, signed=True),)
    if cfg == 4:
        lo, hi = (1e-300, 1e300) if prec == "d" else (1e-37, 3e38)
        return (log_uniform(s, n, lo, hi, dt, signed=True), log_uniform(s ^ 0x7777, n, lo, hi, dt, signed=True))
    if cfg == 5:
        x = overlay_specials(log_uniform(s, n, 1e-300, 1e300, dt, signed=True), s)
        if fn == "pow":
            return (x, uniform(s ^ 0xABCD, n, -30.0, 30.0, dt))
        if fn == "fmod":
            y = overlay_specials(log_uniform(s ^ 0x7777, n, 1e-300, 1e300, dt, signed=True), s ^ 0x7777)
            return (x, y)
        return (x,)
    if cfg == 6:  # SURVEY.md §8(f).1 functions (no BASELINE config): their natural domains
        lo, hi = (1e-300, 1e300) if prec == "d" else (1e-37, 3e38)
        if fn in ("asin", "acos"):
            return (uniform(s, n, -1.0, 1.0, dt),)
        if fn in ("atan2", "fdim"):
            return (log_uniform(s, n, lo, hi, dt, signed=True), log_uniform(s ^ 0x7777, n, lo, hi, dt, signed=True))
        if fn == "atan":
            return (log_uniform(s, n, lo, hi, dt, signed=True),)
    raise ValueError(f"no inputs for cfg{cfg} {fn} {prec}")
