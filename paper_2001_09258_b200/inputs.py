"""Deterministic synthetic inputs for the BASELINE.json configurations.

There is no public dataset: the paper times uniform arguments on fixed
intervals; BASELINE.json's five configs name
the domains used here (seeded synthetic stand-ins).

Every array is a pure function of (recipe, global element index): a
counter-based SplitMix64 stream per (config, function, operand), so any
slice [offset, offset + n) -- a shard, a chunk, a prefix -- can be generated
on its own, on the host (numpy here, `oracle/vem_gen_host.c` for full-size
arrays) or on the device (`csrc/vem_aux.cu`, used by bench.py), and the
three produce the SAME bits.  Only IEEE-754 basic operations in a fixed
order are used (no libm, no fma):

  u       = (splitmix64(seed, i) >> 11) * 2^-53               in [0, 1)
  uniform = a + (b - a) * u
  log-uniform on [lo, hi]:
          L = l0 + (l1 - l0) * u,  l0 = log2(lo), l1 = log2(hi)  (host constants)
          k = floor(L), f = L - k (exact), p = 2^f by a fixed 14-term
          Horner polynomial (mul then add, each rounded), x = p * 2^k (exact)
          -- log-uniform up to the polynomial's ~1e-13 relative error, which
          only perturbs the distribution, never reproducibility
  binary32: computed in binary64, clipped to [FLT_MIN, FLT_MAX] (log-uniform),
          then rounded to nearest
  sign    = top bit of splitmix64(seed ^ 0x5151, i)
  config-5 specials: u' = unit(seed ^ 0xC0FFEE) < 0.01 picks the element,
          splitmix64(seed ^ 0xBEEF) mod 9 picks one of
          {+0, -0, +inf, -inf, NaN, min subnormal, random subnormal, +-DBL_MAX},
          the random subnormal's bits from splitmix64(seed ^ 0xD00D) | 1.
"""
from __future__ import annotations

import math

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
M64 = 0xFFFFFFFFFFFFFFFF


def splitmix64(seed: int, n: int, offset: int = 0) -> np.ndarray:
    """Element i (global index offset..offset+n-1) = SplitMix64 output #(i+1)."""
    with np.errstate(over="ignore"):
        i = np.arange(offset + 1, offset + n + 1, dtype=np.uint64)
        z = np.uint64(seed & M64) + i * GOLDEN
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def unit(seed: int, n: int, offset: int = 0) -> np.ndarray:
    return (splitmix64(seed, n, offset) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


# 2^f on [0, 1): Taylor coefficients (ln 2)^k / k!, k = 0..13, as binary64
# literals (the device and C generators carry the same 14 constants).
EXP2_C = [float.fromhex(h) for h in (
    "0x1.0000000000000p+0", "0x1.62e42fefa39efp-1", "0x1.ebfbdff82c58fp-3", "0x1.c6b08d704a0c0p-5",
    "0x1.3b2ab6fba4e77p-7", "0x1.5d87fe78a6731p-10", "0x1.430912f86c787p-13", "0x1.ffcbfc588b0c7p-17",
    "0x1.62c0223a5c824p-20", "0x1.b5253d395e7c4p-24", "0x1.e4cf5158b8ecap-28", "0x1.e8cac7351bb25p-32",
    "0x1.c3bd650fc2986p-36", "0x1.816193166d0f9p-40")]


def exp2_repro(L: np.ndarray) -> np.ndarray:
    """2^L for |L| < 1022 with normal results: fixed-order IEEE ops only."""
    k = np.floor(L)
    f = L - k
    p = np.full_like(f, EXP2_C[13])
    for c in EXP2_C[12::-1]:
        p = p * f + c
    return np.ldexp(p, k.astype(np.int64))


def uniform(seed, n, a, b, dtype=np.float64, offset: int = 0):
    u = unit(seed, n, offset)
    return (a + (b - a) * u).astype(dtype)


FLT_MIN = float(np.finfo(np.float32).tiny)
FLT_MAX = float(np.finfo(np.float32).max)


def log_uniform(seed, n, a, b, dtype=np.float64, signed=False, offset: int = 0):
    u = unit(seed, n, offset)
    l0, l1 = math.log2(a), math.log2(b)
    v = exp2_repro(l0 + (l1 - l0) * u)
    if dtype == np.float32:
        v = np.minimum(np.maximum(v, FLT_MIN), FLT_MAX)
    v = v.astype(dtype)
    if signed:
        s = (splitmix64(seed ^ 0x5151, n, offset) >> np.uint64(63)).astype(bool)
        v = np.where(s, -v, v)
    return v


SPECIALS_D = np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, 0.0, 1.7976931348623157e308,
                       -1.7976931348623157e308], dtype=np.float64)


def overlay_specials(v: np.ndarray, seed: int, frac: float = 0.01, offset: int = 0) -> np.ndarray:
    """Replace ~frac of the entries by the 9 config-5 specials (uniformly)."""
    n = v.size
    u = unit(seed ^ 0xC0FFEE, n, offset)
    pick = u < frac
    which = (splitmix64(seed ^ 0xBEEF, n, offset) % np.uint64(9)).astype(np.int64)
    out = v.copy()
    sp = SPECIALS_D[which].astype(v.dtype)
    # entry 6: random subnormal
    sub = (splitmix64(seed ^ 0xD00D, n, offset) & np.uint64((1 << 52) - 1)) | np.uint64(1)
    sub = sub.view(np.float64).astype(v.dtype)
    sp = np.where(which == 6, sub, sp)
    out[pick] = sp[pick]
    return out


# --------------------------------------------------------------- recipes
FN_IDX = {"sin": 0, "cos": 1, "tan": 2, "atan": 3, "exp": 4, "log": 5, "pow": 6, "fmod": 7, "asin": 8, "acos": 9,
          "atan2": 10, "fdim": 11}

# recipe kinds (shared with vem_aux.cu / vem_gen_host.c)
K_UNIFORM, K_LOGUNIFORM = 0, 1


def seed_for(cfg: int, fn_idx: int) -> int:
    return 0x5EEF0000 + cfg * 16 + fn_idx


def _U(seed, a, b, f32):
    return {"kind": K_UNIFORM, "seed": seed & M64, "a": float(a), "b": float(b), "sign": 0, "specials": 0,
            "spec_seed": 0, "f32": int(f32)}


def _LU(seed, lo, hi, f32, signed=False, specials=False):
    return {"kind": K_LOGUNIFORM, "seed": seed & M64, "a": math.log2(lo), "b": math.log2(hi), "sign": int(signed),
            "specials": int(specials), "spec_seed": seed & M64, "f32": int(f32)}


def config_recipes(cfg: int, fn: str, prec: str):
    """One recipe per operand for BASELINE.json config `cfg` (1-based)."""
    f32 = prec == "f"
    s = seed_for(cfg, FN_IDX[fn] + (8 if f32 else 0))
    if cfg == 1:
        return [_U(s, -np.pi, np.pi, f32)]
    if cfg == 2:
        if not f32:
            if fn == "exp":
                return [_U(s, -700.0, 700.0, f32)]
            if fn == "log":
                return [_LU(s, 1e-300, 1e300, f32)]
            if fn == "pow":
                return [_LU(s, 1e-10, 1e10, f32), _U(s ^ 0xABCD, -30.0, 30.0, f32)]
        else:
            if fn == "exp":
                return [_U(s, -87.0, 88.0, f32)]
            if fn == "log":
                return [_LU(s, 1e-37, 3e38, f32)]
            if fn == "pow":
                return [_LU(s, 1e-3, 1e3, f32), _U(s ^ 0xABCD, -10.0, 10.0, f32)]
    if cfg == 3:
        return [_LU(s, 1.0, 3e38 if f32 else 1e300, f32, signed=True)]
    if cfg == 4:
        lo, hi = (1e-37, 3e38) if f32 else (1e-300, 1e300)
        return [_LU(s, lo, hi, f32, signed=True), _LU(s ^ 0x7777, lo, hi, f32, signed=True)]
    if cfg == 5:
        if f32:
            raise ValueError("config 5 is binary64 only")
        # the eight functions share ONE x array (BASELINE configs[4]): the
        # stream of config 5 / function index 0
        x = _LU(seed_for(5, 0), 1e-300, 1e300, False, signed=True, specials=True)
        if fn == "pow":
            return [x, _U(seed_for(5, 6) ^ 0xABCD, -30.0, 30.0, False)]
        if fn == "fmod":
            return [x, _LU(seed_for(5, 7) ^ 0x7777, 1e-300, 1e300, False, signed=True, specials=True)]
        return [x]
    if cfg == 6:  # SURVEY.md §8(f).1 functions (no BASELINE config): their natural domains
        lo, hi = (1e-37, 3e38) if f32 else (1e-300, 1e300)
        if fn in ("asin", "acos"):
            return [_U(s, -1.0, 1.0, f32)]
        if fn in ("atan2", "fdim"):
            return [_LU(s, lo, hi, f32, signed=True), _LU(s ^ 0x7777, lo, hi, f32, signed=True)]
        if fn == "atan":
            return [_LU(s, lo, hi, f32, signed=True)]
    raise ValueError(f"no inputs for cfg{cfg} {fn} {prec}")


def materialize(r: dict, n: int, offset: int = 0) -> np.ndarray:
    """numpy evaluation of one recipe over global indices [offset, offset + n)."""
    dt = np.float32 if r["f32"] else np.float64
    if r["kind"] == K_UNIFORM:
        return uniform(r["seed"], n, r["a"], r["b"], dt, offset)
    u = unit(r["seed"], n, offset)
    v = exp2_repro(r["a"] + (r["b"] - r["a"]) * u)
    if r["f32"]:
        v = np.minimum(np.maximum(v, FLT_MIN), FLT_MAX)
    v = v.astype(dt)
    if r["sign"]:
        sg = (splitmix64(r["seed"] ^ 0x5151, n, offset) >> np.uint64(63)).astype(bool)
        v = np.where(sg, -v, v)
    if r["specials"]:
        v = overlay_specials(v, r["spec_seed"], offset=offset)
    return v


def config_inputs(cfg: int, fn: str, prec: str, n: int, offset: int = 0):
    """Return (x,) or (x, y) for BASELINE.json config `cfg` (1-based)."""
    return tuple(materialize(r, n, offset) for r in config_recipes(cfg, fn, prec))


# --------------------------------------------------------------- checksums
def checksum(a: np.ndarray, offset: int = 0, log2chunk: int = 24) -> dict:
    """Position-keyed additive checksums per 2^log2chunk-element chunk of the
    global index space (vem_aux.h): {chunk id: sum_i fmix64(bits_i ^ i*GOLDEN)
    mod 2^64} for the chunks [offset, offset + a.size) touches."""
    bits = a.view(np.uint64) if a.dtype.itemsize == 8 else a.view(np.uint32).astype(np.uint64)
    out = {}
    j = 0
    n = a.size
    with np.errstate(over="ignore"):
        while j < n:
            g = offset + j
            c = g >> log2chunk
            m = min(((c + 1) << log2chunk) - g, n - j)
            i = np.arange(g, g + m, dtype=np.uint64)
            z = bits[j:j + m] ^ (i * GOLDEN)
            z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            z = z ^ (z >> np.uint64(31))
            out[c] = (out.get(c, 0) + int(z.sum(dtype=np.uint64))) & M64
            j += m
    return out


def recipe_struct(r: dict):
    """ctypes image of vem_recipe (csrc/vem_aux.h)."""
    import ctypes

    class VemRecipe(ctypes.Structure):
        _fields_ = [("seed", ctypes.c_uint64), ("spec_seed", ctypes.c_uint64), ("a", ctypes.c_double),
                    ("b", ctypes.c_double), ("kind", ctypes.c_int32), ("sign", ctypes.c_int32),
                    ("specials", ctypes.c_int32), ("f32", ctypes.c_int32)]

    return VemRecipe(r["seed"], r["spec_seed"], r["a"], r["b"], r["kind"], r["sign"], r["specials"], r["f32"])
