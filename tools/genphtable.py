#!/usr/bin/env python3
"""Payne-Hanek tables for the f64 and f32 trig reductions (build-time tool).

Re-derives, with exact big-integer arithmetic, the table the reference builds
in ph_table.cpp:168-180 (layout ph_table.hpp:25-39: 1024 entries x 4 limbs,
entry for exponent E at index E+52, E in [-52, 971], 32768 bytes LE).

The reference's generator has an off-by-one (ph_table.cpp:114, `top = ... + 1`)
and stores only frac(2^E * 2/pi), which loses the quadrant term M*I(E) mod 4
in payne_hanek_reduce (reduction.hpp:106-120); SURVEY.md §0 item 4.  The table
used by the kernels is therefore the *repaired* one:

    T(E) = centred (2^E * 2/pi  mod 4)  in [-2, 2),   limbs F0..F3 cascaded
    nearest doubles: F0 = RN(T), F1 = RN(T-F0), F2 = RN(T-F0-F1), F3 = ...

Also emitted, for parity with the reference generator (after the one-line
off-by-one fix), the frac-only variant whose md5 the survey pinned
(515acbe7c5e28c4087b63b4696a730da).

The f32 table (new; the reference is double-only) serves a
three-limb binary64 Payne-Hanek: 104 entries for the biased exponents 152..255
(|x| = M*2^S, M in [2^23, 2^24), S = fe - 150; smaller exponents use entry 0),
each (2^S * 2/pi mod 4) cut into a 29-bit limb (weights 2^1..2^-27: M times it
is exact in binary64), a second 29-bit limb and a 53-bit tail, stored divided
by 2^S as three doubles plus a zero pad (3328 bytes).  The dropped bits lie
below 2^-109: an absolute error < 2^-85 quadrants, against a smallest reduced
argument of ~2^-30 over all binary32 inputs (tests/test_oracle_accuracy.py).

The f64 integer table (new, for the kernels' own binary64 Payne-Hanek; the
reference-algorithm table above stays the parity anchor of vem_ph_reduce_d):
1025 entries for ue in [-1, 1023], W(E) = floor((2^E 2/pi mod 4) 2^190) as
three little-endian 64-bit words plus a zero pad (32800 bytes).

2/pi itself comes from mpmath at 3400 bits (no constants are copied from the
reference's embedded kTwoOverPiBits, ph_table.cpp:15-26; a test checks that the
first 2560 fractional bits agree with them).
"""
from __future__ import annotations

import hashlib
import math
import os
import struct
import sys
from fractions import Fraction

import mpmath as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NBITS = 3200


def two_over_pi_fixed(nbits=NBITS):
    """floor(2/pi * 2^nbits) as an exact integer."""
    with mp.workprec(nbits + 64):
        v = mp.mpf(2) / mp.pi
        return int(mp.floor(v * mp.mpf(2) ** nbits))


TOP = two_over_pi_fixed()


def value_2e_2pi(E):
    """2^E * 2/pi truncated to 2^(E-NBITS) resolution, as a Fraction."""
    return Fraction(TOP) * Fraction(2) ** (E - NBITS)


def cascade(T, nlimbs):
    out = []
    rem = T
    for _ in range(nlimbs):
        f = float(rem)  # correctly rounded (int/int true division)
        out.append(f)
        rem = rem - Fraction(f)
    return out


def centred_mod4(v):
    # v - 4*round(v/4)  in [-2, 2)
    q = (v / 4)
    n = q.numerator // q.denominator  # floor
    t = v - 4 * n  # in [0, 4)
    if t >= 2:
        t -= 4
    return t


def frac01(v):
    n = v.numerator // v.denominator
    return v - n


def centred_frac(v):
    # the reference window is a signed two's-complement fraction
    # (ph_table.cpp:39 `negative()`), i.e. frac in [-1/2, 1/2)
    t = frac01(v)
    if t >= Fraction(1, 2):
        t -= 1
    return t


def table_f64_mod4():
    out = []
    for i in range(1024):
        E = i - 52
        out.extend(cascade(centred_mod4(value_2e_2pi(E)), 4))
    return out


def table_f64_frac():
    out = []
    for i in range(1024):
        E = i - 52
        out.extend(cascade(centred_frac(value_2e_2pi(E)), 4))
    return out


PH_F_ENTRIES = 104
PH_F_FE0 = 152  # biased exponents <= 152 share entry 0 (no bits above 2^1 to drop)
PH_F_K = 109    # lowest kept weight 2^-109


def table_f32_fp():
    """[t0, t1, t2, 0] per entry (doubles).  |x| = M * 2^S, M in [2^23, 2^24), S
    = fe - 150 for the biased exponent fe (entry fe - 152, fe clamped to >= 152;
    for S < 2 the S = 2 entry applies unchanged, its limbs being relative to x).
    V = (2^S * 2/pi) mod 4 cut at weights 2^1..2^-27 (29 bits: M * a0 is exact in
    binary64), 2^-28..2^-56 (29 bits) and 2^-57..2^-109 (53 bits); each limb is
    stored divided by 2^S, so that x * t_k == M * a_k with the binary32 x
    converted to binary64."""
    out = []
    K = PH_F_K
    for i in range(PH_F_ENTRIES):
        S = i + PH_F_FE0 - 150
        v = TOP >> (NBITS - S - K)  # floor(2^S * 2/pi * 2^K)
        v &= (1 << (K + 2)) - 1     # mod 4
        a0 = v >> (K - 27)
        a1 = (v >> (K - 56)) & ((1 << 29) - 1)
        a2 = v & ((1 << (K - 56)) - 1)
        assert a0 < (1 << 29) and a2 < (1 << 53)
        out.extend([math.ldexp(a0, -27 - S), math.ldexp(a1, -56 - S), math.ldexp(a2, -K - S), 0.0])
    return out


PH_DI_ENTRIES = 1025
PH_DI_UEMIN = -1


def table_f64_int():
    """[w0, w1, w2, 0] per entry (64-bit LE words): W(E) = floor((2^E * 2/pi mod 4)
    * 2^190) for |x| = M * 2^E, M in [2^52, 2^53), E = ue - 52, ue in [-1, 1023]
    (unbiased exponent of x).  M * W(E) mod 2^192 holds the quadrant in its top
    two bits and 190 fraction bits below (integer Payne-Hanek for binary64)."""
    out = []
    for i in range(PH_DI_ENTRIES):
        E = i + PH_DI_UEMIN - 52
        sh = NBITS - E - 190
        v = (TOP >> sh) if sh >= 0 else (TOP << -sh)
        v &= (1 << 192) - 1
        out.extend([v & (2**64 - 1), (v >> 64) & (2**64 - 1), (v >> 128) & (2**64 - 1), 0])
    return out


def serialize_u64(words):
    return b"".join(struct.pack("<Q", w) for w in words)


def serialize_words(words):
    return b"".join(struct.pack("<I", w) for w in words)


def serialize(limbs):
    return b"".join(struct.pack("<d", x) for x in limbs)


def md5(limbs):
    return hashlib.md5(serialize(limbs)).hexdigest()


def emit_header(path, t64, t32, tdi):
    m32 = md5(t32)
    mdi = hashlib.md5(serialize_u64(tdi)).hexdigest()
    lines = [
        "/* GENERATED by tools/genphtable.py -- do not edit.",
        " * Repaired Payne-Hanek tables (centred 2^E*2/pi mod 4, cascaded nearest",
        " * doubles); layout follows ph_table.hpp:8-15 (entry E+52, 4 limbs).",
        f" * md5(f64 table, 32768 B LE) = {md5(t64)}",
        f" * md5(f32 table,  {8 * len(t32)} B LE) = {m32}",
        f" * md5(f64 integer table, {8 * len(tdi)} B LE) = {mdi} */",
        "#ifndef VEM_PH_TABLES_H",
        "#define VEM_PH_TABLES_H",
        "#define VEM_PH_D_ENTRIES 1024",
        "#define VEM_PH_D_EXPBIAS 52",
        f"#define VEM_PH_F_ENTRIES {PH_F_ENTRIES}",
        f"#define VEM_PH_F_FE0 {PH_F_FE0}",
        f'#define VEM_PH_D_MD5 "{md5(t64)}"',
        f'#define VEM_PH_F_MD5 "{m32}"',
        f"#define VEM_PH_DI_ENTRIES {PH_DI_ENTRIES}",
        f"#define VEM_PH_DI_UEMIN ({PH_DI_UEMIN})",
        f'#define VEM_PH_DI_MD5 "{mdi}"',
        "#define VEM_PH_D_INIT \\",
    ]
    for i in range(0, len(t64), 4):
        row = ", ".join(x.hex() for x in t64[i:i + 4])
        lines.append(f"  {row}, \\")
    lines.append("")
    lines.append("#define VEM_PH_F_INIT \\")
    for i in range(0, len(t32), 4):
        row = ", ".join(x.hex() for x in t32[i:i + 4])
        lines.append(f"  {row}, \\")
    lines.append("")
    lines.append("#define VEM_PH_DI_INIT \\")
    for i in range(0, len(tdi), 4):
        row = ", ".join(f"0x{w:016x}ull" for w in tdi[i:i + 4])
        lines.append(f"  {row}, \\")
    lines.append("")
    lines.append("#endif")
    with open(path, "w") as f:
        f.write("\n".join(lines) + "\n")


def main():
    t64 = table_f64_mod4()
    t32 = table_f32_fp()
    tdi = table_f64_int()
    tfr = table_f64_frac()
    print("f64 mod4 md5", md5(t64))
    print("f64 frac md5", md5(tfr))
    m32 = md5(t32)
    print("f32 fp md5", m32)
    mdi = hashlib.md5(serialize_u64(tdi)).hexdigest()
    print("f64 int md5", mdi)
    emit_header(os.path.join(ROOT, "paper_2001_09258_b200", "csrc", "vem_ph_tables.h"), t64, t32, tdi)
    os.makedirs(os.path.join(ROOT, "tests", "golden"), exist_ok=True)
    with open(os.path.join(ROOT, "tests", "golden", "ph_table_digests.txt"), "w") as f:
        f.write(f"f64_mod4 {md5(t64)}\nf64_frac {md5(tfr)}\nf32_fp {m32}\nf64_int {mdi}\n")


if __name__ == "__main__":
    sys.exit(main())
