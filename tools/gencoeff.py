#!/usr/bin/env python3
"""Generate the frozen polynomial coefficient files for every kernel.

Usage:  python tools/gencoeff.py            # regenerate coeffs/*.txt + the C header
        python tools/gencoeff.py --probe NAME lo hi   # error vs term count

Each polynomial P(v) = sum_i c_i v^{p_i} approximates a transformed target
g(v) so that the kernel's final assembly has the smallest relative error; the
weight w(v) converts the polynomial's error into the relative error of the
function value ("relative-error objective").  Term counts follow
the paper where it names them (sin 9, tan 9, atan 20, log 7,
exp 13, pow-internal log 11 / exp 13); see DESIGN.md §4 for where the GPU
design departs (sin/cos are fitted on [-pi/4, pi/4] because the reference
reduction, reduction.hpp:3-6, returns |r| <= pi/4).

Output file format: text, header lines starting with '#'
(name, domain, weighted max error), then one term per line:
    power hex64(hi) [hex64(lo)]
"""
from __future__ import annotations

import argparse
import os
import sys

import mpmath as mp

sys.path.insert(0, os.path.dirname(__file__))
from remez import fit_rounded  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

mp.mp.prec = 200
LN2 = mp.log(2)


def _safe(f, v0, eps="1e-25"):
    def g(v):
        if abs(v) < mp.mpf(eps):
            return v0(v)
        return f(v)
    return g


# ---------------------------------------------------------------- targets
# odd functions f(r) = r + r*z*Q(z), z = r^2 : Q(z) = (f(r)/r - 1)/z
def odd_target(f, q0):
    def g(z):
        r = mp.sqrt(z)
        return (f(r) / r - 1) / z
    return _safe(g, lambda z: mp.mpf(q0))


def odd_weight(f):
    def w(z):
        r = mp.sqrt(z)
        return z * r / abs(f(r))
    return w


# cos(r) = 1 - z/2 + z^2*C(z)
def cos_target():
    return _safe(lambda z: (mp.cos(mp.sqrt(z)) - 1 + z / 2) / (z * z), lambda z: mp.mpf(1) / 24)


def cos_weight():
    return lambda z: z * z / mp.cos(mp.sqrt(z))


# exp(r) = 1 + r + r^2*E(r)
def exp_target():
    return _safe(lambda r: (mp.exp(r) - 1 - r) / (r * r), lambda r: mp.mpf(1) / 2 + r / 6)


def exp_weight():
    return lambda r: r * r / mp.exp(r)


# exp(r) = 1 + r*E(r)   (short forms)
def exp1_target():
    return _safe(lambda r: (mp.exp(r) - 1) / r, lambda r: 1 + r / 2)


def exp1_weight():
    return lambda r: abs(r) / mp.exp(r)


# log(m) = 2s + s*z*L(z), s = (m-1)/(m+1), z = s^2 ; weight relative to log(m)
def log_target():
    def g(z):
        s = mp.sqrt(z)
        return (2 * mp.atanh(s) - 2 * s) / (s * z)
    return _safe(g, lambda z: mp.mpf(2) / 3)


def log_weight():
    def w(z):
        s = mp.sqrt(z)
        return s * z / abs(2 * mp.atanh(s))
    return w


# log1p(r) = r - r^2/2 + r^3*Q(r)   (table-driven log core)
def log1p3_target():
    return _safe(lambda r: (mp.log1p(r) - r + r * r / 2) / (r ** 3), lambda r: mp.mpf(1) / 3 - r / 4)


def log1p3_weight():
    return lambda r: abs(r ** 3 / mp.log1p(r))


# log1p(r) = r + r^2*Q(r)   (f32 table-driven log)
def log1p2_target():
    return _safe(lambda r: (mp.log1p(r) - r) / (r * r), lambda r: -mp.mpf(1) / 2 + r / 3)


def log1p2_weight():
    return lambda r: abs(r * r / mp.log1p(r))


# exp(r) = 1 + r + r^2/2 + r^3*Q(r)   (table-driven exp core)
def exp3_target():
    return _safe(lambda r: (mp.exp(r) - 1 - r - r * r / 2) / (r ** 3), lambda r: mp.mpf(1) / 6 + r / 24)


def exp3_weight():
    return lambda r: abs(r ** 3) / mp.exp(r)


# ---------------------------------------------------------------- registry
# name: (target, weight, domain lo, domain hi, powers, dd_terms, description)
R_TRIG = mp.mpf("0.80")          # |r| bound after CW1/CW2/PH (CW2 slack)
R_TRIG_F = mp.mpf("0.7854")       # f32 reduction in binary64: |r| <= pi/4 (1+2^-30)
H_TAN = R_TRIG / 2
S_LOG = mp.mpf("0.2")             # |s| for m in [0.75, 1.5)
R_EXP = LN2 / 2 * mp.mpf("1.0001")
T_PI8 = mp.tan(mp.pi / 8) * mp.mpf("1.0001")

R_L1P = mp.mpf(2) ** -8 * mp.mpf("1.01")
R_EXPJ = LN2 / 256 * mp.mpf("1.01")

SPECS = {
    # ---- table-driven cores
    "log1p_d": (log1p3_target(), log1p3_weight(), -R_L1P, R_L1P, list(range(6)), 0,
                "log1p(r) = r - r^2/2 + r^3*P(r), |r|<=2^-8 (table-driven log)"),
    "log1p_d_u35": (log1p3_target(), log1p3_weight(), -R_L1P, R_L1P, list(range(5)), 0,
                    "log1p(r) = r - r^2/2 + r^3*P(r), |r|<=2^-8 (u35)"),
    "expj_d": (exp3_target(), exp3_weight(), -R_EXPJ, R_EXPJ, list(range(3)), 0,
               "exp(r) = 1 + r + r^2/2 + r^3*P(r), |r|<=ln2/256 (table-driven exp)"),
    "log1p_f": (log1p2_target(), log1p2_weight(), -R_L1P, R_L1P, list(range(3)), 0,
                "f32 log1p(r) = r + r^2*P(r), |r|<=2^-8"),
    "log1p_f_u35": (log1p2_target(), log1p2_weight(), -R_L1P, R_L1P, list(range(2)), 0,
                    "f32 log1p(r) = r + r^2*P(r), |r|<=2^-8 (u35)"),
    # ---- float64 (u10 unless suffixed)
    "sin_d": (odd_target(mp.sin, -1 / mp.mpf(6)), odd_weight(mp.sin), 0, R_TRIG ** 2, list(range(6)), 0,
              "sin(r) = r + r*z*P(z), z=r^2, |r|<=0.80"),
    "cos_d": (cos_target(), cos_weight(), 0, R_TRIG ** 2, list(range(6)), 0,
              "cos(r) = 1 - z/2 + z^2*P(z), z=r^2, |r|<=0.80"),
    "tan_d": (odd_target(mp.tan, 1 / mp.mpf(3)), odd_weight(mp.tan), 0, H_TAN ** 2, list(range(9)), 0,
              "tan(h) = h + h*z*P(z), z=h^2, |h|<=0.40 (half angle, 10 terms)"),
    "atan_d": (odd_target(mp.atan, -1 / mp.mpf(3)), odd_weight(mp.atan), 0, T_PI8 ** 2, list(range(11)), 0,
               "atan(b) = b + b*z*P(z), z=b^2, |b|<=tan(pi/8) (12 terms)"),
    "exp_d": (exp_target(), exp_weight(), -R_EXP, R_EXP, list(range(11)), 0,
              "exp(r) = 1 + r + r^2*P(r), |r|<=ln2/2 (13 terms)"),
    "exp_d_u35": (exp_target(), exp_weight(), -R_EXP, R_EXP, list(range(10)), 0,
                  "exp(r) = 1 + r + r^2*P(r), |r|<=ln2/2 (12 terms)"),
    # ---- float64, SPEC.md 8(f) additions (asin/acos fold, u35 trig/atan)
    "asin_d": (odd_target(mp.asin, 1 / mp.mpf(6)), odd_weight(mp.asin), 0, mp.mpf("0.2501"), list(range(13)), 0,
               "asin(t) = t + t*z*P(z), z=t^2, |t|<=0.5 (asin/acos fold)"),
    "asin_d_u35": (odd_target(mp.asin, 1 / mp.mpf(6)), odd_weight(mp.asin), 0, mp.mpf("0.2501"), list(range(12)), 0,
                   "asin(t) = t + t*z*P(z), z=t^2, |t|<=0.5 (u35)"),
    "sin_d_u35": (odd_target(mp.sin, -1 / mp.mpf(6)), odd_weight(mp.sin), 0, R_TRIG ** 2, list(range(6)), 0,
                  "sin(r) = r + r*z*P(z), z=r^2, |r|<=0.80 (u35)"),
    "cos_d_u35": (cos_target(), cos_weight(), 0, R_TRIG ** 2, list(range(5)), 0,
                  "cos(r) = 1 - z/2 + z^2*P(z), z=r^2, |r|<=0.80 (u35)"),
    "atan_d_u35": (odd_target(mp.atan, -1 / mp.mpf(3)), odd_weight(mp.atan), 0, T_PI8 ** 2, list(range(10)), 0,
                   "atan(b) = b + b*z*P(z), z=b^2, |b|<=tan(pi/8) (u35)"),
    # ---- float32 (binary64 internals)
    "sin_f": (odd_target(mp.sin, -1 / mp.mpf(6)), odd_weight(mp.sin), 0, R_TRIG_F ** 2, list(range(4)), 0,
              "f32 sin(r) = r + r*z*P(z), |r|<=pi/4"),
    "cos_f": (cos_target(), cos_weight(), 0, R_TRIG_F ** 2, list(range(4)), 0,
              "f32 cos(r) = 1 - z/2 + z^2*P(z), |r|<=pi/4"),
    "tan_f": (odd_target(mp.tan, 1 / mp.mpf(3)), odd_weight(mp.tan), 0, R_TRIG_F ** 2, list(range(9)), 0,
              "f32 tan(r) = r + r*z*P(z), |r|<=pi/4"),
    "exp_f": (exp1_target(), exp1_weight(), -R_EXP, R_EXP, list(range(7)), 0,
              "f32 exp(r) = 1 + r*P(r), |r|<=ln2/2"),
    "exp_f_u35": (exp1_target(), exp1_weight(), -R_EXP, R_EXP, list(range(6)), 0,
                  "f32 exp u35 (r) = 1 + r*P(r)"),
}


def hexd(x: float) -> str:
    return float(x).hex()


def gen_one(name, ngrid=2000):
    g, w, lo, hi, powers, ddn, desc = SPECS[name]
    lo = mp.mpf(lo)
    hi = mp.mpf(hi)
    if lo == 0:
        lo = hi * mp.mpf("1e-12")
    out, err = fit_rounded(g, w, lo, hi, powers, dd_terms=ddn, ngrid=ngrid)
    return out, err, desc, (lo, hi)


def write_all(names):
    os.makedirs(os.path.join(ROOT, "coeffs"), exist_ok=True)
    hdr = [
        "/* GENERATED by tools/gencoeff.py -- do not edit.  Frozen minimax",
        " * coefficients (SPEC.md:318-342); shared data for the CUDA kernels",
        " * (paper_2001_09258_b200/csrc) and the CPU oracle (oracle/). */",
        "#ifndef VEM_COEFFS_H",
        "#define VEM_COEFFS_H",
        "",
    ]
    for name in names:
        out, err, desc, (lo, hi) = gen_one(name)
        le = float(mp.log(err, 2)) if err > 0 else -999.0
        path = os.path.join(ROOT, "coeffs", f"{name}.txt")
        with open(path, "w") as f:
            f.write(f"# name: {name}\n# form: {desc}\n")
            f.write(f"# domain: [{mp.nstr(lo, 8)}, {mp.nstr(hi, 8)}]\n")
            f.write(f"# max weighted (relative) error after rounding: 2^{le:.2f}\n")
            for p, c_hi, c_lo in out:
                if c_lo is None:
                    f.write(f"{p} {hexd(c_hi)}\n")
                else:
                    f.write(f"{p} {hexd(c_hi)} {hexd(c_lo)}\n")
        print(f"{name:12s} terms={len(out):2d} err=2^{le:.2f}", flush=True)
        up = name.upper()
        hdr.append(f"/* {name}: {desc}; rel err 2^{le:.2f} */")
        hdr.append(f"#define VEM_{up}_N {len(out)}")
        for p, c_hi, c_lo in out:
            hdr.append(f"#define VEM_{up}_C{p} {hexd(c_hi)}")
            if c_lo is not None:
                hdr.append(f"#define VEM_{up}_C{p}L {hexd(c_lo)}")
        hdr.append("")
    hdr.append("#endif")
    hpath = os.path.join(ROOT, "paper_2001_09258_b200", "csrc", "vem_coeffs.h")
    with open(hpath, "w") as f:
        f.write("\n".join(hdr) + "\n")


def header_from_files(names):
    """Regenerate the C header from the frozen coeffs/*.txt (no refit)."""
    hdr = [
        "/* GENERATED by tools/gencoeff.py from the coeffs/ files -- do not edit.",
        " * Frozen minimax coefficients (SPEC.md:318-342); shared data for the",
        " * CUDA kernels (paper_2001_09258_b200/csrc) and the CPU oracle (oracle/).",
        " * VEM_<NAME>_ARR lists the binary64 (hi) coefficients by ascending power;",
        " * VEM_<NAME>_C<p>L is the lo limb of a double-double coefficient. */",
        "#ifndef VEM_COEFFS_H",
        "#define VEM_COEFFS_H",
        "",
    ]
    for name in names:
        path = os.path.join(ROOT, "coeffs", f"{name}.txt")
        terms = []
        meta = []
        for line in open(path):
            if line.startswith("#"):
                meta.append(line[1:].strip())
                continue
            parts = line.split()
            if not parts:
                continue
            terms.append((int(parts[0]), parts[1], parts[2] if len(parts) > 2 else None))
        up = name.upper()
        hdr.append("/* " + "; ".join(meta) + " */")
        hdr.append(f"#define VEM_{up}_N {len(terms)}")
        for p, hi, lo in terms:
            hdr.append(f"#define VEM_{up}_C{p} {hi}")
            if lo is not None:
                hdr.append(f"#define VEM_{up}_C{p}L {lo}")
        hdr.append(f"#define VEM_{up}_ARR {{ " + ", ".join(hi for _, hi, _ in terms) + " }")
        hdr.append("")
    hdr.append("#endif")
    hpath = os.path.join(ROOT, "paper_2001_09258_b200", "csrc", "vem_coeffs.h")
    with open(hpath, "w") as f:
        f.write("\n".join(hdr) + "\n")


def probe(name, a, b):
    g, w, lo, hi, powers, ddn, desc = SPECS[name]
    lo = mp.mpf(lo)
    hi = mp.mpf(hi)
    if lo == 0:
        lo = hi * mp.mpf("1e-12")
    for n in range(a, b + 1):
        out, err = fit_rounded(g, w, lo, hi, list(range(n)), dd_terms=ddn, ngrid=1200)
        print(name, n, f"2^{float(mp.log(err, 2)):.2f}", flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--probe", nargs=3)
    ap.add_argument("--only", nargs="*")
    ap.add_argument("--header-only", action="store_true")
    a = ap.parse_args()
    if a.header_only:
        header_from_files(list(SPECS))
    elif a.probe:
        probe(a.probe[0], int(a.probe[1]), int(a.probe[2]))
    else:
        write_all(a.only or list(SPECS))
        header_from_files(list(SPECS))
