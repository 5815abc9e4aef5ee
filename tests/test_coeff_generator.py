"""The coefficient generator reproduces its frozen outputs (SURVEY §8(f).3,
SPEC.md:318-342): tools/gencoeff.py --header-only rebuilds csrc/vem_coeffs.h
byte for byte from coeffs/*.txt, and refitting polynomials with the Remez tool
(tools/remez.py, deterministic: fixed grid, 200-bit mpmath) gives the very
coefficients frozen in coeffs/ -- the short f32 sets in the default suite, every
set under -m slow."""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))


def _frozen(name):
    terms = []
    for line in open(os.path.join(ROOT, "coeffs", f"{name}.txt")):
        if line.startswith("#") or not line.split():
            continue
        p = line.split()
        terms.append((int(p[0]), p[1], p[2] if len(p) > 2 else None))
    return terms


def _refit(name):
    import gencoeff as G
    out, err, desc, dom = G.gen_one(name)
    return [(p, G.hexd(hi), G.hexd(lo) if lo is not None else None) for p, hi, lo in out]


def test_header_is_reproduced_from_coeff_files(tmp_path):
    hdr = os.path.join(ROOT, "paper_2001_09258_b200", "csrc", "vem_coeffs.h")
    keep = tmp_path / "vem_coeffs.h.orig"
    shutil.copy(hdr, keep)
    try:
        subprocess.run([sys.executable, os.path.join(ROOT, "tools", "gencoeff.py"), "--header-only"], check=True,
                       cwd=ROOT)
        assert open(hdr, "rb").read() == open(keep, "rb").read()
    finally:
        shutil.copy(keep, hdr)
        os.utime(hdr, (os.path.getmtime(keep), os.path.getmtime(keep)))  # do not make the built library look stale


@pytest.mark.parametrize("name", ["sin_f", "cos_f", "exp_f_u35"])
def test_refit_reproduces_frozen_coefficients(name):
    assert _refit(name) == _frozen(name), name


@pytest.mark.slow
def test_refit_reproduces_every_frozen_set():
    import gencoeff as G
    bad = [n for n in G.SPECS if _refit(n) != _frozen(n)]
    assert not bad, bad
