#!/usr/bin/env python3
"""Build the reference's own reduction/DD code into oracle/_ref/ (test-only).

Recipe:
  1. copy /root/reference/proj/core/{include,src} into oracle/_ref/src/<variant>/
     (git-ignored build area; nothing from the reference is committed);
  2. apply textual patches:
       gcc      : backend.hpp:156-157,256 -- g++ 13 drops the dependent
                  vector_size attribute; alias through explicit VT<W>
                  specialisations instead (no semantic change);
       repaired : gcc + ph_table.cpp:114 `+ 1` removed (off-by-one, defect i)
                  + `u = two_sum(u.hi, u.lo)` after each rfrac in
                  reduction.hpp:108-112 (precision, defect iii); defect ii
                  (quadrant) is fixed by feeding the mod-4 table through
                  PayneHanekTable::deserialize (see ref_shim.cpp);
  3. g++ -std=c++20 -O2 -ffp-contract=off -mfma -shared ... -> libvemref_<variant>.so

Skips (exit 0, prints why) when /root/reference is absent (the GPU box): the
prebuilt .so files travel there with the repo snapshot.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/proj/core"
OUT = os.path.join(HERE, "_ref")

VT_BLOCK = """
template <int W> struct VT;
template <> struct VT<2> {
  typedef double D __attribute__((vector_size(16)));
  typedef long long L __attribute__((vector_size(16)));
  typedef unsigned long long U __attribute__((vector_size(16)));
};
template <> struct VT<4> {
  typedef double D __attribute__((vector_size(32)));
  typedef long long L __attribute__((vector_size(32)));
  typedef unsigned long long U __attribute__((vector_size(32)));
};
template <> struct VT<8> {
  typedef double D __attribute__((vector_size(64)));
  typedef long long L __attribute__((vector_size(64)));
  typedef unsigned long long U __attribute__((vector_size(64)));
};

}  // namespace detail
"""


def _sub(text, old, new, count=1):
    n = text.count(old)
    if n != count:
        raise SystemExit(f"ref_build: patch anchor found {n}x (want {count}): {old!r}")
    return text.replace(old, new)


def patch_gcc(root):
    p = os.path.join(root, "include", "vem", "backend.hpp")
    t = open(p).read()
    t = _sub(t, "}  // namespace detail\n", VT_BLOCK)
    t = _sub(t, "  using D = double __attribute__((vector_size(W * 8)));\n"
                "  using L = long long __attribute__((vector_size(W * 8)));\n",
             "  using D = typename detail::VT<W>::D;\n  using L = typename detail::VT<W>::L;\n")
    t = _sub(t, "    using U = unsigned long long __attribute__((vector_size(W * 8)));\n",
             "    using U = typename detail::VT<W>::U;\n")
    open(p, "w").write(t)


def patch_repair(root):
    p = os.path.join(root, "src", "ph_table.cpp")
    t = open(p).read()
    t = _sub(t, "int top = int(1023 - biased) + 1;", "int top = int(1023 - biased);")
    open(p, "w").write(t)
    p = os.path.join(root, "include", "vem", "reduction.hpp")
    t = open(p).read()
    t = _sub(t, "  u = rfrac(u, q);\n", "  u = rfrac(u, q);\n  u = two_sum<B>(u.hi, u.lo);\n", count=3)
    open(p, "w").write(t)


def build(variant):
    src = os.path.join(OUT, "src", variant)
    if os.path.exists(src):
        shutil.rmtree(src)
    shutil.copytree(REF, src)
    for dp, _, fs in os.walk(src):
        for f in fs:
            os.chmod(os.path.join(dp, f), 0o644)
    patch_gcc(src)
    if variant == "repaired":
        patch_repair(src)
    so = os.path.join(OUT, f"libvemref_{variant}.so")
    cmd = ["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-mfma", "-fPIC", "-shared",
           "-I", os.path.join(src, "include"), os.path.join(HERE, "ref_shim.cpp"),
           os.path.join(src, "src", "ph_table.cpp"), "-o", so]
    subprocess.run(cmd, check=True)
    return so


def main():
    if not os.path.isdir(REF):
        print("ref_build: /root/reference absent; using prebuilt oracle/_ref/*.so if present")
        return 0
    os.makedirs(OUT, exist_ok=True)
    for v in ("gcc", "repaired"):
        print("built", build(v))
    return 0


if __name__ == "__main__":
    sys.exit(main())
