#!/usr/bin/env python3
"""Attribute an ncu capture's per-SASS-instruction counts to source lines.

Usage: python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX ELEMS [LIB=paper_2001_09258_b200/libvem.so] [TOP=40]

Joins the report's SASS source page (address, instructions executed, stall
samples) with nvdisasm --print-line-info of the same library's cubin (the
library must be the build that was profiled), and prints warp instructions
per element (x32 = thread instructions per element for full warps) and the
share of stall samples per source line, heaviest first.
"""
import collections
import csv
import glob
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def sass_page(rep, kre):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    blocks = re.split(r'^"Kernel Name",', out, flags=re.M)[1:]
    for b in blocks:
        lines = b.splitlines()
        kname = next(csv.reader([lines[0]]))[0]
        if not re.search(kre, kname):
            continue
        rd = csv.reader(lines[1:])
        h = next(rd)
        ia, ie, iss = h.index("Address"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
        isrc = h.index("Source")
        rows = []
        for r in rd:
            if len(r) <= ie:
                continue
            try:
                rows.append((int(r[ia], 16), float(r[ie] or 0), float(r[iss] or 0), r[isrc]))
            except ValueError:
                pass
        return kname, rows
    raise SystemExit(f"no kernel matching {kre}")


def line_map(lib, kname_mangled_hint):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
    cub = glob.glob(os.path.join(d, "*.cubin"))
    maps = {}
    for c in cub:
        txt = subprocess.run(["nvdisasm", "--print-line-info", c], capture_output=True, text=True).stdout
        fn = None
        cur = None
        for ln in txt.splitlines():
            m = re.match(r"\s*\.section\s+\.text\.([^,\s]+),", ln)
            if m:
                fn = m.group(1)
                maps.setdefault(fn, {})
                continue
            m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
            if m:
                cur = (os.path.basename(m.group(1)), int(m.group(2)))
                continue
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+\S", ln)
            if m and fn and cur:
                maps[fn][int(m.group(1), 16)] = cur
    return maps


def main():
    rep, kre, elems = sys.argv[1], sys.argv[2], int(sys.argv[3])
    lib = sys.argv[4] if len(sys.argv) > 4 else os.path.join(ROOT, "paper_2001_09258_b200", "libvem.so")
    top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
    kname, rows = sass_page(rep, kre)
    maps = line_map(lib, kname)
    # runtime addresses -> offsets from the kernel's first instruction; the
    # cubin function with the same instruction count (and the functor's name)
    base = min(a for a, _, _, _ in rows)
    rows = [(a - base, n, s, src) for a, n, s, src in rows]
    ops_in_name = re.findall(r"(Op\w+|FmodQ)", kname)
    cands = [f for f in maps if len(maps[f]) == len(rows)]
    if ops_in_name:
        c2 = [f for f in cands if all(o in f for o in ops_in_name)]
        cands = c2 or cands
    best = cands[0] if cands else max(maps, key=lambda f: len(maps[f]))
    mp = maps[best]
    agg = collections.defaultdict(lambda: [0.0, 0.0])
    ops = collections.defaultdict(collections.Counter)
    for a, n, s, src in rows:
        key = mp.get(a, ("?", 0))
        agg[key][0] += n
        agg[key][1] += s
        ops[key][src.split()[0] if src.split() else "?"] += n
    tot = sum(v[0] for v in agg.values())
    ts = sum(v[1] for v in agg.values()) or 1
    print(f"{kname}\n  function {best}; {tot * 32 / elems:.1f} thread-inst/elem (full warps)")
    for key, (n, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        mix = ", ".join(f"{o}:{c * 32 / elems:.1f}" for o, c in ops[key].most_common(4))
        print(f"  {n * 32 / elems:7.2f}  {100 * s / ts:5.1f}%  {key[0]}:{key[1]}  [{mix}]")


if __name__ == "__main__":
    main()
