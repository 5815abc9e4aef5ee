#!/usr/bin/env python3
"""Static SASS opcode census per kernel of libvem.so (cuobjdump -sass).

Usage: python tools/sass_census.py [regex] [--top N]
Prints, per matching kernel, the instruction count and the most frequent
opcodes (base mnemonic).  Evidence for DESIGN.md §4 (FP64 vs integer/select
overhead) and for tcgen05/TMA usage (UBLKCP = cp.async.bulk).
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2001_09258_b200", "libvem.so")


def census(pattern=".", top=16):
    out = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s*Function : ", out)[1:]
    res = {}
    for f in funcs:
        name = f.split("\n", 1)[0].strip()
        dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
        if not re.search(pattern, dem):
            continue
        ops = re.findall(r"/\*[0-9a-f]{4}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", f)
        c = collections.Counter(ops)
        res[dem] = c
        print(f"{dem[:110]}\n   total {sum(c.values())}: " + ", ".join(f"{o} {n}" for o, n in c.most_common(top)))
    return res


if __name__ == "__main__":
    pat = sys.argv[1] if len(sys.argv) > 1 else "."
    census(pat)
