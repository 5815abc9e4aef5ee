#!/usr/bin/env python3
"""Max ULP error of the oracle's binary32 sin/cos/tan over ALL finite binary32
inputs against (float) of glibc's binary64 function (correctly rounded in
practice at binary32 resolution).  ~3 min per function on 8 cores.
Usage: python tools/f32_trig_maxulp.py [sin cos tan]"""
import os
import sys
from concurrent.futures import ProcessPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
CHUNK = 1 << 26


def work(args):
    fn, c = args
    from oracle_lib import oracle_eval
    x = np.arange(c * CHUNK, (c + 1) * CHUNK, dtype=np.uint64).astype(np.uint32).view(np.float32)
    fin = np.isfinite(x)
    e = oracle_eval(f"{fn}_f_u10", x).astype(np.float64)
    with np.errstate(all="ignore"):
        ref = getattr(np, fn)(x.astype(np.float64))
        ulp = np.spacing(np.abs(ref).astype(np.float32)).astype(np.float64)
        ulp = np.maximum(ulp, 2.0 ** -149)
        err = np.where(fin, np.abs(e - ref) / ulp, 0.0)
    i = int(np.argmax(err))
    return float(err[i]), float(x[i])


def main():
    fns = sys.argv[1:] or ["sin", "cos", "tan"]
    for fn in fns:
        with ProcessPoolExecutor(8) as ex:
            res = list(ex.map(work, [(fn, c) for c in range((1 << 32) // CHUNK)]))
        m = max(res)
        print(f"{fn}_f_u10: max {m[0]:.5f} ulp at x = {m[1]!r} over all finite binary32 inputs", flush=True)


if __name__ == "__main__":
    main()
