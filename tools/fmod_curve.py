#!/usr/bin/env python3
"""fmod throughput vs exponent gap on the GPU (PAPER.md:1178-1189 step curve;
SURVEY.md 8(f).4).

For each gap E, 2^lg pairs with |x|/|y| in [2^E, 2^(E+1)) (random mantissas
and signs), timed through vem_fmod_d / vem_fmod_f with CUDA events; prints
one JSON line per (precision, E): Gelem/s and the long-division step count
ceil(E/50) of the kernels' algorithm (DESIGN.md §4 fmod).
Usage: python tools/fmod_curve.py [lg=24]
"""
import json
import math
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2001_09258_b200 import api, build  # noqa: E402
from paper_2001_09258_b200 import inputs as I  # noqa: E402


def pairs(E, n, dt, seed):
    u = I.uniform(seed, n, 1.0, 2.0, np.float64)
    v = I.uniform(seed + 1, n, 1.0, 2.0, np.float64)
    if dt == np.float32:
        ey = I.uniform(seed + 2, n, -60.0, 60.0 - E, np.float64).astype(np.int64) if E < 120 else np.full(n, -126 + 1)
    else:
        ey = I.uniform(seed + 2, n, -1000.0, 1000.0 - E, np.float64).astype(np.int64) if E < 2000 else \
            np.full(n, -1021)
    y = np.ldexp(v, ey)
    x = np.ldexp(u, ey + E)
    sx = np.where(I.uniform(seed + 3, n, 0, 1) < 0.5, -1.0, 1.0)
    return (x * sx).astype(dt), y.astype(dt)


def main():
    build.build()
    lg = int(sys.argv[1]) if len(sys.argv) > 1 else 24
    n = 1 << lg
    for dt, gaps in ((np.float64, [0, 1, 25, 50, 51, 100, 200, 400, 800, 1200, 1600, 2000]),
                     (np.float32, [0, 1, 25, 50, 51, 100, 150, 200, 240])):
        for E in gaps:
            x, y = pairs(E, n, dt, 1000 + E)
            tx, ty = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
            out = torch.empty_like(tx)
            for _ in range(3):
                api.fmod(tx, ty, out=out)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                api.fmod(tx, ty, out=out)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 10
            steps = 0 if E == 0 else math.ceil(E / 50)
            print(json.dumps({"fn": "fmod_d" if dt == np.float64 else "fmod_f", "gap": E, "steps": steps,
                              "n": n, "ms": round(ms, 4), "gelem_s": round(n / ms / 1e6, 2)}), flush=True)


if __name__ == "__main__":
    main()
