#!/usr/bin/env python3
"""Per-entry-point device throughput sweep (CUDA events, inputs >> L2).

Usage: python tools/perf_sweep.py [log2_n=26] [filter]
Prints one JSON line per entry point: Gelem/s, HBM GB/s (algorithmic bytes),
fraction of the measured HBM peak.
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2001_09258_b200 import _lib, api, build  # noqa: E402
from paper_2001_09258_b200 import inputs as I  # noqa: E402

CFG = {"sin": 3, "cos": 3, "tan": 3, "atan": 5, "exp": 2, "log": 2, "pow": 2, "fmod": 4, "asin": 6, "acos": 6,
       "atan2": 6, "fdim": 6}


def main():
    build.build()
    lg = int(sys.argv[1]) if len(sys.argv) > 1 else 26
    flt = sys.argv[2] if len(sys.argv) > 2 else ""
    n = 1 << lg
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6553.6
    for name in sorted(_lib.ALL):
        if flt and flt not in name:
            continue
        fn, p = name.split("_")[0], name.split("_")[1]
        cfg = CFG[fn]
        if name.startswith(("sin_d", "cos_d")) and not name.endswith("_ph"):
            cfg = 1
        if name.startswith("atan_f"):
            cfg = 6
        arrs = I.config_inputs(cfg, fn, p, n)
        ts = [torch.from_numpy(a).cuda() for a in arrs]
        out = torch.empty_like(ts[0])
        for _ in range(3):
            api.call(name, *ts, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        e0.record()
        for _ in range(reps):
            api.call(name, *ts, out=out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        bpe = ts[0].element_size() * (len(ts) + 1)
        gel = n / ms / 1e6
        gbs = gel * bpe
        print(json.dumps({"fn": name, "cfg": cfg, "n": n, "ms": round(ms, 4), "gelem_s": round(gel, 2),
                          "gb_s": round(gbs, 1), "hbm_frac": round(gbs / peak, 3)}), flush=True)
        del ts, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
