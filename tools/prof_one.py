#!/usr/bin/env python3
"""Run one entry point on one BASELINE config's inputs (dev tool for ncu).

Usage: python tools/prof_one.py NAME[@CFG[@LOG2N]][,...] CFG [log2_n=24] [reps=3]
e.g.  ncu --set full -k regex:k_stream -s 1 -c 1 python tools/prof_one.py sin_d_u10 5 24
reps=0: each entry point runs exactly once, no warm-up (one ncu capture per
entry point with -c <number of names>).
Prints Gelem/s (CUDA events) so the same command also runs without ncu.
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2001_09258_b200 import api  # noqa: E402
from paper_2001_09258_b200 import inputs as I  # noqa: E402


def main():
    cfg = int(sys.argv[2])
    n = 1 << (int(sys.argv[3]) if len(sys.argv) > 3 else 24)
    reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
    for name in sys.argv[1].split(","):
        # NAME@CFG[@LOG2N] overrides the config (and size) per entry point
        parts = name.split("@")
        run(parts[0], int(parts[1]) if len(parts) > 1 else cfg, 1 << int(parts[2]) if len(parts) > 2 else n, reps)
        torch.cuda.empty_cache()


def run(name, cfg, n, reps):
    from paper_2001_09258_b200 import _aux
    fn, p = name.split("_")[0], name.split("_")[1]
    # config inputs generated on the device (bit-identical to inputs.py)
    ts = [_aux.fill(r, torch.empty(n, dtype=torch.float32 if r["f32"] else torch.float64, device="cuda"))
          for r in I.config_recipes(cfg, fn, p)]
    out = torch.empty_like(ts[0])
    if reps == 0:
        api.call(name, *ts, out=out)
        torch.cuda.synchronize()
        print(f"{name} cfg{cfg} n={n}: ran once")
        return
    api.call(name, *ts, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        api.call(name, *ts, out=out)
    e1.record()
    torch.cuda.synchronize()
    print(f"{name} cfg{cfg} n={n}: {n / (e0.elapsed_time(e1) / reps) / 1e6:.1f} Gelem/s")


if __name__ == "__main__":
    main()
