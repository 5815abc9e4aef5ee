#!/usr/bin/env python3
"""Small driver for compute-sanitizer (memcheck / racecheck / synccheck):
one launch of each kernel family on config-domain inputs, 2^20 elements by
default -- k_stream (split fast path, binary, f32), k_trig (selector with
sorting, config 5 mix), k_queue (fmod_d work queue), the plain fallback
kernels (misaligned pointers) and the remainder loops (n not a multiple of
a tile).  Results are compared with the oracle's first-chunk checksums is
NOT done here (tests do that); this only has to run clean under the tool.

Usage: compute-sanitizer --tool memcheck python tools/sanitize_run.py [log2n]
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2001_09258_b200 import _aux, api  # noqa: E402
from paper_2001_09258_b200 import inputs as I  # noqa: E402

CASES = [("exp_d_u10", 2), ("pow_d_u10", 2), ("log_f_u10", 2), ("pow_f_u10", 2), ("sin_d_u10", 5), ("cos_d_u10", 5),
         ("tan_d_u10", 5), ("sin_d_u10", 1), ("sin_d_u10_ph", 3), ("sin_f_u10", 3), ("fmod_d", 4), ("fmod_d", 5),
         ("fmod_f", 4), ("atan2_d_u10", 6), ("fdim_f", 6)]


def main():
    n = 1 << (int(sys.argv[1]) if len(sys.argv) > 1 else 20)
    for name, cfg in CASES:
        fn, p = name.split("_")[0], name.split("_")[1]
        for m, pad in ((n, 0), (n + 77, 0), (4099, 1)):  # tiles only / + remainder / misaligned plain kernel
            ins = []
            for r in I.config_recipes(cfg, fn, p):
                t = torch.empty(m + pad, dtype=torch.float32 if r["f32"] else torch.float64, device="cuda")[pad:]
                ins.append(_aux.fill(r, t, 0))
            out = torch.empty(m + pad, dtype=ins[0].dtype, device="cuda")[pad:]
            api.call(name, *ins, out=out)
        torch.cuda.synchronize()
        print(f"{name} cfg{cfg}: ok", flush=True)


if __name__ == "__main__":
    main()
