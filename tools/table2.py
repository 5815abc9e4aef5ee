#!/usr/bin/env python3
"""The paper's Table 2 rows, run on the B200 (dev tool).

Usage: python tools/table2.py [log2_n=26] [out.md]
For every float64 row of the paper's reciprocal-throughput table (function,
accuracy, argument domain), draws 2^log2_n arguments
uniformly on the domain (seeded, as the paper does),
times the vem entry point with CUDA events (10 launches after warm-up,
inputs > L2) and prints one JSON line per row: GPU Gelem/s and ns/element,
the paper's published SLEEF 3.4 AVX2 1-core figure for the row, and upstream
SLEEF 3.8 AVX-512 on one core of this host on a 2^20-element sample of the
same arguments (oracle/_build/libvem_sleef.so; bench infrastructure).  The
fmod row is a figure in the paper (step function vs ratio): see
tools/fmod_curve.py.  Writes a markdown table to out.md when given.
"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2001_09258_b200 import api  # noqa: E402
from paper_2001_09258_b200 import inputs as I  # noqa: E402

# (function, accuracy, domain lo, hi, paper SLEEF ns per 4-element call, PAPER.md line)
ROWS = [
    ("sin", "u10", 0.4, 0.5, 11.43, 1203), ("sin", "u35", 0.4, 0.5, 7.504, 1206),
    ("sin", "u10", 0.0, 6.28, 11.41, 1209), ("sin", "u35", 0.0, 6.28, 7.507, 1212),
    ("sin", "u10", 0.0, 1e100, 48.79, 1215), ("sin", "u35", 0.0, 1e100, 43.82, 1218),
    ("cos", "u10", 0.4, 0.5, 13.75, 1221), ("cos", "u35", 0.4, 0.5, 7.850, 1224),
    ("cos", "u10", 0.0, 6.28, 13.74, 1227), ("cos", "u35", 0.0, 6.28, 7.850, 1230),
    ("cos", "u10", 0.0, 1e100, 50.38, 1233), ("cos", "u35", 0.0, 1e100, 46.09, 1236),
    ("tan", "u10", 0.4, 0.5, 17.30, 1239), ("tan", "u35", 0.4, 0.5, 9.367, 1242),
    ("tan", "u10", 0.0, 6.28, 17.28, 1245), ("tan", "u35", 0.0, 6.28, 9.367, 1248),
    ("tan", "u10", 0.0, 1e100, 48.82, 1251), ("tan", "u35", 0.0, 1e100, 36.54, 1254),
    ("atan", "u10", -700.0, 700.0, 22.12, 1269), ("atan", "u35", -700.0, 700.0, 9.251, 1272),
    ("log", "u10", 0.0, 1e300, 15.46, 1275), ("log", "u35", 0.0, 1e300, 9.636, 1278),
    ("exp", "u10", -700.0, 700.0, 7.663, 1281), ("exp", "u35", -700.0, 700.0, None, 1284),
    ("pow", "u10", -30.0, 30.0, 55.53, 1287),
]


def sleef_1core(L, name, arrs):
    if L is None:
        return None
    n = arrs[0].size
    out = np.empty_like(arrs[0])
    y = arrs[1].ctypes.data if len(arrs) > 1 else None
    best = None
    for _ in range(3):
        t = L.sleef_run(name.encode(), arrs[0].ctypes.data, y, out.ctypes.data, n, 1)
        if t <= 0:
            return None
        best = t if best is None else min(best, t)
    return n / best / 1e9


def main():
    lg = int(sys.argv[1]) if len(sys.argv) > 1 else 26
    md = sys.argv[2] if len(sys.argv) > 2 else None
    n = 1 << lg
    path = os.path.join(ROOT, "oracle", "_build", "libvem_sleef.so")
    L = None
    if os.path.exists(path):
        L = ctypes.CDLL(path)
        L.sleef_run.restype = ctypes.c_double
        L.sleef_run.argtypes = [ctypes.c_char_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                                ctypes.c_int]
    res = []
    for i, (fn, acc, lo, hi, ns_call, line) in enumerate(ROWS):
        name = f"{fn}_d_{acc}"
        seed = 0x7AB1E200 + i
        arrs = [I.uniform(seed, n, lo, hi, np.float64)]
        if fn == "pow":
            arrs.append(I.uniform(seed ^ 0xABCD, n, lo, hi, np.float64))
        ts = [torch.from_numpy(a).cuda() for a in arrs]
        out = torch.empty_like(ts[0])
        for _ in range(3):
            api.call(name, *ts, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            api.call(name, *ts, out=out)
        e1.record()
        torch.cuda.synchronize()
        gel = n / (e0.elapsed_time(e1) / 10) / 1e6
        cpu = sleef_1core(L, name, [a[: 1 << 20] for a in arrs])
        paper = 4.0 / ns_call if ns_call else None
        r = {"fn": name, "domain": [lo, hi], "gpu_gelem_s": round(gel, 1), "gpu_ns_per_elem": round(1.0 / gel, 5),
             "paper_sleef34_avx2_1core_gelem_s": round(paper, 4) if paper else None,
             "sleef38_avx512_1core_here_gelem_s": round(cpu, 4) if cpu else None,
             "gpu_over_paper": round(gel / paper, 1) if paper else None, "paper_line": f"PAPER.md:{line}"}
        res.append(r)
        print(json.dumps(r), flush=True)
        del ts, out
        torch.cuda.empty_cache()
    if md:
        with open(md, "w") as f:
            f.write(f"# Paper Table 2 rows on one B200 ({n} arguments per row, uniform on the domain)\n\n")
            f.write("Paper column: SLEEF 3.4, AVX2, one i7-6700 core (PAPER.md:1194-1292).  SLEEF 3.8 column: "
                    "AVX-512, one core of the GPU box's host, 2^20-argument sample.  exp u35 has no SLEEF entry.\n\n")
            f.write("| function | domain | B200 Gelem/s | B200 ns/elem | paper SLEEF 1-core Gelem/s | SLEEF 3.8 "
                    "1-core here | B200 / paper |\n|---|---|---|---|---|---|---|\n")
            for r in res:
                f.write(f"| {r['fn']} | [{r['domain'][0]:g}, {r['domain'][1]:g}] | {r['gpu_gelem_s']} | "
                        f"{r['gpu_ns_per_elem']} | {r['paper_sleef34_avx2_1core_gelem_s']} | "
                        f"{r['sleef38_avx512_1core_here_gelem_s']} | {r['gpu_over_paper']} |\n")


if __name__ == "__main__":
    main()
