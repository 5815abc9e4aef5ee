#!/usr/bin/env python3
"""Launch-shape sweep for the streaming kernels (dev tool, runs on a GPU).

Builds a tuning variant of the library (-DVEM_TUNE) into
paper_2001_09258_b200/_tune/libvem_tune.so, then times every entry point
(filtered by argv[2]) at 2^argv[1] elements for each (VPT, STAGES) variant:
 0:(1,2) 1:(1,4) 2:(2,2) 3:(2,3) 4:(2,4) 5:(4,2), -1 = the shipped choice, and
 6/7/8 = the shipped shape with __launch_bounds__ min-blocks 2/3/4, 9/10 = (4,2) with
 min-blocks 2/3, 11 = the shipped shape with the other stage-release scheme
 (per-warp vs CTA barrier), 12/13 = one more stage (same / other release),
 14 = two more stages, 15-20 = (VPT,STAGES,min-blocks) (2,2,3) (2,2,4) (2,3,4) (1,2,6) (1,4,6) (2,2,5).  VEM_TUNE_VARIANTS=-1,11,... picks the variants.
fmod: -1 shipped step-queue kernel; 0-4 warp-private queue (VPT,STAGES[,MINB]) (2,2) (4,2) (2,3) (4,2,2) (2,2,3);
5-6 CTA queue (VPT,STAGES,ROWS) (2,2,2) (4,2,1); 7 = the streaming kernel with
warp step-class regrouping (2,2); 8 = the work-ring kernel; 9/10 = the
streaming kernel with no regrouping (2,2) / (1,2); 11/12/13 = CTA queue (2,2,1) claiming 2/4 units per atomic, and 2 with min-blocks 2; 14-18 = fmodf as one flat streaming body (VPT,STAGES[,MINB]) (2,2) (4,2) (1,2) (2,2,4) (4,2,3); 19-22 = fmodf branch-free six-step body (2,2) (1,2) (2,2,2) (1,4).
VEM_TUNE_CFG=k overrides the BASELINE config whose inputs are used.
Prints one JSON line per entry point with Gelem/s per variant.
"""
import ctypes
import json
import os
import subprocess
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2001_09258_b200 import _lib, build  # noqa: E402
from paper_2001_09258_b200 import inputs as I  # noqa: E402

CFG = {"sin": 1, "cos": 1, "tan": 3, "atan": 5, "exp": 2, "log": 2, "pow": 2, "fmod": 4, "asin": 6, "acos": 6,
       "atan2": 6, "fdim": 6}


def build_tune():
    out = os.path.join(ROOT, "paper_2001_09258_b200", "_tune")
    os.makedirs(out, exist_ok=True)
    if os.environ.get("VEM_TUNE_PREBUILT") and os.path.exists(os.path.join(out, "libvem_tune.so")):
        return os.path.join(out, "libvem_tune.so")
    objs = []
    for src in build.SOURCES:
        o = os.path.join(out, src.replace(".cu", ".o"))
        subprocess.run([build.nvcc(), *build.NVCC_FLAGS, "-DVEM_TUNE", "-c", os.path.join(build.CSRC, src), "-o", o],
                       check=True)
        objs.append(o)
    lib = os.path.join(out, "libvem_tune.so")
    subprocess.run([build.nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static", *objs,
                    "-o", lib], check=True)
    return lib


def main():
    lg = int(sys.argv[1]) if len(sys.argv) > 1 else 26
    flt = sys.argv[2].split(",") if len(sys.argv) > 2 else []
    L = ctypes.CDLL(build_tune())
    L.vem_tune_set.argtypes = [ctypes.c_int]
    n = 1 << lg
    stream = torch.cuda.current_stream().cuda_stream
    for name in sorted(_lib.ALL):
        if flt and not any(f in name for f in flt):
            continue
        fn, p = name.split("_")[0], name.split("_")[1]
        cfg = 3 if name.endswith("_ph") else CFG[fn]
        if p == "f" and cfg in (1, 5):  # binary64-only configs
            cfg = 3 if fn in ("sin", "cos", "tan") else 6
        if os.environ.get("VEM_TUNE_CFG"):
            cfg = int(os.environ["VEM_TUNE_CFG"])
        from paper_2001_09258_b200 import _aux
        ts = [_aux.fill(r, torch.empty(n, dtype=torch.float32 if r["f32"] else torch.float64, device="cuda"))
              for r in I.config_recipes(cfg, fn, p)]
        out = torch.empty_like(ts[0])
        f = getattr(L, "vem_" + name)
        if len(ts) == 2:
            f.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_size_t, ctypes.c_void_p]
            call = lambda: f(ts[0].data_ptr(), ts[1].data_ptr(), out.data_ptr(), n, stream)  # noqa: E731
        else:
            f.argtypes = [ctypes.c_void_p] * 2 + [ctypes.c_size_t, ctypes.c_void_p]
            call = lambda: f(ts[0].data_ptr(), out.data_ptr(), n, stream)  # noqa: E731
        res = {}
        vs = os.environ.get("VEM_TUNE_VARIANTS")
        vs = [int(v) for v in vs.split(",")] if vs else (
            (0, 14, 17, 19, 20, 21, 22) if name.startswith("fmod") else (-1, 0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10))
        for v in vs:
            L.vem_tune_set(v)
            for _ in range(3):
                call()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(10):
                call()
            e1.record()
            torch.cuda.synchronize()
            res[v] = round(n / (e0.elapsed_time(e1) / 10) / 1e6, 1)
        best = max(res, key=res.get)
        print(json.dumps({"fn": name, "cfg": cfg, "gelem_s": res, "best": best}), flush=True)
        del ts, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
