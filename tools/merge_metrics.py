#!/usr/bin/env python3
"""Merge per-config ncu summaries (tools/ncu_summary.py JSON written on the GPU
box, e.g. gpurun_out/r02_full_cfg2.json) into profiles/kernel_metrics.json
under "<entry>@<cfg>" keys (read by bench.py for roofline.traffic and the
FP64-pipe roofline), and copy the markdown summaries to profiles/.
Usage: python tools/merge_metrics.py gpurun_out/r02_full_cfg*.json"""
import json
import os
import re
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    km_path = os.path.join(ROOT, "profiles", "kernel_metrics.json")
    km = json.load(open(km_path)) if os.path.exists(km_path) else {}
    for path in sys.argv[1:]:
        cfg = re.search(r"(cfg\d)", path).group(1)
        base = os.path.splitext(os.path.basename(path))[0]
        d = json.load(open(path))
        for name, m in d.items():
            km[f"{name}@{cfg}"] = {"dram_bytes_per_elem": m["dram_bytes_per_elem"],
                                   "fp64_inst_per_elem": m.get("fp64_inst_per_elem"),
                                   "inst_per_elem": m["inst_per_elem"], "source": base,
                                   "stalls_per_issue": m.get("stalls_per_issue")}
        for ext in (".md", ".json"):
            src = os.path.splitext(path)[0] + ext
            dst = os.path.join(ROOT, "profiles", base + ext)
            if os.path.exists(src) and os.path.abspath(src) != os.path.abspath(dst):
                shutil.copy(src, dst)
    json.dump(km, open(km_path, "w"), indent=1, sort_keys=True)
    print(f"merged {len(sys.argv) - 1} summaries into {km_path}")


if __name__ == "__main__":
    main()
