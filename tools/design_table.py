#!/usr/bin/env python3
"""DESIGN.md §4 table rows from the bench-size ncu summaries
(profiles/r02_full_cfg*.json) and a bench line (per-function Gelem/s).
Usage: python tools/design_table.py profiles/r02_bench_defaultN.jsonl"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BYTES = {"d1": 16, "d2": 24, "f1": 8, "f2": 12}


def main():
    line = [json.loads(l) for l in open(sys.argv[1]) if l.startswith("{")][0]
    hbm = line["roofline"]["peak"]
    dfma = line["roofline"]["fp64_dfma_peak_ginst_s"]
    per = {"cfg2": line["per_function"]}
    for c, v in line.get("per_config", {}).items():
        per[c] = v["per_function"]
    print("| entry (config) | inst/elem | FP64 inst/elem | DRAM B/elem | roof Gelem/s HBM / FP64 | measured | frac | "
          "issue / FP64 / DRAM % | top stalls (per issue) |")
    print("|---|---|---|---|---|---|---|---|---|")
    for cfg in ("cfg2", "cfg1", "cfg3", "cfg4", "cfg5"):
        path = os.path.join(ROOT, "profiles", f"r02_full_{cfg}.json")
        if not os.path.exists(path):
            continue
        m = json.load(open(path))
        for name, k in m.items():
            key = name if name in per[cfg] else name + "_ph" if name + "_ph" in per[cfg] else None
            if key is None:
                continue
            binary = name.startswith(("pow", "fmod"))
            b = BYTES[("f" if "_f" in name else "d") + ("2" if binary else "1")]
            r_hbm = hbm / b
            r_fp = dfma / k["fp64_inst_per_elem"] if k.get("fp64_inst_per_elem") else float("inf")
            g = per[cfg][key]["gelem_s"]
            st = ", ".join(f"{n} {v}" for n, v in list(k["stalls_per_issue"].items())[:4] if n != "selected")
            print(f"| {key} ({cfg}) | {k['inst_per_elem']:.0f} | {k['fp64_inst_per_elem']:.1f} | "
                  f"{k['dram_bytes_per_elem']:.1f} | {r_hbm:.0f} / {r_fp:.0f} | {g:.1f} | {g / min(r_hbm, r_fp):.2f} | "
                  f"{k['issue_active_pct']:.0f} / {k['fp64_pipe_pct']:.0f} / {k['dram_pct']:.0f} | {st} |")


if __name__ == "__main__":
    main()
