#!/usr/bin/env python3
"""Summarise an ncu launch list (gpu__time_duration.sum per launch, CSV).

Usage: python tools/launch_share.py LAUNCHES.csv OUT.md
Groups launches by kernel (vem functor / entry point), prints count, total
and mean device time and each kernel's share of the total.  ncu serialises
launches and runs them cold-cache, so compare SHARES with bench.py's
event-timed step, not absolute times.
"""
import csv
import re
import sys
from collections import defaultdict


VEM = re.compile(r"^(?:void )?(?:vem::)?(k_\w+|vem_\w+)")


def short(name):
    k = VEM.match(name)
    if not k:
        return "(torch / other: input generation, copies)"
    m = re.search(r"(Op\w+|FmodQ<\w+>)", name)
    return f"{k.group(1)}<{m.group(1)}>" if m else k.group(1)


def main():
    src, out = sys.argv[1], sys.argv[2]
    lines = open(src).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(lines[start:]))
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        ns = v * {"ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}.get(unit, 1)
        a = agg[short(r["Kernel Name"])]
        a[0] += 1
        a[1] += ns
    tot = sum(a[1] for a in agg.values())
    vtot = sum(a[1] for k, a in agg.items() if not k.startswith("("))
    with open(out, "w") as f:
        f.write(f"# ncu launch list: {src.split('/')[-1]} ({sum(a[0] for a in agg.values())} launches, "
                f"{tot / 1e6:.2f} ms total device time, serialised)\n\n")
        f.write("| kernel | launches | total ms | mean us | share | share of vem kernels |\n"
                "|---|---|---|---|---|---|\n")
        for k, (c, ns) in sorted(agg.items(), key=lambda t: -t[1][1]):
            vs = "" if k.startswith("(") else f"{ns / vtot:.3f}"
            f.write(f"| {k} | {c} | {ns / 1e6:.3f} | {ns / c / 1e3:.1f} | {ns / tot:.3f} | {vs} |\n")
    print(open(out).read())


if __name__ == "__main__":
    main()
