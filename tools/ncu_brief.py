#!/usr/bin/env python3
"""One-screen summary of an ncu report: per kernel, duration, inst/elem,
pipe / issue / DRAM utilisation, registers, occupancy and the top warp-stall
reasons (per issued instruction).  Usage: ncu_brief.py REPORT ELEMS"""
import csv
import io
import re
import subprocess
import sys

rep, elems = sys.argv[1], int(sys.argv[2])
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, data = rows[0], rows[2:]
kc = hdr.index("Kernel Name")
want = {"us": "gpu__time_duration.sum", "fp64%": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "issue%": "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "dram%": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "regs": "launch__registers_per_thread",
        "warps%": "sm__warps_active.avg.pct_of_peak_sustained_active",
        "dramMB": "dram__bytes_read.sum"}
stall = [i for i, h in enumerate(hdr) if h.startswith("smsp__average_warps_issue_stalled_")
         and h.endswith("_per_issue_active.ratio")]
for r in data:
    m = re.search(r"(Op\w+|FmodQ<\w+>)", r[kc])
    name = m.group(1) if m else r[kc][:50]
    vals = {k: r[hdr.index(v)] for k, v in want.items() if v in hdr}
    ie = float(r[hdr.index("smsp__inst_executed.sum")]) * 32 / elems
    print(f"== {name}: " + ", ".join(f"{k} {float(v):.1f}" for k, v in vals.items()) + f", inst/elem {ie:.1f}")
    st = sorted(((float(r[i]) if r[i] else 0, hdr[i][len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]) for i in stall), reverse=True)[:8]
    print("   stalls/issue: " + ", ".join(f"{n} {v:.2f}" for v, n in st))
