#!/usr/bin/env python3
"""Summarise an ncu report into per-kernel JSON + markdown (profiles/).

Usage: python tools/ncu_summary.py REPORT.ncu-rep ELEMS_PER_LAUNCH OUT_PREFIX [KEY_SUFFIX]

KEY_SUFFIX (e.g. "@cfg5") is appended to the entry-point keys merged into
kernel_metrics.json, for captures whose input mix is workload specific.

For every profiled kernel: duration, DRAM bytes (read+write) per element,
executed instructions per element, the dynamic SASS opcode mix (from the
source page), FP64-pipe instructions per element, pipe/issue utilisation,
occupancy and registers.  Writes OUT_PREFIX.json and OUT_PREFIX.md and
merges {entry point: {dram_bytes_per_elem, fp64_inst_per_elem, ...}} into
profiles/kernel_metrics.json (read by bench.py for roofline.traffic).
"""
import csv
import io
import json
import os
import re
import subprocess
import sys
from collections import Counter

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FP64_OPS = {"DADD", "DMUL", "DFMA", "DSETP", "DMNMX", "FRND", "DSET", "F2I", "I2F", "F2F"}
RAW = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read_mb": "dram__bytes_read.sum",
    "dram_write_mb": "dram__bytes_write.sum",
    "inst_executed": "smsp__inst_executed.sum",
    "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "registers": "launch__registers_per_thread",
    "sm_ghz": "smsp__cycles_elapsed.avg.per_second",
}

ENTRY = {  # kernel functor -> C-ABI entry point
    "OpSinD": "sin_d_u10", "OpCosD": "cos_d_u10", "OpTanD": "tan_d_u10", "OpSinDPh": "sin_d_u10_ph",
    "OpCosDPh": "cos_d_u10_ph", "OpTanDPh": "tan_d_u10_ph", "OpAtanD": "atan_d_u10", "OpExpD": "exp_d_u10",
    "OpExpDU35": "exp_d_u35", "OpLogD": "log_d_u10", "OpLogDU35": "log_d_u35", "OpPowD": "pow_d_u10",
    "OpPowDU35": "pow_d_u35", "OpFmodD": "fmod_d", "OpSinF": "sin_f_u10", "OpCosF": "cos_f_u10",
    "OpTanF": "tan_f_u10", "OpExpF": "exp_f_u10", "OpExpFU35": "exp_f_u35", "OpLogF": "log_f_u10",
    "OpLogFU35": "log_f_u35", "OpPowF": "pow_f_u10", "OpPowFU35": "pow_f_u35", "OpFmodF": "fmod_f", "OpFmodFFlat": "fmod_f",
    "OpSinDU35": "sin_d_u35", "OpCosDU35": "cos_d_u35", "OpTanDU35": "tan_d_u35",
}


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def entry_of(kname):
    q = re.search(r"FmodQ<(double|float)>", kname)
    if q:
        return "fmod_d" if q.group(1) == "double" else "fmod_f"
    m = re.search(r"vem::(Op\w+)|<(Op\w+)", kname)
    if not m:
        return kname
    op = m.group(1) or m.group(2)
    return ENTRY.get(op, op)


def main():
    rep, elems, prefix = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    suffix = sys.argv[4] if len(sys.argv) > 4 else ""
    raw = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv"))))
    hdr, units, data = raw[0], raw[1], raw[2:]
    col = {k: hdr.index(v) for k, v in RAW.items() if v in hdr}
    kcol = hdr.index("Kernel Name")
    # source page: per-kernel blocks
    src = ncu("-i", rep, "--page", "source", "--csv", "--print-source", "sass")
    blocks = re.split(r'^"Kernel Name",', src, flags=re.M)[1:]
    mixes = {}
    for b in blocks:
        lines = b.splitlines()
        kname = next(csv.reader([lines[0]]))[0]
        rd = csv.reader(lines[1:])
        h = next(rd)
        ia = h.index("Source")
        it = h.index("Thread Instructions Executed")
        c = Counter()
        for r in rd:
            if len(r) <= it:
                continue
            op = r[ia].strip().split()
            if not op:
                continue
            o = op[0]
            if o.startswith("@"):
                o = op[1] if len(op) > 1 else o
            base = o.split(".")[0]
            try:
                c[base] += int(r[it])
            except ValueError:
                pass
        mixes[entry_of(kname)] = c
    stall_cols = [(i, h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")])
                  for i, h in enumerate(hdr) if h.startswith("smsp__average_warps_issue_stalled_")
                  and h.endswith("_per_issue_active.ratio")]
    out = {}
    for k, r in enumerate(data):
        name = entry_of(r[kcol])
        d = {}
        st = []
        for i, nm in stall_cols:
            try:
                st.append((float(r[i]), nm))
            except ValueError:
                pass
        d["stalls_per_issue"] = {nm: round(v, 2) for v, nm in sorted(st, reverse=True)[:6]}
        for key, ci in col.items():
            try:
                d[key] = float(r[ci])
            except ValueError:
                d[key] = r[ci]
        def unit_scale(u):  # ncu picks byte / Kbyte / Mbyte / Gbyte per column
            u = u.lower()
            return 1e9 if u.startswith("g") else 1e6 if u.startswith("m") else 1e3 if u.startswith("k") else 1.0
        tu = units[col["duration_us"]].lower()  # ncu picks nsecond / usecond / msecond / second
        d["duration_us"] = d["duration_us"] * {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6}.get(tu, 1.0)
        d["dram_bytes_per_elem"] = round((d["dram_read_mb"] * unit_scale(units[col["dram_read_mb"]]) +
                                          d["dram_write_mb"] * unit_scale(units[col["dram_write_mb"]])) / elems, 3)
        d["inst_per_elem"] = round(d["inst_executed"] * 32 / elems, 2)
        if name in mixes:
            mix = mixes[name]
            fp64 = sum(v for o, v in mix.items() if o in FP64_OPS)
            d["fp64_inst_per_elem"] = round(fp64 / elems, 2)
            d["thread_inst_per_elem"] = round(sum(mix.values()) / elems, 2)
            d["mix_per_elem"] = {o: round(v / elems, 2) for o, v in mix.most_common(24)}
        out[name] = d
    json.dump(out, open(prefix + ".json", "w"), indent=1)
    with open(prefix + ".md", "w") as f:
        f.write(f"# ncu summary: {os.path.basename(rep)} ({elems} elements per launch)\n\n")
        f.write("| entry point | us | DRAM B/elem | inst/elem | FP64 inst/elem | FP64 pipe % | issue % | DRAM % | regs |\n")
        f.write("|---|---|---|---|---|---|---|---|---|\n")
        for n, d in out.items():
            f.write(f"| {n} | {d['duration_us']:.1f} | {d['dram_bytes_per_elem']} | {d['inst_per_elem']} | "
                    f"{d.get('fp64_inst_per_elem')} | {d['fp64_pipe_pct']:.1f} | {d['issue_active_pct']:.1f} | "
                    f"{d['dram_pct']:.1f} | {int(d['registers'])} |\n")
        f.write("\nTop warp-stall reasons (cycles per issued instruction):\n\n")
        for n, d in out.items():
            f.write(f"- {n}: " + ", ".join(f"{k} {v}" for k, v in d.get("stalls_per_issue", {}).items()) + "\n")
        f.write("\nTop opcodes per element (thread instructions):\n\n")
        for n, d in out.items():
            f.write(f"- {n}: " + ", ".join(f"{o} {v}" for o, v in list(d.get('mix_per_elem', {}).items())[:14]) + "\n")
    # only summaries written under profiles/ feed the bench's metrics file
    if os.path.abspath(prefix).startswith(os.path.join(ROOT, "profiles") + os.sep):
        km_path = os.path.join(ROOT, "profiles", "kernel_metrics.json")
        km = json.load(open(km_path)) if os.path.exists(km_path) else {}
        for n, d in out.items():
            km[n + suffix] = {"dram_bytes_per_elem": d["dram_bytes_per_elem"],
                     "fp64_inst_per_elem": d.get("fp64_inst_per_elem"),
                     "inst_per_elem": d["inst_per_elem"], "source": os.path.basename(prefix)}
        json.dump(km, open(km_path, "w"), indent=1, sort_keys=True)
    print(open(prefix + ".md").read())


if __name__ == "__main__":
    main()
