#!/usr/bin/env python3
"""vem-b200 benchmark: Gelem/s of the batched elementwise math path on B200.

Contract (driver): python bench.py --gpus N --steps K --warmup W
  N=1 directly; N>1 under torch.distributed.run (one rank per GPU, NCCL).
Workload (default, BASELINE.json configs[1] -- the config the metric is
quoted on): exp / log / pow x {f32, f64} x {u10, u35}, 2^28 elements each,
inputs drawn from the config's domains.  One STEP = one pass of all 12 entry
points over their resident 2^28-element inputs (12 x 2^28 elements).
  value        = elements processed by all ranks / max-over-ranks step time
  e2e          = same metric through the C ABI with HOST buffers (pinned
                 H2D + kernel + D2H inside the timed region, every step)
  roofline     = dominant kernel (largest share of the step): algorithmic
                 bytes per launch / its CUDA-event duration vs the measured HBM
                 peak; plus its FP64-pipe roofline against the measured DFMA peak
  per_config   = configs 1, 3, 4, 5 timed the same way (config 5: the 2^31
                 element job sharded over the ranks -- strong scaling), each
                 with per-function Gelem/s and roofline fraction
  verify       = every result of every timed workload checked against the CPU
                 ORACLE's checksums of the same full config arrays
                 (tests/golden/config_checksums.json): per-rank partial chunk
                 checksums, one all-reduce (SUM), compared on rank 0
  cpu_baseline = the CPU oracle port (oracle/, all host threads + 1 thread) on
                 a bounded sample; SLEEF 3.8 AVX-512 timed beside it for context
Inputs: the config generator (paper_2001_09258_b200/inputs.py) evaluated on the
device (csrc/vem_aux.cu, bit-identical to the host generator -- verified), rank
r of N taking its own slice of the config's global index space.  Inputs are
1-16 GiB per array (>> 126 MB L2), so no L2 flush is needed.
`--impl reference` times the reference CPU path (oracle port, all host
threads) on the same workload instead (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2001_09258_b200 import configs as C  # noqa: E402

METRIC = "Gelements/s per function (f32/f64, u10/u35) at 1-8 B200 + roofline fraction"
UNIT = "Gelem/s"
GOLDEN = os.path.join(ROOT, "tests", "golden", "config_checksums.json")
M64 = (1 << 64) - 1


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="vem", choices=["vem", "reference"])
    ap.add_argument("--workload", default="cfg2", choices=sorted(C.WORKLOADS))
    ap.add_argument("--only", default="", help="comma list of entry points (profiling)")
    ap.add_argument("--log2n", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-verify", action="store_true")
    ap.add_argument("--no-per-config", action="store_true")
    return ap.parse_args()


# --------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-f", self.path], stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        out = {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        if self.proc is None:
            return out
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 8:
                    rows.append(parts)
            os.unlink(self.path)
        except Exception:
            pass
        if not rows:
            return out
        sm = sorted(float(r[0]) for r in rows if r[0].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            for nm, v in zip(names, r[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        out["sm_mhz"] = sm[len(sm) // 2] if sm else None
        try:
            out["sm_max_mhz"] = float(rows[0][1])
        except Exception:
            pass
        out["reasons"] = sorted(reasons)
        out["samples"] = len(rows)
        return out


# --------------------------------------------------------------- CPU legs
def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def cpu_oracle_rate(workload, names, sample_log2: int, threads: int, budget_s: float = 0.0):
    """Oracle port (oracle/vem_oracle.c, OpenMP on `threads` host threads) over a
    bounded host sample of every entry point: the first 2^sample_log2 elements
    of the config arrays (host generator), passes repeated until each entry
    point has run budget_s/len(names) seconds (at least one pass); returns
    (Gelem/s, seconds, elements, per-function Gelem/s)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_lib as O
    set_omp_threads(threads)
    n = 1 << sample_log2
    total_t = 0.0
    total_n = 0
    per = {}
    for name in names:
        arrs = [O.gen_fill(r, n, 0) for r in C.recipes(workload, name)]
        O.oracle_eval(name, *[a[:4096] for a in arrs])  # warm (threads, pages)
        reps = 0
        t0 = time.perf_counter()
        while True:
            O.oracle_eval(name, *arrs)
            reps += 1
            dt = time.perf_counter() - t0
            if dt >= budget_s / max(1, len(names)):
                break
        per[name] = round(reps * n / dt / 1e9, 4)
        total_t += dt
        total_n += reps * n
    return total_n / total_t / 1e9, total_t, total_n, per


def cpu_sleef_rate(workload, names, sample_log2: int, threads: int):
    """Upstream SLEEF 3.8 AVX-512 (torch's libtorch_cpu.so) on the same sample."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import numpy as np
    import oracle_lib as O
    import sleef_lib as S
    why = S.available()
    if why:
        return {"unavailable": why}
    n = 1 << sample_log2
    tt = 0.0
    per = {}
    L = S.lib()
    for name in names:
        arrs = [O.gen_fill(r, n, 0) for r in C.recipes(workload, name)]
        out = np.empty_like(arrs[0])
        y = arrs[1].ctypes.data if len(arrs) > 1 else None
        best = None
        for _ in range(3):
            t = L.sleef_run(name.encode(), arrs[0].ctypes.data, y, out.ctypes.data, n, threads)
            best = t if best is None or t < best else best
        if best is None or best < 0:
            continue
        per[name] = round(n / best / 1e9, 4)
        tt += best
    return {"value": round(len(per) * n / tt / 1e9, 4) if tt else None, "unit": UNIT, "cores": threads,
            "kind": "sleef-3.8-avx512", "per_function": per,
            "note": "SLEEF has no u35 exp/pow: those rows time the u10 entry"}


def set_omp_threads(k: int):
    os.environ["OMP_NUM_THREADS"] = str(k)
    try:
        import ctypes
        ctypes.CDLL("libgomp.so.1").omp_set_num_threads(k)
    except OSError:
        pass


def run_reference(args, rank, world):
    """--impl reference: the reference CPU path (oracle port; the reference tree
    has no function kernels) on all host threads."""
    if rank != 0:
        return
    names = select(args)
    threads = os.cpu_count() or 1
    set_omp_threads(threads)
    lg = 22
    for _ in range(args.warmup):
        cpu_oracle_rate(args.workload, names[:1], 16, threads)
    vals = []
    t_all = 0.0
    per = {}
    for _ in range(args.steps):
        v, t, n, per = cpu_oracle_rate(args.workload, names, lg, threads, budget_s=3.0)
        vals.append(v)
        t_all += t
    value = sum(vals) / len(vals)
    ms = t_all / max(1, args.steps) * 1e3
    line = {"metric": METRIC, "value": round(value, 4), "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64/f32", "data": "synthetic",
            "config": {"workload": args.workload, "text": C.CONFIG_TEXT[args.workload],
                       "sample": f"the first 2^{lg} elements of each config array (host generator), passes "
                                 f"repeated for ~3 s of CPU work per step"},
            "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": threads, "kind": "port",
                             "cpu_model": cpu_model(),
                             "sample": f"{len(names)} entry points x 2^{lg}-element arrays, ~3 s of CPU work "
                                       f"per step, oracle/vem_oracle.c (OpenMP, {threads} threads)",
                             "per_function": per},
            "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def select(args, workload=None):
    names = C.WORKLOADS[workload or args.workload]
    if args.only:
        keep = set(args.only.split(","))
        names = [w for w in names if w in keep]
    return names


# --------------------------------------------------------------- GPU arm
class Dist:
    def __init__(self, rank, world, local, share, dev):
        self.rank, self.world, self.local, self.share, self.dev = rank, world, local, share, dev

    def tensor(self, vals, dtype):
        import torch
        return torch.tensor(vals, dtype=dtype, device="cpu" if self.share else self.dev)

    def all_reduce(self, t, op):
        import torch.distributed as dist
        if self.world > 1:
            dist.all_reduce(t, op=op)
        return t

    def barrier(self):
        import torch.distributed as dist
        if self.world > 1:
            dist.barrier()


def make_inputs(workload, names, n_log2, D):
    """Device-generated operands of this rank's slice: {entry: [tensors]},
    operands with the same recipe are one tensor (u10/u35 pairs, config 5's
    shared x)."""
    import torch
    from paper_2001_09258_b200 import _aux
    if n_log2:
        off, n = (D.rank << n_log2, 1 << n_log2)
    else:
        off, n = C.shard(workload, D.rank, D.world)
    cache = {}
    bufs = {}
    for name in names:
        ts = []
        for r in C.recipes(workload, name):
            key = (r["kind"], r["seed"], r["a"], r["b"], r["sign"], r["specials"], r["f32"])
            if key not in cache:
                t = torch.empty(n, dtype=torch.float32 if r["f32"] else torch.float64, device=D.dev)
                cache[key] = _aux.fill(r, t, off)
            ts.append(cache[key])
        bufs[name] = ts
    torch.cuda.synchronize()
    return bufs, off, n


def time_workload(workload, names, bufs, n, steps, warmup, D, clocks=False):
    """Warm-up, then `steps` timed passes over every entry point: CUDA events
    on the launching stream around the whole region only (so consecutive
    kernels keep their programmatic-dependent-launch overlap), barrier +
    synchronize on both sides, max over ranks -> ms_step.  Then the same
    number of passes again with an event pair around every launch -> the
    per-kernel durations the roofline and per_function use (their sum is
    reported as instrumented_ms_per_step).  Returns timing dict, outputs."""
    import torch
    import torch.distributed as dist
    from paper_2001_09258_b200 import _lib, api
    outs = {name: torch.empty_like(bufs[name][0]) for name in names}
    stream = torch.cuda.current_stream()

    def step(evs=None):
        for i, name in enumerate(names):
            if evs is not None:
                evs[i][0].record(stream)
            api.call(name, *bufs[name], out=outs[name])
            if evs is not None:
                evs[i][1].record(stream)

    def region(evs_per_step):
        D.barrier()
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        # a short device-side spin ahead of the timed region keeps the GPU busy
        # while the host enqueues the first launches, so host launch latency
        # (Python + ctypes) does not appear as device idle time inside it
        torch.cuda._sleep(int(2e6))
        t0.record(stream)
        for s in range(steps):
            step(evs_per_step[s] if evs_per_step else None)
        t1.record(stream)
        torch.cuda.synchronize()
        D.barrier()
        return t0.elapsed_time(t1)

    for _ in range(max(warmup, 0)):
        step()
    torch.cuda.synchronize()
    sampler = ClockSampler(D.local) if clocks else None
    if sampler:
        sampler.start()
        time.sleep(0.3)
    launches0 = _lib.launch_count()
    ms_total = region(None)
    launches = _lib.launch_count() - launches0
    clk = sampler.stop() if sampler else None
    evs = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in names]
           for _ in range(steps)]
    ms_instr = region(evs)
    per_ms = [sum(evs[s][i][0].elapsed_time(evs[s][i][1]) for s in range(steps)) / steps for i in range(len(names))]
    t = D.tensor([ms_total, ms_instr] + per_ms, torch.float64)
    D.all_reduce(t, dist.ReduceOp.MAX)
    ms_total, ms_instr, per_ms = float(t[0]), float(t[1]), [float(v) for v in t[2:]]
    return {"ms_step": ms_total / steps, "instrumented_ms_step": ms_instr / steps, "per_ms": per_ms,
            "launches": int(launches), "clocks": clk}, outs


def verify_workload(workload, names, bufs, outs, off, n, D, gold):
    """Result (and operand) chunk checksums of this rank's slice, all-reduced
    (SUM) over the ranks -- the path's one collective -- and compared on
    rank 0 with the CPU oracle's checksums of the same config arrays."""
    import torch
    import torch.distributed as dist
    from paper_2001_09258_b200 import _aux
    g = (gold or {}).get("configs", {}).get(workload)
    if g is None:
        return {"skipped": f"no golden checksums for {workload}"}
    lc = C.LOG2CHUNK
    nchunks = len(next(iter(g["outputs"].values())))
    items = [("out", name, outs[name]) for name in names]
    groups = {}
    for name in names:
        groups.setdefault(C.input_key(workload, name), []).append(name)
    for members in groups.values():
        for k, t in enumerate(bufs[members[0]]):
            items.append(("in", f"{members[0]}#{k}", t))
    mine = [C.chunk_vector(_aux.checksum(t, off, lc), nchunks) for _, _, t in items]
    tot = D.tensor(mine, torch.int64)
    D.all_reduce(tot, dist.ReduceOp.SUM)
    # chunks covered by the ranks that ran, within the golden file's range:
    # weak configs [0, world * n), config 5 the whole job
    c_lo = 0
    c_hi = nchunks if workload in C.STRONG else min(nchunks, (D.world * n) >> lc)
    bad = {}
    for (kind, key, _), row in zip(items, tot.cpu().tolist()):
        ref = (g["outputs"] if kind == "out" else g["inputs"]).get(key)
        if ref is None:
            continue
        mis = C.mismatching_chunks(row, ref, c_lo, c_hi)
        if mis:
            bad[f"{kind}:{key}"] = mis[:8]
    checked = (c_hi - c_lo) << lc
    return {"elements_per_entry_point": checked, "entry_points": len(names),
            "mismatching_chunks": sum(len(v) for v in bad.values()), "bad": bad,
            "compared": "chunk checksums (2^24 elements) of every result and operand vs the CPU oracle's over the "
                        "same config arrays (tests/golden/config_checksums.json, tools/make_config_digests.py)",
            "reduction": "per-rank partial checksums, all_reduce SUM over the ranks"}


def roofline_entry(name, workload, n, ms, esz, nops, hbm_peak, fp64_peak, km):
    g = n / (ms * 1e-3) / 1e9
    bpe = esz * (nops + 1)
    hbm_roof = hbm_peak / bpe
    m = km.get(f"{name}@{workload}", km.get(name, {}))
    f64 = m.get("fp64_inst_per_elem")
    fp_roof = fp64_peak / f64 if f64 else None
    roof = min(hbm_roof, fp_roof) if fp_roof else hbm_roof
    return {"gelem_s": round(g, 2), "ms": round(ms, 4), "hbm_frac": round(g * bpe / hbm_peak, 4),
            "roof_gelem_s": round(roof, 1), "roof_frac": round(g / roof, 4),
            "bound": "hbm" if not fp_roof or hbm_roof <= fp_roof else "fp64",
            "fp64_inst_per_elem": f64, "inst_per_elem": m.get("inst_per_elem"), "metrics_source": m.get("source")}


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    from paper_2001_09258_b200 import _lib, build

    # VEM_BENCH_SHARE_GPU=1 (testing only): map every rank to the visible
    # device(s) round-robin and reduce over gloo -- exercises the multi-rank
    # bookkeeping on a box with fewer GPUs than ranks (no kernel waits on
    # another rank: the data path has no collective).
    share = os.environ.get("VEM_BENCH_SHARE_GPU") == "1"
    ndev = max(1, torch.cuda.device_count())
    local = local % ndev if share else local
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    D = Dist(rank, world, local, share, dev)
    if rank == 0:
        build.build()
    D.barrier()
    _lib.lib()
    gold = json.load(open(GOLDEN)) if os.path.exists(GOLDEN) else None

    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    hbm_src = "measured (MEASURED_PEAKS.json)" if "hbm_gbs" in peaks else "fallback (B200_PROFILING.md)"
    fp64_peak = _lib.probe_peak("fp64")
    km = {}
    try:
        km = json.load(open(os.path.join(ROOT, "profiles", "kernel_metrics.json")))
    except Exception:
        pass

    # ---------------- headline workload
    names = select(args)
    bufs, off, n = make_inputs(args.workload, names, args.log2n, D)
    tim, outs = time_workload(args.workload, names, bufs, n, args.steps, args.warmup, D, clocks=True)
    ms_step = tim["ms_step"]
    value = len(names) * n * world / (ms_step * 1e-3) / 1e9
    verify = None
    if not args.no_verify and not args.log2n:
        verify = verify_workload(args.workload, names, bufs, outs, off, n, D, gold)
    e2e = None
    if not args.no_e2e:
        e2e = e2e_leg(names, bufs, outs, n, args, dev, world)
    per_function = {}
    for i, name in enumerate(names):
        per_function[name] = roofline_entry(name, args.workload, n, tim["per_ms"][i], bufs[name][0].element_size(),
                                            len(bufs[name]), hbm_peak, fp64_peak, km)
    dom = max(range(len(names)), key=lambda i: tim["per_ms"][i])
    dname = names[dom]
    esz = bufs[dname][0].element_size()
    bpl = n * esz * (len(bufs[dname]) + 1)
    ach = bpl / (tim["per_ms"][dom] * 1e-3) / 1e9
    m = km.get(f"{dname}@{args.workload}", km.get(dname, {}))
    traffic = m["dram_bytes_per_elem"] * n if m.get("dram_bytes_per_elem") is not None else None
    pipe = None
    if m.get("fp64_inst_per_elem"):
        ach_ops = m["fp64_inst_per_elem"] * n / (tim["per_ms"][dom] * 1e-3) / 1e9
        pipe = {"pipe": "fp64", "achieved": round(ach_ops, 1), "peak": round(fp64_peak, 1), "unit": "Ginst/s",
                "frac": round(ach_ops / fp64_peak, 4), "fp64_inst_per_elem": m["fp64_inst_per_elem"],
                "peak_source": "measured (vem_probe_peak DFMA microbenchmark, this run)"}
    roofline = {"bound": "hbm", "kernel": dname, "achieved": round(ach, 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(ach / hbm_peak, 4), "traffic": traffic, "bytes_per_launch": bpl,
                "bytes_per_elem": esz * (len(bufs[dname]) + 1), "elems_per_launch": n,
                "ms_per_launch": round(tim["per_ms"][dom], 4), "peak_source": hbm_src,
                "traffic_source": m.get("source"), "fp64_pipe": pipe,
                "fp64_dfma_peak_ginst_s": round(fp64_peak, 1)}
    ws = sum(t.numel() * t.element_size() for t in {id(t): t for v in bufs.values() for t in v}.values())
    ws += sum(t.numel() * t.element_size() for t in outs.values())
    del bufs, outs
    torch.cuda.empty_cache()

    # ---------------- the other BASELINE configs (same timing rules)
    per_config = None
    if args.workload == "cfg2" and not args.no_per_config and not args.only and not args.log2n:
        per_config = {}
        for w in ("cfg1", "cfg3", "cfg4", "cfg5"):
            nm = C.WORKLOADS[w]
            b, o, nn = make_inputs(w, nm, 0, D)
            st = max(3, args.steps // 2)
            tw, ow = time_workload(w, nm, b, nn, st, max(3, args.warmup), D)
            vw = None if args.no_verify else verify_workload(w, nm, b, ow, o, nn, D, gold)
            pf = {name: roofline_entry(name, w, nn, tw["per_ms"][i], b[name][0].element_size(), len(b[name]),
                                       hbm_peak, fp64_peak, km) for i, name in enumerate(nm)}
            per_config[w] = {"value": round(len(nm) * nn * world / (tw["ms_step"] * 1e-3) / 1e9, 3), "unit": UNIT,
                             "ms_per_step": round(tw["ms_step"], 4), "steps": st,
                             "instrumented_ms_per_step": round(tw["instrumented_ms_step"], 4),
                             "scaling": "strong" if w in C.STRONG else "weak",
                             "elements_per_entry_point_per_rank": nn, "text": C.CONFIG_TEXT[w],
                             "gpu_launches": tw["launches"], "per_function": pf, "verify": vw}
            del b, ow
            torch.cuda.empty_cache()

    cpu = None
    sleef = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        set_omp_threads(threads)
        v, t, cn, per = cpu_oracle_rate(args.workload, names, 23, threads, budget_s=12.0)
        set_omp_threads(1)
        v1, t1, cn1, _ = cpu_oracle_rate(args.workload, names, 20, 1, budget_s=3.0)
        set_omp_threads(threads)
        cpu = {"value": round(v, 4), "unit": UNIT, "cores": threads, "kind": "port", "cpu_model": cpu_model(),
               "value_1core": round(v1, 4),
               "sample": f"{len(names)} entry points x the first 2^23 elements of the same config arrays (host "
                         f"generator), repeated passes: {cn / 1e9:.2f} G elements in {t:.1f} s of CPU work, "
                         f"oracle/vem_oracle.c, OpenMP {threads} threads; value_1core: 2^20-element samples, "
                         f"{t1:.1f} s on 1 thread",
               "per_function": per}
        try:
            sleef = cpu_sleef_rate(args.workload, names, 23, threads)
        except Exception as ex:  # context only
            sleef = {"error": str(ex)}

    l2_note = (f"no flush: per-step working set {ws / 2**20:.0f} MiB (distinct inputs + outputs of "
               f"{n}-element arrays) > 126 MB L2, each input re-read only after the other kernels' traffic")
    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True,
                "scaling": "strong" if args.workload in C.STRONG else "weak", "vs_baseline": None,
                "dtype": "f64/f32 (per entry point)",
                "data": "synthetic (config-domain inputs, counter-based generator evaluated on the device, "
                        "bit-identical to the host generator)",
                "config": {"workload": args.workload, "text": C.CONFIG_TEXT[args.workload],
                           "elements_per_entry_point_per_rank": n, "entry_points": names, "l2": l2_note,
                           "parallelism": f"data-parallel shards x{world} (no collective on the data path)"},
                "gpu_launches": tim["launches"], "clocks": tim["clocks"],
                "instrumented_ms_per_step": round(tim["instrumented_ms_step"], 4), "roofline": roofline,
                "per_function": per_function, "e2e": e2e, "cpu_baseline": cpu, "sleef_cpu": sleef,
                "verify": verify, "per_config": per_config}
        print(json.dumps(line), flush=True)
    if world > 1:
        D.barrier()
        dist.destroy_process_group()


def e2e_leg(names, bufs, outs, n, args, dev, world):
    """Same step through the C ABI with HOST buffers: every step uploads that
    step's distinct inputs host->device from pinned memory (the u10 and u35
    entry points of one function read the same arrays, so each input array is
    uploaded once), runs every entry point, and reads every result back
    device->host into its own pinned buffer; chunked over four streams so
    copies in both directions overlap the kernels (4 streams, 2^24-element
    chunks: the best of a chunk x stream sweep, profiles/r01_e2e_sweep.log)."""
    import torch
    from paper_2001_09258_b200 import api
    chunk = 1 << int(os.environ.get("VEM_E2E_CHUNK_LOG2", "24"))
    nstreams = int(os.environ.get("VEM_E2E_STREAMS", "4"))
    n = min(n, 1 << 26)  # 2^26 elements per entry point per rank (bounded pinned memory)
    groups = []  # (device input list, [(entry name, work index)])
    for i, name in enumerate(names):
        for g in groups:
            if all(a is b for a, b in zip(g[0], bufs[name])) and len(g[0]) == len(bufs[name]):
                g[1].append((name, i))
                break
        else:
            groups.append((bufs[name], [(name, i)]))
    host_in = {id(g[0]): [t[:n].to("cpu").pin_memory() for t in g[0]] for g in groups}
    dev_in = {id(g[0]): [torch.empty(n, dtype=t.dtype, device=dev) for t in g[0]] for g in groups}
    host_out = [torch.empty(n, dtype=bufs[name][0].dtype).pin_memory() for name in names]
    dev_out = [torch.empty(n, dtype=bufs[name][0].dtype, device=dev) for name in names]
    streams = [torch.cuda.Stream(dev) for _ in range(nstreams)]
    h2d = sum(t.numel() * t.element_size() for v in host_in.values() for t in v)
    d2h = sum(h.numel() * h.element_size() for h in host_out)

    def one_step():
        for dins, members in groups:
            hin, din = host_in[id(dins)], dev_in[id(dins)]
            for j, c0 in enumerate(range(0, n, chunk)):
                c1 = min(n, c0 + chunk)
                s = streams[j % nstreams]  # a given range always uses the same stream
                with torch.cuda.stream(s):
                    for hd, dd_ in zip(hin, din):
                        dd_[c0:c1].copy_(hd[c0:c1], non_blocking=True)
                    for name, i in members:
                        api.call(name, *[d[c0:c1] for d in din], out=dev_out[i][c0:c1])
                        host_out[i][c0:c1].copy_(dev_out[i][c0:c1], non_blocking=True)

    one_step()
    torch.cuda.synchronize()
    steps = max(1, min(args.steps, 3))
    t0 = time.perf_counter()
    for _ in range(steps):
        one_step()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / steps
    # the results that crossed PCIe are the device results (spot check)
    for i, name in enumerate(names):
        if not torch.equal(host_out[i][:4096].view(torch.int32 if host_out[i].dtype == torch.float32 else torch.int64),
                           outs[name][:4096].cpu().view(torch.int32 if host_out[i].dtype == torch.float32
                                                        else torch.int64)):
            raise RuntimeError(f"e2e: {name} host result differs from the device result")
    return {"value": round(len(names) * n * world / dt / 1e9, 3), "unit": UNIT, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": round(dt * 1e3, 2), "steps": steps,
            "elements_per_entry_point_per_rank": n,
            "path": "pinned host -> H2D (each distinct input once, chunked 2^24, 4 streams) -> vem C ABI "
                    "(every entry point) -> D2H of every result, host wall clock"}


if __name__ == "__main__":
    main()
