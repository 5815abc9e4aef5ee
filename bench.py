#!/usr/bin/env python3
"""vem-b200 benchmark: Gelem/s of the batched elementwise math path on B200.

Contract (driver): python bench.py --gpus N --steps K --warmup W
  N=1 directly; N>1 under torch.distributed.run (one rank per GPU, NCCL).
Workload (default, BASELINE.json configs[1] -- the config the metric is
quoted on): exp / log / pow x {f32, f64} x {u10, u35}, 2^28 elements each,
inputs drawn from the config's domains.  One STEP = one pass of all 12 entry
points over their resident 2^28-element inputs (12 x 2^28 elements).
  value      = elements processed by all ranks / max-over-ranks step time
  e2e        = same metric through the C ABI with HOST buffers (pinned
               H2D + kernel + D2H inside the timed region, every step)
  roofline   = dominant kernel (largest share of the step): algorithmic bytes
               per launch / its CUDA-event duration vs measured HBM peak;
               plus its FP64-pipe roofline against the measured DFMA peak
  cpu_baseline = the CPU oracle port (oracle/, all host threads) on a bounded
               sample; SLEEF 3.8 AVX-512 timed beside it for context
Inputs are 2-4 GiB per array (>> 126 MB L2), so no L2 flush is needed.
`--impl reference` times the reference CPU path (oracle port, all host
threads) on the same workload instead (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time
import zlib

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Gelements/s per function (f32/f64, u10/u35) at 1-8 B200 + roofline fraction"
UNIT = "Gelem/s"

# (entry point, config, fn, prec)
WORKLOADS = {
    "cfg2": [("exp_d_u10", 2), ("exp_d_u35", 2), ("log_d_u10", 2), ("log_d_u35", 2), ("pow_d_u10", 2),
             ("pow_d_u35", 2), ("exp_f_u10", 2), ("exp_f_u35", 2), ("log_f_u10", 2), ("log_f_u35", 2),
             ("pow_f_u10", 2), ("pow_f_u35", 2)],
    "cfg1": [("sin_d_u10", 1), ("cos_d_u10", 1)],
    "cfg3": [("sin_d_u10_ph", 3), ("cos_d_u10_ph", 3), ("tan_d_u10_ph", 3), ("sin_f_u10_ph", 3),
             ("cos_f_u10_ph", 3), ("tan_f_u10_ph", 3)],
    "cfg4": [("fmod_d", 4), ("fmod_f", 4)],
    "cfg5": [("sin_d_u10", 5), ("cos_d_u10", 5), ("tan_d_u10", 5), ("atan_d_u10", 5), ("exp_d_u10", 5),
             ("log_d_u10", 5), ("pow_d_u10", 5), ("fmod_d", 5)],
}
LOG2N = {"cfg1": 24, "cfg2": 28, "cfg3": 28, "cfg4": 26, "cfg5": 31}
STRONG = {"cfg5"}  # configs whose element count is the job total (sharded), not per rank
CONFIG_TEXT = {
    "cfg1": "sin/cos f64 u10, 2^24 x U[-pi,pi] (Cody-Waite path)",
    "cfg2": "exp/log/pow x f32/f64 x u10/u35, 2^28 elements each (BASELINE configs[1] domains)",
    "cfg3": "sin/cos/tan u10 f64+f32, 2^28, |x| log-U[1,1e300]/[1,3e38] +-, forced Payne-Hanek",
    "cfg4": "fmod f64+f32, 2^26 pairs, log-U[1e-300,1e300]/[1e-37,3e38] +-",
    "cfg5": "2^31 f64 elements (one shared x array; pow y U[-30,30], fmod y log-U) sharded over the ranks, "
            "through sin/cos/tan/atan/exp/log/pow/fmod u10; log-U[1e-300,1e300] +- with 1% specials",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="vem", choices=["vem", "reference"])
    ap.add_argument("--workload", default="cfg2", choices=sorted(WORKLOADS))
    ap.add_argument("--only", default="", help="comma list of entry points (profiling)")
    ap.add_argument("--log2n", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-verify", action="store_true")
    return ap.parse_args()


# --------------------------------------------------------------- inputs
def device_inputs(fn_name: str, cfg: int, n: int, dev, seed: int):
    """Config-domain inputs generated ON the device (torch Philox): same
    distributions as paper_2001_09258_b200.inputs (the host generator used by
    the parity tests), without shipping 2-4 GiB from the host."""
    import torch
    fn, p = fn_name.split("_")[0], fn_name.split("_")[1]
    dt = torch.float64 if p == "d" else torch.float32
    g = torch.Generator(device=dev)
    g.manual_seed(seed)

    def U(a, b):
        return (a + (b - a) * torch.rand(n, dtype=torch.float64, device=dev, generator=g))

    def LU(a, b, signed=False):
        import math
        la, lb = math.log10(a), math.log10(b)
        v = torch.pow(10.0, U(la, lb))
        if signed:
            s = torch.rand(n, device=dev, generator=g) < 0.5
            v = torch.where(s, -v, v)
        return v

    def specials(v):
        pick = torch.rand(n, device=dev, generator=g) < 0.01
        which = torch.randint(0, 9, (n,), device=dev, generator=g)
        sp = torch.tensor([0.0, -0.0, float("inf"), float("-inf"), float("nan"), 5e-324, 1e-310,
                           1.7976931348623157e308, -1.7976931348623157e308], dtype=torch.float64, device=dev)
        return torch.where(pick, sp[which], v)

    if cfg == 1:
        xs = [U(-3.141592653589793, 3.141592653589793)]
    elif cfg == 2:
        if p == "d":
            xs = {"exp": lambda: [U(-700, 700)], "log": lambda: [LU(1e-300, 1e300)],
                  "pow": lambda: [LU(1e-10, 1e10), U(-30, 30)]}[fn]()
        else:
            xs = {"exp": lambda: [U(-87, 88)], "log": lambda: [LU(1e-37, 3e38)],
                  "pow": lambda: [LU(1e-3, 1e3), U(-10, 10)]}[fn]()
    elif cfg == 3:
        xs = [LU(1.0, 1e300 if p == "d" else 3e38, signed=True)]
    elif cfg == 4:
        lo, hi = (1e-300, 1e300) if p == "d" else (1e-37, 3e38)
        xs = [LU(lo, hi, True), LU(lo, hi, True)]
    else:
        x = specials(LU(1e-300, 1e300, True))
        if fn == "pow":
            xs = [x, U(-30, 30)]
        elif fn == "fmod":
            xs = [x, specials(LU(1e-300, 1e300, True))]
        else:
            xs = [x]
    if dt == torch.float32:
        xs = [torch.clamp(v, -3.4028234663852886e38, 3.4028234663852886e38).to(dt) for v in xs]
    return [v.to(dt).contiguous() for v in xs]


def device_inputs_cfg5(n: int, dev, seed: int, chunk_log2: int = 26):
    """Config 5: ONE x array (log-U[1e-300,1e300] +-, 1% specials) shared by
    all eight functions, plus pow's y (U[-30,30]) and fmod's y (same law as
    x); generated on the device in 2^chunk_log2 chunks to bound temporaries."""
    import torch
    x = torch.empty(n, dtype=torch.float64, device=dev)
    ypow = torch.empty_like(x)
    yfm = torch.empty_like(x)
    step = 1 << chunk_log2
    for c, i in enumerate(range(0, n, step)):
        m = min(step, n - i)
        x[i:i + m] = device_inputs("sin_d_u10", 5, m, dev, seed + 1000003 * c)[0]
        ypow[i:i + m] = device_inputs("pow_d_u10", 5, m, dev, seed + 1000003 * c + 1)[1]
        yfm[i:i + m] = device_inputs("fmod_d", 5, m, dev, seed + 1000003 * c + 2)[1]
    return x, ypow, yfm


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
def cpu_oracle_rate(work, sample_log2: int, threads: int, budget_s: float = 0.0):
    """Oracle port (oracle/vem_oracle.c, OpenMP on `threads` host threads) over a
    bounded host sample of every entry point: 2^sample_log2 elements, passes
    repeated until each entry point has run budget_s/len(work) seconds (at
    least one pass); returns (Gelem/s, seconds, elements, per-function)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import oracle_eval
    from paper_2001_09258_b200 import inputs as I
    os.environ["OMP_NUM_THREADS"] = str(threads)
    n = 1 << sample_log2
    total_t = 0.0
    total_n = 0
    per = {}
    for name, cfg in work:
        fn, p = name.split("_")[0], name.split("_")[1]
        arrs = I.config_inputs(cfg, fn, p, n)
        oracle_eval(name, *[a[:4096] for a in arrs])  # warm (threads, pages)
        reps = 0
        t0 = time.perf_counter()
        while True:
            oracle_eval(name, *arrs)
            reps += 1
            dt = time.perf_counter() - t0
            if dt >= budget_s / max(1, len(work)):
                break
        per[name] = round(reps * n / dt / 1e9, 4)
        total_t += dt
        total_n += reps * n
    return total_n / total_t / 1e9, total_t, total_n, per


def cpu_sleef_rate(work, sample_log2: int, threads: int):
    """Upstream SLEEF 3.8 AVX-512 (torch's libtorch_cpu.so) on the same sample."""
    import ctypes
    import numpy as np
    path = os.path.join(ROOT, "oracle", "_build", "libvem_sleef.so")
    if not os.path.exists(path):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=False)
    if not os.path.exists(path):
        return None
    L = ctypes.CDLL(path)
    L.sleef_run.restype = ctypes.c_double
    L.sleef_run.argtypes = [ctypes.c_char_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                            ctypes.c_int]
    from paper_2001_09258_b200 import inputs as I
    n = 1 << sample_log2
    tt = 0.0
    per = {}
    for name, cfg in work:
        fn, p = name.split("_")[0], name.split("_")[1]
        arrs = I.config_inputs(cfg, fn, p, n)
        out = np.empty_like(arrs[0])
        y = arrs[1].ctypes.data if len(arrs) > 1 else None
        best = None
        for _ in range(3):
            t = L.sleef_run(name.encode(), arrs[0].ctypes.data, y, out.ctypes.data, n, threads)
            best = t if best is None or t < best else best
        per[name] = round(n / best / 1e9, 4)
        tt += best
    return {"value": round(len(work) * n / tt / 1e9, 4), "unit": UNIT, "cores": threads,
            "kind": "sleef-3.8-avx512", "per_function": per,
            "note": "SLEEF has no u35 exp/pow: those rows time the u10 entry"}


def run_reference(args, rank, world):
    """--impl reference: the reference CPU path (oracle port; the reference tree
    has no function kernels) on all host threads."""
    if rank != 0:
        return
    work = WORKLOADS[args.workload]
    if args.only:
        keep = set(args.only.split(","))
        work = [w for w in work if w[0] in keep]
    threads = os.cpu_count() or 1
    lg = 22
    for _ in range(args.warmup):
        cpu_oracle_rate(work[:1], 16, threads)
    vals = []
    t_all = 0.0
    per = {}
    for _ in range(args.steps):
        v, t, n, per = cpu_oracle_rate(work, lg, threads, budget_s=3.0)
        vals.append(v)
        t_all += t
    value = sum(vals) / len(vals)
    ms = t_all / max(1, args.steps) * 1e3
    line = {"metric": METRIC, "value": round(value, 4), "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64/f32", "data": "synthetic",
            "config": {"workload": args.workload, "text": CONFIG_TEXT[args.workload],
                       "sample": f"2^{lg}-element host arrays per entry point, passes repeated for ~3 s "
                                 f"of CPU work per step"},
            "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": f"{len(work)} entry points x 2^{lg}-element arrays, ~3 s of CPU work "
                                       f"per step, oracle/vem_oracle.c (OpenMP, {threads} threads)",
                             "per_function": per},
            "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------- GPU arm
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
    from paper_2001_09258_b200 import _lib, api, build

    # VEM_BENCH_SHARE_GPU=1 (testing only): map every rank to the visible
    # device(s) round-robin and reduce over gloo -- exercises the multi-rank
    # bookkeeping on a box with fewer GPUs than ranks.
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
    if rank == 0:
        build.build()
    if world > 1:
        dist.barrier()
    _lib.lib()

    work = WORKLOADS[args.workload]
    if args.only:
        keep = set(args.only.split(","))
        work = [w for w in work if w[0] in keep]
    n = 1 << (args.log2n or LOG2N[args.workload])
    strong = args.workload in STRONG
    if strong:  # job-total element count, contiguous shard per rank
        n = n // world

    # resident inputs (u10/u35 of one function share inputs)
    cache = {}
    bufs = []
    if args.workload == "cfg5":
        x5, ypow5, yfm5 = device_inputs_cfg5(n, dev, seed=0x5EEF0050 + 7919 * rank)
        cache = {"x": [x5], "ypow": [ypow5], "yfmod": [yfm5]}
        l_x, l_pow, l_fmod = [x5], [x5, ypow5], [x5, yfm5]  # shared lists: e2e uploads x once
    for name, cfg in work:
        if args.workload == "cfg5":
            fn = name.split("_")[0]
            bufs.append(l_pow if fn == "pow" else (l_fmod if fn == "fmod" else l_x))
            continue
        base = name.replace("_u35", "_u10") if "_u35" in name else name
        key = (base.split("_")[0], base.split("_")[1], cfg)
        if key not in cache:
            cache[key] = device_inputs(name, cfg, n, dev, seed=zlib.crc32(repr(key).encode()) + 7919 * rank)
        bufs.append(cache[key])
    outs = {}
    for ins in bufs:
        outs.setdefault(ins[0].dtype, torch.empty_like(ins[0]))
    stream = torch.cuda.current_stream()

    def step(evs=None):
        for i, (name, _) in enumerate(work):
            ins = bufs[i]
            if evs is not None:
                evs[i][0].record(stream)
            api.call(name, *ins, out=outs[ins[0].dtype])
            if evs is not None:
                evs[i][1].record(stream)

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()

    # per-kernel event pairs for every timed step
    evs = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in work]
           for _ in range(args.steps)]
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = _lib.launch_count()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    # a short device-side spin ahead of the timed region keeps the GPU busy
    # while the host enqueues the first launches, so host launch latency
    # (Python + ctypes) does not appear as device idle time inside it
    torch.cuda._sleep(int(2e6))
    t0.record(stream)
    for s in range(args.steps):
        step(evs[s])
    t1.record(stream)
    torch.cuda.synchronize()
    launches = _lib.launch_count() - launches0
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms_total = t0.elapsed_time(t1)
    per_kernel_ms = [sum(evs[s][i][0].elapsed_time(evs[s][i][1]) for s in range(args.steps)) / args.steps
                     for i in range(len(work))]
    if world > 1:
        t = torch.tensor([ms_total], dtype=torch.float64, device="cpu" if share else dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
    ms_step = ms_total / args.steps
    elems_step = len(work) * n * world
    value = elems_step / (ms_step * 1e-3) / 1e9

    # ---------------- verification (outside the timed region): the one
    # collective of the sharded path -- every rank checks its shard, NCCL
    # all-reduces {mismatch count: SUM, max ulp distance: MAX}
    verify = None
    if not args.no_verify:
        verify = verify_leg(work, bufs, outs, n, dev, world, share)

    # ---------------- e2e: C ABI with HOST buffers (pinned), copies timed
    e2e = None
    if not args.no_e2e:
        e2e = e2e_leg(work, bufs, outs, n, args, dev, stream, world)

    # ---------------- roofline of the dominant kernel
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    hbm_src = "measured (MEASURED_PEAKS.json)" if "hbm_gbs" in peaks else "fallback (B200_PROFILING.md)"
    dom = max(range(len(work)), key=lambda i: per_kernel_ms[i])
    dname = work[dom][0]
    esz = bufs[dom][0].element_size()
    bytes_per_launch = n * esz * (len(bufs[dom]) + 1)
    ach = bytes_per_launch / (per_kernel_ms[dom] * 1e-3) / 1e9
    fp64_peak = _lib.probe_peak("fp64")
    traffic = None
    fp64_per_elem = None
    prof = os.path.join(ROOT, "profiles", "kernel_metrics.json")
    if os.path.exists(prof):
        try:
            allm = json.load(open(prof))
            # metrics depend on the input mix: a capture of this workload's
            # inputs (key "name@cfgN") wins over the entry point's default
            km = allm.get(f"{dname}@{args.workload}", allm.get(dname, {}))
            if km.get("dram_bytes_per_elem") is not None:
                traffic = km["dram_bytes_per_elem"] * n
            fp64_per_elem = km.get("fp64_inst_per_elem")
        except Exception:
            pass
    pipe = None
    if fp64_per_elem:
        ach_ops = fp64_per_elem * n / (per_kernel_ms[dom] * 1e-3) / 1e9
        pipe = {"pipe": "fp64", "achieved": round(ach_ops, 1), "peak": round(fp64_peak, 1), "unit": "Ginst/s",
                "frac": round(ach_ops / fp64_peak, 4), "fp64_inst_per_elem": fp64_per_elem,
                "peak_source": "measured (vem_probe_peak DFMA microbenchmark, this run)"}
    roofline = {"bound": "hbm", "kernel": dname, "achieved": round(ach, 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(ach / hbm_peak, 4), "traffic": traffic, "bytes_per_launch": bytes_per_launch,
                "bytes_per_elem": esz * (len(bufs[dom]) + 1), "elems_per_launch": n,
                "ms_per_launch": round(per_kernel_ms[dom], 4), "peak_source": hbm_src,
                "fp64_pipe": pipe, "fp64_dfma_peak_ginst_s": round(fp64_peak, 1)}

    per_function = {}
    for i, (name, cfg) in enumerate(work):
        esz_i = bufs[i][0].element_size() * (len(bufs[i]) + 1)
        g = n / (per_kernel_ms[i] * 1e-3) / 1e9
        per_function[name] = {"gelem_s": round(g, 2), "ms": round(per_kernel_ms[i], 4),
                              "hbm_frac": round(g * esz_i / hbm_peak, 4)}

    cpu = None
    sleef = None
    if rank == 0 and world == 1 and not args.no_cpu:
        threads = os.cpu_count() or 1
        v, t, cn, per = cpu_oracle_rate(work, 23, threads, budget_s=12.0)
        cpu = {"value": round(v, 4), "unit": UNIT, "cores": threads, "kind": "port",
               "sample": f"{len(work)} entry points x 2^23-element arrays of the same config domains, repeated "
                         f"passes: {cn / 1e9:.2f} G elements in {t:.1f} s of CPU work, oracle/vem_oracle.c, "
                         f"OpenMP {threads} threads",
               "per_function": per}
        try:
            sleef = cpu_sleef_rate(work, 23, threads)
        except Exception as ex:  # context only
            sleef = {"error": str(ex)}

    ws = sum(t.numel() * t.element_size() for ins in cache.values() for t in ins) + \
        sum(t.numel() * t.element_size() for t in outs.values())
    l2_note = (f"no flush: per-step working set {ws / 2**20:.0f} MiB (distinct inputs {n}-element arrays + "
               f"outputs) > 126 MB L2, each input re-read only after the other kernels' traffic")
    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True,
                "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": "f64/f32 (per entry point)",
                "data": "synthetic (config-domain inputs generated on device, seeded)",
                "config": {"workload": args.workload, "text": CONFIG_TEXT[args.workload],
                           "elements_per_entry_point_per_rank": n, "entry_points": [w[0] for w in work],
                           "l2": l2_note,
                           "parallelism": f"data-parallel shards x{world} (no collective on the data path)"},
                "gpu_launches": int(launches), "clocks": clk, "roofline": roofline,
                "per_function": per_function, "e2e": e2e, "cpu_baseline": cpu, "sleef_cpu": sleef,
                "verify": verify}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def verify_leg(work, bufs, outs, n, dev, world, share):
    """Every entry point over the rank's whole shard twice: the shipped
    TMA-pipelined / work-queue kernel (16-byte aligned buffers) and the plain
    grid-stride kernel the library takes for misaligned pointers (same math,
    independent load/store path, no staging or regrouping), compared bit for
    bit on the device; per rank: mismatching elements (SUM) and the largest
    ulp distance (MAX), combined over the ranks by one all-reduce each.  Bit
    identity to the CPU oracle is the test suite's job (tests/); this checks,
    at full scale on every shard, that the fast data path returns exactly
    what the per-element function computes."""
    import torch
    import torch.distributed as dist
    from paper_2001_09258_b200 import api
    mism = 0
    max_ulp = 0
    checked = 0
    for i, (name, _) in enumerate(work):
        ins = bufs[i]
        dt = ins[0].dtype
        it = torch.int64 if dt == torch.float64 else torch.int32
        a = api.call(name, *ins, out=outs[dt])
        un = []
        for t in ins:
            u = torch.empty(n + 1, dtype=dt, device=dev)
            u[1:].copy_(t)
            un.append(u[1:])  # 4/8-byte offset: the misaligned (plain) path
        ob = torch.empty(n + 1, dtype=dt, device=dev)
        b = api.call(name, *un, out=ob[1:])
        ai, bi = a.view(it), b.view(it)
        ne = ai != bi
        mism += int(ne.sum().item())
        if bool(ne.any().item()):
            # same-sign finite values: ulp distance = difference of the bit patterns
            d = (ai.to(torch.int64) - bi.to(torch.int64)).abs()
            max_ulp = max(max_ulp, int(d[ne].max().item()))
        checked += n
        del un, ob, b
    torch.cuda.empty_cache()
    if world > 1:
        t = torch.tensor([mism, checked], dtype=torch.int64, device="cpu" if share else dev)
        m = torch.tensor([max_ulp], dtype=torch.int64, device="cpu" if share else dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        dist.all_reduce(m, op=dist.ReduceOp.MAX)
        mism, checked, max_ulp = int(t[0].item()), int(t[1].item()), int(m[0].item())
    return {"elements": checked, "mismatches": mism, "max_ulp": max_ulp,
            "compared": "TMA-pipelined / work-queue kernels vs the plain grid-stride kernel (misaligned "
                        "pointers), bit for bit, every element of every shard",
            "reduction": "all_reduce SUM (mismatches) and MAX (ulp) over the ranks"}


def e2e_leg(work, bufs, outs, n, args, dev, stream, world):
    """Same step through the C ABI with HOST buffers: every step uploads that
    step's distinct inputs host->device from pinned memory (the u10 and u35
    entry points of one function read the same arrays, so each input array is
    uploaded once), runs every entry point, and reads every result back
    device->host into its own pinned buffer; chunked over three streams so
    copies in both directions overlap the kernels (4 streams, 2^24-element
    chunks: the best of a chunk x stream sweep, profiles/r01_e2e_sweep.log)."""
    import torch
    from paper_2001_09258_b200 import api
    chunk = 1 << int(os.environ.get("VEM_E2E_CHUNK_LOG2", "24"))
    nstreams = int(os.environ.get("VEM_E2E_STREAMS", "4"))
    n = min(n, 1 << 26)  # 2^26 elements per entry point per rank (bounded pinned memory)
    groups = []  # (device input list, [(entry name, work index)])
    for i, (name, _) in enumerate(work):
        for g in groups:
            if g[0] is bufs[i]:
                g[1].append((name, i))
                break
        else:
            groups.append((bufs[i], [(name, i)]))
    host_in = {id(g[0]): [t[:n].to("cpu").pin_memory() for t in g[0]] for g in groups}
    host_out = [torch.empty(n, dtype=bufs[i][0].dtype).pin_memory() for i in range(len(work))]
    dev_out = [torch.empty(n, dtype=bufs[i][0].dtype, device=dev) for i in range(len(work))]
    streams = [torch.cuda.Stream(dev) for _ in range(nstreams)]
    h2d = sum(t.numel() * t.element_size() for v in host_in.values() for t in v)
    d2h = sum(h.numel() * h.element_size() for h in host_out)

    def one_step():
        for dins, members in groups:
            hin = host_in[id(dins)]
            for j, c0 in enumerate(range(0, n, chunk)):
                c1 = min(n, c0 + chunk)
                s = streams[j % nstreams]  # a given range always uses the same stream
                with torch.cuda.stream(s):
                    for hd, dd_ in zip(hin, dins):
                        dd_[c0:c1].copy_(hd[c0:c1], non_blocking=True)
                    for name, i in members:
                        api.call(name, *[d[c0:c1] for d in dins], out=dev_out[i][c0:c1])
                        host_out[i][c0:c1].copy_(dev_out[i][c0:c1], non_blocking=True)

    one_step()
    torch.cuda.synchronize()
    steps = max(1, min(args.steps, 3))
    t0 = time.perf_counter()
    for _ in range(steps):
        one_step()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / steps
    return {"value": round(len(work) * n * world / dt / 1e9, 3), "unit": UNIT, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": round(dt * 1e3, 2), "steps": steps,
            "elements_per_entry_point_per_rank": n,
            "path": "pinned host -> H2D (each distinct input once, chunked 2^24, 4 streams) -> vem C ABI "
                    "(every entry point) -> D2H of every result, host wall clock"}


if __name__ == "__main__":
    main()
