#!/usr/bin/env python3
"""Board power and sustained throughput per entry point (dev tool, runs on a GPU).

Usage: python tools/power_probe.py NAME[,NAME...] CFG [log2_n=28] [seconds=1.5]
Loops each entry point alone for `seconds`, samples nvmlDeviceGetPowerUsage and
the SM clock every 10 ms in a thread, and prints the throughput of the first
and the last 100 launches (burst vs sustained), mean power over the second
half of the loop and the energy per 10^9 elements."""
import os
import sys
import threading
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2001_09258_b200 import _aux, api  # noqa: E402
from paper_2001_09258_b200 import inputs as I  # noqa: E402


def main():
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    cfg = int(sys.argv[2])
    n = 1 << (int(sys.argv[3]) if len(sys.argv) > 3 else 28)
    secs = float(sys.argv[4]) if len(sys.argv) > 4 else 1.5
    for name in sys.argv[1].split(","):
        fn, p = name.split("_")[0], name.split("_")[1]
        ts = [_aux.fill(r, torch.empty(n, dtype=torch.float32 if r["f32"] else torch.float64, device="cuda"))
              for r in I.config_recipes(cfg, fn, p)]
        out = torch.empty_like(ts[0])
        api.call(name, *ts, out=out)
        torch.cuda.synchronize()
        time.sleep(1.0)  # idle: let the power average decay
        samples, stop = [], threading.Event()

        def sampler():
            while not stop.is_set():
                samples.append((time.perf_counter(), pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                                pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)))
                time.sleep(0.01)

        th = threading.Thread(target=sampler)
        th.start()
        evs = []
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < secs:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                api.call(name, *ts, out=out)
            e1.record()
            evs.append((e0, e1))
            torch.cuda.synchronize()
        stop.set()
        th.join()
        rates = [20 * n / (a.elapsed_time(b) * 1e6) for a, b in evs]
        half = [s for s in samples if s[0] - t0 > secs / 2]
        pw = sum(s[1] for s in half) / max(1, len(half))
        clk = sorted(s[2] for s in half)[len(half) // 2] if half else 0
        k = max(1, len(rates) // 5)
        first, last = sum(rates[:k]) / k, sum(rates[-k:]) / k
        print(f"{name}: first {first:.1f} last {last:.1f} Gelem/s, power {pw:.0f} W, sm {clk} MHz, "
              f"{pw / last:.2f} J per 1e9 elements", flush=True)
        del ts, out
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
