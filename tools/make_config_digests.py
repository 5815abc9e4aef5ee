#!/usr/bin/env python3
"""Golden oracle checksums over the FULL BASELINE config arrays
(tests/golden/config_checksums.json).

For every workload of paper_2001_09258_b200/configs.py and every 2^24-element
chunk of its global index space (weak configs: ranks 0..7, i.e. 8 x the
per-rank size; config 5: the 2^31-element job), the host generator
(oracle/vem_gen_host.c, bit-identical to inputs.py and to the device twin)
makes the operands, the CPU ORACLE (oracle/vem_oracle.c) evaluates every
entry point, and the chunk checksums (vem_aux.h definition) of operands and
results are recorded; config 1 also gets the MD5 of rank 0's whole 2^24-element
output ("compared bit-for-bit", BASELINE configs[0]).  The GPU side
(tests/test_config_parity.py, bench.py's verify leg) regenerates the operands
on the device and compares its own checksums -- no oracle on the GPU box.

Usage: python tools/make_config_digests.py [cfg1,cfg2,...]   (~5 min, 8 cores)
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle_lib as O  # noqa: E402
from paper_2001_09258_b200 import configs as C  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "config_checksums.json")


def total_elems(w):
    n = 1 << C.LOG2N[w]
    return n if w in C.STRONG else n * C.MAX_RANKS


def run(w):
    names = C.WORKLOADS[w]
    T = total_elems(w)
    chunk = 1 << C.LOG2CHUNK
    groups = {}
    for name in names:
        groups.setdefault(C.input_key(w, name), []).append(name)
    ins = {}
    outs = {name: [] for name in names}
    md5 = {name: hashlib.md5() for name in names} if w == "cfg1" else {}
    in_md5 = {}
    n_rank = 1 << C.LOG2N[w]
    t0 = time.time()
    for c0 in range(0, T, chunk):
        m = min(chunk, T - c0)
        for key, members in groups.items():
            rs = C.recipes(w, members[0])
            arrs = [O.gen_fill(r, m, c0) for r in rs]
            for k, a in enumerate(arrs):
                ins.setdefault(f"{members[0]}#{k}", []).append(O.gen_checksum(a, c0, C.LOG2CHUNK)[c0 >> C.LOG2CHUNK])
                if w == "cfg1" and c0 < n_rank:
                    in_md5.setdefault(f"{members[0]}#{k}", hashlib.md5()).update(a.tobytes())
            for name in members:
                o = O.oracle_eval(name, *arrs)
                outs[name].append(O.gen_checksum(o, c0, C.LOG2CHUNK)[c0 >> C.LOG2CHUNK])
                if name in md5 and c0 < n_rank:
                    md5[name].update(o.tobytes())
        if (c0 // chunk) % 16 == 15:
            print(f"  {w}: {c0 + m}/{T} elements, {time.time() - t0:.0f} s", flush=True)
    hx = lambda v: f"{v:016x}"  # noqa: E731
    rec = {"total_elements": T, "per_rank": n_rank if w not in C.STRONG else None,
           "scaling": "strong" if w in C.STRONG else "weak",
           "inputs": {k: [hx(v) for v in vs] for k, vs in ins.items()},
           "outputs": {k: [hx(v) for v in vs] for k, vs in outs.items()},
           "oracle_seconds": round(time.time() - t0, 1)}
    if md5:
        rec["md5_rank0"] = {k: h.hexdigest() for k, h in md5.items()}
        rec["md5_rank0_inputs"] = {k: h.hexdigest() for k, h in in_md5.items()}
    return rec


def main():
    want = sys.argv[1].split(",") if len(sys.argv) > 1 else list(C.WORKLOADS)
    gold = json.load(open(OUT)) if os.path.exists(OUT) else {}
    gold["log2chunk"] = C.LOG2CHUNK
    gold["generator"] = "paper_2001_09258_b200/inputs.py (host twin oracle/vem_gen_host.c)"
    gold["checker"] = "oracle/vem_oracle.c (CPU oracle)"
    cfgs = gold.setdefault("configs", {})
    for w in want:
        print(f"{w} ...", flush=True)
        cfgs[w] = run(w)
        json.dump(gold, open(OUT + ".tmp", "w"), indent=0, sort_keys=True)
        os.replace(OUT + ".tmp", OUT)
        print(f"{w}: done in {cfgs[w]['oracle_seconds']} s", flush=True)


if __name__ == "__main__":
    main()
