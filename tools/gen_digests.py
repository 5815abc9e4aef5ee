#!/usr/bin/env python3
"""Golden MD5 digests of the CPU oracle over 2^24 random-bit inputs per
entry point (tests/digest_inputs.py) -> tests/golden/oracle_digests.json.
The GPU test (tests/test_gpu_digests.py) recomputes the inputs, runs the
kernels and compares digests: bit identity on ~10^9 points without the
oracle on the GPU box.  Usage: python tools/gen_digests.py [names...]"""
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from digest_inputs import N_DIGEST, digest_inputs  # noqa: E402
from oracle_lib import oracle_eval  # noqa: E402

from paper_2001_09258_b200 import _lib  # noqa: E402


def main():
    path = os.path.join(ROOT, "tests", "golden", "oracle_digests.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    names = sys.argv[1:] or sorted(_lib.ALL)
    for name in names:
        t = time.time()
        r = oracle_eval(name, *digest_inputs(name))
        out[name] = {"n": N_DIGEST, "md5": hashlib.md5(r.tobytes()).hexdigest()}
        print(name, out[name]["md5"], f"{time.time() - t:.1f}s", flush=True)
    json.dump(out, open(path, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
