"""CPU-only checks of the product boundary: libvem.so builds for sm_100a,
loads without a GPU, exports every symbol include/vem.h declares, the host
mirror rejects misuse loudly (no CPU fallback), inputs are deterministic, and
the sharded multi-rank bookkeeping works over gloo with world_size 2."""
from __future__ import annotations

import hashlib
import os
import re
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2001_09258_b200 import _lib, build
    build.build()
    return _lib.lib()


def test_every_declared_symbol_is_exported(lib):
    hdr = open(os.path.join(ROOT, "include", "vem.h")).read()
    names = set(re.findall(r"^\s*(?:int|uint64_t|const char\*)\s+(vem_\w+)\s*\(", hdr, re.M))
    assert len(names) >= 35
    for n in names:
        assert hasattr(lib, n), n
    out = subprocess.run(["nm", "-D", os.path.join(ROOT, "paper_2001_09258_b200", "libvem.so")],
                         capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (vem_\w+)", out))
    assert names <= exported


def test_library_is_sm100a_only():
    so = os.path.join(ROOT, "paper_2001_09258_b200", "libvem.so")
    out = subprocess.run(["cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_no_cpu_fallback_symbols():
    """The product never links the oracle."""
    so = os.path.join(ROOT, "paper_2001_09258_b200", "libvem.so")
    out = subprocess.run(["nm", "-D", so], capture_output=True, text=True).stdout
    assert "vo_" not in out and "mpfr" not in out


def test_host_table_digest(lib):
    from paper_2001_09258_b200 import _lib
    d = dict(line.split() for line in open(os.path.join(ROOT, "tests", "golden", "ph_table_digests.txt")))
    assert hashlib.md5(_lib.ph_table_bytes()).hexdigest() == d["f64_mod4"]


def test_version_and_counter(lib):
    from paper_2001_09258_b200 import _lib
    assert b"sm_100a" in lib.vem_version()
    assert _lib.launch_count() >= 0


def test_api_rejects_cpu_tensors():
    torch = pytest.importorskip("torch")
    from paper_2001_09258_b200 import api
    with pytest.raises(TypeError):
        api.sin(torch.zeros(4, dtype=torch.float64))
    with pytest.raises(TypeError):
        api.exp(torch.zeros(4, dtype=torch.int32))


def test_inputs_deterministic():
    from paper_2001_09258_b200 import inputs as I
    a = I.config_inputs(2, "pow", "d", 1000)
    b = I.config_inputs(2, "pow", "d", 1000)
    assert all(np.array_equal(u, v) for u, v in zip(a, b))
    x = I.config_inputs(5, "sin", "d", 100000)[0]
    frac = np.mean(~np.isfinite(x) | (x == 0) | (np.abs(x) < 2.3e-308) | (np.abs(x) > 1.7e308))
    assert 0.005 < frac < 0.02
    x3 = I.config_inputs(3, "sin", "f", 10000)[0]
    assert x3.dtype == np.float32 and np.all(np.abs(x3) >= 1) and np.all(np.isfinite(x3))


def _gloo_worker(rank, world, port, q):
    """One rank of the sharded path on the CPU: its contiguous shard of the
    first 2^24-element chunk of config 1 (host generator + oracle), partial
    chunk checksums, the path's one collective (all_reduce SUM of the chunk
    vectors, bench.py verify_workload) and the max-over-ranks timing
    reduction; rank 0 compares with the golden oracle checksum."""
    import json

    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_lib as O
    from paper_2001_09258_b200 import configs as C
    m = 1 << C.LOG2CHUNK
    lo, hi = m * rank // world, m * (rank + 1) // world  # contiguous shard, ragged
    (r,) = C.recipes("cfg1", "sin_d_u10")
    x = O.gen_fill(r, hi - lo, lo)
    out = O.oracle_eval("sin_d_u10", x)
    vec = torch.tensor([C.chunk_vector(O.gen_checksum(out, lo, C.LOG2CHUNK), 1)], dtype=torch.int64)
    dist.all_reduce(vec, op=dist.ReduceOp.SUM)
    t = torch.tensor([float(rank + 1)])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)  # max-over-ranks timing reduction
    if rank == 0:
        gold = json.load(open(os.path.join(ROOT, "tests", "golden", "config_checksums.json")))
        ref = gold["configs"]["cfg1"]["outputs"]["sin_d_u10"]
        q.put((C.mismatching_chunks(vec[0].tolist(), ref, 0, 1), float(t.item())))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_checksums_gloo(world):
    import multiprocessing as mp
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_gloo_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    bad, mx = q.get(timeout=180)
    for p in ps:
        p.join(timeout=60)
    assert bad == [] and mx == float(world)
