"""bench.py's multi-rank path: contiguous shards, no
collective on the data path, one all-reduce of the verification checksums and
of the timings.  On a box with one GPU the ranks share it
(VEM_BENCH_SHARE_GPU=1, gloo): no kernel waits on another rank, so this is
safe on one device; the timing is not meaningful there, the bookkeeping is."""
from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

import pytest

from paper_2001_09258_b200 import configs as C

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_shards_partition_the_job():
    for w in C.WORKLOADS:
        n = 1 << C.LOG2N[w]
        for world in (1, 2, 3, 4, 7, 8):
            sl = [C.shard(w, r, world) for r in range(world)]
            if w in C.STRONG:
                assert sl[0][0] == 0 and sum(m for _, m in sl) == n
                assert all(sl[i][0] + sl[i][1] == sl[i + 1][0] for i in range(world - 1))
            else:
                assert sl == [(r * n, n) for r in range(world)]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.gpu
@pytest.mark.parametrize("workload,world", [("cfg1", 2), ("cfg5", 2), ("cfg4", 3)])
def test_bench_torchrun_shared_gpu(cuda, workload, world):
    env = dict(os.environ, VEM_BENCH_SHARE_GPU="1", MASTER_ADDR="127.0.0.1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", str(world),
           "--workload", workload, "--steps", "3", "--warmup", "3", "--no-e2e", "--no-cpu"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    line = json.loads(lines[0])
    assert line["n_gpus"] == world and line["gpu_launches"] > 0
    v = line["verify"]
    assert v["mismatching_chunks"] == 0, v
    n = 1 << C.LOG2N[workload]
    want = n if workload in C.STRONG else min(world, C.MAX_RANKS) * n
    assert v["elements_per_entry_point"] == want
