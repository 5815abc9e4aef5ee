"""The BASELINE.json configurations as bench / parity workloads.

One table shared by bench.py (timing), tools/make_config_digests.py (oracle
golden checksums over the full arrays) and tests/test_config_parity.py (GPU
vs those checksums).  Inputs come from inputs.config_recipes (counter-based:
element i of an operand is a pure function of (recipe, i)).

Sharding:
  * weak configs (1-4): rank r of N evaluates elements [r*n, (r+1)*n) of
    the config's streams, n = the config's size per rank; golden checksums
    cover ranks 0..7;
  * strong config 5: the 2^31-element job is split contiguously,
    rank r gets [r*T/N, (r+1)*T/N).
"""
from __future__ import annotations

LOG2CHUNK = 24  # checksum chunk: 2^24 elements of the global index space
MAX_RANKS = 8

WORKLOADS = {
    "cfg2": ["exp_d_u10", "exp_d_u35", "log_d_u10", "log_d_u35", "pow_d_u10", "pow_d_u35", "exp_f_u10",
             "exp_f_u35", "log_f_u10", "log_f_u35", "pow_f_u10", "pow_f_u35"],
    "cfg1": ["sin_d_u10", "cos_d_u10"],
    "cfg3": ["sin_d_u10_ph", "cos_d_u10_ph", "tan_d_u10_ph", "sin_f_u10_ph", "cos_f_u10_ph", "tan_f_u10_ph"],
    "cfg4": ["fmod_d", "fmod_f"],
    "cfg5": ["sin_d_u10", "cos_d_u10", "tan_d_u10", "atan_d_u10", "exp_d_u10", "log_d_u10", "pow_d_u10", "fmod_d"],
}
CFG_NUM = {"cfg1": 1, "cfg2": 2, "cfg3": 3, "cfg4": 4, "cfg5": 5}
LOG2N = {"cfg1": 24, "cfg2": 28, "cfg3": 28, "cfg4": 26, "cfg5": 31}
STRONG = {"cfg5"}
CONFIG_TEXT = {
    "cfg1": "sin/cos f64 u10, 2^24 x U[-pi,pi] (Cody-Waite path)",
    "cfg2": "exp/log/pow x f32/f64 x u10/u35, 2^28 elements each (BASELINE configs[1] domains)",
    "cfg3": "sin/cos/tan u10 f64+f32, 2^28, |x| log-U[1,1e300]/[1,3e38] +-, forced Payne-Hanek",
    "cfg4": "fmod f64+f32, 2^26 pairs, log-U[1e-300,1e300]/[1e-37,3e38] +-",
    "cfg5": "2^31 f64 elements (one shared x array; pow y U[-30,30], fmod y log-U) sharded over the ranks, "
            "through sin/cos/tan/atan/exp/log/pow/fmod u10; log-U[1e-300,1e300] +- with 1% specials",
}


def fn_prec(name: str):
    fn, p = name.split("_")[0], name.split("_")[1]
    return fn, p


def recipes(workload: str, name: str):
    from . import inputs as I
    fn, p = fn_prec(name)
    return I.config_recipes(CFG_NUM[workload], fn, p)


def input_key(workload: str, name: str) -> str:
    """Entry points whose operands are the same arrays share a key (u10/u35
    of one function; every config-5 function shares x)."""
    rs = recipes(workload, name)
    return "|".join(f"{r['kind']}:{r['seed']:x}:{r['a']!r}:{r['b']!r}:{r['sign']}{r['specials']}{r['f32']}"
                    for r in rs)


def shard(workload: str, rank: int, world: int):
    """(offset, n) of this rank's slice of the config's global index space."""
    n = 1 << LOG2N[workload]
    if workload in STRONG:
        lo, hi = n * rank // world, n * (rank + 1) // world
        return lo, hi - lo
    return rank * n, n


# ---------------------------------------- checksum vectors (the one collective)
M64 = (1 << 64) - 1


def chunk_vector(partials: dict, nchunks: int) -> list:
    """{chunk: uint64 partial} -> a dense int64 (two's complement) vector, the
    operand of the ranks' all_reduce(SUM): sums wrap mod 2^64 exactly like the
    checksum definition."""
    v = [0] * nchunks
    for c, s in partials.items():
        if 0 <= c < nchunks:
            v[c] = s - (1 << 64) if s >= (1 << 63) else s
    return v


def mismatching_chunks(row, ref_hex, c_lo: int, c_hi: int) -> list:
    """Chunks in [c_lo, c_hi) whose reduced checksum differs from the golden hex."""
    return [c for c in range(c_lo, c_hi) if f"{int(row[c]) & M64:016x}" != ref_hex[c]]
