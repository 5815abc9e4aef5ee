#!/usr/bin/env python3
"""Oracle accuracy sweep vs MPFR (max ULP per function/domain); dev tool."""
import sys, os, time
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
from oracle_lib import oracle_eval, ulp_errors
from paper_2001_09258_b200 import inputs as I

def rnd_bits(seed, n, dt):
    b = I.splitmix64(seed, n)
    if dt == np.float32:
        return (b & np.uint64(0xffffffff)).astype(np.uint32).view(np.float32)
    return b.view(np.float64)

def check(name, fn, args, bound):
    t=time.time()
    out = oracle_eval(name, *args)
    e = ulp_errors(fn, args[0], out, args[1] if len(args) > 1 else None)
    i = int(np.argmax(e))
    ok = "OK " if e[i] <= bound else "BAD"
    extra = f" y={args[1][i]!r}" if len(args)>1 else ""
    print(f"{ok} {name:14s} max {e[i]:.4f} ulp at x={args[0][i]!r}{extra} out={out[i]!r} ({time.time()-t:.1f}s)", flush=True)
    return e[i]

N = int(sys.argv[2]) if len(sys.argv) > 2 else 200000
which = sys.argv[1] if len(sys.argv) > 1 else "all"
D, F = np.float64, np.float32
tests = []
def add(name, fn, bound, gens): tests.append((name, fn, bound, gens))
add("sin_d_u10", "sin", 1.0, [lambda: (I.uniform(1,N,-np.pi,np.pi),), lambda: (I.log_uniform(2,N,1,1e300,signed=True),), lambda:(I.uniform(3,N,-15,15),), lambda:(I.log_uniform(4,N,15,1e14,signed=True),), lambda:(rnd_bits(5,N,D),)])
add("cos_d_u10", "cos", 1.0, [lambda: (I.uniform(1,N,-np.pi,np.pi),), lambda: (I.log_uniform(2,N,1,1e300,signed=True),), lambda:(I.log_uniform(4,N,15,1e14,signed=True),), lambda:(rnd_bits(5,N,D),)])
add("tan_d_u10", "tan", 1.0, [lambda: (I.uniform(1,N,-np.pi,np.pi),), lambda: (I.log_uniform(2,N,1,1e300,signed=True),), lambda:(I.log_uniform(4,N,15,1e14,signed=True),), lambda:(rnd_bits(5,N,D),)])
add("sin_d_u10_ph", "sin", 1.0, [lambda: (I.uniform(1,N,-np.pi,np.pi),), lambda: (I.log_uniform(2,N,1,1e300,signed=True),)])
add("cos_d_u10_ph", "cos", 1.0, [lambda: (I.log_uniform(2,N,1,1e300,signed=True),)])
add("tan_d_u10_ph", "tan", 1.0, [lambda: (I.log_uniform(2,N,1,1e300,signed=True),)])
add("atan_d_u10", "atan", 1.0, [lambda: (I.uniform(1,N,-700,700),), lambda: (I.log_uniform(2,N,1e-300,1e300,signed=True),), lambda:(I.uniform(3,N,-2,2),), lambda:(rnd_bits(5,N,D),)])
add("exp_d_u10", "exp", 1.0, [lambda: (I.uniform(1,N,-700,700),), lambda:(I.uniform(3,N,-1,1),), lambda:(I.uniform(3,N,-745.2,-700),), lambda:(rnd_bits(5,N,D),)])
add("exp_d_u35", "exp", 3.5, [lambda: (I.uniform(1,N,-700,700),), lambda:(rnd_bits(5,N,D),)])
add("log_d_u10", "log", 1.0, [lambda: (I.log_uniform(1,N,1e-300,1e300),), lambda:(I.uniform(3,N,0.3,3),), lambda:(rnd_bits(5,N,D),)])
add("log_d_u35", "log", 3.5, [lambda: (I.log_uniform(1,N,1e-300,1e300),), lambda:(I.uniform(3,N,0.3,3),), lambda:(rnd_bits(5,N,D),)])
add("pow_d_u10", "pow", 1.0, [lambda: (I.log_uniform(1,N,1e-10,1e10), I.uniform(2,N,-30,30)), lambda:(I.uniform(3,N,0,30), I.uniform(4,N,-30,30)), lambda:(I.log_uniform(5,N,1e-300,1e300,signed=True), I.uniform(6,N,-30,30)), lambda:(rnd_bits(7,N,D), rnd_bits(8,N,D))])
add("pow_d_u35", "pow", 3.5, [lambda: (I.log_uniform(1,N,1e-10,1e10), I.uniform(2,N,-30,30)), lambda:(I.uniform(3,N,0,30), I.uniform(4,N,-30,30))])
add("sin_f_u10", "sin", 1.0, [lambda: (I.log_uniform(2,N,1,3e38,F,signed=True),), lambda:(I.uniform(3,N,-10,10,F),), lambda:(rnd_bits(5,N,F),)])
add("cos_f_u10", "cos", 1.0, [lambda: (I.log_uniform(2,N,1,3e38,F,signed=True),), lambda:(I.uniform(3,N,-10,10,F),), lambda:(rnd_bits(5,N,F),)])
add("tan_f_u10", "tan", 1.0, [lambda: (I.log_uniform(2,N,1,3e38,F,signed=True),), lambda:(I.uniform(3,N,-10,10,F),), lambda:(rnd_bits(5,N,F),)])
add("exp_f_u10", "exp", 1.0, [lambda: (I.uniform(1,N,-87,88,F),), lambda:(I.uniform(3,N,-104,-87,F),), lambda:(rnd_bits(5,N,F),)])
add("exp_f_u35", "exp", 3.5, [lambda: (I.uniform(1,N,-87,88,F),), lambda:(rnd_bits(5,N,F),)])
add("log_f_u10", "log", 1.0, [lambda: (I.log_uniform(1,N,1e-37,3e38,F),), lambda:(rnd_bits(5,N,F),)])
add("log_f_u35", "log", 3.5, [lambda: (I.log_uniform(1,N,1e-37,3e38,F),), lambda:(rnd_bits(5,N,F),)])
add("pow_f_u10", "pow", 1.0, [lambda: (I.log_uniform(1,N,1e-3,1e3,F), I.uniform(2,N,-10,10,F)), lambda:(rnd_bits(7,N,F), rnd_bits(8,N,F))])
add("pow_f_u35", "pow", 3.5, [lambda: (I.log_uniform(1,N,1e-3,1e3,F), I.uniform(2,N,-10,10,F))])
add("fmod_d", "fmod", 0.0, [lambda: (I.log_uniform(1,N,1e-300,1e300,signed=True), I.log_uniform(2,N,1e-300,1e300,signed=True)), lambda:(rnd_bits(7,N,D), rnd_bits(8,N,D))])
add("fmod_f", "fmod", 0.0, [lambda: (I.log_uniform(1,N,1e-37,3e38,F,signed=True), I.log_uniform(2,N,1e-37,3e38,F,signed=True)), lambda:(rnd_bits(7,N,F), rnd_bits(8,N,F))])
for name, fn, bound, gens in tests:
    if which != "all" and not name.startswith(which): continue
    for g in gens:
        check(name, fn, g(), bound)
