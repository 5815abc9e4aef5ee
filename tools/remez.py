"""Discrete Remez exchange for weighted minimax polynomial fits (build-time tool).

Implements the coefficient generator the reference specifies but does not ship
("minimax_fit"; §5 "a tool for generating coefficients
that minimizes the maximum relative error").  The paper publishes no
coefficients, so every table in this repo is produced here and then
frozen as hex floats (coefficient file format SPEC.md:341-342).

Problem solved:  minimise  max_{x in grid} | w(x) * (sum_i c_i x^{p_i} + F(x) - g(x)) |
where F is the (already rounded, fixed) part of the polynomial.  The grid is a
dense set of Chebyshev nodes on [a, b]; the exchange runs on that grid, which
gives a near-minimax fit (within a grid-resolution factor of the true optimum).

Coefficient rounding follows the usual sequential scheme: fit with all terms
free, round the lowest-power free term to binary64 (or to a double-double when
the kernel evaluates that term in DD), freeze it, refit the rest, and repeat.
"""
from __future__ import annotations

import mpmath as mp


def cheb_grid(a, b, n):
    a = mp.mpf(a)
    b = mp.mpf(b)
    out = []
    for k in range(n):
        t = mp.cos(mp.pi * k / (n - 1))
        out.append((a + b) / 2 + (b - a) / 2 * t)
    out.sort()
    return out


def _solve(A, rhs):
    M = mp.matrix(A)
    v = mp.matrix(rhs)
    return mp.lu_solve(M, v)


class Fit:
    def __init__(self, coeffs, powers, err, fixed):
        self.coeffs = coeffs
        self.powers = powers
        self.err = err
        self.fixed = fixed


def remez(g_vals, w_vals, grid, powers, fixed=None, iters=40, tol=1e-4, ref=None):
    """Weighted discrete Remez.

    g_vals / w_vals: target and weight on grid.  powers: free monomial powers.
    fixed: list of (power, value) already frozen.  Returns (coeffs, maxerr, ref).
    """
    fixed = fixed or []
    n = len(powers)
    N = len(grid)
    # residual target after removing fixed terms
    tgt = []
    for k, x in enumerate(grid):
        s = g_vals[k]
        for p, c in fixed:
            s -= c * x ** p
        tgt.append(s)
    xp = [[x ** p for p in powers] for x in grid]
    if ref is None or len(ref) != n + 1:
        ref = [int(round(j * (N - 1) / n)) for j in range(n + 1)]
    best = None
    for _ in range(iters):
        A = []
        rhs = []
        for j, k in enumerate(ref):
            row = list(xp[k]) + [(-1) ** j / w_vals[k]]
            A.append(row)
            rhs.append(tgt[k])
        sol = _solve(A, rhs)
        c = [sol[i] for i in range(n)]
        E = abs(sol[n])
        err = []
        for k in range(N):
            s = mp.mpf(0)
            row = xp[k]
            for i in range(n):
                s += c[i] * row[i]
            err.append(w_vals[k] * (s - tgt[k]))
        maxe = max(abs(e) for e in err)
        if best is None or maxe < best[1]:
            best = (c, maxe, list(ref))
        if maxe <= E * (1 + tol):
            break
        # new reference: extremum of each same-sign run
        ext = []
        k = 0
        while k < N:
            sgn = err[k] >= 0
            j = k
            bi = k
            while j < N and (err[j] >= 0) == sgn:
                if abs(err[j]) > abs(err[bi]):
                    bi = j
                j += 1
            ext.append(bi)
            k = j
        if len(ext) > n + 1:
            # choose the window of n+1 consecutive (hence alternating) extrema
            # that contains the global maximum and has the largest minimum
            gi = max(range(len(ext)), key=lambda i: abs(err[ext[i]]))
            best_w = None
            for s0 in range(max(0, gi - n), min(gi, len(ext) - n - 1) + 1):
                m = min(abs(err[ext[i]]) for i in range(s0, s0 + n + 1))
                if best_w is None or m > best_w[0]:
                    best_w = (m, s0)
            ext = ext[best_w[1]:best_w[1] + n + 1]
        if len(ext) < n + 1:
            break
        if ext == ref:
            break
        ref = ext
    return best


def to_double(x):
    return float(mp.mpf(x))


def to_dd(x):
    hi = float(mp.mpf(x))
    lo = float(mp.mpf(x) - mp.mpf(hi))
    return hi, lo


def fit_rounded(g, w, a, b, powers, dd_terms=0, ngrid=3000, prec=192, lead_fixed=None):
    """Sequentially-rounded minimax fit.

    g, w: callables on mpf.  powers: ascending list of monomial powers.
    dd_terms: the first `dd_terms` powers are emitted as (hi, lo) pairs.
    lead_fixed: optional dict power->exact value to freeze before fitting
    (e.g. the exactly-known leading Taylor coefficient).
    Returns list of (power, hi, lo_or_None) and the max weighted error after
    rounding (evaluated on the grid in `prec`-bit arithmetic).
    """
    with mp.workprec(prec):
        grid = cheb_grid(a, b, ngrid)
        gv = [g(x) for x in grid]
        wv = [w(x) for x in grid]
        fixed = []
        out = []
        free = list(powers)
        if lead_fixed:
            for p, v in lead_fixed.items():
                fixed.append((p, mp.mpf(v)))
                free.remove(p)
        ref = None
        idx = 0
        while free:
            c, e, ref_full = remez(gv, wv, grid, free, fixed=fixed, ref=ref)
            p = free[0]
            if idx < dd_terms:
                hi, lo = to_dd(c[0])
                val = mp.mpf(hi) + mp.mpf(lo)
                out.append((p, hi, lo))
            else:
                hi = to_double(c[0])
                val = mp.mpf(hi)
                out.append((p, hi, None))
            fixed.append((p, val))
            free = free[1:]
            # shrink reference to n+1 points for the smaller system
            ref = None
            idx += 1
        def grid_err(fx):
            m = mp.mpf(0)
            for k, x in enumerate(grid):
                s = mp.mpf(0)
                for p, cv in fx:
                    s += cv * x ** p
                e = abs(wv[k] * (s - gv[k]))
                if e > m:
                    m = e
            return m

        maxe = grid_err(fixed)
        # alternative: round the unconstrained minimax fit directly; keep
        # whichever rounded coefficient set has the smaller grid error
        base = [(p, mp.mpf(v)) for p, v in (lead_fixed or {}).items()]
        free0 = [p for p in powers if p not in dict(base)]
        c_all, _, _ = remez(gv, wv, grid, free0, fixed=base)
        alt_fixed = list(base)
        alt_out = []
        for i, p in enumerate(free0):
            if i < dd_terms:
                hi, lo = to_dd(c_all[i])
                alt_fixed.append((p, mp.mpf(hi) + mp.mpf(lo)))
                alt_out.append((p, hi, lo))
            else:
                hi = to_double(c_all[i])
                alt_fixed.append((p, mp.mpf(hi)))
                alt_out.append((p, hi, None))
        alt_e = grid_err(alt_fixed)
        if alt_e < maxe:
            maxe = alt_e
            out = alt_out
        if lead_fixed:
            for p, v in lead_fixed.items():
                out.append((p, float(v), None))
            out.sort(key=lambda t: t[0])
        return out, maxe
