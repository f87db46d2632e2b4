"""Constant-search tool of the paper, on the oracle.

TEST INFRASTRUCTURE ONLY (see oracle/oracle.h): tests/ and tools/ may call
it; the product path never does.

The paper tunes the precision constants by a greedy search on a coarse
problem: fix b1 = b3 = b4 = 30 and N = 12, raise b2 from 1 until the success
criteria Eq 7.3 / 7.4 hold up to L_max, add one bit;
then tune b1, b4, b3 and lastly N (from 1) the same way, each with one extra
bit / iteration.  In this implementation b3 (matrix precision) and b4 (the
coarsest-section precision) are not free parameters: every temporary and
operator is FP64 (reading R9), so the search runs over b2 = b_r,
b1 = b_u and N, in the paper's order.

Criteria (reading R3 maps the paper's level L to our L - 1):
  Eq 7.3  e_L <= 2 e^disc_L            for every L with h <= 1/16
  Eq 7.4  -log2(e_L / e_{L-1}) >= p - 0.05  (H1, m = 1)
where e is the relative full H1 error (reading R13) and e^disc the error of
the FP64 discretisation solution (reading R14).
"""
from __future__ import annotations

import numpy as np

from . import CFMG, errors, schedule, std_solve


def _criteria(d, p, levels, s, edisc, first=3):
    c = CFMG(d, p, levels, s)
    prev = None
    ok = True
    for L in range(1, levels):
        c.solve_upto(L, s.n_ir)
        e = c.errors(L)[2]
        if L >= first:
            ok &= e <= 2.0 * edisc[L]
            ok &= prev is not None and -np.log2(e / prev) >= p - 0.05
        prev = e
        if not ok:
            return False
    return True


def disc_errors(d, p, levels, s):
    """Relative H1 errors of the FP64 discretisation solutions (reading R14)."""
    return {L: errors(d, p, L, std_solve(d, p, L + 1, s, 12))[2] for L in range(1, levels)}


def search_constants(d: int, p: int, levels: int, start: int = 30, n_start: int = 12, max_bits: int = 30,
                     max_n: int = 12, **sched):
    """The greedy search of PAPER.md:1461-1477 on the oracle.  Returns
    (N, b1 = b_u, b2 = b_r) and the trial log [(name, value, passed)]."""
    base = schedule(d, p, **sched)
    edisc = disc_errors(d, p, levels, base)
    log = []

    def ok(b_u, b_r, n):
        s = schedule(d, p, b_u=b_u, b_r=b_r, n_ir=n, **sched)
        return _criteria(d, p, levels, s, edisc)

    def tune(name, fixed):
        # (the paper starts at 1; our widths include the sign bit, PAPER.md:1486,
        # reading R7, so the smallest representable width is 2)
        for v in range(2, max_bits + 1):
            passed = ok(**{**fixed, name: v})
            log.append((name, v, passed))
            if passed:
                v1 = v + 1  # one extra bit (iteration) of stability, then re-check
                passed1 = ok(**{**fixed, name: v1})
                log.append((name, v1, passed1))
                if passed1:
                    return v1
        raise RuntimeError(f"search for {name} failed")

    b_r = tune("b_r", dict(b_u=start, n=n_start))
    b_u = tune("b_u", dict(b_r=b_r, n=n_start))
    n = None
    for v in range(1, max_n + 1):
        passed = ok(b_u, b_r, v)
        log.append(("n", v, passed))
        if passed:
            n = v + 1
            log.append(("n", n, ok(b_u, b_r, n)))
            break
    if n is None:
        raise RuntimeError("search for N failed")
    return (n, b_u, b_r), log
