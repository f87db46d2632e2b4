"""Pins for the 1D B-spline compact FMG oracle (oracle/bspline1d.py; §8(f)
row N4): the paper's other workloads, Poisson (m = 1) and the biharmonic
(m = 2) problem in 1D with B-splines.

* Basis and assembly against closed forms: partition of unity, the p = 1
  stiffness (1/h) [-1 2 -1] and mass (h/6) [1 4 1].
* The two-scale matrix against direct evaluation (coarse B-splines are the P
  combinations of fine ones) and the Galerkin identity R A P = A_c.
* Polynomial reproduction: a solution in the spline space is recovered.
* The paper's own result: every 1D row of tab:experiments-params (Table 3,
  PAPER.md:1481-1515; tests/golden) meets Eq 7.3 / 7.4
  for L >= 4, up to the level FP64 carries the paper's progressive matrix
  precision b3 + (p+m+1) L <= 53 (reading R9; the paper itself uses MPFR).
"""
import json
import math
import os

import numpy as np
import pytest

import oracle.bspline1d as B

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "table3_poisson.json")))


def test_partition_of_unity_and_derivative_sums():
    for p in (1, 3, 5, 7):
        t = B.knots(p, 8)
        for x in np.linspace(0, 1, 37):
            v = B.basis_all(t, p, float(x), min(2, p))
            assert abs(v[0].sum() - 1) < 1e-14 and np.all(v[0] >= -1e-15)
            for k in range(1, v.shape[0]):
                assert abs(v[k].sum()) < 1e-9 * 8 ** k


def test_p1_matrices_closed_form():
    lv = B.assemble(1, 1, 3)
    h = 1.0 / lv.nel
    n = len(lv.free)
    K = (2 * np.eye(n) - np.eye(n, k=1) - np.eye(n, k=-1)) / h
    assert np.max(np.abs(lv.K - K)) < 1e-12 / h
    M = lv.M_all[np.ix_(lv.free, lv.free)]
    Mref = h / 6 * (4 * np.eye(n) + np.eye(n, k=1) + np.eye(n, k=-1))
    assert np.max(np.abs(M - Mref)) < 1e-15


@pytest.mark.parametrize("p,m", [(1, 1), (2, 1), (3, 2), (5, 2)])
def test_two_scale_matrix(p, m):
    f, c = B.assemble(p, m, 4), B.assemble(p, m, 3)
    P = B.two_scale(f, c)
    rng = np.random.default_rng(p)
    for x in rng.random(20):
        bf = B.basis_all(f.t, p, float(x), 0)[0][f.free]
        bc = B.basis_all(c.t, p, float(x), 0)[0][c.free]
        assert np.max(np.abs(bf @ P - bc)) < 1e-13
    assert np.max(np.abs(P.T @ f.K @ P - c.K)) < 1e-12 * np.max(np.abs(c.K))


def test_polynomial_reproduction():
    # Poisson, u = x(1 - x) in the space for p >= 2; biharmonic u = x^2 (1 - x)^2 for p >= 4
    for p, m, u, f in [(2, 1, lambda x, k=0: [x - x * x, 1 - 2 * x, -2.0][k], lambda x: 2.0),
                       (4, 2, lambda x, k=0: [x * x * (1 - x) ** 2, 2 * x - 6 * x * x + 4 * x ** 3,
                                              2 - 12 * x + 12 * x * x][k], lambda x: 24.0)]:
        lv = B.assemble(p, m, 3)
        ud = np.linalg.solve(lv.K, B.load(lv, f))
        assert B.hm_error(lv, ud, u, m) < 1e-10


def _table_row_errors(p, m, row, Ltop):
    uf, ff = (B.poisson_u, B.poisson_f) if m == 1 else (B.biharm_u, B.biharm_f)
    s = B.CFMG1D(p, m, Ltop + 1, row["N"], row["b1"], row["b2"], ff)
    sols = s.solve()
    ec, ed = {}, {}
    for L in range(3, Ltop + 1):
        lv = s.lv[L]
        ec[L] = B.hm_error(lv, sols[L], uf, m)
        ed[L] = B.hm_error(lv, np.linalg.solve(lv.K, s.f[L]), uf, m)
    return ec, ed


@pytest.mark.parametrize("m,p", [(1, 1), (1, 2), (1, 3), (1, 4), (1, 5), (2, 3), (2, 4), (2, 5), (2, 6), (2, 7)])
def test_table3_1d_rows_meet_eq73_eq74(m, p):
    row = GOLD["poisson_1d" if m == 1 else "biharmonic_1d"][str(p)]
    Lfp = (53 - row["b3"]) // (p + m + 1)  # FP64 carries b3 + (p+m+1) L bits
    Ltop = min(7, Lfp)
    if (p, m) == (7, 2):
        Ltop = 4  # L = 5: the discretisation error (h^6 ~ 2^-36) meets FP64's floor
    ec, ed = _table_row_errors(p, m, row, Ltop)
    for L in range(4, Ltop + 1):
        assert ec[L] <= 2 * ed[L], (L, ec[L] / ed[L])                     # Eq 7.3
        assert -math.log2(ec[L] / ec[L - 1]) >= (p - m + 1) - 0.05, L     # Eq 7.4


def test_wide_widths_reach_the_discrete_solution():
    """b1 = b2 = 54 with no increments and many IR iterations: the compact FMG
    converges to the exact discrete solution (the compact form loses nothing)."""
    s = B.CFMG1D(2, 1, 6, 12, 54, 54, B.poisson_f)
    s.wu = lambda l, L: 54
    s.wr = lambda l, L: 54
    sols = s.solve()
    lv = s.lv[5]
    ud = np.linalg.solve(lv.K, s.f[5])
    assert np.max(np.abs(sols[5] - ud)) < 1e-11 * np.max(np.abs(ud))
