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


# ---------------------------------------------- operator layouts (R27) --

@pytest.mark.parametrize("p,m", [(1, 1), (2, 1), (3, 1), (3, 2), (5, 2), (7, 2)])
def test_layouts_reproduce_the_dense_operators(p, m):
    """band / ELL storage and their canonical products against dense numpy
    products; the entries of P dropped outside the support structure are
    rounding noise of the L2 solve."""
    f, c = B.assemble(p, m, 4), B.assemble(p, m, 3)
    P = B.two_scale(f, c)
    st = B.two_scale_structure(f, c)
    mask = np.zeros_like(P, dtype=bool)
    for i, (j0, j1) in enumerate(st):
        mask[i, j0:j1 + 1] = True
    assert np.max(np.abs(P[~mask])) < 1e-12  # genuine coefficients are >= 2^-p
    # interior rows: a fine support, (p+1)/2 coarse elements long and starting
    # at a coarse knot or a midpoint, lies in the supports starting at the
    # coarse knots j in [a - (p+1)/2, a]: (p+1)/2 or (p+3)/2 of them for odd p,
    # p/2 + 1 for even p; near the ends the open knots widen it, never past p + 1
    wid = [j1 - j0 + 1 for j0, j1 in st]
    n = len(wid)
    inner = {(p + 1) // 2, (p + 3) // 2} if p % 2 else {p // 2 + 1}
    assert set(wid[n // 4: 3 * n // 4]) == inner and max(wid) <= p + 1
    rng = np.random.default_rng(p + 10 * m)
    xc = rng.standard_normal(P.shape[1])
    xf = rng.standard_normal(P.shape[0])
    Pv, c0 = B.ell(P, st)
    Rv, r0 = B.ell_transpose(P, st, P.shape[1])
    Pm = np.where(mask, P, 0.0)
    assert np.allclose(B.ell_mv(Pv, c0, xc), Pm @ xc, rtol=0, atol=1e-14)
    assert np.allclose(B.ell_mv(Rv, r0, xf), Pm.T @ xf, rtol=0, atol=1e-14)
    Ab = B.band(f.K, p)
    x = rng.standard_normal(f.K.shape[0])
    assert np.allclose(B.band_mv(Ab, x, p), f.K @ x, rtol=1e-13, atol=1e-13 * np.abs(f.K).max())
    A = rng.standard_normal((5, 7))
    assert np.allclose(B.dense_mv(A, x[:7]), A @ x[:7], rtol=1e-14, atol=1e-14)


def test_p1_two_scale_closed_form():
    # linear B-splines: coarse hat j = fine hats (1/2, 1, 1/2) around node 2j+1
    f, c = B.assemble(1, 1, 3), B.assemble(1, 1, 2)
    st = B.two_scale_structure(f, c)
    Pv, c0 = B.ell(B.two_scale(f, c), st)
    P = np.zeros((len(f.free), len(c.free)))
    for j in range(len(c.free)):
        P[2 * j, j], P[2 * j + 1, j], P[2 * j + 2, j] = 0.5, 1.0, 0.5
    for i in range(len(f.free)):
        for k in range(Pv.shape[1]):
            if c0[i] + k < len(c.free):
                assert abs(Pv[i, k] - P[i, c0[i] + k]) < 1e-15


@pytest.mark.parametrize("p", [1, 2, 4])
def test_gauss_seidel_sweeps_are_triangular_solves(p):
    """From y = 0 a lexicographic GS sweep solves (D + L) y = b; the multicolour
    sweep does the same on the colour-permuted system."""
    from scipy.linalg import solve_triangular
    lv = B.assemble(p, 1 if p < 3 else 2, 4)
    K = lv.K
    n = K.shape[0]
    b = np.random.default_rng(p).standard_normal(n)
    Ab = B.band(K, p)
    y = B.lex_gs(Ab, b, p)
    assert np.allclose(y, solve_triangular(np.tril(K), b, lower=True), rtol=1e-12, atol=1e-12)
    perm = np.concatenate([np.arange(c, n, p + 1) for c in range(p + 1)])
    Kp = K[np.ix_(perm, perm)]
    yp = solve_triangular(np.tril(Kp), b[perm], lower=True)
    ym = B.mc_gs(Ab, b, p)
    assert np.allclose(ym[perm], yp, rtol=1e-12, atol=1e-12)
    assert not np.allclose(ym, y)  # the two orders differ


@pytest.mark.parametrize("m,p", [(1, 1), (1, 3), (2, 3), (2, 5)])
def test_multicolour_gs_meets_eq73(m, p):
    """The GPU-parallel multicolour sweep keeps the Table-3 rows' accuracy
    (Eq 7.3) with one more IR iteration than the paper's lexicographic sweep."""
    row = dict(GOLD["poisson_1d" if m == 1 else "biharmonic_1d"][str(p)])
    row["N"] += 1
    uf, ff = (B.poisson_u, B.poisson_f) if m == 1 else (B.biharm_u, B.biharm_f)
    Ltop = min(6, (53 - row["b3"]) // (p + m + 1))
    s = B.CFMG1D(p, m, Ltop + 1, row["N"], row["b1"], row["b2"], ff, smoother="mcgs")
    sols = s.solve()
    for L in range(4, Ltop + 1):
        lv = s.lv[L]
        ec = B.hm_error(lv, sols[L], uf, m)
        ed = B.hm_error(lv, np.linalg.solve(lv.K, s.f[L]), uf, m)
        assert ec <= 2 * ed, (L, ec / ed)
