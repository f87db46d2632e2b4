"""Pins for the oracle compact FMG (oracle/orc_cfmg.c): what the paper and the
mathematics fix, independently of the oracle's own code.

* Eq 7.3 / 7.4 success criteria: error within twice the
  discretisation error and H1 order >= p - 0.05 on every level with h <= 1/16
  (the paper's L >= 4; reading R3 maps paper L to our L+1).
* Discretisation orders L2 p+1, H1 p (BASELINE.json north star).
* Width-54 degeneration: compact V(0,1) from y = 0 equals a standard
  correction-scheme V(0,1) with zero initial guess, written here in numpy
  (block-system remark PAPER.md:686-690).
* fmgResidual with u = 0 gives r_l = enc(R..R f_L) (restricts t, not r;
  PAPER.md:742-744); the exact discrete solution leaves a round-off residual.
* Storage: bits/DoF inside the paper's ranges and below the
  Eq 6.1 bound with constants 4/3, 8/7.
"""
import json
import os

import numpy as np
import pytest

import oracle as O
import fe_exact as X

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "table3_poisson.json")))


def fmg_errors_per_level(d, p, levels, s):
    c = O.CFMG(d, p, levels, s)
    errs = {}
    for L in range(1, levels):
        c.solve_upto(L, s.n_ir)
        errs[L] = c.errors(L)[2]
    return errs


def disc_errors(d, p, levels, s):
    return {L: O.errors(d, p, L, O.std_solve(d, p, L + 1, s, 12))[2] for L in range(1, levels)}


CASES = [(2, 1, 8), (2, 2, 6), (2, 3, 5), (3, 1, 6), (3, 2, 5), (3, 3, 4)]


@pytest.mark.parametrize("d,p,levels", CASES)
def test_success_criteria_eq73_eq74(d, p, levels):
    s = O.schedule(d, p)
    e = fmg_errors_per_level(d, p, levels, s)
    ed = disc_errors(d, p, levels, s)
    for L in range(3, levels):
        assert e[L] <= 2.0 * ed[L], (L, e[L], ed[L])                      # Eq 7.3
        order = -np.log2(e[L] / e[L - 1])
        assert order >= p - 0.05, (L, order)                              # Eq 7.4


def test_paper_table3_p1_schedule_2d():
    """2D p=1 with the paper's own Table 3 constants (N=3, b1=4, b2=4): Q1 equals
    the degree-1 B-spline space, so the row transfers (smoother: Chebyshev,
    DESIGN.md R4)."""
    row = GOLD["poisson_2d"]["1"]
    s = O.schedule(2, 1, b_u=row["b1"], b_r=row["b2"], n_ir=row["N"])
    e = fmg_errors_per_level(2, 1, 9, s)
    ed = disc_errors(2, 1, 9, s)
    for L in range(3, 9):
        assert e[L] <= 2.0 * ed[L]
        assert -np.log2(e[L] / e[L - 1]) >= 1 - 0.05


@pytest.mark.parametrize("d,p,levels", [(2, 1, 8), (2, 2, 6), (2, 3, 5), (3, 1, 5), (3, 2, 4)])
def test_discretisation_orders(d, p, levels):
    s = O.schedule(d, p)
    u1 = O.std_solve(d, p, levels - 1, s, 12)
    u2 = O.std_solve(d, p, levels, s, 12)
    e1 = O.errors(d, p, levels - 2, u1)
    e2 = O.errors(d, p, levels - 1, u2)
    assert -np.log2(e2[0] / e1[0]) > p + 1 - 0.15   # L2
    assert -np.log2(e2[1] / e1[1]) > p - 0.1        # H1 semi


@pytest.mark.parametrize("d,p", [(2, 1), (2, 2), (2, 3), (3, 1), (3, 2), (3, 3)])
def test_std_solver_converges(d, p):
    levels = 5 if d == 2 else 3
    s = O.schedule(d, p)
    L = levels - 1
    u = O.std_solve(d, p, levels, s, 30)
    r = O.rhs(d, p, L) - O.apply_A(d, p, L, u)
    assert np.linalg.norm(r) <= 1e-12 * np.linalg.norm(O.rhs(d, p, L))


def numpy_vcycle01(d, p, L, t, s):
    """Standard correction-scheme V(0,1), zero initial guess: returns x_L."""
    inv_theta, al, be = O.cheb_coefs(s)
    rs = {L: t}
    for l in range(L - 1, -1, -1):
        rs[l] = O.restrict(d, p, l + 1, rs[l + 1])
    Ai = O.coarse_inverse(d, p)
    g0 = O.Geom(d, p, 0)
    x0 = X.to_grid(d, p, 0, Ai @ X.from_grid(d, p, 0, rs[0]))
    x = x0
    for l in range(1, L + 1):
        x = O.prolong(d, p, l, x)
        iD = O.inv_diag(d, p, l)
        b = rs[l] - O.apply_A(d, p, l, x)
        dv = inv_theta * (iD * b)
        y = dv.copy()
        for j in range(2, s.cheb_degree + 1):
            q = b - O.apply_A(d, p, l, y)
            dv = al[j - 1] * dv + be[j - 1] * (iD * q)
            y = y + dv
        x = x + y
    return x


@pytest.mark.parametrize("d,p,levels", [(2, 1, 6), (2, 2, 5), (2, 3, 4), (3, 1, 4), (3, 3, 3)])
def test_width54_cfas_equals_standard_vcycle(d, p, levels):
    s = O.schedule(d, p, b_u=54, b_r=54, k_u=0, k_r=0)
    c = O.CFMG(d, p, levels, s)
    L = levels - 1
    c.solve_upto(L - 1, s.n_ir)
    # push level L without iterating, then one residual + cFas
    c.solve_upto(L, 0)
    c.residual(L)
    t = c.array(1, L)
    c.cfas_correct(L)
    # decode the compact correction to standard representation
    yh = None
    for l in range(0, L + 1):
        mant, exps, w = c.section(2, l)
        g = O.Geom(d, p, l)
        _, v = O.bfp_decode(mant, exps, g.size, w)
        v = v.reshape(g.shape)
        yh = v if yh is None else O.prolong(d, p, l, yh) + v
    ref = numpy_vcycle01(d, p, L, t, s)
    assert np.max(np.abs(yh - ref)) <= 1e-11 * np.max(np.abs(ref))


@pytest.mark.parametrize("d,p,levels", [(2, 2, 5), (3, 1, 4)])
def test_zero_solution_residual_restricts_t(d, p, levels):
    s = O.schedule(d, p)
    c = O.CFMG(d, p, levels, s)
    L = levels - 1
    norms = c.residual(L)      # all sections are zero after create
    t = O.rhs(d, p, L)
    for l in range(L, -1, -1):
        if l < L:
            t = O.restrict(d, p, l + 1, t)
        mant, exps, w = c.section(1, l)
        assert w == s.b_r + (L - l)
        rc, m2, e2 = O.bfp_encode(t.reshape(-1), w)
        assert np.array_equal(mant, m2) and np.array_equal(exps, e2)
        assert abs(norms[l] - np.linalg.norm(t)) <= 1e-14 * np.linalg.norm(t)


@pytest.mark.parametrize("d,p,levels", [(2, 1, 6), (2, 3, 4), (3, 2, 3)])
def test_exact_discrete_solution_has_roundoff_residual(d, p, levels):
    s = O.schedule(d, p)
    L = levels - 1
    u = O.std_solve(d, p, levels, s, 40)
    c = O.CFMG(d, p, levels, s)
    c.set_section(0, L, u, 54)
    norms = c.residual(L)
    assert norms[L] <= 1e-11 * np.linalg.norm(O.rhs(d, p, L))


def test_determinism():
    s = O.schedule(2, 2)
    a = O.CFMG(2, 2, 5, s); a.solve()
    b = O.CFMG(2, 2, 5, s); b.solve()
    assert np.array_equal(a.norms(), b.norms())
    for l in range(5):
        assert np.array_equal(a.section(0, l)[0], b.section(0, l)[0])


@pytest.mark.parametrize("d,p", [(2, 1), (2, 2), (2, 3), (3, 1), (3, 2), (3, 3)])
def test_bits_per_dof_in_paper_ranges(d, p):
    s = O.schedule(d, p)
    lo, hi = GOLD["bits_per_dof_claim"]["solution_bits_range"]
    rlo, rhi = GOLD["bits_per_dof_claim"]["residual_bits_range"]
    assert lo <= s.b_u <= hi and rlo <= s.b_r <= rhi
    # Eq 6.1: sum_l n_l (k(L-l) + b) < (2^d/(2^d-1) b + 2^d/(2^d-1)^2 k) n_L
    c = GOLD["storage_constants"][str(d)]
    for L in (4, 8):
        n = [(p * 2 ** (l + 1) - 1) ** d for l in range(L + 1)]
        tot = sum(n[l] * (s.b_u + s.k_u * (L - l)) for l in range(L + 1))
        bound = (c * s.b_u + c / (2 ** d - 1) * s.k_u) * n[L]
        assert tot < bound


def test_norm_log_shape_and_monotone_decrease_on_finest():
    s = O.schedule(2, 1)
    c = O.CFMG(2, 1, 7, s)
    c.solve()
    nr = c.norms()
    assert nr.shape == (7, 3, 7)
    for L in range(1, 7):
        assert np.all(nr[L, :, L + 1:] == 0)
        assert nr[L, -1, L] < nr[L, 0, L]   # IR reduces the finest residual
