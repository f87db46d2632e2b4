"""Pins for nu > 1 compact V-cycles per IR iteration (§8(f) row N2; Alg 3.1
PAPER.md:633-661 with its fine-to-coarse s sweep and nonzero-initial-guess
terms; reading R23).  Oracle only this round (the GPU path runs nu = 1).

* nu = 1 is the existing method, bit for bit.
* At width 54 (rounding far below the tolerance) the compact cFas with nu = 2
  equals two standard correction-scheme V(0,1) cycles written in numpy,
  x1 = V(t), x2 = x1 + V(t - A x1): the block-system residual of the first
  correction is the restriction of t - A x1 (Galerkin R A P = A),
  so a dropped s term, a sign or a wrong z / ý coupling breaks it.
* A second cycle reduces the algebraic residual of the correction equation.
"""
import numpy as np
import pytest

import oracle as O
from test_oracle_cfmg import numpy_vcycle01


def _correction_std(c, d, p, L):
    """Decode the compact correction ý_0..L into the standard representation."""
    yh = None
    for l in range(0, L + 1):
        mant, exps, w = c.section(2, l)
        g = O.Geom(d, p, l)
        _, v = O.bfp_decode(mant, exps, g.size, w)
        v = v.reshape(g.shape)
        yh = v if yh is None else O.prolong(d, p, l, yh) + v
    return yh


def _one_iteration(d, p, levels, nu, **kw):
    s = O.schedule(d, p, nu=nu, **kw)
    c = O.CFMG(d, p, levels, s)
    L = levels - 1
    c.solve_upto(L - 1, s.n_ir)
    c.solve_upto(L, 0)
    c.residual(L)
    t = c.array(1, L)
    c.cfas_correct(L)
    return c, s, t, L


@pytest.mark.parametrize("d,p,levels", [(2, 1, 6), (2, 2, 5), (2, 3, 4), (3, 1, 4), (3, 2, 3)])
def test_nu2_width54_equals_two_standard_vcycles(d, p, levels):
    c, s, t, L = _one_iteration(d, p, levels, 2, b_u=54, b_r=54, k_u=0, k_r=0)
    yh = _correction_std(c, d, p, L)
    x1 = numpy_vcycle01(d, p, L, t, s)
    x2 = x1 + numpy_vcycle01(d, p, L, t - O.apply_A(d, p, L, x1), s)
    assert np.max(np.abs(yh - x2)) <= 1e-10 * np.max(np.abs(x2))
    # and it is not the one-cycle result
    assert np.max(np.abs(yh - x1)) > 1e-6 * np.max(np.abs(x2))


@pytest.mark.parametrize("d,p,levels", [(2, 2, 5), (3, 1, 4)])
def test_nu1_is_the_single_cycle_method(d, p, levels):
    a = O.CFMG(d, p, levels, O.schedule(d, p))
    b = O.CFMG(d, p, levels, O.schedule(d, p, nu=1))
    a.solve()
    b.solve()
    assert np.array_equal(a.norms(), b.norms())
    for l in range(levels):
        for which in (0, 1):
            assert np.array_equal(a.section(which, l)[0], b.section(which, l)[0])


@pytest.mark.parametrize("smoother", ["chebyshev", "mcgs"])
@pytest.mark.parametrize("d,p,levels", [(2, 1, 6), (2, 2, 5), (3, 1, 4)])
def test_more_cycles_reduce_the_correction_residual(smoother, d, p, levels):
    res = []
    for nu in (1, 2, 3):
        c, s, t, L = _one_iteration(d, p, levels, nu, b_u=54, b_r=54, k_u=0, k_r=0, smoother=smoother)
        yh = _correction_std(c, d, p, L)
        res.append(np.linalg.norm(t - O.apply_A(d, p, L, yh)))
    assert res[1] < 0.5 * res[0] and res[2] < 0.5 * res[1], res


@pytest.mark.parametrize("d,p", [(2, 1), (2, 2)])
def test_nu2_fmg_meets_the_accuracy_criterion(d, p):
    """Default precisions: the nu = 2 solve is at least as accurate as nu = 1
    (H1 error of the final level within 1 %)."""
    lv = 7 if p == 1 else 6
    e = []
    for nu in (1, 2):
        c = O.CFMG(d, p, lv, O.schedule(d, p, nu=nu))
        c.solve()
        e.append(c.errors()[2])
    assert e[1] <= 1.01 * e[0], e
