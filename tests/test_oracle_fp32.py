"""FP32 cFas in the oracle (reading R28; tab:precisions PAPER.md:820-841: the
cFas working precision is at most L + b_r <= 15 bits at the configurations,
well inside float's 24).  Pins: the float operator and prolongation trees
against the FP64 ones (same tree, so within a few float ulps of the rows'
absolute sums); the FP32-cFas solve meets the success criteria Eq 7.3 / 7.4
 and its errors stay within 1 % of the FP64-cFas solve;
the float path is really taken (w_l are floats)."""
import numpy as np
import pytest

import oracle as O

CASES = [(2, 1, 8), (2, 2, 6), (2, 3, 5), (3, 1, 6), (3, 2, 5), (3, 3, 4)]


def _smooth(d, p, l, seed):
    g = O.Geom(d, p, l)
    rng = np.random.default_rng(seed)
    u = np.zeros(g.shape)
    n = g.n
    x = np.arange(n) / n
    k = rng.integers(1, 4, 3)
    f = [np.sin(np.pi * k[i] * x) for i in range(3)]
    if d == 2:
        u[0, :, :n] = np.outer(f[1], f[0])
    else:
        u[:, :, :n] = f[2][:, None, None] * f[1][None, :, None] * f[0][None, None, :]
    return u


@pytest.mark.parametrize("d,p,l", [(2, 2, 4), (3, 1, 3), (3, 3, 2)])
def test_float_operator_and_prolongation_trees(d, p, l):
    u = _smooth(d, p, l, 1).astype(np.float32)
    a64 = O.apply_A(d, p, l, u.astype(np.float64))
    a32 = O.apply_A_f32(d, p, l, u).astype(np.float64)
    # every entry of the float tree is within ~2R float ulps of the row's absolute sum
    absA = O.apply_A(d, p, l, np.abs(u).astype(np.float64))  # (not a bound on |A| |u|, but the same scale)
    tol = 64 * np.finfo(np.float32).eps * (np.abs(a64).max() + np.abs(absA).max())
    assert np.abs(a32 - a64).max() <= tol
    c = _smooth(d, p, l - 1 if l > 0 else 0, 2).astype(np.float32)
    if l >= 1:
        p64 = O.prolong(d, p, l, c.astype(np.float64))
        p32 = O.prolong_f32(d, p, l, c).astype(np.float64)
        assert np.abs(p32 - p64).max() <= 8 * np.finfo(np.float32).eps * np.abs(p64).max()


def _errs(d, p, levels, s):
    c = O.CFMG(d, p, levels, s)
    out = {}
    for L in range(1, levels):
        c.solve_upto(L, s.n_ir)
        out[L] = c.errors(L)[2]
    return out, c


@pytest.mark.parametrize("d,p,levels", CASES)
def test_fp32_cfas_meets_success_criteria(d, p, levels):
    s32 = O.schedule(d, p, cfas_fp32=1)
    s64 = O.schedule(d, p)
    e32, c32 = _errs(d, p, levels, s32)
    e64, c64 = _errs(d, p, levels, s64)
    ed = {L: O.errors(d, p, L, O.std_solve(d, p, L + 1, s64, 12))[2] for L in range(1, levels)}
    for L in range(3, levels):
        assert e32[L] <= 2.0 * ed[L], (L, e32[L], ed[L])             # Eq 7.3
        assert -np.log2(e32[L] / e32[L - 1]) >= p - 0.05, L           # Eq 7.4
        assert abs(e32[L] - e64[L]) <= 0.01 * e64[L], (L, e32[L], e64[L])
    # the float path is taken: w_l (l >= 1) are floats (the sections may well
    # coincide with FP64's: the float rounding sits far below the quantisation
    # of ý, and for Q1 the dyadic prolongation keeps FP64's w float-exact too)
    for l in range(1, levels):
        w32 = c32.array(2, l)
        assert np.array_equal(w32, w32.astype(np.float32).astype(np.float64)), l


def test_fp32_cfas_changes_w_somewhere():
    s32, s64 = O.schedule(2, 2, cfas_fp32=1), O.schedule(2, 2)
    _, c32 = _errs(2, 2, 6, s32)
    _, c64 = _errs(2, 2, 6, s64)
    assert not np.array_equal(c32.array(2, 5), c64.array(2, 5))


def test_fp32_cfas_rejects_other_smoothers():
    with pytest.raises(ValueError):
        O.CFMG(2, 1, 4, O.schedule(2, 1, cfas_fp32=1, smoother="mcgs"))
