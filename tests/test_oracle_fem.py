"""Pins for the oracle discretisation (oracle/orc_fem.c) against the exact,
independently written formulation in tests/fe_exact.py and against closed forms.

Paper passages: nested spaces and Φ_{l-1} = Φ_l P_l; R = P^T
and Galerkin coarsening A_{l-1} = R_l A_l P_l; Poisson problem
eq:pde-poisson; RHS "free of any error besides that stemming
from quantization".
"""
from fractions import Fraction as F

import mpmath
import numpy as np
import pytest

import oracle as O
import fe_exact as X

DP = [(2, 1), (2, 2), (2, 3), (3, 1), (3, 2), (3, 3)]


@pytest.mark.parametrize("p", [1, 2, 3])
def test_element_matrices_exact(p):
    K, M = X.element_matrices(p)
    Kc, Mc = O.coef_A(p)
    # assembled rows of the oracle vs exact assembly of the exact element matrices
    Kg, Mg = X.assembled_1d(p, 2)
    n = p << 3
    for i in range(p, 2 * p):  # one full period of interior node types
        tau = i % p
        for o in range(-p, p + 1):
            assert Kc[tau, o + p] == float(Kg[i][i + o])
            assert Mc[tau, o + p] == float(Mg[i][i + o])
    # survey table values as a second pin
    if p == 1:
        assert K == [[1, -1], [-1, 1]] and M == [[F(1, 3), F(1, 6)], [F(1, 6), F(1, 3)]]
    if p == 3:
        assert K[0][0] == F(148, 40) and M[1][1] == F(648, 1680)


def rand_grid(d, p, l, seed):
    rng = np.random.default_rng(seed)
    n = p << (l + 1)
    m = n - 1
    v = rng.standard_normal(m ** d)
    return X.to_grid(d, p, l, v), v


@pytest.mark.parametrize("d,p", DP)
def test_apply_A_equals_dense_kronecker(d, p):
    l = 2 if d == 2 else 1
    if d == 3 and p == 1:
        l = 2
    g, v = rand_grid(d, p, l, 1)
    A = X.dense_A(d, p, l)
    ref = A @ v
    out = O.apply_A(d, p, l, g)
    got = X.from_grid(d, p, l, out)
    assert np.max(np.abs(got - ref)) <= 1e-13 * np.max(np.abs(ref))
    # non-unknowns (boundary, padding) are exactly zero
    mask = X.to_grid(d, p, l, np.ones_like(v)) == 0
    assert not out[mask].any()


@pytest.mark.parametrize("d,p", DP)
def test_A_symmetric_positive(d, p):
    l = 1
    A = X.dense_A(d, p, l)
    n0 = A.shape[0]
    cols = np.stack([X.from_grid(d, p, l, O.apply_A(d, p, l, X.to_grid(d, p, l, e)))
                     for e in np.eye(n0)], axis=1)
    assert np.allclose(cols, cols.T, rtol=0, atol=1e-14 * np.abs(cols).max())
    assert np.linalg.eigvalsh((cols + cols.T) / 2).min() > 0


@pytest.mark.parametrize("d,p", DP)
def test_prolongation_is_nodal_interpolation(d, p):
    lf = 2 if d == 2 else 1
    P1 = X.dense_P_1d(p, lf)
    P = np.kron(P1, P1) if d == 2 else np.kron(np.kron(P1, P1), P1)
    gc, vc = rand_grid(d, p, lf - 1, 2)
    out = O.prolong(d, p, lf, gc)
    got = X.from_grid(d, p, lf, out)
    ref = P @ vc
    assert np.max(np.abs(got - ref)) <= 1e-14 * np.max(np.abs(ref))
    W = O.coef_P(p)
    assert np.all(W * 2 ** 8 == np.round(W * 2 ** 8))  # dyadic weights (exact doubles)


@pytest.mark.parametrize("d,p", DP)
def test_restriction_is_transpose(d, p):
    lf = 2 if d == 2 else 1
    gf, vf = rand_grid(d, p, lf, 3)
    gc, vc = rand_grid(d, p, lf - 1, 4)
    Rt = X.from_grid(d, p, lf - 1, O.restrict(d, p, lf, gf))
    Pv = X.from_grid(d, p, lf, O.prolong(d, p, lf, gc))
    assert abs(Rt @ vc - vf @ Pv) <= 1e-13 * abs(vf @ Pv) + 1e-13


@pytest.mark.parametrize("d,p", DP)
def test_galerkin_identity(d, p):
    lf = 2 if d == 2 else 1
    gc, vc = rand_grid(d, p, lf - 1, 5)
    lhs = O.restrict(d, p, lf, O.apply_A(d, p, lf, O.prolong(d, p, lf, gc)))
    rhs = O.apply_A(d, p, lf - 1, gc)
    assert np.max(np.abs(lhs - rhs)) <= 1e-13 * np.max(np.abs(rhs))


@pytest.mark.parametrize("d,p", [(2, 2), (2, 3), (3, 2), (3, 3)])
def test_A_exact_on_quadratic(d, p):
    """For u = prod x_k(1-x_k) in Q_p (p >= 2): (A I_h u)_i = ∫ (-Δu) φ_i exactly."""
    l = 1
    n = p << (l + 1)
    xs = [F(i, n) for i in range(n + 1)]
    q = [F(0), F(1), F(-1)]                 # x(1-x)
    two = [F(2)]                            # -(x(1-x))'' = 2
    Lq = X.load_1d(p, l, q)
    L2 = X.load_1d(p, l, two)
    vals = np.array([float(x * (1 - x)) for x in xs])
    NX = (n + 31) // 32 * 32
    if d == 2:
        u = np.zeros((1, n, NX)); u[0, :, :n] = np.outer(vals[:n], vals[:n])
        b = np.zeros_like(u)
        for j in range(1, n):
            for i in range(1, n):
                b[0, j, i] = float(L2[j] * Lq[i] + Lq[j] * L2[i])
    else:
        u = np.zeros((n, n, NX))
        u[:, :, :n] = vals[:n, None, None] * vals[None, :n, None] * vals[None, None, :n]
        b = np.zeros_like(u)
        for k in range(1, n):
            for j in range(1, n):
                for i in range(1, n):
                    b[k, j, i] = float(L2[k] * Lq[j] * Lq[i] + Lq[k] * L2[j] * Lq[i] + Lq[k] * Lq[j] * L2[i])
    out = O.apply_A(d, p, l, u)
    assert np.max(np.abs(out - b)) <= 1e-13 * np.max(np.abs(b))


@pytest.mark.parametrize("p,l", [(1, 0), (1, 3), (2, 2), (3, 1), (3, 6)])
def test_rhs_table_correctly_rounded(p, l):
    """g_l(i) = ∫ sin(pi x) phi_i(x) dx, correctly rounded (mpmath, 60 digits)."""
    g = O.rhs_table(p, l)
    n = p << (l + 1)
    H = mpmath.mpf(1) / 2 ** (l + 1)
    mpmath.mp.dps = 60
    Lg = X.lagrange(p)
    idx = list(range(1, min(n, 12))) + [n // 2, n - 1]
    for i in idx:
        tot = mpmath.mpf(0)
        elems = [i // p] if i % p else [i // p - 1, i // p]
        for e in elems:
            t = i - p * e
            c = [mpmath.mpf(x.numerator) / x.denominator for x in Lg[t]]
            f = lambda xi: mpmath.sin(mpmath.pi * (e * H + H * xi)) * sum(cc * xi ** k for k, cc in enumerate(c))
            tot += H * mpmath.quad(f, [0, 1])
        assert g[i] == float(tot), (i, g[i], float(tot))
    mpmath.mp.dps = 15


def test_rhs_const():
    assert O.lib().orc_rhs_const(2) == float(2 * mpmath.pi ** 2) or \
        abs(O.lib().orc_rhs_const(2) - 2 * np.pi ** 2) < 1e-14


@pytest.mark.parametrize("d,p", DP)
def test_inverse_diagonal(d, p):
    l = 1
    A = X.dense_A(d, p, l)
    iD = X.from_grid(d, p, l, O.inv_diag(d, p, l))
    assert np.allclose(iD * np.diag(A), 1.0, rtol=2e-16 * 4, atol=0)


@pytest.mark.parametrize("d,p", DP)
def test_coarse_inverse(d, p):
    A0 = X.dense_A(d, p, 0)
    assert np.allclose(O.coarse_matrix(d, p), A0, rtol=1e-14, atol=0)
    Ai = O.coarse_inverse(d, p)
    assert np.max(np.abs(Ai @ A0 - np.eye(A0.shape[0]))) < 1e-12


@pytest.mark.parametrize("k,alpha", [(2, 4.0), (3, 8.0), (4, 6.0)])
def test_chebyshev_coefficients_give_chebyshev_polynomial(k, alpha):
    """Error propagation of the k-step recurrence from y=0 on the scalar problem
    lam*y = b equals T_k((theta - lam)/delta) / T_k(theta/delta) (textbook
    Chebyshev acceleration), for lam in [lo, hi]."""
    s = O.schedule(2, 1, cheb_degree=k, alpha=alpha, lambda_hi=1.6)
    inv_theta, al, be = O.cheb_coefs(s)
    hi, lo = 1.6, 1.6 / alpha
    theta, delta = (hi + lo) / 2, (hi - lo) / 2
    for lam in np.linspace(lo, hi, 13):
        b = 1.0
        d_ = inv_theta * b
        y = d_
        for j in range(2, k + 1):
            q = b - lam * y
            d_ = al[j - 1] * d_ + be[j - 1] * q
            y = y + d_
        err = 1 - lam * y  # e = (1/lam - y) lam
        Tk = np.polynomial.chebyshev.Chebyshev.basis(k)
        ref = Tk((theta - lam) / delta) / Tk(theta / delta)
        assert abs(err - ref) < 1e-12
