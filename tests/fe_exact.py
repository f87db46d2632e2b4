"""Independent exact finite-element formulation used to PIN the oracle.

Written from the definitions, with Python Fractions: the equispaced Lagrange
basis of degree p on the reference element, its exact element integrals, dense
assembled 1D matrices on level l (h = 2^-(l+1)), dense Kronecker-product
operators, prolongation as nodal interpolation of the coarse FE function
(Φ_{l-1} = Φ_l P_l) and load-vector integrals.  Shares no code
with the oracle (which hard-codes the element matrices and applies operators
factor by factor).
"""
from __future__ import annotations

from fractions import Fraction as F
from functools import lru_cache

import numpy as np


def poly_mul(a, b):
    out = [F(0)] * (len(a) + len(b) - 1)
    for i, x in enumerate(a):
        for j, y in enumerate(b):
            out[i + j] += x * y
    return out


def poly_der(a):
    return [a[k] * k for k in range(1, len(a))] or [F(0)]


def poly_int01(a):
    return sum(c / (k + 1) for k, c in enumerate(a))


def poly_eval(a, x):
    return sum(c * x ** k for k, c in enumerate(a))


@lru_cache(None)
def lagrange(p):
    """Monomial coefficients of phi_t on nodes j/p, t = 0..p."""
    out = []
    for t in range(p + 1):
        c = [F(1)]
        for j in range(p + 1):
            if j != t:
                c = poly_mul(c, [F(-j, t - j), F(p, t - j)])
        out.append(tuple(c))
    return tuple(out)


@lru_cache(None)
def element_matrices(p):
    L = lagrange(p)
    K = [[poly_int01(poly_mul(poly_der(list(L[a])), poly_der(list(L[b])))) for b in range(p + 1)]
         for a in range(p + 1)]
    M = [[poly_int01(poly_mul(list(L[a]), list(L[b]))) for b in range(p + 1)] for a in range(p + 1)]
    return K, M


def assembled_1d(p, l):
    """Dense 1D stiffness (times h) and mass (over h) on all nodes 0..n of level l."""
    n = p << (l + 1)
    K, M = element_matrices(p)
    Kg = [[F(0)] * (n + 1) for _ in range(n + 1)]
    Mg = [[F(0)] * (n + 1) for _ in range(n + 1)]
    for e in range(n // p):
        for a in range(p + 1):
            for b in range(p + 1):
                Kg[p * e + a][p * e + b] += K[a][b]
                Mg[p * e + a][p * e + b] += M[a][b]
    return Kg, Mg


def dense_ops_1d(p, l):
    """Float dense 1D K_ref, M_ref restricted to unknowns 1..n-1."""
    Kg, Mg = assembled_1d(p, l)
    n = p << (l + 1)
    Kf = np.array([[float(Kg[i][j]) for j in range(1, n)] for i in range(1, n)])
    Mf = np.array([[float(Mg[i][j]) for j in range(1, n)] for i in range(1, n)])
    return Kf, Mf


def dense_A(d, p, l):
    """A_l = h^(d-2) sum_k (K in slot k, M elsewhere) on unknowns, x fastest."""
    K, M = dense_ops_1d(p, l)
    h = 2.0 ** -(l + 1)
    if d == 2:
        return np.kron(K, M) + np.kron(M, K)  # (y, x) ordering: kron(Y, X)
    return h * (np.kron(np.kron(K, M), M) + np.kron(np.kron(M, K), M) + np.kron(np.kron(M, M), K))


def basis_value(p, l, i, x):
    """Value of the level-l nodal basis function of node i at x (exact Fraction)."""
    H = F(1, 2 ** (l + 1))
    e_lo = (i - 1) // p if i % p == 0 else i // p
    for e in {e_lo, i // p}:
        if e < 0 or e >= 2 ** (l + 1):
            continue
        a, b = e * H, (e + 1) * H
        if a <= x <= b:
            t = i - p * e
            if 0 <= t <= p:
                xi = (x - a) / H
                return poly_eval(lagrange(p)[t], xi)
    return F(0)


def dense_P_1d(p, lf):
    """Dense 1D prolongation on unknowns: P[i, c] = phi^coarse_c(x_i) (fine nodes x_i)."""
    nf = p << (lf + 1)
    nc = nf // 2
    hf = F(1, nf)
    P = np.zeros((nf - 1, nc - 1))
    for i in range(1, nf):
        for c in range(1, nc):
            P[i - 1, c - 1] = float(basis_value(p, lf - 1, c, i * hf))
    return P


def load_1d(p, l, g):
    """∫ g(x) phi_i(x) dx for polynomial g (coefficients), exact, i = 0..n."""
    n = p << (l + 1)
    H = F(1, 2 ** (l + 1))
    L = lagrange(p)
    out = [F(0)] * (n + 1)
    for e in range(n // p):
        # g(eH + H xi) as a polynomial in xi (Horner)
        shifted = [F(0)]
        for c in reversed(g):
            shifted = poly_mul(shifted, [F(e) * H, H])
            shifted[0] += c
        for t in range(p + 1):
            out[p * e + t] += H * poly_int01(poly_mul(shifted, list(L[t])))
    return out


def to_grid(d, p, l, vec_unknowns):
    """Scatter an unknown-ordered vector (x fastest) into the stored grid layout."""
    n = p << (l + 1)
    NX = (n + 31) // 32 * 32
    shape = (n, n, NX) if d == 3 else (1, n, NX)
    g = np.zeros(shape)
    m = n - 1
    if d == 2:
        g[0, 1:n, 1:n] = vec_unknowns.reshape(m, m)
    else:
        g[1:n, 1:n, 1:n] = vec_unknowns.reshape(m, m, m)
    return g


def from_grid(d, p, l, g):
    n = p << (l + 1)
    if d == 2:
        return g[0, 1:n, 1:n].reshape(-1).copy()
    return g[1:n, 1:n, 1:n].reshape(-1).copy()
