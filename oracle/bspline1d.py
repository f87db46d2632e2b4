"""1D B-spline compact FMG oracle (§8(f) row N4; TEST INFRASTRUCTURE ONLY --
only tests/ may import it; the product package never does).

The paper's other workloads: homogeneous Dirichlet
Poisson -u'' = f (m = 1) and the biharmonic u'''' = f with u = u' = 0 (m = 2)
on (0, 1), discretised with B-splines of degree p on uniform open knot
vectors, solved by the compact FMG of Alg 3.3 / 3.2 / 3.1
with the paper's smoother, one lexicographic Gauss-Seidel sweep
(PAPER.md:689-690, 1624), an exact coarsest solve, and the solution,
residual and correction stored as BFP sections of regressive widths
w_u = b1 + (p+1)(L-l), w_r = b2 + m(L-l) (tab:experiments-params,
PAPER.md:1481-1515).  The BFP format is the oracle's 32-entry block codec
(orc_bfp.c, reading R8); temporaries, matrices and f are FP64 (reading R9:
FP64 covers b3/b4 only while b3 + (p+m+1) l <= 53 -- the pins stay inside
that range).

Readings (R24-R26): level l has 2^(l+1) elements (R3); the
prolongation is the exact two-scale (knot-insertion) matrix, computed as the
L2 projection M_f^{-1} M_fc, exact in exact arithmetic because the coarse
space is nested in the fine one; R = P^T; A_l is assembled on each level.

Plain sequential code; Gauss-Legendre quadrature with p + 3 points per
element (exact for the polynomial integrands of K and M).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import bfp_decode, bfp_encode

# ----------------------------------------------------------------- basis --


def knots(p: int, nel: int) -> np.ndarray:
    """Open uniform knot vector on [0, 1]: p+1 repeated end knots."""
    inner = np.arange(1, nel) / nel
    return np.concatenate([np.zeros(p + 1), inner, np.ones(p + 1)])


def basis_all(t: np.ndarray, p: int, x: float, nder: int) -> np.ndarray:
    """Values and derivatives (rows 0..nder) of all n = len(t)-p-1 B-splines
    at x, by the Cox-de Boor recursion and its derivative formula."""
    n = len(t) - p - 1
    # span index s with t[s] <= x < t[s+1] (x = 1 belongs to the last span)
    s = np.searchsorted(t, x, side="right") - 1
    s = min(max(s, p), n - 1)
    # degree-0 .. degree-p values on the span (standard triangular table)
    N = np.zeros((p + 1, p + 1))
    N[0, 0] = 1.0
    left = np.zeros(p + 1)
    right = np.zeros(p + 1)
    for j in range(1, p + 1):
        left[j] = x - t[s + 1 - j]
        right[j] = t[s + j] - x
        saved = 0.0
        for r in range(j):
            N[j, r] = right[r + 1] + left[j - r]        # knot differences (lower triangle)
            tmp = N[r, j - 1] / N[j, r]
            N[r, j] = saved + right[r + 1] * tmp
            saved = left[j - r] * tmp
        N[j, j] = saved
    out = np.zeros((nder + 1, n))
    for r in range(p + 1):
        out[0, s - p + r] = N[r, p]
    # derivatives (The NURBS Book A2.3)
    a = np.zeros((2, p + 1))
    for r in range(p + 1):
        s1, s2 = 0, 1
        a[0, 0] = 1.0
        for k in range(1, nder + 1):
            d = 0.0
            rk, pk = r - k, p - k
            if r >= k:
                a[s2, 0] = a[s1, 0] / N[pk + 1, rk]
                d = a[s2, 0] * N[rk, pk]
            j1 = 1 if rk >= -1 else -rk
            j2 = k - 1 if r - 1 <= pk else p - r
            for j in range(j1, j2 + 1):
                a[s2, j] = (a[s1, j] - a[s1, j - 1]) / N[pk + 1, rk + j]
                d += a[s2, j] * N[rk + j, pk]
            if r <= pk:
                a[s2, k] = -a[s1, k - 1] / N[pk + 1, r]
                d += a[s2, k] * N[r, pk]
            if k <= p:
                out[k, s - p + r] = d
            s1, s2 = s2, s1
    f = p
    for k in range(1, nder + 1):
        out[k] *= f
        f *= p - k
    return out


# ------------------------------------------------------------ discretise --


@dataclass
class Level:
    p: int
    m: int
    l: int
    nel: int
    t: np.ndarray
    n_all: int      # all B-splines
    free: np.ndarray  # indices of the unknowns (end functions removed)
    K: np.ndarray   # stiffness on the unknowns (dense; 1D sizes are small)
    M_all: np.ndarray  # mass over all functions (for the two-scale matrix)


def gauss(npts: int):
    xg, wg = np.polynomial.legendre.leggauss(npts)
    return xg, wg


def assemble(p: int, m: int, l: int) -> Level:
    """K_ij = int B_i^(m) B_j^(m) over the unknowns;
    homogeneous Dirichlet data removes m functions at each end."""
    nel = 2 ** (l + 1)
    t = knots(p, nel)
    n_all = len(t) - p - 1
    free = np.arange(m, n_all - m)
    K = np.zeros((n_all, n_all))
    M = np.zeros((n_all, n_all))
    xg, wg = gauss(p + 3)
    h = 1.0 / nel
    for e in range(nel):
        a = e * h
        for q in range(len(xg)):
            x = a + 0.5 * h * (xg[q] + 1.0)
            w = 0.5 * h * wg[q]
            B = basis_all(t, p, x, m)
            K += w * np.outer(B[m], B[m])
            M += w * np.outer(B[0], B[0])
    return Level(p, m, l, nel, t, n_all, free, K[np.ix_(free, free)], M)


def load(lv: Level, f) -> np.ndarray:
    """f_i = int f B_i over the unknowns."""
    xg, wg = gauss(lv.p + 6)
    h = 1.0 / lv.nel
    b = np.zeros(lv.n_all)
    for e in range(lv.nel):
        a = e * h
        for q in range(len(xg)):
            x = a + 0.5 * h * (xg[q] + 1.0)
            b += 0.5 * h * wg[q] * f(x) * basis_all(lv.t, lv.p, x, 0)[0]
    return b[lv.free]


def two_scale(fine: Level, coarse: Level) -> np.ndarray:
    """P with coarse B-spline j = sum_i P_ij fine B-spline i (all functions),
    restricted to the unknowns: the L2 projection M_f^{-1} M_fc, exact for
    the nested spaces."""
    xg, wg = gauss(fine.p + 3)
    h = 1.0 / fine.nel
    Mfc = np.zeros((fine.n_all, coarse.n_all))
    for e in range(fine.nel):
        a = e * h
        for q in range(len(xg)):
            x = a + 0.5 * h * (xg[q] + 1.0)
            w = 0.5 * h * wg[q]
            Mfc += w * np.outer(basis_all(fine.t, fine.p, x, 0)[0], basis_all(coarse.t, coarse.p, x, 0)[0])
    Pall = np.linalg.solve(fine.M_all, Mfc)
    return Pall[np.ix_(fine.free, coarse.free)]


# --------------------------------------------------------------- BFP I/O --


def _pad(n: int) -> int:
    return (n + 31) // 32 * 32


def enc(x: np.ndarray, w: int):
    """32-entry block BFP (orc_bfp.c) of x padded with zeros."""
    xp = np.zeros(_pad(len(x)))
    xp[: len(x)] = x
    rc, mant, exps = bfp_encode(xp, w)
    assert rc == 0
    return (mant, exps, w, len(x))


def dec(sec) -> np.ndarray:
    mant, exps, w, n = sec
    rc, x = bfp_decode(mant, exps, _pad(n), w)
    assert rc == 0
    return x[:n]


# ------------------------------------------------------------ compact FMG --


def lex_gs(A: np.ndarray, b: np.ndarray, bw: int) -> np.ndarray:
    """One forward Gauss-Seidel sweep from y = 0;
    A is banded with half-bandwidth bw (B-splines of degree p: bw = p)."""
    n = len(b)
    y = np.zeros(n)
    for i in range(n):
        s = b[i]
        for j in range(max(0, i - bw), min(n, i + bw + 1)):
            if j != i:
                s -= A[i, j] * y[j]
        y[i] = s / A[i, i]
    return y


class CFMG1D:
    """Alg 3.3 in 1D with B-splines, m in {1, 2}."""

    def __init__(self, p, m, levels, N, b1, b2, f):
        self.p, self.m, self.levels, self.N, self.b1, self.b2 = p, m, levels, N, b1, b2
        self.lv = [assemble(p, m, l) for l in range(levels)]
        self.P = [None] + [two_scale(self.lv[l], self.lv[l - 1]) for l in range(1, levels)]
        self.f = [load(lv, f) for lv in self.lv]

    def wu(self, l, L):
        return self.b1 + (self.p + 1) * (L - l)

    def wr(self, l, L):
        return self.b2 + self.m * (L - l)

    def std(self, secs, L):
        """Standard representation of a compact vector: u_l = dec ú_l + P_l u_{l-1}."""
        u = dec(secs[0])
        for l in range(1, L + 1):
            u = dec(secs[l]) + self.P[l] @ u
        return u

    def solve(self, Lstop=None):
        L0 = self.levels - 1 if Lstop is None else Lstop
        # coarse-grid solve PAPER.md:785-786
        u0 = np.linalg.solve(self.lv[0].K, self.f[0])
        self.u = [enc(u0, self.wu(0, 0))]
        self.sols = {0: dec(self.u[0])}
        for L in range(1, L0 + 1):
            self.u.append(enc(np.zeros(len(self.f[L])), self.wu(L, L)))  # push level: ú_L = 0
            for _ in range(self.N):
                self.iteration(L)
            self.sols[L] = self.std(self.u, L)
        return self.sols

    def iteration(self, L):
        # fmgResidual (Alg 3.2): t_L = f_L - A_L u_L, r_l = enc R ... R t_L
        uL = self.std(self.u, L)
        t = self.f[L] - self.lv[L].K @ uL
        r = [None] * (L + 1)
        r[L] = enc(t, self.wr(L, L))
        for l in range(L - 1, -1, -1):
            t = self.P[l + 1].T @ t
            r[l] = enc(t, self.wr(l, L))
        # cFas V(0,1) from zero (Alg 3.1)
        y = [None] * (L + 1)
        y0 = np.linalg.solve(self.lv[0].K, dec(r[0]))
        y[0] = enc(y0, self.wr(0, L))
        w = dec(y[0])
        for l in range(1, L + 1):
            z = self.P[l] @ w
            b = dec(r[l]) - self.lv[l].K @ z
            yl = lex_gs(self.lv[l].K, b, self.p)
            y[l] = enc(yl, self.wr(l, L))
            w = z + dec(y[l])
        # correction PAPER.md:798
        for l in range(L + 1):
            self.u[l] = enc(dec(self.u[l]) + dec(y[l]), self.wu(l, L))


# ------------------------------------------------------------- accuracy --


def hm_error(lv: Level, coef: np.ndarray, du, m: int) -> float:
    """|| (sum_i c_i B_i)^(m) - u^(m) ||_L2 (the H^m seminorm error; du(x, m)
    is the m-th derivative of the exact solution)."""
    full = np.zeros(lv.n_all)
    full[lv.free] = coef
    xg, wg = gauss(lv.p + 6)
    h = 1.0 / lv.nel
    s = 0.0
    for e in range(lv.nel):
        a = e * h
        for q in range(len(xg)):
            x = a + 0.5 * h * (xg[q] + 1.0)
            v = basis_all(lv.t, lv.p, x, m)[m] @ full
            s += 0.5 * h * wg[q] * (v - du(x, m)) ** 2
    return math.sqrt(s)


# manufactured solutions
def poisson_u(x, k=0):
    # u = x (1 - x) cos(pi x / 2)
    a = math.pi / 2
    c, sn = math.cos(a * x), math.sin(a * x)
    g, g1, g2 = x - x * x, 1 - 2 * x, -2.0
    if k == 0:
        return g * c
    if k == 1:
        return g1 * c - a * g * sn
    if k == 2:
        return g2 * c - 2 * a * g1 * sn - a * a * g * c
    raise ValueError(k)


def poisson_f(x):
    return -poisson_u(x, 2)


def biharm_u(x, k=0):
    # u = 1 - cos(2 pi x)
    a = 2 * math.pi
    if k == 0:
        return 1 - math.cos(a * x)
    if k == 1:
        return a * math.sin(a * x)
    if k == 2:
        return a * a * math.cos(a * x)
    if k == 4:
        return -a ** 4 * math.cos(a * x)
    raise ValueError(k)


def biharm_f(x):
    return biharm_u(x, 4)
