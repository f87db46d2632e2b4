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


def span(t: np.ndarray, p: int, x: float) -> int:
    """Span index s with t[s] <= x < t[s+1] (x = 1 belongs to the last span);
    only B-splines s-p .. s are nonzero at x."""
    n = len(t) - p - 1
    s = np.searchsorted(t, x, side="right") - 1
    return int(min(max(s, p), n - 1))


def basis_all(t: np.ndarray, p: int, x: float, nder: int) -> np.ndarray:
    """Values and derivatives (rows 0..nder) of all n = len(t)-p-1 B-splines
    at x, by the Cox-de Boor recursion and its derivative formula."""
    n = len(t) - p - 1
    s = span(t, p, x)
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
            # only the (p+1) x (p+1) block of the functions nonzero at x: the
            # other products are exact zeros, which leave every sum unchanged
            sl = slice(span(t, p, x) - p, span(t, p, x) + 1)
            K[sl, sl] += w * np.outer(B[m][sl], B[m][sl])
            M[sl, sl] += w * np.outer(B[0][sl], B[0][sl])
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
            sf = span(fine.t, fine.p, x)
            sc = span(coarse.t, coarse.p, x)
            fs = slice(sf - fine.p, sf + 1)
            cs = slice(sc - coarse.p, sc + 1)
            Mfc[fs, cs] += w * np.outer(basis_all(fine.t, fine.p, x, 0)[0][fs], basis_all(coarse.t, coarse.p, x, 0)[0][cs])
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


# ------------------------------------------------- operator layouts (R27) --
#
# The GPU path (include/fmg1d.h) consumes the level operators in these
# layouts, and the oracle evaluates every product in the order they define
# (reading R27): a row's terms are summed from 0.0 in ascending storage index,
# so both sides round identically.


def band(K: np.ndarray, p: int) -> np.ndarray:
    """A_l as an n x (2p+1) band: Ab[i, k] = K[i, i-p+k], 0 outside 0..n-1."""
    n = K.shape[0]
    Ab = np.zeros((n, 2 * p + 1))
    for i in range(n):
        for k in range(2 * p + 1):
            j = i - p + k
            if 0 <= j < n:
                Ab[i, k] = K[i, j]
    return Ab


def two_scale_structure(fine: Level, coarse: Level):
    """(j0, j1) per fine unknown i: the coarse unknowns j whose B-spline support
    contains that of fine B-spline i, j0 <= j <= j1 -- the only columns where
    the two-scale coefficient can be nonzero (a coarse B-spline is a
    combination of the fine B-splines inside its support).  Knots are dyadic,
    so the comparisons are exact."""
    p, m = fine.p, fine.m
    nf, nc = len(fine.free), len(coarse.free)
    lo = coarse.t[m: m + nc]                   # coarse supports [lo_j, hi_j]
    hi = coarse.t[m + p + 1: m + p + 1 + nc]
    out = []
    for i in range(nf):
        I = i + m
        a, b = fine.t[I], fine.t[I + p + 1]
        js = np.nonzero((lo <= a) & (b <= hi))[0]
        assert np.array_equal(js, np.arange(js[0], js[-1] + 1))
        out.append((int(js[0]), int(js[-1])))
    return out


def ell(P: np.ndarray, st) -> tuple:
    """P in ELL form: vals[i, k] = P[i, c0[i] + k] for c0[i] + k <= j1(i), 0 beyond."""
    kp = max(j1 - j0 + 1 for j0, j1 in st)
    vals = np.zeros((len(st), kp))
    c0 = np.array([j0 for j0, _ in st], dtype=np.int64)
    for i, (j0, j1) in enumerate(st):
        vals[i, : j1 - j0 + 1] = P[i, j0 : j1 + 1]
    return vals, c0


def ell_transpose(P: np.ndarray, st, nc: int) -> tuple:
    """R = P^T in ELL form: for coarse j the fine rows i with j in st[i],
    ascending."""
    j0s = np.array([a for a, _ in st])
    j1s = np.array([b for _, b in st])
    rows = [np.nonzero((j0s <= j) & (j <= j1s))[0].tolist() for j in range(nc)]
    kr = max(len(r) for r in rows)
    vals = np.zeros((nc, kr))
    r0 = np.array([r[0] for r in rows], dtype=np.int64)
    for j, r in enumerate(rows):
        assert r == list(range(r[0], r[-1] + 1))
        vals[j, : len(r)] = P[r, j]
    return vals, r0


def band_mv(Ab: np.ndarray, x: np.ndarray, p: int) -> np.ndarray:
    """y_i = sum_k Ab[i, k] x[i-p+k], from 0.0, k ascending (R27)."""
    n = len(x)
    xp = np.concatenate([np.zeros(p), x, np.zeros(p)])
    y = np.zeros(n)
    for k in range(2 * p + 1):
        y = y + Ab[:, k] * xp[k : k + n]
    return y


def ell_mv(vals: np.ndarray, c0: np.ndarray, x: np.ndarray) -> np.ndarray:
    """y_i = sum_k vals[i, k] x[c0[i] + k], from 0.0, k ascending (R27)."""
    xp = np.concatenate([x, np.zeros(vals.shape[1])])
    y = np.zeros(vals.shape[0])
    for k in range(vals.shape[1]):
        y = y + vals[:, k] * xp[c0 + k]
    return y


def dense_mv(A: np.ndarray, x: np.ndarray) -> np.ndarray:
    """y_i = sum_j A[i, j] x[j], from 0.0, j ascending (R27)."""
    y = np.zeros(A.shape[0])
    for j in range(A.shape[1]):
        y = y + A[:, j] * x[j]
    return y


# ------------------------------------------------------------ compact FMG --


def gs_row(Ab: np.ndarray, b: np.ndarray, y: np.ndarray, i: int, p: int) -> float:
    """One Gauss-Seidel row update: (b_i - sum_{j != i} A_ij y_j) / A_ii, the
    terms subtracted in ascending j over the band (R27)."""
    n = len(b)
    s = b[i]
    for k in range(2 * p + 1):
        j = i - p + k
        if k != p and 0 <= j < n:
            s = s - Ab[i, k] * y[j]
    return s / Ab[i, p]


def lex_gs(Ab: np.ndarray, b: np.ndarray, p: int) -> np.ndarray:
    """One forward (lexicographic) Gauss-Seidel sweep from y = 0
    (PAPER.md:689-690, 1624)."""
    y = np.zeros(len(b))
    for i in range(len(b)):
        y[i] = gs_row(Ab, b, y, i, p)
    return y


def mc_gs(Ab: np.ndarray, b: np.ndarray, p: int) -> np.ndarray:
    """One multicolour Gauss-Seidel sweep from y = 0 (§8(f) N1 carried to 1D):
    colours c = 0..p, rows i = c mod (p+1) in ascending colour order.  Rows of
    one colour are more than p apart, so they do not couple and the sweep is
    parallel within a colour."""
    y = np.zeros(len(b))
    for c in range(p + 1):
        for i in range(c, len(b), p + 1):
            y[i] = gs_row(Ab, b, y, i, p)
    return y


class CFMG1D:
    """Alg 3.3 in 1D with B-splines, m in {1, 2}.
    smoother: "lex" (the paper's lexicographic Gauss-Seidel) or "mcgs"."""

    def __init__(self, p, m, levels, N, b1, b2, f, smoother="lex"):
        assert smoother in ("lex", "mcgs")
        self.p, self.m, self.levels, self.N, self.b1, self.b2 = p, m, levels, N, b1, b2
        self.smoother = smoother
        self.lv = [assemble(p, m, l) for l in range(levels)]
        self.P = [None] + [two_scale(self.lv[l], self.lv[l - 1]) for l in range(1, levels)]
        self.f = [load(lv, f) for lv in self.lv] if callable(f) else [np.asarray(v, dtype=float) for v in f]
        # operators in the GPU layouts (R27); P entries outside the support
        # structure are the L2 solve's rounding noise and are dropped
        self.Ab = [band(lv.K, p) for lv in self.lv]
        self.Pe = [None]
        self.Re = [None]
        for l in range(1, levels):
            st = two_scale_structure(self.lv[l], self.lv[l - 1])
            self.Pe.append(ell(self.P[l], st))
            self.Re.append(ell_transpose(self.P[l], st, len(self.lv[l - 1].free)))
        self.A0inv = np.linalg.inv(self.lv[0].K)

    def wu(self, l, L):
        return self.b1 + (self.p + 1) * (L - l)

    def wr(self, l, L):
        return self.b2 + self.m * (L - l)

    def prolong(self, l, x):
        return ell_mv(*self.Pe[l], x)

    def restrict(self, l, x):
        return ell_mv(*self.Re[l], x)

    def std(self, secs, L):
        """Standard representation of a compact vector: u_l = dec ú_l + P_l u_{l-1}."""
        u = dec(secs[0])
        for l in range(1, L + 1):
            u = dec(secs[l]) + self.prolong(l, u)
        return u

    def solve(self, Lstop=None):
        L0 = self.levels - 1 if Lstop is None else Lstop
        # coarse-grid solve PAPER.md:785-786
        u0 = dense_mv(self.A0inv, self.f[0])
        self.u = [enc(u0, self.wu(0, 0))]
        self.sols = {0: dec(self.u[0])}
        for L in range(1, L0 + 1):
            self.u.append(enc(np.zeros(len(self.f[L])), self.wu(L, L)))  # push level: ú_L = 0
            for _ in range(self.N):
                self.iteration(L)
            self.sols[L] = self.std(self.u, L)
        return self.sols

    def iteration(self, L):
        p = self.p
        # fmgResidual (Alg 3.2): t_L = f_L - A_L u_L, r_l = enc R ... R t_L
        uL = self.std(self.u, L)
        t = self.f[L] - band_mv(self.Ab[L], uL, p)
        r = [None] * (L + 1)
        r[L] = enc(t, self.wr(L, L))
        for l in range(L - 1, -1, -1):
            t = self.restrict(l + 1, t)
            r[l] = enc(t, self.wr(l, L))
        # cFas V(0,1) from zero (Alg 3.1)
        y = [None] * (L + 1)
        y0 = dense_mv(self.A0inv, dec(r[0]))
        y[0] = enc(y0, self.wr(0, L))
        w = dec(y[0])
        gs = lex_gs if self.smoother == "lex" else mc_gs
        for l in range(1, L + 1):
            z = self.prolong(l, w)
            b = dec(r[l]) - band_mv(self.Ab[l], z, p)
            yl = gs(self.Ab[l], b, p)
            y[l] = enc(yl, self.wr(l, L))
            w = z + dec(y[l])
        self.y = y
        self.r = r
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
