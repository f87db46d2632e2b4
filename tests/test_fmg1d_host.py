"""CPU checks of the 1D B-spline path's host side (§8(f) row N4,
include/fmg1d.h): the library's native assembly (fmg1d_assembly.cpp, written
independently of the oracle -- knot insertion instead of an L2 projection for
P, its own quadrature) against the oracle's operators and closed forms, and the
argument validation of fmg1d_create, which runs before any device call."""
import ctypes as C

import numpy as np
import pytest

import oracle.bspline1d as B

P = pytest.importorskip("paper_2511_19036_b200")

CASES = [(1, 1), (2, 1), (3, 1), (5, 1), (3, 2), (4, 2), (5, 2), (7, 2)]


@pytest.mark.parametrize("p,m", CASES)
def test_sizes_and_structure(p, m):
    for l in range(0, 6):
        lv = B.assemble(p, m, l)
        assert P.fmg1d_size(p, m, l) == len(lv.free)
        if l:
            st = B.two_scale_structure(lv, B.assemble(p, m, l - 1))
            assert P._lib.fmg1d_ell_width(p, m, l) == max(j1 - j0 + 1 for j0, j1 in st)


@pytest.mark.parametrize("p,m", CASES)
def test_native_assembly_matches_oracle(p, m):
    f = B.poisson_f if m == 1 else B.biharm_f
    for l in (0, 1, 3, 5):
        lv = B.assemble(p, m, l)
        Ab = B.band(lv.K, p)
        An = P.fmg1d_operator(p, m, l)
        assert np.abs(An - Ab).max() <= 1e-14 * np.abs(Ab).max()
        assert np.array_equal(An == 0, Ab == 0)  # the same band structure
        fo = B.load(lv, f)
        assert np.abs(P.fmg1d_load(p, m, l) - fo).max() <= 1e-14 * np.abs(fo).max()
        if l:
            c = B.assemble(p, m, l - 1)
            Po, _ = B.ell(B.two_scale(lv, c), B.two_scale_structure(lv, c))
            assert np.abs(P.fmg1d_prolongation(p, m, l) - Po).max() <= 1e-12


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5])
def test_native_two_scale_interior_closed_form(p):
    """Away from the open ends, uniform B-splines refine by the binomial mask:
    coarse B_j = 2^-p sum_k C(p+1, k) fine B_{2j+k} (up to the index shift)."""
    from math import comb
    Pv = P.fmg1d_prolongation(p, 1, 5)
    mask = np.array([comb(p + 1, k) / 2 ** p for k in range(p + 2)])
    n = Pv.shape[0]
    # each interior fine row holds the mask entries of every other position
    for i in range(n // 4, 3 * n // 4):
        row = Pv[i][Pv[i] != 0]
        ok = any(np.allclose(row, mask[s::2][: len(row)], rtol=0, atol=2e-16) for s in (0, 1))
        assert ok, (i, row)


def test_create_validates_before_any_device_call():
    s = P.Schedule1D(4, 5, 3, 0)
    h = C.c_void_p()
    lib = P._lib
    assert lib.fmg1d_create(8, 1, 4, C.byref(s), 1, None, None, None, None, C.byref(h)) == P.FMG_EINVAL
    assert lib.fmg1d_create(2, 2, 4, C.byref(s), 1, None, None, None, None, C.byref(h)) == P.FMG_EINVAL  # n_0 = 0
    assert lib.fmg1d_create(3, 1, 0, C.byref(s), 1, None, None, None, None, C.byref(h)) == P.FMG_EINVAL
    assert lib.fmg1d_create(3, 1, 4, C.byref(s), 0, None, None, None, None, C.byref(h)) == P.FMG_EINVAL
    wide = P.Schedule1D(4, 50, 3, 0)  # b1 + (p+1) L > 54
    assert lib.fmg1d_create(3, 1, 4, C.byref(wide), 1, None, None, None, None, C.byref(h)) == P.FMG_EINVAL
    bad = P.Schedule1D(4, 5, 3, 7)
    assert lib.fmg1d_create(3, 1, 4, C.byref(bad), 1, None, None, None, None, C.byref(h)) == P.FMG_EINVAL
    assert lib.fmg1d_size(3, 3, 2) == -1 and lib.fmg1d_ell_width(3, 1, 0) == -1


def test_bench_n4_alg_bytes_by_hand():
    """bench.py's N4 roofline numerator on a two-level case,
    counted by hand: p = 1, m = 1, levels 2 (n_0 = 1, n_1 = 3), N = 2, b1 = 5,
    b2 = 3.  One FMG level L = 1 with two iterations; per iteration f_1
    (8 * 3 B) plus, for l = 0 (w_u = 5 + 2 = 7, w_r = 3 + 1 = 4) and l = 1
    (w_u = 5, w_r = 3), n_l (3 w_u + 5 w_r) / 8; then the final solution."""
    import bench
    per_it = 8 * 3 + 1 * (3 * 7 + 5 * 4) / 8 + 3 * (3 * 5 + 5 * 3) / 8
    assert bench.n4_alg_bytes(1, 1, 2, 2, 5, 3) == 2 * per_it + 8 * 3
    assert bench.N4_ROWS[(1, 1)] == (4, 5, 3) and bench.N4_ROWS[(7, 2)] == (11, 12, 6)


def test_bench_n4_rows_are_table3():
    """The N4 bench schedules are Table 3's 1D rows (tests/golden)."""
    import json
    import os
    import bench
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "table3_poisson.json")))
    for m, key in ((1, "poisson_1d"), (2, "biharmonic_1d")):
        for p, row in g[key].items():
            if not p.startswith("_"):
                assert bench.N4_ROWS[(int(p), m)] == (row["N"], row["b1"], row["b2"])
