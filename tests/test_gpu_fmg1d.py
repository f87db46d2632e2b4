"""GPU parity of the 1D B-spline compact FMG (§8(f) row N4, include/fmg1d.h)
against the oracle (oracle/bspline1d.py), through the C-ABI.

The GPU context gets the oracle's operators (band A_l, ELL P_l, A_0^-1: the
layouts of reading R27) and load vectors, so both sides run the same
arithmetic; the finest-level solution and every section of the last IR
iteration (u_l, r_l, y_l: mantissa words and exponents) must be BIT-identical.
Cases: Table 3's 1D rows with both smoothers, ragged
level sizes (n_l = 2^(l+1) + p - 2m is never a multiple of 32), one level
(coarse solve only), the widest widths (54 bits), batches with distinct
loads, the native-assembly path against Eq 7.3, and the error path."""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

import oracle.bspline1d as B

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "table3_poisson.json")))


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")


def _gpu_from_oracle(o, batch=1, loads=None):
    import paper_2511_19036_b200 as P
    s = P.Solver1D(o.p, o.m, o.levels, o.N, o.b1, o.b2, smoother=o.smoother, batch=batch,
                   Ab=o.Ab, Pv=[None] + [o.Pe[l][0] for l in range(1, o.levels)], A0inv=o.A0inv)
    s.set_load(loads if loads is not None else o.f)
    s.solve()
    return s


def _compare(o, s, b=0):
    L = o.levels - 1
    assert np.array_equal(s.solution(b), o.sols[L])
    for l in range(o.levels):
        for which, sec in ((0, o.u[l]), (1, o.r[l] if L else None), (2, o.y[l] if L else None)):
            if sec is None:
                continue
            mg, eg, wg = s.section(which, l, b)
            mo, eo, wo, _ = sec
            assert wg == wo, (which, l)
            assert np.array_equal(eg, eo), (which, l)
            assert np.array_equal(mg, mo), (which, l)


def _row(m, p):
    return GOLD["poisson_1d" if m == 1 else "biharmonic_1d"][str(p)]


@pytest.mark.parametrize("smoother", ["lex", "mcgs"])
@pytest.mark.parametrize("m,p,levels", [(1, 1, 7), (1, 2, 6), (1, 3, 7), (1, 4, 6), (1, 5, 6),
                                        (2, 3, 6), (2, 4, 6), (2, 5, 5), (2, 6, 5), (2, 7, 5)])
def test_table3_rows_bit_exact(m, p, levels, smoother):
    _need_gpu()
    r = _row(m, p)
    o = B.CFMG1D(p, m, levels, r["N"], r["b1"], r["b2"], B.poisson_f if m == 1 else B.biharm_f, smoother=smoother)
    o.solve()
    _compare(o, _gpu_from_oracle(o))


@pytest.mark.parametrize("smoother", ["lex", "mcgs"])
def test_larger_level_count(smoother):
    """10 levels: n_L = 2049 unknowns, 65 blocks with a ragged tail, every
    phase spans several CTA-stride passes."""
    _need_gpu()
    o = B.CFMG1D(1, 1, 10, 4, 5, 3, B.poisson_f, smoother=smoother)
    o.solve()
    _compare(o, _gpu_from_oracle(o))


def test_single_level_is_the_coarse_solve():
    _need_gpu()
    o = B.CFMG1D(3, 1, 1, 4, 7, 4, B.poisson_f)
    o.solve()
    s = _gpu_from_oracle(o)
    assert np.array_equal(s.solution(), o.sols[0])
    mg, eg, wg = s.section(0, 0)
    assert wg == o.u[0][2] and np.array_equal(mg, o.u[0][0]) and np.array_equal(eg, o.u[0][1])


def test_widest_widths():
    """b1 + (p+1) L = 54 and b2 + m L = 54 at the coarsest level: the 54-bit
    (two-word-per-lane) codec path."""
    _need_gpu()
    L = 4
    o = B.CFMG1D(2, 1, L + 1, 3, 54 - 3 * L, 54 - L, B.poisson_f)
    o.solve()
    _compare(o, _gpu_from_oracle(o))


def test_batch_of_distinct_loads():
    """Problems of one batch are independent: each equals the oracle run on its
    own load (seeded random loads, not only the manufactured one)."""
    _need_gpu()
    p, m, levels = 3, 2, 6
    rng = np.random.default_rng(7)
    base = B.CFMG1D(p, m, levels, 6, 4, 4, B.biharm_f)
    loads = [base.f]
    for _ in range(4):
        loads.append([rng.standard_normal(len(v)) * 10.0 ** rng.uniform(-3, 3) for v in base.f])
    batch = len(loads)
    stacked = [np.stack([ld[l] for ld in loads]) for l in range(levels)]
    s = None
    for b, ld in enumerate(loads):
        o = B.CFMG1D(p, m, levels, 6, 4, 4, ld)
        o.solve()
        if s is None:
            s = _gpu_from_oracle(o, batch=batch, loads=stacked)
        _compare(o, s, b)


def test_solve_host_end_to_end_matches_device_path():
    _need_gpu()
    o = B.CFMG1D(2, 1, 6, 3, 5, 4, B.poisson_f)
    o.solve()
    s = _gpu_from_oracle(o, batch=3)
    u = s.solve_host([np.stack([v] * 3) for v in o.f])
    for b in range(3):
        assert np.array_equal(u[b], o.sols[5])


@pytest.mark.parametrize("m,p", [(1, 1), (1, 3), (2, 3), (2, 5)])
def test_native_assembly_meets_eq73(m, p):
    """With the library's own operators and loads (no oracle input), the GPU
    solution meets Eq 7.3 at the finest level: H^m error within 2x the
    discretisation error of the exact discrete solution."""
    _need_gpu()
    import paper_2511_19036_b200 as P
    r = _row(m, p)
    Ltop = min(7, (53 - r["b3"]) // (p + m + 1))
    if (p, m) == (7, 2):
        Ltop = 4
    levels = Ltop + 1
    s = P.Solver1D(p, m, levels, r["N"], r["b1"], r["b2"], batch=2)
    s.set_load([P.fmg1d_load(p, m, l) for l in range(levels)])
    s.solve()
    u = s.solution(1)
    lv = B.assemble(p, m, Ltop)
    uf = B.poisson_u if m == 1 else B.biharm_u
    ec = B.hm_error(lv, u, uf, m)
    ed = B.hm_error(lv, np.linalg.solve(lv.K, B.load(lv, B.poisson_f if m == 1 else B.biharm_f)), uf, m)
    assert ec <= 2 * ed, ec / ed
    assert np.array_equal(u, s.solution(0))


def test_non_finite_load_reports_erange():
    _need_gpu()
    import paper_2511_19036_b200 as P
    s = P.Solver1D(1, 1, 4, 2, 5, 3)
    f = [P.fmg1d_load(1, 1, l) for l in range(4)]
    f[3] = f[3].copy()
    f[3][5] = np.inf
    s.set_load(f)
    s.solve_async()
    with pytest.raises(P.FmgError) as e:
        s.sync()
    assert e.value.code == P.FMG_ERANGE


@pytest.mark.parametrize("tp", ["32", "256"])
@pytest.mark.parametrize("smoother", ["lex", "mcgs"])
@pytest.mark.parametrize("m,p,levels", [(1, 1, 9), (2, 5, 5), (1, 3, 7)])
def test_thread_layouts_bit_exact(monkeypatch, tp, smoother, m, p, levels):
    """Both thread layouts (one warp per problem; one CTA per problem:
    FMG1D_TP) give the oracle's bits, batched with distinct loads."""
    _need_gpu()
    monkeypatch.setenv("FMG1D_TP", tp)
    r = _row(m, p)
    o = B.CFMG1D(p, m, levels, r["N"], r["b1"], r["b2"], B.poisson_f if m == 1 else B.biharm_f, smoother=smoother)
    o.solve()
    rng = np.random.default_rng(11)
    other = [rng.standard_normal(len(v)) for v in o.f]
    o2 = B.CFMG1D(p, m, levels, r["N"], r["b1"], r["b2"], other, smoother=smoother)
    o2.solve()
    s = _gpu_from_oracle(o, batch=5, loads=[np.stack([a, b, a, b, a]) for a, b in zip(o.f, other)])
    for b in range(5):
        _compare(o if b % 2 == 0 else o2, s, b)
