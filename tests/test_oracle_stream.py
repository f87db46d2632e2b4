"""The oracle's plane-streamed mode (oracle/orc_stream.c: Alg 5.3 cFas and
Alg 5.4 fmgResidual at plane granularity) against its simple
mode: every section (ú, r, ý at every level) and every residual norm identical
bit for bit ("a plane-streamed mode ... which must be
bit-identical to the simple mode"), with FP64 temporaries that grow with the
plane, not the grid (linear space)."""
import numpy as np
import pytest

import oracle as O


def _same(a, b, levels):
    assert np.array_equal(a.norms(), b.norms())
    for which in range(3):
        for l in range(levels):
            ma, ea, wa = a.section(which, l)
            mb, eb, wb = b.section(which, l)
            assert wa == wb, (which, l)
            assert np.array_equal(ea, eb), (which, l)
            assert np.array_equal(ma, mb), (which, l)


CASES = [
    (2, 1, 7, {}),
    (2, 2, 6, {}),
    (2, 3, 5, {}),
    (2, 1, 6, dict(cheb_degree=1)),
    (2, 2, 6, dict(cheb_degree=4, n_ir=3)),
    (3, 1, 5, {}),
    (3, 2, 4, {}),
    (3, 3, 4, {}),
    (3, 3, 4, dict(cheb_degree=2, b_u=5, b_r=3)),
    (3, 2, 4, dict(cheb_degree=5, n_ir=1)),
    (3, 1, 4, dict(b_u=20, b_r=20)),
]


@pytest.mark.parametrize("d,p,levels,kw", CASES)
def test_streamed_solve_bit_identical(d, p, levels, kw):
    s = O.schedule(d, p, **kw)
    a = O.CFMG(d, p, levels, s)
    a.solve()
    b = O.CFMG(d, p, levels, s, streamed=True)
    b.solve()
    assert b.stream_bytes() > 0 and a.stream_bytes() == 0
    assert a.norms()[-1, -1, -1] > 0
    _same(a, b, levels)


@pytest.mark.parametrize("d,p,levels", [(2, 2, 6), (3, 1, 5), (3, 3, 4)])
def test_streamed_partial_solve_and_residual(d, p, levels):
    """A partial solve (mid-FMG, sections narrower than at the end) then one
    more residual: the streamed residual reads the same compact state."""
    s = O.schedule(d, p)
    a = O.CFMG(d, p, levels, s)
    b = O.CFMG(d, p, levels, s, streamed=True)
    for c in (a, b):
        c.solve_upto(levels - 2, 1)
    _same(a, b, levels)
    na, nb = a.residual(levels - 2), b.residual(levels - 2)
    assert np.array_equal(na, nb)
    for l in range(levels - 1):
        assert np.array_equal(a.section(1, l)[0], b.section(1, l)[0])


def test_streamed_temporaries_grow_with_the_plane():
    """Linear space: one more 3D level multiplies a full array by 8 and the
    streamed windows by about 4 (they hold planes)."""
    s = O.schedule(3, 1)
    sizes = []
    for levels in (5, 6, 7):
        c = O.CFMG(3, 1, levels, s, streamed=True)
        c.solve_upto(levels - 1, 1)
        sizes.append(c.stream_bytes())
    full = [O.Geom(3, 1, lv - 1).size * 8 for lv in (5, 6, 7)]
    assert full[2] / full[1] > 7.5
    assert 3.0 < sizes[2] / sizes[1] < 4.6
    assert 3.0 < sizes[1] / sizes[0] < 4.8
    # at 2048^3 the same windows would be ~ (2048/128)^2 x sizes[2]: a few GB,
    # against 69 GB for one full FP64 array
    assert sizes[2] * 16 ** 2 < 0.1 * O.Geom(3, 1, 10).size * 8


@pytest.mark.parametrize("kw", [dict(smoother="mcgs"), dict(nu=2), dict(cfas_fp32=1)])
def test_streamed_mode_scope(kw):
    with pytest.raises(ValueError):
        O.CFMG(3, 1, 3, O.schedule(3, 1, **kw), streamed=True)
