"""GPU parity for nu > 1 compact V(0,1) cycles per IR iteration (§8(f) row N2;
Alg 3.1, reading R23) against the oracle: every solution and
residual section bit for bit, per-level norms within 1e-6, the decoded
solution bit-identical.  The GPU path covers 2D and 3D (one GPU) with the
Chebyshev (degree >= 2) or multicolour Gauss-Seidel smoother; Chebyshev of
degree 1 and z slabs are refused."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

import oracle as O
from fmg_inputs import CONFIGS, default_schedule


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2511_19036_b200 as P
    return P


def _compare(P, d, p, levels, nu, **kw):
    so = O.schedule(d, p, nu=nu, **kw)
    oc = O.CFMG(d, p, levels, so)
    oc.solve()
    s = default_schedule(d, p)
    s.update(kw)
    s["nu"] = nu
    gs = P.Solver(d, p, levels, P.Schedule.from_dict(s))
    gs.solve()
    no, ng = oc.norms(), gs.norms()
    m = no != 0
    assert np.array_equal(m, ng != 0)
    assert np.max(np.abs(ng[m] - no[m]) / no[m]) <= 1e-6
    for l in range(levels):
        for which in (0, 1):
            mo, eo, wo = oc.section(which, l)
            mg, eg, wg = gs.section(which, l)
            assert wo == wg and np.array_equal(eo, eg) and np.array_equal(mo, mg), (which, l)
    assert np.array_equal(oc.solution(), gs.solution().cpu().numpy())
    return oc, gs


@pytest.mark.parametrize("nu", [2, 3])
@pytest.mark.parametrize("d,p,levels", [(2, 1, 2), (2, 1, 6), (2, 2, 5), (2, 3, 4),
                                        (3, 1, 2), (3, 1, 5), (3, 2, 4), (3, 3, 3)])
def test_nu_parity(P, d, p, levels, nu):
    _compare(P, d, p, levels, nu)


@pytest.mark.parametrize("kw", [dict(cheb_degree=3), dict(k_u=0, k_r=0), dict(b_u=12, b_r=6, n_ir=1)])
def test_nu_parity_schedules(P, kw):
    _compare(P, 2, 2, 5, 2, **kw)


@pytest.mark.parametrize("d,p,levels", [(2, 1, 6), (2, 2, 5), (3, 1, 4), (3, 2, 3)])
def test_nu_parity_multicolour_gs(P, d, p, levels):
    """nu = 2 with the multicolour Gauss-Seidel smoother (N1 x N2)."""
    _compare(P, d, p, levels, 2, smoother="mcgs")


def test_nu_parity_C2_full(P):
    c = CONFIGS["C2"]
    _compare(P, c["dim"], c["p"], c["levels"], 2)


def test_nu_parity_C3_full(P):
    c = CONFIGS["C3"]
    _compare(P, c["dim"], c["p"], 7, 2)  # (C3's geometry on 7 levels: the oracle stays in seconds)


def test_nu_refused_outside_the_gpu_scope(P):
    for d, p, over in [(2, 1, {"cheb_degree": 1}), (3, 1, {"cheb_degree": 1})]:
        s = default_schedule(d, p)
        s.update(over)
        s["nu"] = 2
        with pytest.raises(P.FmgError):
            P.Solver(d, p, 3, P.Schedule.from_dict(s))
    s = default_schedule(3, 1)
    s["nu"] = 2
    with pytest.raises(P.FmgError):  # z slabs: nu = 1 only this round
        P.Solver(3, 1, 4, P.Schedule.from_dict(s), slabs=2)
