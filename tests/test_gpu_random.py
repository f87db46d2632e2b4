"""Randomised-schedule GPU parity: seeded draws of dimension, degree, level
count, width law (b_u, k_u, b_r, k_r), IR iteration count, Chebyshev degree,
smoother and staging path (FMG_TMA), each checked bit for bit against the
oracle on the same schedule (sections, decoded solution; norms within 1e-6).
Schedules outside the method's convergence regime are fine here: parity is a
property of the arithmetic, not of the accuracy the schedule reaches."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

import oracle as O
from fmg_inputs import default_schedule


def _draw(seed):
    rng = np.random.default_rng(seed)
    d = int(rng.choice([2, 3]))
    p = int(rng.integers(1, 4))
    if d == 2:
        levels = int(rng.integers(2, {1: 8, 2: 7, 3: 6}[p]))
    else:
        levels = int(rng.integers(2, {1: 6, 2: 5, 3: 4}[p]))
    s = default_schedule(d, p)
    s["b_u"] = int(rng.integers(2, 12))
    s["k_u"] = int(rng.integers(0, p + 3))
    s["b_r"] = int(rng.integers(2, 8))
    s["k_r"] = int(rng.integers(0, 3))
    s["n_ir"] = int(rng.integers(1, 5))
    s["cheb_degree"] = int(rng.integers(1, 5))
    L = levels - 1
    s["b_u"] = min(s["b_u"], 54 - s["k_u"] * L)
    s["b_r"] = min(s["b_r"], 54 - s["k_r"] * L)
    smoother = "mcgs" if rng.random() < 0.3 else "chebyshev"
    tma = str(int(rng.integers(0, 2)))
    return d, p, levels, s, smoother, tma


@pytest.mark.parametrize("seed", range(48))
def test_random_schedule_parity(monkeypatch, seed):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2511_19036_b200 as P
    d, p, levels, s, smoother, tma = _draw(seed)
    monkeypatch.setenv("FMG_TMA", tma)
    so = O.schedule(d, p, b_u=s["b_u"], b_r=s["b_r"], n_ir=s["n_ir"], k_u=s["k_u"], k_r=s["k_r"],
                    cheb_degree=s["cheb_degree"], smoother=smoother)
    oc = O.CFMG(d, p, levels, so)
    oc.solve()
    gs = P.Solver(d, p, levels, P.Schedule.from_dict(dict(s, smoother=smoother)))
    gs.solve()
    no, ng = oc.norms(), gs.norms()
    m = no != 0
    assert np.array_equal(m, ng != 0)
    if m.any():
        assert np.max(np.abs(ng[m] - no[m]) / no[m]) <= 1e-6
    for l in range(levels):
        for which in (0, 1):
            mo, eo, wo = oc.section(which, l)
            mg, eg, wg = gs.section(which, l)
            assert wo == wg and np.array_equal(eo, eg) and np.array_equal(mo, mg), (which, l)
    assert np.array_equal(oc.solution(), gs.solution().cpu().numpy())
