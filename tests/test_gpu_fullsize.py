"""Full-size GPU checks for the BASELINE configs the oracle cannot solve in a
test (C3 opt-in only, C4 never): properties that hold at any size.

Convergence order, PAPER.md:1449-1459 (Eq 7.3/7.4).  When the compact FMG reaches the
discretisation error at every FMG level, the relative H1-seminorm error of
the manufactured solution u = prod sin(pi x_k) falls by 2^-p per level (Q_p),
and the L2 error by about 2^-(p+1).  The L2 bound is looser: the width
schedules target the H1 error.  The finest level runs through the bench's
path (the captured CUDA graph, fmg_solve); the coarser ones through
fmg_solve_upto.  Measured (tools/rates_full.py): the H1 log2 ratios are
within 0.07 of -p for C2-C4."""
import math

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

from fmg_inputs import CONFIGS, default_schedule


@pytest.mark.parametrize("cfg", ["C2", "C3", "C4"])
def test_full_size_convergence_order(cfg):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2511_19036_b200 as P
    c = CONFIGS[cfg]
    d, p, lv = c["dim"], c["p"], c["levels"]
    s = P.Solver(d, p, lv, default_schedule(d, p))
    errs = {}
    for L in range(lv - 4, lv - 1):
        s.solve_upto(L, s.schedule.n_ir)
        errs[L] = s.errors()
    s.solve()
    errs[lv - 1] = s.errors()
    for L in range(lv - 3, lv):
        h1 = math.log2(errs[L][1] / errs[L - 1][1])
        l2 = math.log2(errs[L][0] / errs[L - 1][0])
        assert abs(h1 + p) <= 0.1, (cfg, L, h1)
        assert l2 <= -(p + 1) + 0.5, (cfg, L, l2)
    s.close()


def test_c5h_convergence_order_and_full_solve():
    """C5's per-GPU share (2048^3 Q1, 11 levels, 8.6 G unknowns) on one B200,
    lean finest-level kernels: the H1 error falls by 2^-1 per
    FMG level up to level 10, and the full solve completes and is
    bit-reproducible.  (The level-11 error needs a decoded 69 GB u array on
    top of the context's 135 GB, so it is not taken.)"""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import numpy as np
    import paper_2511_19036_b200 as P
    c = CONFIGS["C5h"]
    d, p, lv = c["dim"], c["p"], c["levels"]
    s = P.Solver(d, p, lv, default_schedule(d, p))
    errs = {}
    for L in range(lv - 5, lv - 1):
        s.solve_upto(L, s.schedule.n_ir)
        errs[L] = s.errors()
    for L in range(lv - 4, lv - 1):
        h1 = math.log2(errs[L][1] / errs[L - 1][1])
        assert abs(h1 + p) <= 0.1, (L, h1)
    s.solve()
    n1 = s.norms().copy()
    top = s.section(0, lv - 1)
    s.solve()
    assert np.array_equal(n1, s.norms())
    again = s.section(0, lv - 1)
    assert np.array_equal(top[0], again[0]) and np.array_equal(top[1], again[1])
    s.close()
