"""The oracle's OpenMP mode (C4/C5 need more than one core) is
deterministic: every output is one canonical chain computed by one thread
and every norm a sequential sum, so one thread and many give bit-identical
sections and norms."""
import numpy as np
import pytest

import oracle as O


@pytest.mark.parametrize("d,p,levels", [(3, 1, 5), (3, 3, 3), (2, 2, 6)])
def test_thread_count_does_not_change_results(d, p, levels):
    L = O.lib()
    n0 = L.orc_threads()
    out = []
    try:
        for t in (1, 4):
            L.orc_set_threads(t)
            assert L.orc_threads() == t
            c = O.CFMG(d, p, levels, O.schedule(d, p))
            c.solve()
            out.append((c.norms().copy(), [c.section(0, l) for l in range(levels)]))
    finally:
        L.orc_set_threads(n0)
    (n1, s1), (n4, s4) = out
    assert np.array_equal(n1, n4)
    for a, b in zip(s1, s4):
        assert a[2] == b[2] and np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
