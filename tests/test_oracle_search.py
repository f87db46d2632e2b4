"""The paper's constant search run on the oracle
(oracle/search.py): greedy b2 (= b_r), then b1 (= b_u), then N, each the
first value meeting Eq 7.3 / 7.4 plus one.  Pins: the search terminates with
a schedule that meets the criteria on the search levels, and the frozen
schedules of fmg_inputs (every bench number uses them) are
never below what the search finds, i.e. at least as conservative."""
import pytest

import oracle as O
from fmg_inputs import default_schedule
from oracle.search import _criteria, disc_errors, search_constants

CASES = [(2, 1, 5), (2, 2, 5), (2, 3, 5), (3, 1, 4), (3, 3, 4)]


@pytest.mark.parametrize("d,p,levels", CASES)
def test_search_result_meets_criteria_and_frozen_schedule_is_not_below(d, p, levels):
    (n, b_u, b_r), log = search_constants(d, p, levels)
    assert 2 <= b_r <= 12 and 2 <= b_u <= 12 and 1 <= n <= 12
    # the trial log: every tuned value below the result failed, the result passed
    for name, v, passed in log:
        if name == "b_r" and v < b_r - 1:
            assert not passed
    s = O.schedule(d, p, b_u=b_u, b_r=b_r, n_ir=n)
    assert _criteria(d, p, levels, s, disc_errors(d, p, levels, s))
    fz = default_schedule(d, p)
    assert fz["b_u"] >= b_u and fz["b_r"] >= b_r and fz["n_ir"] >= n, ((n, b_u, b_r), fz)


def test_search_finds_the_frozen_q3_schedule():
    """For Q3 the search reproduces DESIGN.md §5's frozen (N, b_u, b_r) = (3, 6, 4)."""
    (n, b_u, b_r), _ = search_constants(2, 3, 5)
    f = default_schedule(2, 3)
    assert (n, b_u, b_r) == (f["n_ir"], f["b_u"], f["b_r"])
