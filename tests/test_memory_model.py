"""Storage accounting (§8(f) row N3; Eq 6.1-6.3):
``fmg_memory_model`` (host-only C ABI call) against the oracle's actual
section storage, the paper's Eq 6.1 inequality with its printed constants
(tests/golden/table3_poisson.json), and the sub-linear
temporaries of Eq 6.2/6.3."""
import json
import os

import numpy as np
import pytest

import oracle as O
from fmg_inputs import CONFIGS, default_schedule

P = pytest.importorskip("paper_2511_19036_b200")
GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "table3_poisson.json")))


@pytest.mark.parametrize("d,p,lv", [(2, 1, 6), (2, 2, 5), (2, 3, 4), (3, 1, 4), (3, 2, 3)])
def test_stored_bits_equal_oracle_sections(d, p, lv):
    """The model's stored mantissa and exponent bits are exactly what the
    oracle holds after a solve (its sections have the same padded layout)."""
    s = O.schedule(d, p)
    c = O.CFMG(d, p, lv, s)
    c.solve()
    um = sum(c.section(0, l)[0].size * 32 for l in range(lv))
    rm = sum(c.section(1, l)[0].size * 32 for l in range(lv))
    ex = sum((c.section(0, l)[1].size + c.section(1, l)[1].size) * 8 for l in range(lv))
    m = P.memory_model(d, p, lv, default_schedule(d, p))
    assert (m["u_mantissa_bits"], m["r_mantissa_bits"], m["exponent_bits_fixed"]) == (um, rm, ex)
    assert m["section_bytes"] == um / 8 + rm / 8 + ex / 8


@pytest.mark.parametrize("cfg", sorted(CONFIGS))
@pytest.mark.parametrize("k", [None, 0, 3])
def test_eq61_inequality(cfg, k):
    """Eq 6.1: sum_l (k(L-l)+b) n_l < (2^d/(2^d-1) b + 2^d/(2^d-1)^2 k) n_L with
    the constants the paper prints (2, 4/3, 8/7)."""
    c = CONFIGS[cfg]
    d, p, lv = c["dim"], c["p"], c["levels"]
    s = default_schedule(d, p)
    if k is not None:
        s["k_u"] = k
        s["k_r"] = k
        if s["b_u"] + k * (lv - 1) > 54 or s["b_r"] + k * (lv - 1) > 54:
            pytest.skip("width above 54")
    m = P.memory_model(d, p, lv, s)
    const = GOLD["storage_constants"][str(d)]
    L = lv - 1
    n = [(p * 2 ** (l + 1) - 1) ** d for l in range(L + 1)]
    assert m["unknowns"] == n[L]
    assert m["eq61_u"] == sum(n[l] * (s["b_u"] + s["k_u"] * (L - l)) for l in range(L + 1))
    assert m["eq61_u_bound"] == pytest.approx((const * s["b_u"] + const / (2 ** d - 1) * s["k_u"]) * n[L],
                                              rel=1e-12)
    assert m["eq61_u"] < m["eq61_u_bound"] and m["eq61_r"] < m["eq61_r_bound"]
    # stored (padded rows, boundary planes) is at least the unknown count
    assert m["u_mantissa_bits"] >= m["eq61_u"]


@pytest.mark.parametrize("d", [2, 3])
def test_eq61_constant_is_approached(d):
    """With k = 0 the ratio sum_l n_l / n_L tends to 2^d/(2^d-1) from below
    (PAPER.md:1207-1208)."""
    s = default_schedule(d, 1)
    s["k_u"] = 0
    const = GOLD["storage_constants"][str(d)]
    prev = 0.0
    for lv in range(4, 12 if d == 2 else 10):
        m = P.memory_model(d, 1, lv, s)
        ratio = m["eq61_u"] / (s["b_u"] * m["unknowns"])
        assert prev < ratio < const
        prev = ratio
    assert ratio > const * (1 - 2e-3)


@pytest.mark.parametrize("cfg", ["C2", "C3", "C4", "C5"])
def test_exponents_and_temporaries_sublinear(cfg):
    """Streaming exponents (N3) cost O(w) bits per section, far below one
    exponent per 32 entries; the streaming-window temporaries of Eq 6.2/6.3
    are o(n_L) bits, while this implementation's FP64 temporaries are
    Theta(n_L) bytes."""
    c = CONFIGS[cfg]
    d, p, lv = c["dim"], c["p"], c["levels"]
    m = P.memory_model(d, p, lv)
    n = m["unknowns"]
    assert m["exponent_bits_streaming"] < 0.01 * m["exponent_bits_fixed"]
    assert m["eq63_z_bits"] <= m["eq62_ut_bits"] / 2 + 1e-9
    assert m["eq62_ut_bits"] / n < 0.2 * (m["u_mantissa_bits"] / n)
    # hand count of the FP64 arrays create_impl allocates (stored points per level)
    st = [(((p << (l + 1)) + 31) // 32 * 32) * (p << (l + 1)) ** (d - 1) for l in range(lv)]
    L = lv - 1
    k = default_schedule(d, p)["cheb_degree"]
    if d == 3 and k in (2, 3):  # finest-level kernels (lean): t_L (+ d_2 for degree 3); u, t, w below; Z, PU at L-1
        want = st[L] * (1 + (k >= 3)) + 3 * sum(st[:L]) + 2 * st[L - 1] + st[0]
    else:                       # level-by-level kernels: u, t, w per level, six finest-size scratch arrays
        want = 3 * sum(st) + 6 * st[L]
    assert m["fp64_temporary_bytes"] == 8 * want
    assert m["fp64_temporary_bytes"] >= 8 * n


def test_memory_model_rejects_bad_arguments():
    s = P.Schedule.from_dict(default_schedule(2, 2))
    out = np.zeros(P.FMG_MEM_COUNT if hasattr(P, "FMG_MEM_COUNT") else 13)
    import ctypes as C
    lib = P._lib
    dp = C.POINTER(C.c_double)
    assert lib.fmg_memory_model(4, 2, 5, C.byref(s), out.ctypes.data_as(dp), 13) == 1
    assert lib.fmg_memory_model(2, 2, 5, C.byref(s), out.ctypes.data_as(dp), 12) == 1
    assert lib.fmg_memory_model(2, 2, 5, None, out.ctypes.data_as(dp), 13) == 1


def test_c5_fits_eight_gpus_per_rank():
    """C5 (4096^3 Q1, 12 levels) at 8 GPUs: with the z-slab memory partition
    (a rank holds NZ_l / G planes + 2p ghost planes each side of
    every level array and section) and the finest-level kernels (DESIGN.md
    §4.3), one rank's device bytes fit a 180 GB B200.  Hand count of the
    allocations in create_impl, every level partitioned (the replicated
    coarse levels are a few MB)."""
    c = CONFIGS["C5"]
    d, p, lv = c["dim"], c["p"], c["levels"]
    G, L = 8, lv - 1
    sch = default_schedule(d, p)
    tot = 0
    for l in range(lv):
        n = p << (l + 1)
        NX = (n + 31) // 32 * 32
        planes = min(n, n // G + 4 * p)
        plane = NX * n
        arrays = 1 if l == L else 3                      # t_L; u, t, w below
        arrays += 2 if l == L - 1 else 0                 # Z, PU scratch
        tot += 8 * plane * planes * arrays
        wu, wr = sch["b_u"] + sch["k_u"] * (L - l), sch["b_r"] + sch["k_r"] * (L - l)
        tot += (plane // 32) * planes * (4 * (wu + wr) + 2)  # section words + exponents
    assert tot < 180e9 * 0.9, tot / 1e9
