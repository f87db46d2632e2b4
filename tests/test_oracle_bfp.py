"""Pins for the oracle BFP codec (oracle/orc_bfp.c) against an independent exact
formulation written here with Python integers and fractions.

Format: PAPER.md:1246-1249 (blocks sharing one exponent), rounding PAPER.md:846
(round to nearest, ties to even), sign bit included in the width
(PAPER.md:1486); block size 32, exponent rule and layout DESIGN.md R8 / §2.
The exponent is characterised here as "the smallest E >= -127 such that
RNE(max|x| 2^(q-E)) <= 2^q - 1" -- a different statement from the oracle's
ilogb-plus-bump computation, so a mistake in either shows up.
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle as O
from fmg_inputs import codec_vectors


def rne(fr: Fraction) -> int:
    return round(fr)  # Python rounds Fractions half-to-even


def ref_block(x, w):
    q = w - 1
    fx = [Fraction(float(v)) for v in x]
    mx = max(abs(v) for v in fx)
    if mx == 0:
        return -128, [0] * 32
    E = None
    for e in range(-127, 128):
        if rne(mx * Fraction(2) ** (q - e)) <= 2 ** q - 1:
            E = e
            break
    assert E is not None
    return E, [rne(v * Fraction(2) ** (q - E)) for v in fx]


def ref_pack(m, w):
    stream = 0
    for j, mj in enumerate(m):
        stream |= (mj & ((1 << w) - 1)) << (j * w)
    return [(stream >> (32 * k)) & 0xFFFFFFFF for k in range(w)]


@pytest.mark.parametrize("kind", ["smooth", "gauss", "adversarial"])
@pytest.mark.parametrize("w", [2, 3, 4, 5, 6, 8, 13, 21, 32, 33, 40, 54])
def test_encode_matches_exact_definition(kind, w):
    x = codec_vectors(32 * 24, seed=w * 7 + len(kind), kind=kind)
    rc, mant, exps = O.bfp_encode(x, w)
    assert rc == 0
    for b in range(24):
        E, m = ref_block(x[32 * b:32 * b + 32], w)
        assert exps[b] == E
        assert list(mant[b * w:(b + 1) * w]) == ref_pack(m, w)
    rc, y = O.bfp_decode(mant, exps, x.size, w)
    assert rc == 0
    for b in range(24):
        E, m = ref_block(x[32 * b:32 * b + 32], w)
        exp_vals = [float(Fraction(mj) * Fraction(2) ** (E - (w - 1))) for mj in m]
        assert np.array_equal(y[32 * b:32 * b + 32], np.array(exp_vals))


def test_rne_tie_example():
    # 1.01_2 at width 3 (2 significand bits) -> 1.0_2 (tie to even)
    x = np.zeros(32); x[0] = 1.25
    rc, mant, exps = O.bfp_encode(x, 3)
    _, y = O.bfp_decode(mant, exps, 32, 3)
    assert exps[0] == 1 and y[0] == 1.0
    # 1.11_2 * 2^-1 = 0.875 next to max 1.0 at width 3: 0.875*2 = 1.75 -> 2 (up)
    x[1] = 0.875
    rc, mant, exps = O.bfp_encode(x, 3)
    _, y = O.bfp_decode(mant, exps, 32, 3)
    assert y[1] == 1.0


def test_exponent_bump():
    # max rounds up to 2^q at E0: block exponent must bump by one
    w, q = 4, 3
    x = np.zeros(32); x[0] = 2.0 - 2.0 ** -5  # 1.11111b: *2^(3-1) = 7.875 -> 8 = 2^q
    rc, mant, exps = O.bfp_encode(x, w)
    assert exps[0] == 2
    _, y = O.bfp_decode(mant, exps, 32, w)
    assert y[0] == 2.0


def test_powers_of_two_exact_and_zero_block():
    # powers of two within the block's w-1 magnitude bits are exact
    x = np.zeros(64)
    k = np.arange(32) % 5
    x[:32] = np.where(np.arange(32) % 2, 1.0, -1.0) * 2.0 ** (3 - k)
    rc, mant, exps = O.bfp_encode(x, 6)
    _, y = O.bfp_decode(mant, exps, 64, 6)
    assert rc == 0 and np.array_equal(y, x)
    assert exps[1] == -128 and not mant[6:].any()


@pytest.mark.parametrize("w", [2, 4, 6, 12, 30, 54])
def test_roundtrip_half_lsb_bound(w):
    x = codec_vectors(32 * 512, seed=99 + w, kind="smooth")
    rc, mant, exps = O.bfp_encode(x, w)
    _, y = O.bfp_decode(mant, exps, x.size, w)
    bound = np.repeat(2.0 ** (exps.astype(np.float64) - (w - 1) - 1), 32)
    assert np.all(np.abs(y - x) <= bound)


def test_errors():
    x = np.zeros(32); x[3] = np.inf
    assert O.bfp_encode(x, 4)[0] == 2
    x[3] = np.nan
    assert O.bfp_encode(x, 4)[0] == 2
    x[3] = 2.0 ** 200
    assert O.bfp_encode(x, 4)[0] == 2
    assert O.bfp_encode(np.zeros(31), 4)[0] == 1
    assert O.bfp_encode(np.zeros(32), 1)[0] == 1
    assert O.bfp_encode(np.zeros(32), 55)[0] == 1


def test_underflow_saturates():
    x = np.zeros(32); x[0] = 2.0 ** -140; x[1] = 2.0 ** -130
    rc, mant, exps = O.bfp_encode(x, 8)
    assert rc == 0 and exps[0] == -127
    E, m = ref_block(x, 8)
    _, y = O.bfp_decode(mant, exps, 32, 8)
    assert E == -127 and y[1] == 2.0 ** -130 and y[0] == 0.0
