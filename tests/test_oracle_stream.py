"""Pins for the oracle streaming-exponent BFP codec (oracle/orc_bfp.c,
orc_stream_encode / orc_stream_decode; §8(f) row N3).

Scheme: PAPER.md:1252-1266 -- running-maximum exponent while streaming, a new
block at each increase, only the b largest exponents stored, the rest of the
entries "truncated to zero in single-exponent BFP precision".  Readings R19-R22
(DESIGN.md).  The pins below do not re-state the oracle's loop.  They check it
against:

* a hand-worked example (derivation in the comments);
* the paper's accuracy claim, entry by entry: the streaming encoding is never
  less accurate than single-exponent BFP of the whole vector, which is computed
  here exactly with Python fractions;
* the special case that reduces to single-exponent BFP (largest entry first);
* structural facts: the block count, the block-start positions of a doubling
  sequence, and what is dropped;
* the error and edge cases.
"""
from fractions import Fraction
import math

import numpy as np
import pytest

import oracle as O


def unpack(mant, n, w):
    """Two's-complement w-bit fields, entry i at stream bits [i w, i w + w)."""
    big = 0
    for k, word in enumerate(np.asarray(mant, dtype=np.uint64).tolist()):
        big |= int(word) << (32 * k)
    out = []
    for i in range(n):
        f = (big >> (i * w)) & ((1 << w) - 1)
        out.append(f - (1 << w) if f >> (w - 1) else f)
    return out


def single_exponent_bfp(x, w):
    """One exponent for the whole vector: the smallest E
    with RNE(max|x| 2^(q-E)) <= 2^q - 1; entries RNE(x 2^(q-E)) 2^(E-q)."""
    q = w - 1
    fx = [Fraction(float(v)) for v in x]
    mx = max(abs(v) for v in fx)
    if mx == 0:
        return [Fraction(0)] * len(fx)
    E = math.floor(math.log2(mx)) - 2  # safely below, then walk up
    while round(mx * Fraction(2) ** (q - E)) > 2 ** q - 1:
        E += 1
    return [round(v * Fraction(2) ** (q - E)) * Fraction(2) ** (E - q) for v in fx]


def test_worked_example():
    # w = 4, q = 3 (mantissas -7..7).  Entry exponents (ilogb+1, bump if RNE hits 8):
    #   1 -> 1 (4/8 of 2^1)   3 -> 2   0.5 -> 0   10 -> 4   -7 -> 3   100 -> 7
    # running max 1,2,2,4,4,7 -> blocks (1,@0) (2,@1) (4,@3) (7,@5), K = 4 <= b = 4.
    # mantissas: 1*2^2=4; 3*2^1=6; 0.5*2^1=1; 10*2^-1=5; -7*2^-1=-3.5 -> -4 (even);
    # 100*2^-4=6.25 -> 6.  Decoded: 1, 3, 0.5, 10, -8, 96.
    x = np.zeros(32)
    x[:6] = [1, 3, 0.5, 10, -7, 100]
    rc, mant, xe, xs = O.stream_encode(x, 4)
    assert rc == 0
    assert xe.tolist() == [1, 2, 4, 7] and xs.tolist() == [0, 1, 3, 5]
    assert unpack(mant, 32, 4)[:7] == [4, 6, 1, 5, -4, 6, 0]
    rc, y = O.stream_decode(mant, xe, xs, 32, 4)
    assert rc == 0 and y[:6].tolist() == [1, 3, 0.5, 10, -8, 96] and not y[6:].any()


def test_worked_example_drops_small_blocks():
    # w = 3 (b = 3 exponents kept).  |x| doubles: 1, 2, 4, 8, 16 -> five blocks
    # with exponents 1..5 starting at 0..4; the b = 3 largest are 3, 4, 5 (@2, 3, 4).
    # Entries 0, 1 (exponent <= 5 - 3) are dropped: single-exponent BFP (E = 5,
    # q = 2) stores them as RNE(1/8), RNE(2/8) = 0 too.
    x = np.zeros(32)
    x[:5] = [1, 2, 4, 8, 16]
    rc, mant, xe, xs = O.stream_encode(x, 3)
    assert rc == 0
    assert xe.tolist() == [3, 4, 5] and xs.tolist() == [2, 3, 4]
    # R22: the dropped entries' mantissas stay as written (1 2^(2-1) = 2 and
    # 2 2^(2-2) = 2 at q = 2); only their exponent records are gone
    assert unpack(mant, 32, 3)[:5] == [2, 2, 2, 2, 2]
    rc, y = O.stream_decode(mant, xe, xs, 32, 3)
    assert y[:5].tolist() == [0, 0, 4, 8, 16]
    se = single_exponent_bfp(x, 3)
    assert [float(v) for v in se[:5]] == [0, 0, 0, 8, 16]


def _wide_range(rng, n, decades):
    mag = 10.0 ** rng.uniform(-decades, decades, n)
    x = mag * rng.choice([-1.0, 1.0], n)
    x[rng.random(n) < 0.05] = 0.0
    return x


@pytest.mark.parametrize("w", [2, 3, 4, 5, 8, 13, 24, 33, 53, 54])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_never_less_accurate_than_single_exponent(w, seed):
    # the scheme recovers every entry to at least
    # single-exponent BFP accuracy.  Entry-wise, exactly.
    rng = np.random.default_rng(1000 * w + seed)
    n = 256
    x = _wide_range(rng, n, 6 if seed < 2 else 40)
    if seed == 1:
        x = np.sort(np.abs(x)) * rng.choice([-1.0, 1.0], n)  # increasing: many blocks
    rc, mant, xe, xs = O.stream_encode(x, w)
    assert rc == 0
    rc, y = O.stream_decode(mant, xe, xs, n, w)
    assert rc == 0
    se = single_exponent_bfp(x, w)
    for i in range(n):
        fx = Fraction(float(x[i]))
        assert abs(fx - Fraction(float(y[i]))) <= abs(fx - se[i]), (i, x[i], y[i], float(se[i]))


@pytest.mark.parametrize("w", [3, 6, 17, 54])
def test_largest_first_is_single_exponent_bfp(w):
    # One block when the first entry carries the largest exponent: the scheme
    # then IS single-exponent BFP.
    rng = np.random.default_rng(w)
    x = rng.standard_normal(128)
    x[0] = 4 * np.abs(x).max()
    rc, mant, xe, xs = O.stream_encode(x, w)
    assert rc == 0 and len(xe) == 1 and xs.tolist() == [0]
    rc, y = O.stream_decode(mant, xe, xs, 128, w)
    assert [Fraction(float(v)) for v in y] == single_exponent_bfp(x, w)


@pytest.mark.parametrize("w", [2, 4, 9, 30])
def test_block_structure_doubling_sequence(w):
    # |x_i| = 2^i (i < 60): every entry raises the exponent, K = 60 blocks,
    # the b = w last are kept and start at their own index.
    n = 64
    x = np.zeros(n)
    x[:60] = [2.0 ** i for i in range(60)]
    rc, mant, xe, xs = O.stream_encode(x, w)
    assert rc == 0
    keep = min(w, 60)
    assert xs.tolist() == list(range(60 - keep, 60))
    assert xe.tolist() == [i + 1 for i in range(60 - keep, 60)]
    rc, y = O.stream_decode(mant, xe, xs, n, w)
    assert y[:60 - keep].tolist() == [0.0] * (60 - keep)
    assert y[60 - keep:60].tolist() == x[60 - keep:60].tolist()  # powers of two: exact


def test_block_count_and_dropped_entries_bound():
    rng = np.random.default_rng(7)
    for w in (2, 3, 5, 12):
        x = np.sort(_wide_range(rng, 512, 30))
        x = x * rng.choice([-1.0, 1.0], 512)
        rc, mant, xe, xs = O.stream_encode(x, w)
        assert rc == 0 and 1 <= len(xe) <= w
        assert np.all(np.diff(xe) > 0) and np.all(np.diff(xs) > 0)
        rc, y = O.stream_decode(mant, xe, xs, 512, w)
        xmax = int(xe[-1])
        dropped = np.arange(512) < xs[0]
        # what is not stored is below 2^(X_max - b)
        assert np.all(np.abs(x[dropped]) < 2.0 ** (xmax - w))
        assert not y[dropped].any()
        # the stored block exponent is the running maximum at each start
        for k in range(len(xe)):
            i = int(xs[k])
            assert math.frexp(abs(x[i]))[1] <= xe[k] <= math.frexp(abs(x[i]))[1] + 1


def test_edge_cases():
    # all zero: no block, zeros back
    rc, mant, xe, xs = O.stream_encode(np.zeros(64), 5)
    assert rc == 0 and len(xe) == 0 and not mant.any()
    rc, y = O.stream_decode(mant, xe, xs, 64, 5)
    assert rc == 0 and not y.any()
    # empty input
    rc, mant, xe, xs = O.stream_encode(np.zeros(0), 5)
    assert rc == 0 and len(xe) == 0
    # ragged length is an argument error
    assert O.stream_encode(np.ones(33), 5)[0] == 1
    # non-finite input, and an exponent past 1024 (R21)
    for bad in (np.inf, -np.inf, np.nan):
        x = np.ones(32)
        x[5] = bad
        assert O.stream_encode(x, 5)[0] == 2
    x = np.ones(32)
    x[3] = np.finfo(np.float64).max  # RNE(max 2^(3-1024)) = 8 = 2^q -> E = 1025
    assert O.stream_encode(x, 4)[0] == 2
    assert O.stream_encode(x, 54)[0] == 0  # 53 magnitude bits hold it
    # subnormals alone round-trip exactly (int32 exponents, no saturation)
    x = np.zeros(32)
    x[:4] = [5e-324, -1e-320, 3e-310, 2.5e-308]
    for w in (8, 54):
        rc, mant, xe, xs = O.stream_encode(x, w)
        rc, y = O.stream_decode(mant, xe, xs, 32, w)
        assert rc == 0
        se = single_exponent_bfp(x, w)
        for i in range(32):
            assert abs(Fraction(float(x[i])) - Fraction(float(y[i]))) <= abs(Fraction(float(x[i])) - se[i])
    rc, mant, xe, xs = O.stream_encode(np.array([5e-324] + [0.0] * 31), 2)
    assert xe.tolist() == [-1073] and O.stream_decode(mant, xe, xs, 32, 2)[1][0] == 5e-324


def test_storage_bits():
    # Storage: n w mantissa bits plus at most b exponents and
    # block starts -- O(1) per vector, against n/32 exponents for fixed blocks.
    rng = np.random.default_rng(3)
    n, w = 4096, 5
    x = np.sort(np.abs(_wide_range(rng, n, 50)))
    rc, mant, xe, xs = O.stream_encode(x, w)
    assert rc == 0 and mant.size * 32 == n * w and len(xe) <= w
    bits_stream = n * w + len(xe) * (32 + 64)
    bits_fixed = n * w + (n // 32) * 8
    assert bits_stream < bits_fixed
