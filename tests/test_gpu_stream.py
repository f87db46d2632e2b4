"""GPU parity of the streaming-exponent BFP codec (§8(f) row N3,
PAPER.md:1252-1266) against the oracle (oracle/orc_bfp.c orc_stream_*):
bit-exact mantissa stream, block table and decoded values."""
import numpy as np
import pytest

import oracle as O
from fmg_inputs import codec_vectors

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2511_19036_b200 as P
    return P


def _check(P, x, w):
    n = x.size
    rc, m_ref, e_ref, s_ref = O.stream_encode(x, w)
    assert rc == 0
    xt = torch.from_numpy(x).cuda()
    mant, xexp, xstart, nb = P.bfp_stream_encode(xt, w)
    assert P.bfp_status() == 0
    k = int(nb.item())
    assert k == len(e_ref)
    assert np.array_equal(xexp.cpu().numpy()[:k], e_ref)
    assert np.array_equal(xstart.cpu().numpy()[:k], s_ref)
    assert np.array_equal(mant.cpu().numpy().view(np.uint32), m_ref)
    y = P.bfp_stream_decode(mant, xexp, xstart, nb, n, w)
    _, y_ref = O.stream_decode(m_ref, e_ref, s_ref, n, w)
    assert np.array_equal(y.cpu().numpy().view(np.uint64), y_ref.view(np.uint64))


@pytest.mark.parametrize("kind", ["smooth", "gauss", "adversarial", "staircase"])
@pytest.mark.parametrize("w", [2, 3, 4, 5, 7, 8, 9, 13, 24, 32, 33, 53, 54])
def test_stream_codec_bit_exact(P, kind, w):
    n = 32 * 4099  # 16 CTA chunks of 256 groups + a ragged chunk
    _check(P, codec_vectors(n, seed=2000 + w, kind=kind), w)


@pytest.mark.parametrize("w", [2, 5, 54])
def test_stream_codec_small_and_degenerate(P, w):
    rng = np.random.default_rng(w)
    _check(P, rng.standard_normal(32), w)                   # one group
    _check(P, np.zeros(32 * 300), w)                        # no block at all
    x = np.zeros(32 * 300)
    x[-1] = -3.0                                            # one block at the very end
    _check(P, x, w)
    x = np.zeros(32 * 600)
    x[:60] = [2.0 ** i for i in range(60)]                  # 60 blocks in two groups
    x[32 * 256 + 5] = 2.0 ** 70                             # + one in the second CTA chunk
    _check(P, x, w)
    x = np.ldexp(np.ones(32 * 257), -1074)                  # subnormal-only vector
    _check(P, x, w)
    x = np.arange(32 * 513, dtype=np.float64)[::-1].copy()  # largest first: one block
    _check(P, x, w)


def test_stream_codec_empty_and_errors(P):
    mant, xexp, xstart, nb = P.bfp_stream_encode(torch.zeros(0, dtype=torch.float64, device="cuda"), 4)
    assert mant.numel() == 0 and int(nb.item()) == 0
    x = torch.ones(64, dtype=torch.float64, device="cuda")
    x[7] = float("nan")
    P.bfp_stream_encode(x, 4)
    assert P.bfp_status() == P.FMG_ERANGE
    assert P.bfp_status() == 0
    x[7] = np.finfo(np.float64).max  # E = 1025 at w = 4 (R21)
    P.bfp_stream_encode(x, 4)
    assert P.bfp_status() == P.FMG_ERANGE
    P.bfp_stream_encode(x, 54)
    assert P.bfp_status() == 0


@pytest.mark.parametrize("w", [4, 8])
def test_stream_codec_large(P, w):
    """2^26 entries (8192 CTA chunks; the scan's chunk loop runs 8 rounds)."""
    n = 1 << 26
    _check(P, codec_vectors(n, seed=77 + w, kind="staircase"), w)
