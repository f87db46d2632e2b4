/*
 * orc_bfp.c -- oracle BFP codec.  TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * Follows the block-floating-point format of PAPER.md:1240-1249 ("the vector
 * is divided into few blocks ... only a single exponent scaling all
 * mantissas") with the paper's rounding rule PAPER.md:846 (round to nearest,
 * ties to even; widening appends zero bits) and the sign-bit-included width
 * convention of tab:experiments-params PAPER.md:1486.  Block structure fixed
 * at 32 entries (reading R8); storage layout DESIGN.md §2.
 *
 * Pins (tests/test_oracle_bfp.py): exact rational brute force with Python
 * fractions, RNE tie cases, powers of two, round-trip bound 2^(E-q-1).
 */
#include <math.h>
#include <stdlib.h>
#include <stdint.h>
#include <string.h>
#include "oracle.h"

/* Block encode, R8:
 *   q = w-1; E0 = ilogb(max|x|)+1; E = E0+1 if RNE(max|x| 2^(q-E0)) == 2^q else E0;
 *   E < -127 saturates to -127; E > 127 -> ORC_ERANGE; all-zero block -> E = -128;
 *   m_i = RNE(x_i 2^(q-E)). */
int orc_block_encode(const double* x, int w, int64_t* m, int* E) {
  int q = w - 1;
  double mx = 0.0;
  for (int i = 0; i < 32; ++i) {
    if (!isfinite(x[i])) return ORC_ERANGE;
    double a = fabs(x[i]);
    if (a > mx) mx = a;
  }
  if (mx == 0.0) {
    *E = -128;
    for (int i = 0; i < 32; ++i) m[i] = 0;
    return ORC_OK;
  }
  int e = ilogb(mx) + 1;
  if (rint(ldexp(mx, q - e)) == ldexp(1.0, q)) e = e + 1;
  if (e > 127) return ORC_ERANGE;
  if (e < -127) e = -127;
  *E = e;
  for (int i = 0; i < 32; ++i) m[i] = (int64_t)rint(ldexp(x[i], q - e));
  return ORC_OK;
}

/* Decode one entry: x = m 2^(E-q) (exact; |m| < 2^53). */
double orc_block_decode_one(int64_t m, int E, int w) { return ldexp((double)m, E - (w - 1)); }

/* Bit packing: entry j occupies bits [j w, j w + w) of the
 * block's 32 w-bit stream, two's complement; stream bit k = bit (k mod 32)
 * of word k/32. A block is exactly w words. */
void orc_pack_block(const int64_t* m, int w, uint32_t* words) {
  for (int k = 0; k < w; ++k) words[k] = 0;
  for (int j = 0; j < 32; ++j) {
    uint64_t field = (uint64_t)m[j];
    for (int b = 0; b < w; ++b) {
      if ((field >> b) & 1u) {
        int64_t pos = (int64_t)j * w + b;
        words[pos >> 5] |= (uint32_t)1u << (pos & 31);
      }
    }
  }
}

void orc_unpack_block(const uint32_t* words, int w, int64_t* m) {
  for (int j = 0; j < 32; ++j) {
    uint64_t field = 0;
    for (int b = 0; b < w; ++b) {
      int64_t pos = (int64_t)j * w + b;
      if ((words[pos >> 5] >> (pos & 31)) & 1u) field |= (uint64_t)1 << b;
    }
    /* sign-extend from w bits */
    if ((field >> (w - 1)) & 1u) field |= ~(uint64_t)0 << w;
    m[j] = (int64_t)field;
  }
}

int orc_bfp_encode(const double* x, int64_t n, int width, uint32_t* mant, int8_t* exps) {
  if (width < 2 || width > 54 || n < 0 || (n % 32) != 0) return ORC_EINVAL;
  int64_t m[32];
  for (int64_t b = 0; b < n / 32; ++b) {
    int E;
    int rc = orc_block_encode(x + 32 * b, width, m, &E);
    if (rc) return rc;
    exps[b] = (int8_t)E;
    orc_pack_block(m, width, mant + b * width);
  }
  return ORC_OK;
}

int orc_bfp_decode(const uint32_t* mant, const int8_t* exps, int64_t n, int width, double* x) {
  if (width < 2 || width > 54 || n < 0 || (n % 32) != 0) return ORC_EINVAL;
  int64_t m[32];
  for (int64_t b = 0; b < n / 32; ++b) {
    orc_unpack_block(mant + b * width, width, m);
    for (int j = 0; j < 32; ++j) x[32 * b + j] = orc_block_decode_one(m[j], exps[b], width);
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------------
 * Streaming-exponent BFP (§8(f) row N3): "As the entries
 * of the vector are computed, we keep track of the currently largest known
 * exponent and normalize the current mantissa to that exponent. This exponent
 * and associated mantissas constitute one block of the BFP vector. The next
 * block starts when a larger exponent is encountered. [...] storing only the b
 * largest exponents suffices [...] The other exponents are smaller by at least
 * b compared to the largest exponent. Therefore, those entries would be
 * truncated to zero in single-exponent BFP precision."
 *
 * Readings (R19-R21):
 *   R19 the exponent an entry needs is the block codec's rule applied to that
 *       entry alone: E_i = ilogb|x_i| + 1, plus 1 when RNE(|x_i| 2^(q-E_i))
 *       reaches 2^q; zero entries need no exponent and never start a block;
 *   R20 b = w (the paper's "number of bits in each mantissa", sign included):
 *       an entry whose block exponent is <= X_max - w has |x| < 2^(X_max - w),
 *       i.e. below half a unit of the single-exponent mantissa, so it is stored
 *       as 0;
 *   R21 exponents are int32 in [-1073, 1024] (no int8 saturation); E_i > 1024
 *       (a decode would overflow) and non-finite inputs are ORC_ERANGE;
 *   R22 every mantissa is written once, normalised to the running maximum at
 *       its position; dropping a block discards only its exponent record, and
 *       decoding reads the entries before the first kept block as 0.
 * Output: the packed mantissa stream (same packing as the block codec: entry i
 * at stream bits [i w, i w + w)), the kept blocks' exponents X_k and first
 * indices s_k in increasing order, and their count K' <= w.
 * ------------------------------------------------------------------------ */
#define ORC_NOEXP (-0x40000000)

/* R19: the exponent entry x needs on its own (ORC_NOEXP for zero). */
static int entry_exponent(double x, int q) {
  double a = fabs(x);
  if (a == 0.0) return ORC_NOEXP;
  int e = ilogb(a) + 1;
  if (rint(ldexp(a, q - e)) == ldexp(1.0, q)) e = e + 1;
  return e;
}

int orc_stream_encode(const double* x, int64_t n, int width, uint32_t* mant, int32_t* xexp,
                      int64_t* xstart, int32_t* nblocks) {
  if (width < 2 || width > 54 || n < 0 || (n % 32) != 0) return ORC_EINVAL;
  int q = width - 1;
  /* pass 1 (the paper's stream): running maximum exponent, a block per increase */
  int* M = (int*)malloc(sizeof(int) * (size_t)(n > 0 ? n : 1));
  int64_t cap = 2200, K = 0;
  int32_t* bx = (int32_t*)malloc(sizeof(int32_t) * cap);
  int64_t* bs = (int64_t*)malloc(sizeof(int64_t) * cap);
  if (!M || !bx || !bs) { free(M); free(bx); free(bs); return ORC_ENOMEM; }
  int cur = ORC_NOEXP;
  for (int64_t i = 0; i < n; ++i) {
    if (!isfinite(x[i])) { free(M); free(bx); free(bs); return ORC_ERANGE; }
    int e = entry_exponent(x[i], q);
    if (e > 1024) { free(M); free(bx); free(bs); return ORC_ERANGE; }
    if (e > cur) {       /* "the next block starts when a larger exponent is encountered" */
      cur = e;
      bx[K] = e;         /* K <= 2098 distinct increasing exponents < cap */
      bs[K] = i;
      K = K + 1;
    }
    M[i] = cur;
  }
  /* keep the b = w largest exponents: the last b blocks (exponents increase) */
  int64_t k0 = K > width ? K - width : 0;
  for (int64_t k = k0; k < K; ++k) {
    xexp[k - k0] = bx[k];
    xstart[k - k0] = bs[k];
  }
  *nblocks = (int32_t)(K - k0);
  /* mantissas: each normalised once, to the running maximum at its position
   * ("normalize the current mantissa to that exponent"); those of dropped
   * blocks are not rewritten (R22: no re-normalisation) --
   * the decoder reads every entry before the first kept block as 0 */
  int64_t m[32];
  for (int64_t g = 0; g < n / 32; ++g) {
    for (int j = 0; j < 32; ++j) {
      int64_t i = 32 * g + j;
      m[j] = M[i] == ORC_NOEXP ? 0 : (int64_t)rint(ldexp(x[i], q - M[i]));
    }
    orc_pack_block(m, width, mant + g * width);
  }
  free(M); free(bx); free(bs);
  return ORC_OK;
}

/* x_i = m_i 2^(X_k - q) for the kept block k containing i (s_k <= i < s_{k+1});
 * entries before s_0 are 0. */
int orc_stream_decode(const uint32_t* mant, const int32_t* xexp, const int64_t* xstart, int32_t nblocks,
                      int64_t n, int width, double* x) {
  if (width < 2 || width > 54 || n < 0 || (n % 32) != 0 || nblocks < 0 || nblocks > width) return ORC_EINVAL;
  int q = width - 1;
  int64_t m[32];
  int k = -1;
  for (int64_t g = 0; g < n / 32; ++g) {
    orc_unpack_block(mant + g * width, width, m);
    for (int j = 0; j < 32; ++j) {
      int64_t i = 32 * g + j;
      while (k + 1 < nblocks && xstart[k + 1] <= i) k = k + 1;
      x[i] = k < 0 ? 0.0 : ldexp((double)m[j], xexp[k] - q);
    }
  }
  return ORC_OK;
}
