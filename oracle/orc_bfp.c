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
