// fmg_device.cuh -- device-side helpers shared by the sm_100a kernels of the
// compact-FMG hot path (fmg_kernels.cu: grid tile ops; fmg_kc.cu: the cluster
// kernel of the coarse levels): BFP codec (RNE PAPER.md:846),
// cp.async / PDL helpers and the device context.  Product path only.
#pragma once
#include <cstdint>
#include <cstdio>
#include <cstring>

#include "fmg_internal.h"

namespace fmg {

constexpr unsigned FULL = 0xffffffffu;
constexpr int NWARP = 8;
constexpr int NT = 32 * NWARP;

__device__ __forceinline__ double pow2(int k) {  // exact 2^k, k in [-1022, 1023]
  return __longlong_as_double((long long)(k + 1023) << 52);
}
__device__ __forceinline__ bool unk1(int i, int n) { return i >= 1 && i <= n - 1; }
__device__ __forceinline__ int floordiv(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// cp.async (LDGSTS) helpers: every global load of a tile is issued up front and
// awaited once; out-of-range elements are zero-filled (src-size 0).
__device__ __forceinline__ void cpa8(double* dst, const double* src, bool ok) {
  unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(src), "r"(ok ? 8 : 0) : "memory");
}
__device__ __forceinline__ void cpa4(uint32_t* dst, const uint32_t* src) {
  unsigned s = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(src) : "memory");
}
__device__ __forceinline__ void cpa_wait_sync() {
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();
}

// ------------------------------------------------------------------ TMA --
// Tensor-map (cp.async.bulk.tensor) staging with mbarrier completion: one
// elected thread arms the slot's barrier with the box bytes and issues the
// copy; out-of-range box elements are zero-filled by the hardware (the march
// kernels' "zero outside the stored level").  The map is a __grid_constant__
// kernel parameter (MArgs::tm).
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// order this thread's generic-proxy shared accesses before a following TMA write
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n.reg .pred P1;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, int x, int y, unsigned long long* bar,
                                            unsigned bytes) {
  unsigned long long st;
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 %0, [%1], %2;"
               : "=l"(st)
               : "r"(smem_u32(bar)), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(smem_u32(dst)),
      "l"((unsigned long long)tmap), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(void* dst, const void* tmap, int x, int y, int z,
                                            unsigned long long* bar, unsigned bytes) {
  unsigned long long st;
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 %0, [%1], %2;"
               : "=l"(st)
               : "r"(smem_u32(bar)), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
      "[%5];" ::"r"(smem_u32(dst)),
      "l"((unsigned long long)tmap), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

// ----------------------------------------------------------------- codec --
// Exact int -> double for |m| < 2^31 by the 1.5*2^52 magic constant (an FP64
// add instead of an I2F conversion); wider mantissas use the conversion.
__device__ __forceinline__ double i2d(long long m, int w) {
  if (w <= 32) return __longlong_as_double(0x4338000000000000LL + m) - 6755399441055744.0;
  return (double)m;
}
// RNE of x to an integer for |x| < 2^31 (x + 1.5*2^52 rounds to nearest even at
// integer granularity; the low word is the two's-complement result).
__device__ __forceinline__ long long rne_int(double x, int w) {
  if (w <= 32) return (long long)(int)__double2loint(x + 6755399441055744.0);
  return (long long)rint(x);
}

// Warp-cooperative unpack: lane j returns the w-bit two's-complement mantissa
// of entry j of the 32-entry group whose w words start at `words` (DESIGN.md
// §2).  All 32 lanes must call.
__device__ __forceinline__ long long warp_unpack(const uint32_t* words, int w, int lane) {
  uint32_t my0 = lane < w ? words[lane] : 0u;
  uint32_t my1 = 0u;
  if (w > 32) my1 = lane + 32 < w ? words[lane + 32] : 0u;
  int o = lane * w, j0 = o >> 5, s = o & 31;
  uint32_t w0, w1, w2;
  if (w <= 32) {
    w0 = __shfl_sync(FULL, my0, j0 & 31);
    w1 = __shfl_sync(FULL, my0, (j0 + 1) & 31);
    w2 = __shfl_sync(FULL, my0, (j0 + 2) & 31);
  } else {
    uint32_t a0 = __shfl_sync(FULL, my0, j0 & 31), b0 = __shfl_sync(FULL, my1, j0 & 31);
    uint32_t a1 = __shfl_sync(FULL, my0, (j0 + 1) & 31), b1 = __shfl_sync(FULL, my1, (j0 + 1) & 31);
    uint32_t a2 = __shfl_sync(FULL, my0, (j0 + 2) & 31), b2 = __shfl_sync(FULL, my1, (j0 + 2) & 31);
    w0 = j0 < 32 ? a0 : b0;
    w1 = j0 + 1 < 32 ? a1 : b1;
    w2 = j0 + 2 < 32 ? a2 : b2;
  }
  unsigned long long lo = (unsigned long long)w0 | ((unsigned long long)w1 << 32);
  unsigned long long field = lo >> s;
  if (s + w > 64) field |= (unsigned long long)w2 << (64 - s);
  return (long long)(field << (64 - w)) >> (64 - w);
}

// Warp-cooperative decode: lane j returns entry j of the block whose w words
// start at `words`.  All 32 lanes must call.
__device__ __forceinline__ double warp_decode(const uint32_t* words, int E, int w, int lane) {
  return i2d(warp_unpack(words, w, lane), w) * pow2(E - (w - 1));
}
// The same with a compile-time width W <= 32, the words in SHARED memory:
// lane j loads the one or two words holding its field directly (broadcast
// loads, no shuffles; the field never reaches a third word for W <= 32).
// Bit-identical to warp_decode.
template <int W>
__device__ __forceinline__ double warp_decode_w(const uint32_t* words, int E, int lane) {
  static_assert(W >= 1 && W <= 32, "compile-time widths <= 32");
  const int o = lane * W, j0 = o >> 5, s = o & 31;
  unsigned long long field;
  if (32 % W == 0) {
    field = words[j0] >> s;
  } else {  // (j0 + 1 <= W: the exponent word at most, whose bits the shift drops)
    field = ((unsigned long long)words[j0] | ((unsigned long long)words[j0 + 1] << 32)) >> s;
  }
  const long long m = (long long)(field << (64 - W)) >> (64 - W);
  return i2d(m, W) * pow2(E - (W - 1));
}

// Single-entry decode (entry j of a block), for halo points.
__device__ __forceinline__ double point_decode(const uint32_t* words, int E, int w, int j) {
  int o = j * w, j0 = o >> 5, s = o & 31;
  int jl = (o + w - 1) >> 5;
  unsigned long long lo = words[j0];
  if (jl > j0) lo |= (unsigned long long)words[j0 + 1] << 32;
  unsigned long long field = lo >> s;
  if (jl > j0 + 1) field |= (unsigned long long)words[j0 + 2] << (64 - s);
  long long m = (long long)(field << (64 - w)) >> (64 - w);
  return i2d(m, w) * pow2(E - (w - 1));
}

// Packed words of a narrow block (w = W <= 8): lane j returns word j (j < W).
template <int W>
__device__ __forceinline__ uint32_t pack_narrow(unsigned long long field, int lane) {
  const int p = lane * W, j0 = p >> 5;
  const unsigned long long cf = field << (p & 31);
  const uint32_t c0 = (uint32_t)cf, c1 = (uint32_t)(cf >> 32);
  uint32_t mine = 0u;
#pragma unroll
  for (int j = 0; j < W; ++j) {
    const uint32_t word = __reduce_or_sync(FULL, j == j0 ? c0 : (j == j0 + 1 ? c1 : 0u));
    mine = lane == j ? word : mine;
  }
  return mine;
}

// Warp-cooperative pack: lane j holds the masked w-bit field of entry j; the
// group's w words are written to `words`.  All lanes must call.
__device__ __forceinline__ void warp_pack(unsigned long long field, int w, uint32_t* words, int lane) {
  uint32_t mine0 = 0u, mine1 = 0u;
  if (w <= 8) {
    // narrow: entry `lane` occupies stream bits [lane w, lane w + w) = (low, high)
    // parts of words j0, j0 + 1; one redux.or per output word (width-specialised)
    switch (w) {
      case 2: mine0 = pack_narrow<2>(field, lane); break;
      case 3: mine0 = pack_narrow<3>(field, lane); break;
      case 4: mine0 = pack_narrow<4>(field, lane); break;
      case 5: mine0 = pack_narrow<5>(field, lane); break;
      case 6: mine0 = pack_narrow<6>(field, lane); break;
      case 7: mine0 = pack_narrow<7>(field, lane); break;
      default: mine0 = pack_narrow<8>(field, lane); break;
    }
  } else {
    // wide: word j gathers its <= ceil(32/w)+1 entries by shuffles
    const int K = (32 + w - 1) / w + 1;
    const uint32_t flo = (uint32_t)field, fhi = (uint32_t)(field >> 32);
#pragma unroll 1
    for (int half = 0; half < (w > 32 ? 2 : 1); ++half) {
      const int j = lane + 32 * half;
      const int e0 = (32 * j) / w;
      uint32_t acc = 0u;
#pragma unroll
      for (int k = 0; k < 5; ++k) {  // K <= 5 for w >= 9
        if (k >= K) break;
        const int e = e0 + k;
        const int src = e < 32 ? e : 31;
        const uint32_t lo_ = __shfl_sync(FULL, flo, src), hi_ = __shfl_sync(FULL, fhi, src);
        const unsigned long long f = ((unsigned long long)hi_ << 32) | lo_;
        const int sh = e * w - 32 * j;
        if (e < 32 && sh < 32 && sh > -w) acc |= sh >= 0 ? (uint32_t)(f << sh) : (uint32_t)(f >> (-sh));
      }
      if (half == 0) mine0 = acc; else mine1 = acc;
    }
  }
  if (lane < w) words[lane] = mine0;
  if (lane + 32 < w) words[lane + 32] = mine1;
}

// Warp-cooperative encode of one block; lane j holds entry j.
// Writes the w words and the exponent when `words` is non-null; returns the
// quantised value m 2^(E-q).  Non-finite input or E > 127 sets *status.
__device__ __forceinline__ double warp_encode(double v, int w, uint32_t* words, int8_t* eptr, int lane,
                                              int* status, long long* mout = nullptr, int* Eout = nullptr) {
  unsigned long long bits = (unsigned long long)__double_as_longlong(v) & 0x7fffffffffffffffULL;
  const unsigned hi = (unsigned)(bits >> 32);
  const unsigned mh = __reduce_max_sync(FULL, hi);
  // The exponent needs only the maximum's high word; its bump test
  //   RNE(mx 2^(q-E0)) == 2^q  <=>  frac(mx) >= 2^52 - 2^(52-q)   (mx normal; never for q = 53)
  // is monotone in the bits, so it holds for the maximum iff it holds for some
  // lane carrying the maximal high word: one redux and three independent
  // ballots instead of two dependent reduxes.
  const int q = w - 1;
  const unsigned long long thr = q <= 52 ? (1ULL << 52) - (1ULL << (52 - q)) : ~0ULL;
  const unsigned vbad = __ballot_sync(FULL, bits >= 0x7ff0000000000000ULL);
  const unsigned vnz = __ballot_sync(FULL, bits != 0ULL);
  const unsigned vbump = __ballot_sync(FULL, hi == mh && (bits & 0x000fffffffffffffULL) >= thr);
  bool err = vbad != 0u;
  int E = -128;
  if (!err && vnz != 0u) {
    int ebits = (int)((mh >> 20) & 0x7FFu);
    int E0 = ebits == 0 ? -1100 : ebits - 1022;  // ilogb(mx) + 1; subnormal max -> saturates below
    if (E0 > 127) {
      err = true;
    } else if (E0 < -127) {
      E = -127;
    } else {
      E = E0 + (vbump != 0u ? 1 : 0);
      if (E > 127) err = true;
    }
  }
  long long m = 0;
  if (err) {
    E = -128;
    if (lane == 0 && status) atomicOr(status, 1);
  } else if (E != -128) {
    m = rne_int(v * pow2(q - E), w);
  }
  if (words) {
    warp_pack((unsigned long long)m & ((1ULL << w) - 1ULL), w, words, lane);
    if (lane == 0) *eptr = (int8_t)E;
  }
  if (mout) {  // (the mantissa and exponent themselves: k_f3_cheb's FIN = 2 mode)
    *mout = m;
    *Eout = E;
  }
  return E == -128 ? 0.0 : i2d(m, w) * pow2(E - q);
}

// ------------------------------------------------- thread-per-block codec --
// One THREAD encodes / decodes one whole 32-entry block held in shared memory
// (a warp handles 32 blocks per instruction stream), so the exponent search
// is a serial max and the packing a running 64-bit bit accumulator: about 13
// warp instructions per block against ~100 for the warp-cooperative codec
// above.  Same format and arithmetic (R8, §3.8); w <= 32 only.
// `row`: the block's 32 doubles in shared memory (callers pad the row stride
// to an odd number of doubles so the 32 lanes' rows fall in distinct banks);
// `wrow`: its w packed words (callers pad the row stride to w + 1 words).

// Exponent of one block (R8): E = -128 for an all-zero block; *bad on a
// non-finite entry or E > 127.
// E from the block's largest |x| bit pattern mx (R8; see tpb_exponent).
__device__ __forceinline__ int tpb_exp_of_max(unsigned long long mx, int w, bool& bad) {
  if (mx >= 0x7ff0000000000000ULL) { bad = true; return -128; }
  if (mx == 0ULL) return -128;
  const int q = w - 1;
  const int ebits = (int)(mx >> 52);
  const int E0 = ebits == 0 ? -1100 : ebits - 1022;
  if (E0 > 127) { bad = true; return -128; }
  if (E0 < -127) return -127;
  int E = E0;
  if (rint(__longlong_as_double((long long)mx) * pow2(q - E0)) == pow2(q)) E = E0 + 1;
  if (E > 127) { bad = true; return -128; }
  return E;
}
__device__ __forceinline__ int tpb_exponent(const double* row, int w, bool& bad) {
  unsigned long long mx = 0ULL;
#pragma unroll 8
  for (int e = 0; e < 32; ++e) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(row[e]) & 0x7fffffffffffffffULL;
    mx = b > mx ? b : mx;
  }
  return tpb_exp_of_max(mx, w, bad);
}

// One pass of the correction (S9 + S10 on one block): row holds y_k; with
// the ý exponent Ey, row[e] <- dec ú_e + enc_{wr}(y_e) (the sum the ú encode
// takes, same operands and order as tpb_quant + tpb_unpack_add); returns the
// largest |sum| bit pattern for tpb_exp_of_max.
__device__ __forceinline__ unsigned long long tpb_quant_add(double* row, int Ey, int wr, const uint32_t* wrow, int Eu,
                                                            int wu) {
  const int q = wr - 1;
  const double s = Ey == -128 ? 0.0 : pow2(q - Ey);
  const double sbq = Ey == -128 ? 0.0 : pow2(Ey - q);
  const double sbu = Eu == -128 ? 0.0 : pow2(Eu - (wu - 1));
  unsigned long long acc = 0ULL, mx = 0ULL;
  int nb = 0, k = 0;
#pragma unroll 4
  for (int e = 0; e < 32; ++e) {
    if (nb < wu) {
      acc |= (unsigned long long)wrow[k++] << nb;
      nb += 32;
    }
    const long long m = (long long)(acc << (64 - wu)) >> (64 - wu);
    acc >>= wu;
    nb -= wu;
    const double yq = i2d(rne_int(row[e] * s, wr), wr) * sbq;
    const double v = i2d(m, wu) * sbu + yq;
    row[e] = v;
    const unsigned long long b = (unsigned long long)__double_as_longlong(v) & 0x7fffffffffffffffULL;
    mx = b > mx ? b : mx;
  }
  return mx;
}

// Quantise and pack one block with exponent E (E = -128: zeros).  When
// `qrow` is non-null the decoded value m 2^(E-q) of entry e is stored to
// qrow[e] (qrow may alias row).
__device__ __forceinline__ void tpb_pack(const double* row, int E, int w, uint32_t* wrow, double* qrow) {
  const int q = w - 1;
  const double s = E == -128 ? 0.0 : pow2(q - E);
  const double sb = E == -128 ? 0.0 : pow2(E - q);
  const unsigned long long mask = (1ULL << w) - 1ULL;
  unsigned long long acc = 0ULL;
  int nb = 0, k = 0;
#pragma unroll 4
  for (int e = 0; e < 32; ++e) {
    const long long m = rne_int(row[e] * s, w);
    if (qrow) qrow[e] = i2d(m, w) * sb;
    acc |= ((unsigned long long)m & mask) << nb;
    nb += w;
    if (nb >= 32) {
      wrow[k++] = (uint32_t)acc;
      acc >>= 32;
      nb -= 32;
    }
  }
}

// Quantise one block in place with exponent E (E = -128: zeros): row[e] =
// m 2^(E-q), the value warp_encode returns, without packing.
__device__ __forceinline__ void tpb_quant(double* row, int E, int w) {
  const int q = w - 1;
  const double s = E == -128 ? 0.0 : pow2(q - E);
  const double sb = E == -128 ? 0.0 : pow2(E - q);
#pragma unroll 8
  for (int e = 0; e < 32; ++e) row[e] = i2d(rne_int(row[e] * s, w), w) * sb;
}

// row[e] = dec(entry e) + row[e] (the unpack of tpb_unpack, added in place).
__device__ __forceinline__ void tpb_unpack_add(const uint32_t* wrow, int E, int w, double* row) {
  const double sb = E == -128 ? 0.0 : pow2(E - (w - 1));
  unsigned long long acc = 0ULL;
  int nb = 0, k = 0;
#pragma unroll 4
  for (int e = 0; e < 32; ++e) {
    if (nb < w) {
      acc |= (unsigned long long)wrow[k++] << nb;
      nb += 32;
    }
    const long long m = (long long)(acc << (64 - w)) >> (64 - w);
    acc >>= w;
    nb -= w;
    row[e] = i2d(m, w) * sb + row[e];
  }
}

// Unpack and scale one block into row[0..32).
__device__ __forceinline__ void tpb_unpack(const uint32_t* wrow, int E, int w, double* row) {
  const double sb = E == -128 ? 0.0 : pow2(E - (w - 1));
  unsigned long long acc = 0ULL;
  int nb = 0, k = 0;
#pragma unroll 4
  for (int e = 0; e < 32; ++e) {
    if (nb < w) {
      acc |= (unsigned long long)wrow[k++] << nb;
      nb += 32;
    }
    const long long m = (long long)(acc << (64 - w)) >> (64 - w);
    acc >>= w;
    nb -= w;
    row[e] = i2d(m, w) * sb;
  }
}

// ---- compile-time-width lane routines (W <= 32): every bit position of the
// packed stream is a constant, the 32 entries are unrolled, the words live in
// registers.  Same arithmetic as the runtime-width routines above.
__device__ __forceinline__ double i2d32(int m) {  // exact int -> double (the 1.5 2^52 magic)
  return __longlong_as_double(0x4338000000000000LL + (long long)m) - 6755399441055744.0;
}
__device__ __forceinline__ int rne32(double x) { return (int)__double2loint(x + 6755399441055744.0); }
__device__ __forceinline__ unsigned long long absbits(double v) {
  return (unsigned long long)__double_as_longlong(v) & 0x7fffffffffffffffULL;
}
template <int W>
__device__ __forceinline__ int tpb_field(const uint32_t (&wv)[W], int e) {  // entry e (e constant after unrolling)
  const int p = e * W, j0 = p >> 5, sh = p & 31;
  uint32_t f = wv[j0] >> sh;
  if (sh + W > 32) f |= wv[j0 + 1] << (32 - sh);
  return (int)(f << (32 - W)) >> (32 - W);
}
template <int W>
__device__ __forceinline__ void tpb_put(uint32_t (&ov)[W], int e, int m) {
  const int p = e * W, j0 = p >> 5, sh = p & 31;
  const uint32_t f = (uint32_t)m & (W == 32 ? 0xffffffffu : ((1u << W) - 1u));
  ov[j0] |= f << sh;
  if (sh + W > 32) ov[j0 + 1] |= f >> (32 - sh);
}
// Encode one block (row: 32 values) at width W with exponent E: the words to
// wout, the quantised values to qrow (may alias row, may be null).
template <int W>
__device__ __forceinline__ void tpb_pack_w(const double* row, int E, uint32_t* wout, double* qrow) {
  const double s = E == -128 ? 0.0 : pow2(W - 1 - E);
  const double sb = E == -128 ? 0.0 : pow2(E - (W - 1));
  uint32_t ov[W];
#pragma unroll
  for (int j = 0; j < W; ++j) ov[j] = 0u;
#pragma unroll
  for (int e = 0; e < 32; ++e) {
    const int m = rne32(row[e] * s);
    if (qrow) qrow[e] = i2d32(m) * sb;
    tpb_put<W>(ov, e, m);
  }
#pragma unroll
  for (int j = 0; j < W; ++j) wout[j] = ov[j];
}
// The correction of one block (k_f3_tpb<1>, no w_l): row holds y_k; ý =
// enc_{WR}(y), row <- enc_{W}(dec ú + ý) (values), the new words to wout;
// returns the new exponent.  The operand order of tpb_quant_add / tpb_pack.
template <int W, int WR>
__device__ __forceinline__ int tpb_correct_w(double* row, const uint32_t* win, int Eu, uint32_t* wout, bool& bad) {
  unsigned long long mx = 0ULL;
#pragma unroll
  for (int e = 0; e < 32; ++e) {
    const unsigned long long b = absbits(row[e]);
    mx = b > mx ? b : mx;
  }
  const int Ey = tpb_exp_of_max(mx, WR, bad);
  const double s = Ey == -128 ? 0.0 : pow2(WR - 1 - Ey);
  const double sbq = Ey == -128 ? 0.0 : pow2(Ey - (WR - 1));
  const double sbu = Eu == -128 ? 0.0 : pow2(Eu - (W - 1));
  uint32_t wv[W];
#pragma unroll
  for (int j = 0; j < W; ++j) wv[j] = win[j];
  unsigned long long m2 = 0ULL;
#pragma unroll
  for (int e = 0; e < 32; ++e) {
    const double yq = i2d32(rne32(row[e] * s)) * sbq;
    const double v = i2d32(tpb_field<W>(wv, e)) * sbu + yq;
    row[e] = v;
    const unsigned long long b = absbits(v);
    m2 = b > m2 ? b : m2;
  }
  const int En = tpb_exp_of_max(m2, W, bad);
  tpb_pack_w<W>(row, En, wout, row);
  return En;
}

// The correction of one block from ý given as mantissas (int8, the k_f3_cheb
// FIN = 2 store) and its exponent Ey: row <- enc_{W}(dec ú + ý) values are
// not kept; the new words to wout; returns the new exponent.  Same operands
// and order as tpb_correct_w (ý = m 2^(Ey - q_r) is what warp_encode returns).
template <int W, int WR>
__device__ __forceinline__ int tpb_correct_m(const int8_t* my, int Ey, const uint32_t* win, int Eu, uint32_t* wout,
                                             bool& bad) {
  const double sbq = Ey == -128 ? 0.0 : pow2(Ey - (WR - 1));
  const double sbu = Eu == -128 ? 0.0 : pow2(Eu - (W - 1));
  uint32_t wv[W];
#pragma unroll
  for (int j = 0; j < W; ++j) wv[j] = win[j];
  int4 q0 = *(const int4*)my, q1 = *(const int4*)(my + 16);
  const int8_t* mb0 = (const int8_t*)&q0;
  const int8_t* mb1 = (const int8_t*)&q1;
  double v[32];
  unsigned long long m2 = 0ULL;
#pragma unroll
  for (int e = 0; e < 32; ++e) {
    const int mq = e < 16 ? (int)mb0[e] : (int)mb1[e - 16];
    const double yq = i2d32(mq) * sbq;
    v[e] = i2d32(tpb_field<W>(wv, e)) * sbu + yq;
    const unsigned long long b = absbits(v[e]);
    m2 = b > m2 ? b : m2;
  }
  const int En = tpb_exp_of_max(m2, W, bad);
  const double s = En == -128 ? 0.0 : pow2(W - 1 - En);
  uint32_t ov[W];
#pragma unroll
  for (int j = 0; j < W; ++j) ov[j] = 0u;
#pragma unroll
  for (int e = 0; e < 32; ++e) tpb_put<W>(ov, e, rne32(v[e] * s));
#pragma unroll
  for (int j = 0; j < W; ++j) wout[j] = ov[j];
  return En;
}

// ------------------------------------------------------------- contexts --
// Device-side context (lives in global memory, built by fmg_api.cpp).
// (LevelDev: fmg_internal.h)

struct __align__(16) DevCtx {
  LevelDev lv[kMaxLev];
  double* pbase; // norm partials of the grid levels (one slot per FMG level, iteration, level)
  int lc;        // the cluster kernel (fmg_kc.cu) handles levels 0..lc
  int n_cheb;    // Chebyshev degree k
  int smoother;  // 0 Chebyshev, 1 multicolour Gauss-Seidel
  double* Z;     // z_l (only for l < L)
  double* B;     // b_l = dec r_l - A z_l
  double* Y[2];  // Chebyshev iterates (k >= 3)
  double* Dv;    // Chebyshev direction (k >= 3)
  double* PU;    // P_l u_{l-1} (cluster kernel)
  double* KS[2]; // (unused)
  KcLayout kc;   // cluster-kernel shared-memory layout
  const double* Ainv;
  int n0;
  double* norms;
  int levels, n_ir;
  int* status;
  Coefs cf;
};


}  // namespace fmg
