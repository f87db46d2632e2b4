// fmg_stream.cu -- streaming-exponent BFP codec for sm_100a (§8(f) row N3).
//
// while the entries stream by, the running maximum of the
// entry exponents is the exponent the current mantissa is normalised to; a
// new block starts at each increase, and only the b largest exponents (b = w,
// reading R20) are stored -- entries of earlier blocks are below half a unit
// of the single-exponent mantissa and are stored as 0.  Entry exponent rule
// R19, int32 exponent range R21.
//
// The running maximum is a prefix-max scan.  The encode is ONE pass over x
// (DESIGN.md §N3), in the spirit of the paper's one-pass motivation
// (no re-normalisation, no re-computation):
//   k_sx_encode  chunks of 256 groups of 32 entries in ticket order; each CTA
//                reads its chunk once, publishes its maximum exponent, looks
//                back over its predecessors' published values (decoupled
//                look-back; max is idempotent) for the running maximum before
//                the chunk, then normalises every mantissa to the running
//                maximum at its position (R22) and packs it.  Groups that
//                raise the maximum record their block starts in an
//                exponent-indexed table (each exponent starts at most one block).
//   k_sx_select  one CTA: the w largest recorded exponents -> xexp/xstart and
//                the block count.
// Decode: k_sx_decode, per group: unpack, binary search of the block start
// table (<= 54 entries, shared memory), x_i = m_i 2^(X_k - q); 0 before the
// first kept block.
// Product path only; bit-exact against oracle/orc_bfp.c orc_stream_*.
#include <cuda_runtime.h>
#include <stdint.h>

#include "fmg_device.cuh"
#include "fmg_internal.h"

namespace fmg {

static int sx_num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

#ifdef SX_PROBE
__device__ unsigned long long* sx_probe_buf;  // per chunk: land, lookback done, end, rounds
__device__ __forceinline__ unsigned long long sx_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define SX_STAMP(c, k, v) \
  if (sx_probe_buf && threadIdx.x == 0) sx_probe_buf[(c) * 4 + (k)] = (v)
#else
#define SX_STAMP(c, k, v)
#endif

constexpr int SX_OFF = 1100;          // table index = X + SX_OFF, X in [-1073, 1024]
constexpr int SX_N = 2176;            // > 1024 + SX_OFF
constexpr int SX_NOEXP = -0x40000000;  // zero entries: no exponent (R19)
constexpr int SX_WARPS = 2;
constexpr int SX_GPC = 32 * SX_WARPS;  // groups per CTA chunk (one 32-group tile per warp)
constexpr int SX_RS = 33;              // staged row stride (doubles): lanes' rows in distinct banks
constexpr int SX_WS = 57;              // packed row stride (words) >= w + 1, odd
constexpr int SX_SMEM = SX_WARPS * 32 * (SX_RS * 8 + SX_WS * 4);

// x 2^k exactly as C's ldexp (correctly rounded; one rounding at most).
__device__ __forceinline__ double sx_scale(double x, int k) {
  if (k >= -1022 && k <= 1023) return x * pow2(k);
  return ldexp(x, k);
}

// R19: exponent entry v needs on its own; SX_NOEXP for zero; *bad for
// non-finite input or E > 1024 (R21).
__device__ __forceinline__ int sx_entry_exp(double v, int q, bool& bad) {
  const unsigned long long bits = (unsigned long long)__double_as_longlong(v) & 0x7fffffffffffffffULL;
  if (bits >= 0x7ff0000000000000ULL) { bad = true; return SX_NOEXP; }
  if (bits == 0ULL) return SX_NOEXP;
  const int ebits = (int)(bits >> 52);
  const int il = ebits ? ebits - 1023 : -1074 + 63 - __clzll((long long)bits);  // ilogb
  int e = il + 1;
  if (rint(sx_scale(__longlong_as_double((long long)bits), q - e)) == pow2(q)) e = e + 1;
  if (e > 1024) bad = true;
  return e;
}

__device__ __forceinline__ int warp_incl_max(int v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(FULL, v, o);
    if (lane >= o) v = max(v, u);
  }
  return v;
}

__device__ __forceinline__ void sx_publish(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long sx_peek(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// chunk status word: flag in bits 62..63 (0 none, 1 chunk maximum, 2 running
// maximum through the chunk), the int value in the low 32 bits
constexpr unsigned long long SX_AGG = 1ULL << 62, SX_INC = 2ULL << 62;
__device__ __forceinline__ unsigned long long sx_word(unsigned long long flag, int v) {
  return flag | (unsigned long long)(unsigned)v;
}

// R19 from the bits of |x| (non-zero, finite): for normal x the exponent bump
// RNE(|x| 2^(q-E0)) = 2^q is exactly frac(x) >= 2^52 - 2^(52-q) (never for
// q = 53); subnormals take the general path.
__device__ __forceinline__ int sx_exp_bits(unsigned long long bits, int q) {
  const int ebits = (int)(bits >> 52);
  if (ebits == 0) {
    bool bad = false;
    return sx_entry_exp(__longlong_as_double((long long)bits), q, bad);
  }
  const int bump = q <= 52 && (bits & 0x000fffffffffffffULL) >= (1ULL << 52) - (1ULL << (52 - q));
  return ebits - 1022 + bump;
}

// Decoupled look-back (warp 0): the running maximum before chunk c, given
// its own maximum agg; publishes agg, then the running maximum through c.
__device__ __forceinline__ int sx_lookback(unsigned long long* tiles, long long c, int agg, int lane) {
  int pre = SX_NOEXP;
  if (c == 0) {
    if (lane == 0) sx_publish(tiles, sx_word(SX_INC, agg));
    return pre;
  }
  if (lane == 0) sx_publish(tiles + c, sx_word(SX_AGG, agg));
  // window of 32 predecessors per poll (wider windows contend on the hot
  // status lines and measured slower)
  long long j = c - 1;
  while (true) {
    const long long idx = j - lane;
    unsigned long long sw = idx >= 0 ? sx_peek(tiles + idx) : sx_word(SX_INC, SX_NOEXP);
    while (__any_sync(FULL, (sw >> 62) == 0)) {
      if ((sw >> 62) == 0) {
        __nanosleep(20);
        sw = sx_peek(tiles + idx);
      }
    }
    const unsigned incm = __ballot_sync(FULL, (sw >> 62) == 2);
    const int v = (int)(unsigned)sw;
    if (incm) {
      const int first = __ffs(incm) - 1;  // nearest predecessor holding its running maximum
      pre = max(pre, __reduce_max_sync(FULL, lane <= first ? v : SX_NOEXP));
      break;
    }
    pre = max(pre, __reduce_max_sync(FULL, v));
    j -= 32;
  }
  SX_STAMP(c, 3, (unsigned long long)(c - 1 - j));
  if (lane == 0) sx_publish(tiles + c, sx_word(SX_INC, max(pre, agg)));
  return pre;
}

// Thread-per-group layout: a warp stages its 32 groups (8 KB) in shared memory
// with cp.async; lane j owns group g0 + j for the exponent search and the
// packing (serial, a running bit accumulator), and the packed words leave
// through a coalesced copy.  One small CTA (2 warps, ~19 KB of shared memory)
// per chunk, so that ~11 CTAs per SM hide each other's look-back latency; a
// CTA publishes its chunk maximum as soon as its data lands.
__device__ __forceinline__ void sx_stage(double* tile, const double* x, long long g0, int ngw, int lane) {
#pragma unroll 8
  for (int r = 0; r < 32; ++r) cpa8(tile + r * SX_RS + lane, x + (g0 + r) * 32 + lane, r < ngw);
}

__global__ void __launch_bounds__(SX_WARPS * 32) k_sx_encode(const double* __restrict__ x, long long ng,
                                                             long long nc, int w, int ws,
                                                             uint32_t* __restrict__ mant, int* __restrict__ present,
                                                             long long* __restrict__ start,
                                                             unsigned long long* __restrict__ tiles, int* ticket,
                                                             int* status) {
  extern __shared__ __align__(16) unsigned char sx_smem[];
  __shared__ long long s_chunk;
  __shared__ int s_pre;
  __shared__ int wsum[SX_WARPS];
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5, q = w - 1;
  double* tile = (double*)sx_smem + wp * 32 * SX_RS;
  uint32_t* wt = (uint32_t*)((double*)sx_smem + SX_WARPS * 32 * SX_RS) + wp * 32 * ws;
  const unsigned magic = (unsigned)((0x100000000ULL + w - 1) / w);
  const unsigned long long mask = (1ULL << w) - 1ULL;
  // chunks in ticket order: every lower ticket belongs to a CTA already running
  if (threadIdx.x == 0) s_chunk = atomicAdd(ticket, 1);
  __syncthreads();
  const long long c = s_chunk;
  const long long g0 = c * SX_GPC + wp * 32;
  const int ngw = (int)(ng - g0 < 0 ? 0 : (ng - g0 < 32 ? ng - g0 : 32));
  sx_stage(tile, x, g0, ngw, lane);
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncwarp();
  SX_STAMP(c, 0, sx_now());
  // group maximum exponent (monotone in |x|: the exponent of the max bits)
  const double* row = tile + lane * SX_RS;
  unsigned long long mx = 0ULL;
#pragma unroll 8
  for (int e = 0; e < 32; ++e) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(row[e]) & 0x7fffffffffffffffULL;
    mx = b > mx ? b : mx;
  }
  bool bad = mx >= 0x7ff0000000000000ULL;
  int gm = SX_NOEXP;
  if (!bad && mx != 0ULL) {
    gm = sx_exp_bits(mx, q);
    if (gm > 1024) bad = true;
  }
  if (__any_sync(FULL, bad) && lane == 0) atomicOr(status, 1);
  const int inc = warp_incl_max(gm, lane);
  if (lane == 31) wsum[wp] = inc;
  __syncthreads();
  if (wp == 0) {  // publish the chunk maximum at once, then look back
    int agg = wsum[0];
#pragma unroll
    for (int i = 1; i < SX_WARPS; ++i) agg = max(agg, wsum[i]);
    const int pre = sx_lookback(tiles, c, agg, lane);
    if (lane == 0) s_pre = pre;
    SX_STAMP(c, 1, sx_now());
  }
  __syncthreads();
  int excl = __shfl_up_sync(FULL, inc, 1);
  if (lane == 0) excl = SX_NOEXP;
  int M = max(s_pre, excl);  // running maximum before group g0 + lane
  for (int i = 0; i < wp; ++i) M = max(M, wsum[i]);
  // normalise each entry to the running maximum at its position (R22) and
  // pack; a group whose maximum exceeds M raises it entry by entry and
  // records the block starts ("a larger exponent is encountered")
  const bool raise = gm > M;
  uint32_t* wrow = wt + lane * ws;
  if (!raise && w <= 32 && M != SX_NOEXP && q - M >= -1022 && q - M <= 1023) {
    // common case: one exponent for the whole group, at most one word per entry
    const double sc = pow2(q - M);
    unsigned long long acc = 0ULL;
    int nb = 0, o = 0;
#pragma unroll 4
    for (int e = 0; e < 32; ++e) {
      const long long m = rne_int(row[e] * sc, w);
      acc |= ((unsigned long long)m & mask) << nb;
      nb += w;
      if (nb >= 32) {
        wrow[o++] = (uint32_t)acc;
        acc >>= 32;
        nb -= 32;
      }
    }
  } else {
    int k = q - M;
    bool fast = k >= -1022 && k <= 1023;
    double sc = fast ? pow2(k) : 0.0;
    unsigned long long acc = 0ULL;
    int nb = 0, o = 0;
    for (int e = 0; e < 32; ++e) {
      const double v = row[e];
      if (raise) {
        const unsigned long long b = (unsigned long long)__double_as_longlong(v) & 0x7fffffffffffffffULL;
        const int Ee = b ? sx_exp_bits(b, q) : SX_NOEXP;
        if (Ee > M) {
          M = Ee;
          present[M + SX_OFF] = 1;
          start[M + SX_OFF] = (g0 + lane) * 32 + e;
          k = q - M;
          fast = k >= -1022 && k <= 1023;
          sc = fast ? pow2(k) : 0.0;
        }
      }
      long long m = 0;
      if (M != SX_NOEXP) m = rne_int(fast ? v * sc : ldexp(v, k), w);
      const unsigned long long f = (unsigned long long)m & mask;
      acc |= f << nb;
      unsigned long long hi = nb ? f >> (64 - nb) : 0ULL;  // bits past 64 (w > 32 only)
      nb += w;
      while (nb >= 32) {
        wrow[o++] = (uint32_t)acc;
        acc = (acc >> 32) | (hi << 32);
        hi >>= 32;
        nb -= 32;
      }
    }
  }
  __syncwarp();
  uint32_t* dst = mant + g0 * w;
  for (int t = lane; t < ngw * w; t += 32) {
    const int j = (int)__umulhi((unsigned)t, magic);
    dst[t] = wt[j * ws + (t - j * w)];
  }
  SX_STAMP(c, 2, sx_now());
}

// Keep the w largest block exponents (ascending in xexp/xstart), *nblocks =
// count.  One CTA of 1024 threads, 3 consecutive table entries per thread.
__global__ void __launch_bounds__(1024) k_sx_select(const int* __restrict__ present,
                                                    const long long* __restrict__ start, int w,
                                                    int32_t* __restrict__ xexp, int64_t* __restrict__ xstart,
                                                    int32_t* __restrict__ nblocks) {
  __shared__ int wsum[32];
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  // suffix counts: thread t' = 1023 - t scans the table from the top
  const int t = 1023 - (int)threadIdx.x;
  int f[3], c = 0;
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const int i = 3 * t + j;
    f[j] = i < SX_N ? present[i] : 0;
    c += f[j];
  }
  int inc = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int u = __shfl_up_sync(FULL, inc, o);
    if (lane >= o) inc += u;
  }
  if (lane == 31) wsum[wp] = inc;
  __syncthreads();
  if (wp == 0) {
    int v = wsum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(FULL, v, o);
      if (lane >= o) v += u;
    }
    wsum[lane] = v;
  }
  __syncthreads();
  const int total = wsum[31];
  int above = inc - c + (wp > 0 ? wsum[wp - 1] : 0);  // present entries above this thread's three
  const int nb = total < w ? total : w;
#pragma unroll
  for (int j = 2; j >= 0; --j) {
    const int i = 3 * t + j;
    if (f[j]) {
      const int rank = above;  // 0 = largest exponent
      if (rank < nb) {
        const int slot = nb - 1 - rank;
        xexp[slot] = i - SX_OFF;
        xstart[slot] = start[i];
      }
      above += 1;
    }
  }
  if (threadIdx.x == 0) *nblocks = nb;
}

// Decode, thread per group: cp.async the warp's packed words to shared memory,
// lane j unpacks group g0 + j entry by entry (bit extraction as point_decode)
// with its block found by one binary search and advanced as starts pass, and
// the values leave through coalesced stores.
__global__ void __launch_bounds__(SX_WARPS * 32) k_sx_decode(const uint32_t* __restrict__ mant,
                                                             const int32_t* __restrict__ xexp,
                                                             const int64_t* __restrict__ xstart,
                                                             const int32_t* __restrict__ nblocks, long long ng,
                                                             int w, int ws, double* __restrict__ x) {
  extern __shared__ __align__(16) unsigned char sx_smem[];
  __shared__ long long s_start[64];
  __shared__ int s_exp[64];
  const int nbk = *nblocks;
  if ((int)threadIdx.x < nbk) {
    s_start[threadIdx.x] = xstart[threadIdx.x];
    s_exp[threadIdx.x] = xexp[threadIdx.x];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5, q = w - 1;
  double* tile = (double*)sx_smem + wp * 32 * SX_RS;
  uint32_t* wt = (uint32_t*)((double*)sx_smem + SX_WARPS * 32 * SX_RS) + wp * 32 * ws;
  const unsigned magic = (unsigned)((0x100000000ULL + w - 1) / w);
  const long long ntile = (ng + 31) / 32;
  const long long wg = (long long)blockIdx.x * SX_WARPS + wp, nw = (long long)gridDim.x * SX_WARPS;
  for (long long t = wg; t < ntile; t += nw) {
    const long long g0 = t * 32;
    const int ngw = (int)(ng - g0 < 32 ? ng - g0 : 32);
    const uint32_t* src = mant + g0 * w;
    for (int o = lane; o < ngw * w; o += 32) {
      const int j = (int)__umulhi((unsigned)o, magic);
      cpa4(wt + j * ws + (o - j * w), src + o);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncwarp();
    const long long i0 = (g0 + lane) * 32;
    int lo = 0, hi = nbk;  // kb = number of starts <= i0
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (s_start[mid] <= i0) lo = mid + 1; else hi = mid;
    }
    int kb = lo;
    long long nxt = kb < nbk ? s_start[kb] : 0x7fffffffffffffffLL;
    int ks = kb > 0 ? s_exp[kb - 1] - q : 0;
    const uint32_t* wrow = wt + lane * ws;
    double* row = tile + lane * SX_RS;
    for (int e = 0; e < 32; ++e) {
      if (i0 + e >= nxt) {
        ks = s_exp[kb] - q;
        ++kb;
        nxt = kb < nbk ? s_start[kb] : 0x7fffffffffffffffLL;
      }
      const int pos = e * w, j0 = pos >> 5, sh = pos & 31;
      unsigned long long f = ((unsigned long long)wrow[j0] | ((unsigned long long)wrow[j0 + 1] << 32)) >> sh;
      if (sh + w > 64) f |= (unsigned long long)wrow[j0 + 2] << (64 - sh);
      const long long m = (long long)(f << (64 - w)) >> (64 - w);
      double v = 0.0;
      if (kb > 0) v = (ks >= -1022 && ks <= 1023) ? i2d(m, w) * pow2(ks) : ldexp((double)m, ks);
      row[e] = v;
    }
    __syncwarp();
#pragma unroll 8
    for (int r = 0; r < 32; ++r)
      if (r < ngw) __stcs(x + (g0 + r) * 32 + lane, tile[r * SX_RS + lane]);
    __syncwarp();
  }
}

// ------------------------------------------------------------- launchers --
// work: [ticket | present[SX_N] | tiles[nc]] (zeroed by one memset) + start[SX_N]
static long long sx_zeroed_bytes(long long nc) { return 256 + SX_N * 4 + nc * 8; }

long long stream_work_bytes(long long n) {
  const long long ng = n / 32, nc = (ng + SX_GPC - 1) / SX_GPC;
  return (sx_zeroed_bytes(nc) + 255) / 256 * 256 + SX_N * 8;
}

void launch_stream_encode(const double* x, long long n, int w, uint32_t* mant, int32_t* xexp, int64_t* xstart,
                          int32_t* nblocks, void* work, int* status, cudaStream_t st) {
  const long long ng = n / 32, nc = (ng + SX_GPC - 1) / SX_GPC;
  char* p = (char*)work;
  int* ticket = (int*)p;
  int* present = (int*)(p + 256);
  unsigned long long* tiles = (unsigned long long*)(p + 256 + SX_N * 4);
  long long* start = (long long*)(p + (sx_zeroed_bytes(nc) + 255) / 256 * 256);
  const int ws = (w + 1) | 1;  // odd packed-row stride >= w + 1
  const int smem = SX_WARPS * 32 * SX_RS * 8 + SX_WARPS * 32 * ws * 4;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_sx_encode, cudaFuncAttributeMaxDynamicSharedMemorySize, SX_SMEM);
    attr = true;
  }
  cudaMemsetAsync(p, 0, sx_zeroed_bytes(nc), st);
  k_sx_encode<<<(unsigned)nc, SX_WARPS * 32, smem, st>>>(x, ng, nc, w, ws, mant, present, start, tiles, ticket,
                                                         status);
  k_sx_select<<<1, 1024, 0, st>>>(present, start, w, xexp, xstart, nblocks);
}

void launch_stream_decode(const uint32_t* mant, const int32_t* xexp, const int64_t* xstart, const int32_t* nblocks,
                          long long n, int w, double* x, cudaStream_t st) {
  const long long ng = n / 32;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k_sx_decode, cudaFuncAttributeMaxDynamicSharedMemorySize, SX_SMEM);
    attr = true;
  }
  const int ws = (w + 1) | 1;
  const int smem = SX_WARPS * 32 * SX_RS * 8 + SX_WARPS * 32 * ws * 4;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sx_decode, SX_WARPS * 32, smem);
  if (per_sm < 1) per_sm = 1;
  long long want = (ng + 32 * SX_WARPS - 1) / (32 * SX_WARPS);
  const long long cap = (long long)sx_num_sms() * per_sm;
  const int grid = (int)(want < cap ? (want > 0 ? want : 1) : cap);
  k_sx_decode<<<grid, SX_WARPS * 32, smem, st>>>(mant, xexp, xstart, nblocks, ng, w, ws, x);
}

}  // namespace fmg
