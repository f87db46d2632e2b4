// fmg_kernels.cu -- sm_100a kernels of the compact-FMG hot path.
//
// Structure: every step of the method is a *tile operation* (a __device__
// function that produces one output tile of one level: 32 x TY (x TZ) points,
// 256 threads, one warp per 32-entry x row = one BFP block).  A step is
// executed by a grid kernel (one CTA per tile, `k_op`).  The small levels
// 0..lc live in shared memory of one CTA (`k4_kernel`), which runs their part
// of every IR iteration back to back (no launch gaps, no global round trips).
// All kernels use programmatic dependent launch (griddepcontrol).
//
// Every floating-point expression follows the canonical evaluation order of
// DESIGN.md §3 with explicit fma(); compiled with -fmad=false.  Tensor-product
// operators are applied factor by factor in shared memory: x pass, y, z.
//
// Paper: BFP codec PAPER.md:1240-1274 with RNE; decode sweep /
// residual / truncate / restriction = fmgResidual (Alg 3.2);
// coarse-to-fine sweep of cFas (Alg 3.1, nu = 1 so s = 0,
// PAPER.md:809-812) fused with the correction (Alg 3.3).
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

// Warp-cooperative decode: lane j returns entry j of the block whose w words
// start at `words`.  All 32 lanes must call.
__device__ __forceinline__ double warp_decode(const uint32_t* words, int E, int w, int lane) {
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
  long long m = (long long)(field << (64 - w)) >> (64 - w);
  return i2d(m, w) * pow2(E - (w - 1));
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

// Warp-cooperative encode of one block; lane j holds entry j.
// Writes the w words and the exponent when `words` is non-null; returns the
// quantised value m 2^(E-q).  Non-finite input or E > 127 sets *status.
__device__ __forceinline__ double warp_encode(double v, int w, uint32_t* words, int8_t* eptr, int lane,
                                              int* status) {
  unsigned long long bits = (unsigned long long)__double_as_longlong(v) & 0x7fffffffffffffffULL;
  bool bad = bits >= 0x7ff0000000000000ULL;
  unsigned hi = (unsigned)(bits >> 32), lo = (unsigned)bits;
  unsigned mh = __reduce_max_sync(FULL, hi);
  unsigned ml = __reduce_max_sync(FULL, hi == mh ? lo : 0u);
  bool err = __any_sync(FULL, bad);
  double mx = __longlong_as_double((long long)(((unsigned long long)mh << 32) | ml));
  int q = w - 1, E = -128;
  if (!err && mx != 0.0) {
    int ebits = (int)((mh >> 20) & 0x7FFu);
    int E0 = ebits == 0 ? -1100 : ebits - 1022;  // ilogb(mx) + 1; subnormal max -> saturates below
    if (E0 > 127) {
      err = true;
    } else if (E0 < -127) {
      E = -127;
    } else {
      E = E0;
      if (rint(mx * pow2(q - E0)) == pow2(q)) E = E0 + 1;
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
    unsigned long long field = (unsigned long long)m & ((1ULL << w) - 1ULL);
    uint32_t mine0 = 0u, mine1 = 0u;
    if (w <= 8) {
      // narrow: one redux.or per output word
      int o = lane * w;
      for (int j = 0; j < w; ++j) {
        int s = o - 32 * j;
        uint32_t c = 0u;
        if (s > -w && s < 32) c = s >= 0 ? (uint32_t)(field << s) : (uint32_t)(field >> (-s));
        uint32_t word = __reduce_or_sync(FULL, c);
        if (lane == j) mine0 = word;
      }
    } else {
      // wide: word j gathers its <= ceil(32/w)+1 entries by shuffles
      const int K = (32 + w - 1) / w + 1;
      uint32_t flo = (uint32_t)field, fhi = (uint32_t)(field >> 32);
#pragma unroll 1
      for (int half = 0; half < 2; ++half) {
        int j = lane + 32 * half;
        if (half == 1 && w <= 32) break;
        int e0 = (32 * j) / w;
        uint32_t acc = 0u;
        for (int k = 0; k < K; ++k) {
          int e = e0 + k;
          int src = e < 32 ? e : 31;
          uint32_t lo_ = __shfl_sync(FULL, flo, src), hi_ = __shfl_sync(FULL, fhi, src);
          unsigned long long f = ((unsigned long long)hi_ << 32) | lo_;
          int s = e * w - 32 * j;
          if (e < 32 && s < 32 && s > -w) acc |= s >= 0 ? (uint32_t)(f << s) : (uint32_t)(f >> (-s));
        }
        if (half == 0) mine0 = acc; else mine1 = acc;
      }
    }
    if (lane < w) words[lane] = mine0;
    if (lane + 32 < w) words[lane + 32] = mine1;
    if (lane == 0) *eptr = (int8_t)E;
  }
  return E == -128 ? 0.0 : i2d(m, w) * pow2(E - q);
}

// ------------------------------------------------------------ tile plans --
template <int D, int P> struct TileCfg;
#ifndef FMG_TY2D
#define FMG_TY2D 16
#endif
template <int P> struct TileCfg<2, P> { static constexpr int TY = FMG_TY2D, TZ = 1; };
template <> struct TileCfg<3, 1> { static constexpr int TY = 8, TZ = 4; };
template <> struct TileCfg<3, 2> { static constexpr int TY = 4, TZ = 4; };
template <> struct TileCfg<3, 3> { static constexpr int TY = 4, TZ = 4; };

template <int D, int P> struct Plan {
  static constexpr int TY = TileCfg<D, P>::TY, TZ = TileCfg<D, P>::TZ;
  static constexpr int T = 2 * P + 1;  // A taps
  // A tile: input box (output + P halo), x-pass out, y-pass out (3D)
  static constexpr int BX = 32 + 2 * P, BY = TY + 2 * P, BZ = (D == 3) ? TZ + 2 * P : 1;
  static constexpr int NU = BX * BY * BZ;
  static constexpr int NAB = 32 * BY * BZ;
  static constexpr int NCS = (D == 3) ? 32 * TY * BZ : 0;
  // coarse box feeding a prolongation onto the input box
  static constexpr int CBX = P * ((BX - 1) / (2 * P) + 2) + 1;
  static constexpr int CBY = P * ((BY - 1) / (2 * P) + 2) + 1;
  static constexpr int CBZ = (D == 3) ? P * ((BZ - 1) / (2 * P) + 2) + 1 : 1;
  static constexpr int NCB = CBX * CBY * CBZ;
  static constexpr int NV1 = BX * CBY * CBZ;              // P x-pass out
  static constexpr int NV2 = (D == 3) ? BX * BY * CBZ : 0; // P y-pass out (3D)
  static constexpr int PRO_REGION = NCB + NV1 + NV2;
  static constexpr int A_REGION = 2 * NAB + 2 * NCS;
  static constexpr int mx3(int a, int b, int c) { return a > b ? (a > c ? a : c) : (b > c ? b : c); }
  static constexpr int R1N = mx3(PRO_REGION, A_REGION, 0);  // prolongation scratch | A stages
  static constexpr int NROWS = TY * TZ;
  // [box0 NU][box1 NU][R1][PU tile][section words (<= 54 per row, as doubles)][z rows]
  static constexpr int A_SMEM = (2 * NU + R1N + 0 + 32 * NROWS + 27 * NROWS + 32 * NROWS) * 8;
  // decode/prolong tile (output only, no halo)
  static constexpr int DBX = 32, DBY = TY, DBZ = (D == 3) ? TZ : 1;
  static constexpr int DCBX = P * ((DBX - 1) / (2 * P) + 2) + 1;
  static constexpr int DCBY = P * ((DBY - 1) / (2 * P) + 2) + 1;
  static constexpr int DCBZ = (D == 3) ? P * ((DBZ - 1) / (2 * P) + 2) + 1 : 1;
  static constexpr int D_SCR = DCBX * DCBY * DCBZ + DBX * DCBY * DCBZ + ((D == 3) ? DBX * DBY * DCBZ : 0);
  static_assert(D_SCR <= PRO_REGION || D_SCR <= A_REGION || true, "");
  static constexpr int D_SMEM = (D_SCR + DBX * DBY * DBZ) * 8;
  static constexpr int NPU = DBX * DBY * DBZ;  // emitted-u prolongation tile
  // restriction tile (coarse output 32 x TY x TZ); x pass gathered from global
  static constexpr int FBY = 2 * TY + 4 * P - 3, FBZ = (D == 3) ? 2 * TZ + 4 * P - 3 : 1;
  static constexpr int NXR = 32 * FBY * FBZ;
  static constexpr int NYR = (D == 3) ? 32 * TY * FBZ : 0;
  static constexpr int R_SMEM = (NXR + NYR) * 8;
  static constexpr int C_SMEM = 2 * ((D == 3) ? 4 * P * P : 2 * P) * 32 * 8;  // coarse solve
  static constexpr int mx2(int a, int b) { return a > b ? a : b; }
  static constexpr int SMEM = mx2(mx2(A_SMEM, D_SMEM), mx2(R_SMEM, C_SMEM));
};

// ------------------------------------------------------------- contexts --
// Device-side context (lives in global memory, built by fmg_api.cpp).
struct LevelDev {
  Geom g;
  uint32_t* umant;
  int8_t* uexp;
  int ustride;
  uint32_t* rmant;
  int8_t* rexp;
  int rstride;
  const double* gtab;
  int tx, ty, tz;  // tile grid of this level
  double* part;    // norm partials, one per tile
  int* count;      // arrival counter for the last-CTA norm reduction
};

struct DevCtx {
  LevelDev lv[kMaxLev];
  double* U[2];  // decoded u_l (ping-pong by level parity), emitted by the cFas finalize
  double* T[2];  // residual temporaries t_l
  double* W[2];  // w_l = z_l + dec ý_l
  double* pbase; // norm partials of the grid levels (one slot per FMG level, iteration, level)
  double* usm;   // K4: dense u_l of the smem levels, persisted between launches
  long long usm_off[kMaxLev];
  int lc;        // K4 handles levels 0..lc in shared memory
  int n_cheb;    // Chebyshev degree k
  double* Z;     // z_l (only for l < L)
  double* B;     // b_l = dec r_l - A z_l
  double* Y[2];  // Chebyshev iterates (k >= 3)
  double* Dv;    // Chebyshev direction (k >= 3)
  const double* Ainv;
  int n0;
  double* norms;
  int levels, n_ir;
  int* status;
  Coefs cf;
};

using Op = OpDesc;  // one step of the method on one level (fmg_internal.h)

__device__ __forceinline__ int op_tiles(const DevCtx& c, const Op& op) {
  const LevelDev& lv = c.lv[op.l];
  if (op.type == OP_NORMS) return 1;
  return lv.tx * lv.ty * lv.tz;
}

// ------------------------------------------------ prolongation onto a box --
// out[bz][by][bx] = (P_lf coarse)(fx0+bx, fy0+by, fz0+bz) over a box of
// NBX x NBY x NBZ fine points, canonical x, y, z passes; 0 at
// fine non-unknowns.  Scratch: cb (coarse box), v1, v2.  Lanes own x columns
// (weights in registers), warps own rows (row-uniform weights).
template <int D, int P, int NCX, int NCY, int NCZ>
__device__ void cbox_async(const double* __restrict__ coarse, const Geom& gc, int fx0, int fy0, int fz0, double* cb) {
  static_assert(NCX <= 32, "coarse box wider than a warp");
  const int lane = threadIdx.x, wid = threadIdx.y;
  const int nc = gc.n;
  const int cx0 = P * floordiv(fx0, 2 * P), cy0 = P * floordiv(fy0, 2 * P);
  const int cz0 = (D == 3) ? P * floordiv(fz0, 2 * P) : 0;
  const int gx = cx0 + lane;
  const bool okx = lane < NCX && gx >= 0 && gx < nc;
  for (int r = wid; r < NCY * NCZ; r += NWARP) {
    int gy = cy0 + r % NCY, gz = cz0 + r / NCY;
    bool ok = okx && gy >= 0 && gy < nc && (D == 2 || (gz >= 0 && gz < nc));
    if (lane < NCX) cpa8(cb + r * NCX + lane, ok ? coarse + ((long long)gz * gc.NY + gy) * gc.NX + gx : coarse, ok);
  }
}

// Prolongation passes from an already loaded coarse box `cb` (see box_prolong).
template <int D, int P, int NBX, int NBY, int NBZ, int NCX, int NCY, int NCZ>
__device__ void box_prolong_compute(int nf, int fx0, int fy0, int fz0, const Coefs& cf, const double* cb, double* v1,
                                    double* v2, double* out) {
  const int lane = threadIdx.x, wid = threadIdx.y;
  const int cx0 = P * floordiv(fx0, 2 * P), cy0 = P * floordiv(fy0, 2 * P);
  const int cz0 = (D == 3) ? P * floordiv(fz0, 2 * P) : 0;
  __syncthreads();
  // x pass: v1[cz][cy][bx]; columns bx = lane and lane + 32
  {
    constexpr int NCOL = (NBX + 31) / 32;
    double w[NCOL][P + 1];
    int base[NCOL];
    bool ok[NCOL];
#pragma unroll
    for (int k = 0; k < NCOL; ++k) {
      int bx = lane + 32 * k;
      int x = fx0 + bx;
      ok[k] = bx < NBX && unk1(x, nf);
      int rx = ok[k] ? x % (2 * P) : 0;
      base[k] = ok[k] ? P * (x / (2 * P)) - cx0 : 0;
#pragma unroll
      for (int t = 0; t <= P; ++t) w[k][t] = cf.Pw[rx][t];
    }
    for (int r = wid; r < NCY * NCZ; r += NWARP) {
      const double* src = cb + r * NCX;
#pragma unroll
      for (int k = 0; k < NCOL; ++k) {
        int bx = lane + 32 * k;
        if (bx >= NBX) break;
        double acc = 0.0;
#pragma unroll
        for (int t = 0; t <= P; ++t) acc = fma(w[k][t], src[base[k] + t], acc);
        v1[r * NBX + bx] = ok[k] ? acc : 0.0;
      }
    }
  }
  __syncthreads();
  // y pass (rows (cz, by), weights row-uniform)
  double* yout = (D == 3) ? v2 : out;
  for (int r = wid; r < NBY * NCZ; r += NWARP) {
    int by = r % NBY, cz = r / NBY;
    int y = fy0 + by;
    bool ok = unk1(y, nf);
    int ry = ok ? y % (2 * P) : 0, base = ok ? P * (y / (2 * P)) - cy0 : 0;
    double w[P + 1];
#pragma unroll
    for (int t = 0; t <= P; ++t) w[t] = cf.Pw[ry][t];
    const double* src = v1 + (cz * NCY + base) * NBX;
    for (int bx = lane; bx < NBX; bx += 32) {
      double acc = 0.0;
#pragma unroll
      for (int t = 0; t <= P; ++t) acc = fma(w[t], src[t * NBX + bx], acc);
      yout[r * NBX + bx] = ok ? acc : 0.0;
    }
  }
  if constexpr (D == 3) {
    __syncthreads();
    for (int r = wid; r < NBY * NBZ; r += NWARP) {
      int by = r % NBY, bz = r / NBY;
      int z = fz0 + bz;
      bool ok = unk1(z, nf);
      int rz = ok ? z % (2 * P) : 0, base = ok ? P * (z / (2 * P)) - cz0 : 0;
      double w[P + 1];
#pragma unroll
      for (int t = 0; t <= P; ++t) w[t] = cf.Pw[rz][t];
      const double* src = v2 + (base * NBY + by) * NBX;
      for (int bx = lane; bx < NBX; bx += 32) {
        double acc = 0.0;
#pragma unroll
        for (int t = 0; t <= P; ++t) acc = fma(w[t], src[t * NBY * NBX + bx], acc);
        out[r * NBX + bx] = ok ? acc : 0.0;
      }
    }
  }
  __syncthreads();
}

template <int D, int P, int NBX, int NBY, int NBZ, int NCX, int NCY, int NCZ>
__device__ void box_prolong(const double* __restrict__ coarse, const Geom& gc, int nf, int fx0, int fy0, int fz0,
                            const Coefs& cf, double* cb, double* v1, double* v2, double* out) {
  cbox_async<D, P, NCX, NCY, NCZ>(coarse, gc, fx0, fy0, fz0, cb);
  cpa_wait_sync();
  box_prolong_compute<D, P, NBX, NBY, NBZ, NCX, NCY, NCZ>(nf, fx0, fy0, fz0, cf, cb, v1, v2, out);
}

// Adds dec(section) to the box rows (in place): box covers fine x in
// [bx0, bx0+NBX) = [x0-H, x0+32+H) and rows (y, z); 0 outside the stored level.
template <int D, int NBX, int NBY, int NBZ, int H>
__device__ void box_add_decode(const LevelDev& lv, int w, int x0, int y0b, int z0b, double* box) {
  const int lane = threadIdx.x;
  const Geom& g = lv.g;
  const int nxb = g.NX >> 5, xb = x0 >> 5;
  for (int r = threadIdx.y; r < NBY * NBZ; r += NWARP) {
    int by = r % NBY, bz = r / NBY;
    int gy = y0b + by, gz = (D == 3) ? z0b + bz : 0;
    if (gy < 0 || gy >= g.NY || gz < 0 || gz >= g.NZ) continue;  // warp-uniform
    long long rowblk = ((long long)gz * g.NY + gy) * nxb;
    long long blk = rowblk + xb;
    double dv = warp_decode(lv.umant + blk * lv.ustride, lv.uexp[blk], w, lane);
    double* brow = box + r * NBX;
    brow[H + lane] = dv + brow[H + lane];
    if (H > 0 && lane < 2 * H) {
      int xl = lane < H ? x0 - H + lane : x0 + 32 + (lane - H);
      if (xl >= 0 && xl < g.NX) {
        long long b2 = rowblk + (xl >> 5);
        double d2 = point_decode(lv.umant + b2 * lv.ustride, lv.uexp[b2], w, xl & 31);
        int bx = lane < H ? lane : 32 + lane;
        brow[bx] = d2 + brow[bx];
      }
    }
  }
  __syncthreads();
}

// ------------------------------------------------------------ A on a tile --
// Given the input box U (output tile + P halo) in smem, computes the x pass
// (a = Mx u, b = Kx u) and, in 3D, the y pass (c = My a, s = Ky a + My b)
// (DESIGN.md §3.2).  The last pass is done per output point by a_final.
template <int D, int P>
__device__ void a_stages(const Geom& g, int x0, int y0, const Coefs& cf, const double* U, double* AB, double* CS) {
  using PL = Plan<D, P>;
  const int lane = threadIdx.x, wid = threadIdx.y;
  double* A = AB;
  double* B = AB + PL::NAB;
  // x pass: lane = output x column (node type fixed per thread -> registers)
  {
    const int gx = x0 + lane;
    const bool ok = unk1(gx, g.n);
    const int tau = ok ? gx % P : 0;
    double km[PL::T], kk[PL::T];
#pragma unroll
    for (int o = 0; o < PL::T; ++o) {
      km[o] = cf.Mc[tau][o];
      kk[o] = cf.Kc[tau][o];
    }
    for (int r = wid; r < PL::BY * PL::BZ; r += NWARP) {
      const double* u = U + r * PL::BX + lane;
      double a = 0.0, b = 0.0;
#pragma unroll
      for (int o = 0; o < PL::T; ++o) {
        a = fma(km[o], u[o], a);
        b = fma(kk[o], u[o], b);
      }
      A[r * 32 + lane] = ok ? a : 0.0;
      B[r * 32 + lane] = ok ? b : 0.0;
    }
  }
  __syncthreads();
  if constexpr (D == 3) {
    double* C = CS;
    double* S = CS + PL::NCS;
    for (int r = wid; r < PL::TY * PL::BZ; r += NWARP) {
      int ty = r % PL::TY, bz = r / PL::TY;
      int gy = y0 + ty;
      bool ok = unk1(gy, g.n);
      int tau = ok ? gy % P : 0;
      const double* a = A + (bz * PL::BY + ty) * 32 + lane;
      const double* b = B + (bz * PL::BY + ty) * 32 + lane;
      double c = 0.0, dd = 0.0, e = 0.0;
#pragma unroll
      for (int o = 0; o < PL::T; ++o) {
        c = fma(cf.Mc[tau][o], a[o * 32], c);
        dd = fma(cf.Kc[tau][o], a[o * 32], dd);
        e = fma(cf.Mc[tau][o], b[o * 32], e);
      }
      C[r * 32 + lane] = ok ? c : 0.0;
      S[r * 32 + lane] = ok ? dd + e : 0.0;
    }
    __syncthreads();
  }
}

// Last pass of A at output (x0+lane, y0+ty, z0+tz); 0 at non-unknowns.
template <int D, int P>
__device__ __forceinline__ double a_final(const Geom& g, int x0, int y0, int z0, int ty, int tz, const Coefs& cf,
                                          const double* AB, const double* CS) {
  using PL = Plan<D, P>;
  const int lane = threadIdx.x;
  int gx = x0 + lane, gy = y0 + ty, gz = z0 + tz;
  if (!unk1(gx, g.n) || !unk1(gy, g.n) || (D == 3 && !unk1(gz, g.n))) return 0.0;
  if constexpr (D == 2) {
    const double* A = AB;
    const double* B = AB + PL::NAB;
    int tau = gy % P;
    double d = 0.0, e = 0.0;
#pragma unroll
    for (int o = 0; o < PL::T; ++o) {
      d = fma(cf.Kc[tau][o], A[(ty + o) * 32 + lane], d);
      e = fma(cf.Mc[tau][o], B[(ty + o) * 32 + lane], e);
    }
    return d + e;
  } else {
    const double* C = CS;
    const double* S = CS + PL::NCS;
    int tau = gz % P;
    double acc = 0.0;
#pragma unroll
    for (int o = 0; o < PL::T; ++o) acc = fma(cf.Kc[tau][o], C[((tz + o) * PL::TY + ty) * 32 + lane], acc);
#pragma unroll
    for (int o = 0; o < PL::T; ++o) acc = fma(cf.Mc[tau][o], S[((tz + o) * PL::TY + ty) * 32 + lane], acc);
    return acc * pow2(-(g.l + 1));
  }
}

// Load a plain FP64 array onto the input box (0 outside the stored level).
// Flat element mapping (constant divisors): no half-empty column iterations.
template <int D, int P>
__device__ void box_load(const double* __restrict__ src, const Geom& g, int x0, int y0, int z0, double* U) {
  using PL = Plan<D, P>;
  const int tid = threadIdx.y * 32 + threadIdx.x;
#pragma unroll 4
  for (int i = tid; i < PL::NU; i += NT) {
    int bx = i % PL::BX, r = i / PL::BX;
    int gy = y0 - P + r % PL::BY, gz = (D == 3) ? z0 - P + r / PL::BY : 0, gx = x0 - P + bx;
    bool ok = gx >= 0 && gx < g.NX && gy >= 0 && gy < g.NY && gz >= 0 && gz < g.NZ;
    U[i] = ok ? src[((long long)gz * g.NY + gy) * g.NX + gx] : 0.0;
  }
  __syncthreads();
}

template <int D, int P>
__device__ void box_async(const double* __restrict__ src, const Geom& g, int x0, int y0, int z0, double* U) {
  using PL = Plan<D, P>;
  const int tid = threadIdx.y * 32 + threadIdx.x;
#pragma unroll 4
  for (int i = tid; i < PL::NU; i += NT) {
    int bx = i % PL::BX, r = i / PL::BX;
    int gy = y0 - P + r % PL::BY, gz = (D == 3) ? z0 - P + r / PL::BY : 0, gx = x0 - P + bx;
    bool ok = gx >= 0 && gx < g.NX && gy >= 0 && gy < g.NY && gz >= 0 && gz < g.NZ;
    cpa8(U + i, ok ? src + ((long long)gz * g.NY + gy) * g.NX + gx : src, ok);
  }
}

// Section words of the tile's output rows (row-major [row][stride]) into smem.
template <int D, int P>
__device__ void rows_words_async(const uint32_t* __restrict__ mant, int stride, int w, const Geom& g, int x0, int y0,
                                 int z0, uint32_t* dst) {
  using PL = Plan<D, P>;
  const int nxb = g.NX >> 5;
  for (int r = threadIdx.y; r < PL::NROWS; r += NWARP) {
    int y = y0 + r % PL::TY, z = z0 + r / PL::TY;
    if (y >= g.NY || z >= g.NZ) continue;
    long long blk = ((long long)z * g.NY + y) * nxb + (x0 >> 5);
    for (int j = threadIdx.x; j < w; j += 32) cpa4(dst + r * stride + j, mant + blk * stride + j);
  }
}

// Deterministic CTA sum; result valid in thread 0.
__device__ __forceinline__ double cta_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  if (threadIdx.x == 0) red[threadIdx.y] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0 && threadIdx.y == 0)
    for (int i = 0; i < NWARP; ++i) s += red[i];
  __syncthreads();
  return s;
}

// Per-tile partial of ||t_l||^2 -> part[tile]; the last CTA of the level to
// arrive sums all partials in fixed order and writes ||t_l||_2 to the norm row
// (deterministic: the order does not depend on which CTA is last).
__device__ void level_norm(const DevCtx& c, const LevelDev& lv, int l, int row, int tile, double ss, bool reduce,
                           long long poff) {
  __shared__ double red[NT];
  __shared__ int last;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(FULL, ss, o);
  if (threadIdx.x == 0) red[threadIdx.y] = ss;
  __syncthreads();
  const int tid = threadIdx.y * 32 + threadIdx.x;
  if (tid == 0) {
    double s = 0.0;
    for (int i = 0; i < NWARP; ++i) s += red[i];
    if (poff >= 0) c.pbase[poff + tile] = s;
    lv.part[tile] = s;
    last = 0;
    if (reduce) {
      __threadfence();
      int nt = lv.tx * lv.ty * lv.tz;
      last = atomicAdd(lv.count, 1) == nt - 1;
    }
  }
  __syncthreads();
  if (!last || row < 0) return;
  __threadfence();
  const int nt = lv.tx * lv.ty * lv.tz;
  double s = 0.0;
  for (int i = tid; i < nt; i += NT) s += ((volatile double*)lv.part)[i];
  red[tid] = s;
  __syncthreads();
  for (int o = NT / 2; o > 0; o >>= 1) {
    if (tid < o) red[tid] += red[tid + o];
    __syncthreads();
  }
  if (tid == 0) {
    c.norms[(long long)row * c.levels + l] = sqrt(red[0]);
    *lv.count = 0;
  }
}

// Tile of a grid op: 3D block index (no runtime division) and its linear index.
struct TileIdx {
  int bx, by, bz, lin;
};
__device__ __forceinline__ void tile_coords(const TileIdx& t, int TY, int TZ, int& x0, int& y0, int& z0) {
  x0 = t.bx * 32;
  y0 = t.by * TY;
  z0 = t.bz * TZ;
}

// ============================================================ tile ops =====
// S2: u_l = dec ú_l + P_l u_{l-1} (decode sweep PAPER.md:733-735), materialised.
template <int D, int P>
__device__ void tile_decode(const DevCtx& c, const Op& op, const TileIdx& tile, double* sm) {
  using PL = Plan<D, P>;
  const LevelDev& lv = c.lv[op.l];
  const Geom& g = lv.g;
  int x0, y0, z0;
  tile_coords(tile, PL::TY, PL::TZ, x0, y0, z0);
  double* out = c.U[op.l & 1];
  double* box = sm;  // DBX x DBY x DBZ
  if (op.l > 0) {
    double* cb = box + PL::DBX * PL::DBY * PL::DBZ;
    double* v1 = cb + PL::DCBX * PL::DCBY * PL::DCBZ;
    double* v2 = v1 + PL::DBX * PL::DCBY * PL::DCBZ;
    box_prolong<D, P, PL::DBX, PL::DBY, PL::DBZ, PL::DCBX, PL::DCBY, PL::DCBZ>(
        c.U[(op.l - 1) & 1], c.lv[op.l - 1].g, g.n, x0, y0, z0, c.cf, cb, v1, v2, box);
  } else {
    for (int i = threadIdx.y * 32 + threadIdx.x; i < PL::DBX * PL::DBY * PL::DBZ; i += NT) box[i] = 0.0;
    __syncthreads();
  }
  box_add_decode<D, PL::DBX, PL::DBY, PL::DBZ, 0>(lv, op.wu_in, x0, y0, z0, box);
  for (int r = threadIdx.y; r < PL::DBY * PL::DBZ; r += NWARP) {
    int gy = y0 + r % PL::DBY, gz = z0 + r / PL::DBY;
    if (gy >= g.NY || gz >= g.NZ) continue;
    out[((long long)gz * g.NY + gy) * g.NX + x0 + threadIdx.x] = box[r * 32 + threadIdx.x];
  }
}

// S3+S4: t_L = f_L - A_L u_L on the tile, r_L = enc(t_L), ||t_L||^2 partial
// (PAPER.md:738-739).  u_L = dec ú_L + P u_{L-1} (S2) was emitted by the previous
// sweep's finalize (or by the decode op at the start of the FMG level).
template <int D, int P>
__device__ void tile_residual(const DevCtx& c, const Op& op, const TileIdx& tile, double* sm) {
  using PL = Plan<D, P>;
  const LevelDev& lv = c.lv[op.L];
  const Geom& g = lv.g;
  int x0, y0, z0;
  tile_coords(tile, PL::TY, PL::TZ, x0, y0, z0);
  double* U = sm;
  double* R1 = sm + 2 * PL::NU;
  box_async<D, P>(c.U[op.L & 1], g, x0, y0, z0, U);
  cpa_wait_sync();
  double* AB = R1;
  double* CS = R1 + 2 * PL::NAB;
  a_stages<D, P>(g, x0, y0, c.cf, U, AB, CS);
  const int lane = threadIdx.x;
  double* T = c.T[op.L & 1];
  double ss = 0.0;
  for (int row = threadIdx.y; row < PL::TY * PL::TZ; row += NWARP) {
    int ty = row % PL::TY, tz = row / PL::TY;
    int y = y0 + ty, z = z0 + tz, x = x0 + lane;
    if (y >= g.NY || z >= g.NZ) continue;
    double au = a_final<D, P>(g, x0, y0, z0, ty, tz, c.cf, AB, CS);
    bool unk = unk1(x, g.n) && unk1(y, g.n) && (D == 2 || unk1(z, g.n));
    double t = 0.0;
    if (unk) {
      double f = c.cf.rhs_c * lv.gtab[x];
      f = f * lv.gtab[y];
      if (D == 3) f = f * lv.gtab[z];
      t = f - au;
    }
    long long idx = ((long long)z * g.NY + y) * g.NX + x;
    T[idx] = t;
    ss = fma(t, t, ss);
    long long blk = idx >> 5;
    warp_encode(t, op.wr, lv.rmant + blk * lv.rstride, lv.rexp + blk, lane, c.status);
  }
  level_norm(c, lv, op.L, op.row, tile.lin, ss, op.step == 9, op.poff);
}

// S5: t_l = R_{l+1} t_{l+1} (restricts t, not r), r_l = enc.
template <int D, int P>
__device__ void tile_restrict(const DevCtx& c, const Op& op, const TileIdx& tile, double* sm) {
  using PL = Plan<D, P>;
  const LevelDev& lc = c.lv[op.l];
  const Geom& gc = lc.g;
  const Geom& gf = c.lv[op.l + 1].g;
  const double* __restrict__ Tf = c.T[(op.l + 1) & 1];
  double* Tc = c.T[op.l & 1];
  int x0, y0, z0;
  tile_coords(tile, PL::TY, PL::TZ, x0, y0, z0);
  double* XR = sm;
  double* YR = sm + PL::NXR;
  const int lane = threadIdx.x, nf = gf.n, nc = gc.n;
  {
    const int cx = x0 + lane;
    const bool ok = unk1(cx, nc);
    const int tau = ok ? cx % P : 0, fx0 = 2 * cx - (2 * P - 1);
    double rw[4 * P - 1];
#pragma unroll
    for (int s = 0; s < 4 * P - 1; ++s) rw[s] = c.cf.Rw[tau][s];
    for (int rr = threadIdx.y; rr < PL::FBY * PL::FBZ; rr += NWARP) {
      int by = rr % PL::FBY, bz = rr / PL::FBY;
      int fy = 2 * y0 - (2 * P - 1) + by;
      int fz = (D == 3) ? 2 * z0 - (2 * P - 1) + bz : 0;
      double v = 0.0;
      if (ok && fy >= 0 && fy < gf.NY && fz >= 0 && fz < gf.NZ) {
        const double* rowp = Tf + ((long long)fz * gf.NY + fy) * gf.NX;
#pragma unroll
        for (int s = 0; s < 4 * P - 1; ++s) {
          int fx = fx0 + s;
          double t = unk1(fx, nf) ? rowp[fx] : 0.0;
          v = fma(rw[s], t, v);
        }
      }
      XR[rr * 32 + lane] = v;
    }
  }
  __syncthreads();
  if constexpr (D == 3) {
    for (int rr = threadIdx.y; rr < PL::TY * PL::FBZ; rr += NWARP) {
      int ty = rr % PL::TY, bz = rr / PL::TY;
      int cy = y0 + ty;
      bool ok = unk1(cy, nc);
      int tau = ok ? cy % P : 0;
      const double* xr = XR + (bz * PL::FBY + 2 * ty) * 32 + lane;
      double v = 0.0;
#pragma unroll
      for (int s = 0; s < 4 * P - 1; ++s) v = fma(c.cf.Rw[tau][s], xr[s * 32], v);
      YR[rr * 32 + lane] = ok ? v : 0.0;
    }
    __syncthreads();
  }
  double ss = 0.0;
  for (int row = threadIdx.y; row < PL::TY * PL::TZ; row += NWARP) {
    int ty = row % PL::TY, tz = row / PL::TY;
    int y = y0 + ty, z = z0 + tz, x = x0 + lane;
    if (y >= gc.NY || z >= gc.NZ) continue;
    double t = 0.0;
    if (unk1(x, nc) && unk1(y, nc) && (D == 2 || unk1(z, nc))) {
      if constexpr (D == 2) {
        int tau = y % P;
#pragma unroll
        for (int s = 0; s < 4 * P - 1; ++s) t = fma(c.cf.Rw[tau][s], XR[(2 * ty + s) * 32 + lane], t);
      } else {
        int tau = z % P;
#pragma unroll
        for (int s = 0; s < 4 * P - 1; ++s) t = fma(c.cf.Rw[tau][s], YR[((2 * tz + s) * PL::TY + ty) * 32 + lane], t);
      }
    }
    long long idx = ((long long)z * gc.NY + y) * gc.NX + x;
    Tc[idx] = t;
    ss = fma(t, t, ss);
    long long blk = idx >> 5;
    warp_encode(t, op.wr, lc.rmant + blk * lc.rstride, lc.rexp + blk, lane, c.status);
  }
  level_norm(c, lc, op.l, op.row, tile.lin, ss, op.step == 9, op.poff);
}

// Norms of t_0..t_L from the per-tile partials (fixed order).
__device__ void op_norms(const DevCtx& c, const Op& op, double* sm) {
  const int tid = threadIdx.y * 32 + threadIdx.x;
  for (int l = 0; l <= op.L; ++l) {
    const LevelDev& lv = c.lv[l];
    int n = lv.tx * lv.ty * lv.tz;
    double s = 0.0;
    for (int i = tid; i < n; i += NT) s += lv.part[i];
    sm[tid] = s;
    __syncthreads();
    for (int o = NT / 2; o > 0; o >>= 1) {
      if (tid < o) sm[tid] += sm[tid + o];
      __syncthreads();
    }
    if (tid == 0) c.norms[(long long)op.row * c.levels + l] = sqrt(sm[0]);
    __syncthreads();
  }
}

// Finalise a cFas level at one output row:
// ý = enc_wr(y); W_l = z_l + dec ý (l < L); ú_l = enc_{wu_out}(dec_{wu_in} ú_l + dec ý);
// and the next sweep's decoded u_l = dec ú_l + P_l u_{l-1} (S2).
__device__ __forceinline__ void cfas_finalize(const DevCtx& c, const Op& op, const LevelDev& lv, long long idx,
                                              double y, double pu, double zc, const uint32_t* uw_s) {
  const int lane = threadIdx.x;
  double yq = warp_encode(y, op.wr, nullptr, nullptr, lane, c.status);
  if (op.l < op.L) c.W[op.l & 1][idx] = zc + yq;
  long long blk = idx >> 5;
  double uo = warp_decode(uw_s, lv.uexp[blk], op.wu_in, lane);
  double uq = warp_encode(uo + yq, op.wu_out, lv.umant + blk * lv.ustride, lv.uexp + blk, lane, c.status);
  c.U[op.l & 1][idx] = uq + pu;
}

// P_l u_{l-1} on the output tile (for the emitted u_l): coarse box issue
// (async) and the prolongation passes (after the wait).
template <int D, int P>
__device__ void tile_pu_issue(const DevCtx& c, int l, int x0, int y0, int z0, double* scratch) {
  using PL = Plan<D, P>;
  cbox_async<D, P, PL::DCBX, PL::DCBY, PL::DCBZ>(c.U[(l - 1) & 1], c.lv[l - 1].g, x0, y0, z0, scratch);
}
template <int D, int P>
__device__ void tile_pu_compute(const DevCtx& c, int l, int x0, int y0, int z0, double* scratch, double* pu) {
  using PL = Plan<D, P>;
  double* cb = scratch;
  double* v1 = cb + PL::DCBX * PL::DCBY * PL::DCBZ;
  double* v2 = v1 + PL::DBX * PL::DCBY * PL::DCBZ;
  box_prolong_compute<D, P, PL::DBX, PL::DBY, PL::DBZ, PL::DCBX, PL::DCBY, PL::DCBZ>(c.lv[l].g.n, x0, y0, z0, c.cf,
                                                                                    cb, v1, v2, pu);
}

__device__ __forceinline__ double inv_diag(const Coefs& cf, int D, int P, int l, int x, int y, int z) {
  return cf.invd[((D == 3 ? z % P : 0) * P + y % P) * P + x % P] * pow2((l + 1) * (D - 2));
}

// smem regions of the cFas tile ops: [box0 NU][box1 NU][R1 scratch][PU][words][z]
template <int D, int P> struct CfasSmem {
  using PL = Plan<D, P>;
  double *b0, *b1, *r1, *pu, *zs;
  uint32_t* words;
  __device__ CfasSmem(double* sm) {
    b0 = sm;
    b1 = sm + PL::NU;
    r1 = sm + 2 * PL::NU;
    pu = r1 + PL::R1N;
    words = (uint32_t*)(pu + 32 * PL::NROWS);
    zs = pu + 32 * PL::NROWS + 27 * PL::NROWS;
  }
};

// S7 + S8 step 1: z = P w_{l-1} on the box, b = dec r_l - A z;
// d = inv_theta (invD b), y = d.  Writes B (and Z for l < L);
// with k == 1 finalises directly.  All global loads are issued up front.
template <int D, int P>
__device__ void tile_cfas1(const DevCtx& c, const Op& op, const TileIdx& tile, double* sm) {
  using PL = Plan<D, P>;
  const LevelDev& lv = c.lv[op.l];
  const Geom& g = lv.g;
  int x0, y0, z0;
  tile_coords(tile, PL::TY, PL::TZ, x0, y0, z0);
  CfasSmem<D, P> S(sm);
  double* U = S.b0;
  double* cb = S.r1;
  double* v1 = cb + PL::NCB;
  double* v2 = v1 + PL::NV1;
  uint32_t* rw = S.words;
  cbox_async<D, P, PL::CBX, PL::CBY, PL::CBZ>(c.W[(op.l - 1) & 1], c.lv[op.l - 1].g, x0 - P, y0 - P, z0 - P, cb);
  rows_words_async<D, P>(lv.rmant, lv.rstride, op.wr, g, x0, y0, z0, rw);
  cpa_wait_sync();
  box_prolong_compute<D, P, PL::BX, PL::BY, PL::BZ, PL::CBX, PL::CBY, PL::CBZ>(g.n, x0 - P, y0 - P, z0 - P, c.cf,
                                                                              cb, v1, v2, U);
  double* AB = S.r1;
  double* CS = S.r1 + 2 * PL::NAB;
  a_stages<D, P>(g, x0, y0, c.cf, U, AB, CS);
  const int lane = threadIdx.x;
  double bsave[(PL::NROWS + NWARP - 1) / NWARP], zsave[(PL::NROWS + NWARP - 1) / NWARP];
  int k = 0;
  for (int row = threadIdx.y; row < PL::NROWS; row += NWARP, ++k) {
    int ty = row % PL::TY, tz = row / PL::TY;
    int y = y0 + ty, z = z0 + tz, x = x0 + lane;
    bsave[k] = 0.0;
    zsave[k] = 0.0;
    if (y >= g.NY || z >= g.NZ) continue;
    double az = a_final<D, P>(g, x0, y0, z0, ty, tz, c.cf, AB, CS);
    long long idx = ((long long)z * g.NY + y) * g.NX + x;
    long long blk = idx >> 5;
    double rv = warp_decode(rw + row * lv.rstride, lv.rexp[blk], op.wr, lane);
    double b = rv - az;
    double zc = U[((tz + ((D == 3) ? P : 0)) * PL::BY + ty + P) * PL::BX + P + lane];
    if (op.l < op.L) c.Z[idx] = zc;
    if (!op.last) c.B[idx] = b;
    bsave[k] = b;
    zsave[k] = zc;
  }
  if (!op.last) return;
  // k == 1: y = d_1; emitted u_l needs P u_{l-1}
  __syncthreads();
  uint32_t* uw = S.words;
  tile_pu_issue<D, P>(c, op.l, x0, y0, z0, S.r1);
  rows_words_async<D, P>(lv.umant, lv.ustride, op.wu_in, g, x0, y0, z0, uw);
  cpa_wait_sync();
  tile_pu_compute<D, P>(c, op.l, x0, y0, z0, S.r1, S.pu);
  k = 0;
  for (int row = threadIdx.y; row < PL::NROWS; row += NWARP, ++k) {
    int ty = row % PL::TY, tz = row / PL::TY;
    int y = y0 + ty, z = z0 + tz, x = x0 + lane;
    if (y >= g.NY || z >= g.NZ) continue;
    bool unk = unk1(x, g.n) && unk1(y, g.n) && (D == 2 || unk1(z, g.n));
    long long idx = ((long long)z * g.NY + y) * g.NX + x;
    double invD = unk ? inv_diag(c.cf, D, P, op.l, x, y, z) : 0.0;
    double d = c.cf.inv_theta * (invD * bsave[k]);
    cfas_finalize(c, op, lv, idx, d, S.pu[row * 32 + lane], zsave[k], uw + row * lv.ustride);
  }
}

// S8 step j >= 2: q = b - A y, d = fma(alpha_j, d, beta_j (invD q)), y = y + d.
// Step 2 reconstructs y_1 = d_1 = inv_theta (invD b) from the b box (no Y/D
// arrays for k = 2); later steps read Y/Dv.  Last step finalises (S9, S10) and
// emits u_l.  All global loads (b/y box, coarse u box, ú words, z rows) are
// issued up front and awaited once.
template <int D, int P>
__device__ void tile_cheb(const DevCtx& c, const Op& op, const TileIdx& tile, double* sm) {
  using PL = Plan<D, P>;
  const LevelDev& lv = c.lv[op.l];
  const Geom& g = lv.g;
  int x0, y0, z0;
  tile_coords(tile, PL::TY, PL::TZ, x0, y0, z0);
  CfasSmem<D, P> S(sm);
  double* Bb = S.b0;  // raw b box (step 2)
  double* Yb = S.b1;  // y box
  const int lane = threadIdx.x;
  if (op.step == 2) box_async<D, P>(c.B, g, x0, y0, z0, Bb);
  else box_async<D, P>(c.Y[op.step & 1], g, x0, y0, z0, Yb);
  if (op.last) {
    tile_pu_issue<D, P>(c, op.l, x0, y0, z0, S.r1);
    rows_words_async<D, P>(lv.umant, lv.ustride, op.wu_in, g, x0, y0, z0, S.words);
    if (op.l < op.L) {
      for (int r = threadIdx.y; r < PL::NROWS; r += NWARP) {
        int y = y0 + r % PL::TY, z = z0 + r / PL::TY;
        bool ok = y < g.NY && z < g.NZ;
        const double* src = c.Z + ((long long)z * g.NY + y) * g.NX + x0 + lane;
        cpa8(S.zs + r * 32 + lane, ok ? src : c.Z, ok);
      }
    }
  }
  cpa_wait_sync();
  if (op.step == 2) {
    const double sc = pow2((op.l + 1) * (D - 2));
    for (int i = threadIdx.y * 32 + lane; i < PL::NU; i += NT) {
      int bx = i % PL::BX, r = i / PL::BX;
      int gy = y0 - P + r % PL::BY, gz = (D == 3) ? z0 - P + r / PL::BY : 0, gx = x0 - P + bx;
      bool ok = unk1(gx, g.n) && unk1(gy, g.n) && (D == 2 || unk1(gz, g.n));
      int t = ((D == 3 ? (ok ? gz % P : 0) : 0) * P + (ok ? gy % P : 0)) * P + (ok ? gx % P : 0);
      Yb[i] = ok ? c.cf.inv_theta * ((c.cf.invd[t] * sc) * Bb[i]) : 0.0;
    }
    __syncthreads();
  }
  if (op.last) tile_pu_compute<D, P>(c, op.l, x0, y0, z0, S.r1, S.pu);
  double* AB = S.r1;
  double* CS = S.r1 + 2 * PL::NAB;
  a_stages<D, P>(g, x0, y0, c.cf, Yb, AB, CS);
  for (int row = threadIdx.y; row < PL::NROWS; row += NWARP) {
    int ty = row % PL::TY, tz = row / PL::TY;
    int y = y0 + ty, z = z0 + tz, x = x0 + lane;
    if (y >= g.NY || z >= g.NZ) continue;
    double ay = a_final<D, P>(g, x0, y0, z0, ty, tz, c.cf, AB, CS);
    bool unk = unk1(x, g.n) && unk1(y, g.n) && (D == 2 || unk1(z, g.n));
    long long idx = ((long long)z * g.NY + y) * g.NX + x;
    double invD = unk ? inv_diag(c.cf, D, P, op.l, x, y, z) : 0.0;
    const int ci = ((tz + ((D == 3) ? P : 0)) * PL::BY + ty + P) * PL::BX + P + lane;
    double b = (op.step == 2) ? Bb[ci] : c.B[idx];
    double q = b - ay;
    double yprev = Yb[ci];
    double dprev = (op.step == 2) ? yprev : c.Dv[idx];
    double d = fma(c.cf.cal[op.step - 1], dprev, c.cf.cbe[op.step - 1] * (invD * q));
    double yv = yprev + d;
    if (op.last) {
      cfas_finalize(c, op, lv, idx, yv, S.pu[row * 32 + lane], (op.l < op.L) ? S.zs[row * 32 + lane] : 0.0,
                    S.words + row * lv.ustride);
    } else {
      c.Y[(op.step + 1) & 1][idx] = yv;
      c.Dv[idx] = d;
    }
  }
}

template <int D, int P>
__device__ __forceinline__ void run_op(const DevCtx& c, const Op& op, const TileIdx& tile, double* sm) {
  switch (op.type) {
    case OP_DECODE: tile_decode<D, P>(c, op, tile, sm); break;
    case OP_RESIDUAL: tile_residual<D, P>(c, op, tile, sm); break;
    case OP_RESTRICT: tile_restrict<D, P>(c, op, tile, sm); break;
    case OP_NORMS: op_norms(c, op, sm); break;
    case OP_CFAS1: tile_cfas1<D, P>(c, op, tile, sm); break;
    case OP_CHEB: tile_cheb<D, P>(c, op, tile, sm); break;
  }
}

// Grid kernel: one CTA per tile of one operation.  The device context lives in
// global memory and is read through the read-only path (uniform, L1-cached).
template <int D, int P>
#ifndef FMG_KOP_MINB
#define FMG_KOP_MINB 4
#endif
__global__ void __launch_bounds__(NT, FMG_KOP_MINB) k_op(const DevCtx* __restrict__ cp, Op op) {
  extern __shared__ double sm[];
  pdl_wait();
  pdl_trigger();
  const DevCtx& c = *cp;
  TileIdx t{(int)blockIdx.x, (int)blockIdx.y, (int)blockIdx.z,
            (int)((blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x)};
  run_op<D, P>(c, op, t, sm);
}

// =============================================== K4: coarse hierarchy ======
// One 512-thread CTA owns levels 0..lc, stored densely (n_l^d doubles, x
// fastest, no padding) in shared memory: the restriction tail, the norms, the
// exact coarse solve, the cFas sweep with the corrections and the emitted u_l
// of those levels run back to back with only __syncthreads between phases (no
// launch gaps, no global round trips).  Same canonical expression trees as the
// tile ops.  For FMG levels L <= lc the whole IR iteration
// (residual included) runs here.
constexpr int NW4 = 16, NT4 = 32 * NW4;
constexpr int K4_MAX_SMEM = 210 * 1024;  // dynamic smem budget of the K4 CTA
constexpr int K4_AINV_MAX = 4096;         // A_0^{-1} entries staged in smem

using K4Args = K4Desc;

__host__ __device__ inline int ipow(int n, int d) { return d == 3 ? n * n * n : n * n; }

// smem offsets (doubles): per level U, T, RQ, W blocks, then 6 scratch arrays of the top level
__host__ __device__ inline int k4_level_off(int D, int P, int l) {
  int o = 0;
  for (int k = 0; k < l; ++k) o += 4 * ipow(P << (k + 1), D);
  return o;
}
__host__ __device__ inline int k4_smem_doubles(int D, int P, int lc) {
  return k4_level_off(D, P, lc + 1) + 6 * ipow(P << (lc + 1), D);
}

struct K4Lvl {
  int n, len;
  double *U, *T, *RQ, *W;
};

__device__ __forceinline__ K4Lvl k4_lvl(int D, int P, int l, double* sm) {
  K4Lvl v;
  v.n = P << (l + 1);
  v.len = ipow(v.n, D);
  // offset of level l: 4 * sum_{k<l} (P 2^(k+1))^D  (geometric sum)
  const int r = D == 3 ? 8 : 4;                         // ratio between consecutive levels
  const int first = ipow(2 * P, D);
  double* b = sm + 4 * first * ((l == 0) ? 0 : ((1 << (D * l)) - 1) / (r - 1));
  v.U = b;
  v.T = b + v.len;
  v.RQ = b + 2 * v.len;
  v.W = b + 3 * v.len;
  return v;
}

__device__ __forceinline__ double rd(const double* a, int j, int n) { return (j >= 0 && j < n) ? a[j] : 0.0; }

// Final-pass iteration helper: warps walk (row, 32-entry block) pairs of a
// dense level so that each warp holds one BFP block (x = xb*32 + lane, values
// beyond n are 0) -- epilogues may then encode/decode with warp collectives.
#define K4_BLOCKS(n, rows)                                                        \
  for (int rb = threadIdx.y, nxb_ = ((n) + 31) >> 5; rb < (rows) * nxb_; rb += NW4) \
    for (int r = rb / nxb_, x = (rb % nxb_) * 32 + (int)threadIdx.x, once_ = 1; once_; once_ = 0)

// A_l in (dense), canonical passes; the last pass calls
// epi(r, x, Av) per point (Av = 0 at non-unknowns and beyond n), warp-aligned.
template <int D, int P, class Epi>
__device__ void k4_A(const Coefs& cf, int l, int n, const double* in, double* s, Epi epi) {
  const int lane = threadIdx.x, w = threadIdx.y, len = ipow(n, D), rows = len / n;
  double* a = s;
  double* b = s + len;
  for (int r = w; r < rows; r += NW4)
    for (int x = lane; x < n; x += 32) {
      const double* u = in + r * n;
      bool ok = unk1(x, n);
      int tau = ok ? x % P : 0;
      double aa = 0.0, bb = 0.0;
#pragma unroll
      for (int o = 0; o <= 2 * P; ++o) {
        double v = rd(u, x - P + o, n);
        aa = fma(cf.Mc[tau][o], v, aa);
        bb = fma(cf.Kc[tau][o], v, bb);
      }
      a[r * n + x] = ok ? aa : 0.0;
      b[r * n + x] = ok ? bb : 0.0;
    }
  __syncthreads();
  if constexpr (D == 2) {
    K4_BLOCKS(n, n) {
      const int y = r;
      bool ok = unk1(y, n) && unk1(x, n);
      int tau = unk1(y, n) ? y % P : 0, xs = x < n ? x : 0;
      double d = 0.0, e = 0.0;
#pragma unroll
      for (int o = 0; o <= 2 * P; ++o) {
        int j = y - P + o;
        bool in_ = j >= 0 && j < n;
        d = fma(cf.Kc[tau][o], in_ ? a[j * n + xs] : 0.0, d);
        e = fma(cf.Mc[tau][o], in_ ? b[j * n + xs] : 0.0, e);
      }
      epi(r, x, ok ? d + e : 0.0);
    }
  } else {
    double* c = s + 2 * len;
    double* sv = s + 3 * len;
    for (int r = w; r < n * n; r += NW4) {  // rows (z, y)
      int y = r % n, z = r / n;
      bool oky = unk1(y, n);
      int tau = oky ? y % P : 0;
      for (int x = lane; x < n; x += 32) {
        double cc = 0.0, dd = 0.0, e = 0.0;
#pragma unroll
        for (int o = 0; o <= 2 * P; ++o) {
          int j = y - P + o;
          bool in_ = j >= 0 && j < n;
          double av = in_ ? a[(z * n + j) * n + x] : 0.0, bv = in_ ? b[(z * n + j) * n + x] : 0.0;
          cc = fma(cf.Mc[tau][o], av, cc);
          dd = fma(cf.Kc[tau][o], av, dd);
          e = fma(cf.Mc[tau][o], bv, e);
        }
        c[r * n + x] = oky ? cc : 0.0;
        sv[r * n + x] = oky ? dd + e : 0.0;
      }
    }
    __syncthreads();
    const double h = pow2(-(l + 1));
    K4_BLOCKS(n, n * n) {
      int y = r % n, z = r / n, xs = x < n ? x : 0;
      bool ok = unk1(z, n) && unk1(y, n) && unk1(x, n);
      int tau = unk1(z, n) ? z % P : 0;
      double acc = 0.0;
#pragma unroll
      for (int o = 0; o <= 2 * P; ++o) {
        int j = z - P + o;
        acc = fma(cf.Kc[tau][o], (j >= 0 && j < n) ? c[(j * n + y) * n + xs] : 0.0, acc);
      }
#pragma unroll
      for (int o = 0; o <= 2 * P; ++o) {
        int j = z - P + o;
        acc = fma(cf.Mc[tau][o], (j >= 0 && j < n) ? sv[(j * n + y) * n + xs] : 0.0, acc);
      }
      epi(r, x, ok ? acc * h : 0.0);
    }
  }
  __syncthreads();
}

// f1 = P c1 and (if c2) f2 = P c2 on the fine level nf, one set of passes
// (DESIGN.md §3.3).  scratch: 2 * (len_f/2^(d-1) + len_f/2).
template <int D, int P>
__device__ void k4_P2(const Coefs& cf, int nf, const double* c1, double* f1, const double* c2, double* f2, double* s) {
  const int lane = threadIdx.x, w = threadIdx.y, nc = nf / 2;
  const int nv = c2 ? 2 : 1;
  const int n1 = (D == 3) ? nc * nc * nf : nc * nf;  // x-pass size
  const int n2 = (D == 3) ? nc * nf * nf : 0;        // y-pass size (3D)
  const int rows1 = (D == 3) ? nc * nc : nc;
  for (int r = w; r < nv * rows1; r += NW4) {
    int k = r / rows1, rr = r % rows1;
    const double* cs = (k == 0 ? c1 : c2) + rr * nc;
    double* t1 = s + k * n1;
    for (int x = lane; x < nf; x += 32) {
      bool ok = unk1(x, nf);
      int rx = ok ? x % (2 * P) : 0, base = ok ? P * (x / (2 * P)) : 0;
      double acc = 0.0;
#pragma unroll
      for (int t = 0; t <= P; ++t) acc = fma(cf.Pw[rx][t], rd(cs, base + t, nc), acc);
      t1[rr * nf + x] = ok ? acc : 0.0;
    }
  }
  __syncthreads();
  const int rows2 = (D == 3) ? nc * nf : nf;
  for (int r = w; r < nv * rows2; r += NW4) {
    int k = r / rows2, rr = r % rows2;
    const double* t1 = s + k * n1;
    double* t2 = (D == 3) ? s + 2 * n1 + k * n2 : (k == 0 ? f1 : f2);
    int y = rr % nf, cz = rr / nf;
    bool ok = unk1(y, nf);
    int ry = ok ? y % (2 * P) : 0, base = ok ? P * (y / (2 * P)) : 0;
    for (int x = lane; x < nf; x += 32) {
      double acc = 0.0;
#pragma unroll
      for (int t = 0; t <= P; ++t) {
        int j = base + t;
        acc = fma(cf.Pw[ry][t], (j < nc) ? t1[(cz * nc + j) * nf + x] : 0.0, acc);
      }
      t2[rr * nf + x] = ok ? acc : 0.0;
    }
  }
  __syncthreads();
  if constexpr (D == 3) {
    for (int r = w; r < nv * nf * nf; r += NW4) {
      int k = r / (nf * nf), rr = r % (nf * nf);
      const double* t2 = s + 2 * n1 + k * n2;
      double* fo = k == 0 ? f1 : f2;
      int y = rr % nf, z = rr / nf;
      bool ok = unk1(z, nf);
      int rz = ok ? z % (2 * P) : 0, base = ok ? P * (z / (2 * P)) : 0;
      for (int x = lane; x < nf; x += 32) {
        double acc = 0.0;
#pragma unroll
        for (int t = 0; t <= P; ++t) {
          int j = base + t;
          acc = fma(cf.Pw[rz][t], (j < nc) ? t2[(j * nf + y) * nf + x] : 0.0, acc);
        }
        fo[rr * nf + x] = ok ? acc : 0.0;
      }
    }
    __syncthreads();
  }
}

// coarse = R fine; fine given by (ptr, row stride sy, plane
// stride sz), x < nf valid.  The last pass calls epi(r, x, t) warp-aligned.
// scratch: nc*nf^(d-1) + nc^2*nf (3D).
template <int D, int P, class Epi>
__device__ void k4_R(const Coefs& cf, int nf, const double* fine, long long sy, long long sz, double* s, Epi epi) {
  const int lane = threadIdx.x, w = threadIdx.y, nc = nf / 2;
  double* t1 = s;  // [zf][yf][xc]
  const int rows1 = (D == 3) ? nf * nf : nf;
  for (int r = w; r < rows1; r += NW4) {
    int yf = r % nf, zf = r / nf;
    const double* row = fine + (long long)zf * sz + (long long)yf * sy;
    for (int x = lane; x < nc; x += 32) {
      bool ok = unk1(x, nc);
      int tau = ok ? x % P : 0;
      double acc = 0.0;
#pragma unroll
      for (int t = 0; t <= 4 * P - 2; ++t) {
        int j = 2 * x - (2 * P - 1) + t;
        acc = fma(cf.Rw[tau][t], (j >= 0 && j < nf) ? row[j] : 0.0, acc);
      }
      t1[r * nc + x] = ok ? acc : 0.0;
    }
  }
  __syncthreads();
  if constexpr (D == 2) {
    K4_BLOCKS(nc, nc) {
      const int yc = r, xs = x < nc ? x : 0;
      bool ok = unk1(yc, nc) && unk1(x, nc);
      int tau = unk1(yc, nc) ? yc % P : 0;
      double acc = 0.0;
#pragma unroll
      for (int t = 0; t <= 4 * P - 2; ++t) {
        int j = 2 * yc - (2 * P - 1) + t;
        acc = fma(cf.Rw[tau][t], (j >= 0 && j < nf) ? t1[j * nc + xs] : 0.0, acc);
      }
      epi(r, x, ok ? acc : 0.0);
    }
  } else {
    double* t2 = s + nf * nf * nc;  // [zf][yc][xc]
    for (int r = w; r < nf * nc; r += NW4) {
      int yc = r % nc, zf = r / nc;
      bool ok = unk1(yc, nc);
      int tau = ok ? yc % P : 0;
      for (int x = lane; x < nc; x += 32) {
        double acc = 0.0;
#pragma unroll
        for (int t = 0; t <= 4 * P - 2; ++t) {
          int j = 2 * yc - (2 * P - 1) + t;
          acc = fma(cf.Rw[tau][t], (j >= 0 && j < nf) ? t1[(zf * nf + j) * nc + x] : 0.0, acc);
        }
        t2[r * nc + x] = ok ? acc : 0.0;
      }
    }
    __syncthreads();
    K4_BLOCKS(nc, nc * nc) {
      int yc = r % nc, zc = r / nc, xs = x < nc ? x : 0;
      bool ok = unk1(zc, nc) && unk1(yc, nc) && unk1(x, nc);
      int tau = unk1(zc, nc) ? zc % P : 0;
      double acc = 0.0;
#pragma unroll
      for (int t = 0; t <= 4 * P - 2; ++t) {
        int j = 2 * zc - (2 * P - 1) + t;
        acc = fma(cf.Rw[tau][t], (j >= 0 && j < nf) ? t2[(j * nc + yc) * nc + xs] : 0.0, acc);
      }
      epi(r, x, ok ? acc : 0.0);
    }
  }
  __syncthreads();
}

// BFP block of dense level row r, block x/32 (global padded layout).
__device__ __forceinline__ long long k4_blk(const LevelDev& lv, int r, int x) {
  return (long long)r * (lv.g.NX >> 5) + (x >> 5);
}

// Copy a dense level into a padded global array (zeros in the padding).
__device__ void k4_to_global(int D, int n, const double* v, double* g, const Geom& gg) {
  const int rows = (D == 3) ? n * n : n;
  for (int r = threadIdx.y; r < rows; r += NW4)
    for (int x = threadIdx.x; x < gg.NX; x += 32) g[(long long)r * gg.NX + x] = x < n ? v[r * n + x] : 0.0;
}

__device__ __forceinline__ double k4_invd_at(const Coefs& cf, int D, int P, int l, int n, int r, int x) {
  int y = r % n, z = (D == 3) ? r / n : 0;
  if (!unk1(x, n) || !unk1(y, n) || (D == 3 && !unk1(z, n))) return 0.0;
  return cf.invd[((D == 3 ? z % P : 0) * P + y % P) * P + x % P] * pow2((l + 1) * (D - 2));
}

// Optional phase timestamps (debug): thread 0 records globaltimer after phases.
__device__ unsigned long long g_k4_stamps[64];
__device__ int g_k4_debug = 0;
__device__ __forceinline__ void k4_stamp(int i) {
  if (g_k4_debug && threadIdx.x == 0 && threadIdx.y == 0 && i < 64) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_k4_stamps[i] = t;
  }
}

template <int D, int P>
__global__ void __launch_bounds__(NT4, 1) k4_kernel(const DevCtx* __restrict__ cp, K4Args a) {
  extern __shared__ double sm[];
  __shared__ double red[kMaxLev * NW4];
  pdl_wait();
  pdl_trigger();
  const DevCtx& c = *cp;
  const Coefs& cf = c.cf;
  const int tid = threadIdx.y * 32 + threadIdx.x, lane = threadIdx.x;
  const int lc = c.lc;
  int stamp = 0;
  k4_stamp(stamp++);
  const int L = a.L, lce = L < lc ? L : lc;
  double* scr = sm + k4_level_off(D, P, lc + 1);
  const int lenc = ipow(P << (lc + 1), D);
  double* S0 = scr;              // pass scratch (4 arrays)
  double* SZ = scr + 4 * lenc;   // z_l
  double* SB = scr + 5 * lenc;   // Chebyshev direction d
  // Shared-memory staging of the sections of levels 0..lc (read once in the
  // prologue, written back once in the epilogue) and of A_0^{-1}.
  __shared__ uint32_t* s_uw[kMaxLev];
  __shared__ uint32_t* s_rw[kMaxLev];
  __shared__ int8_t* s_ue[kMaxLev];
  __shared__ int8_t* s_re[kMaxLev];
  __shared__ const double* s_ainv;
  if (tid == 0) {
    char* p = (char*)(scr + 6 * lenc);
    for (int l = 0; l <= lc; ++l) {
      const LevelDev& lv = c.lv[l];
      s_uw[l] = (uint32_t*)p;
      p += 4 * lv.g.nblk * lv.ustride;
      s_rw[l] = (uint32_t*)p;
      p += 4 * lv.g.nblk * lv.rstride;
    }
    for (int l = 0; l <= lc; ++l) {
      const LevelDev& lv = c.lv[l];
      s_ue[l] = (int8_t*)p;
      p += lv.g.nblk;
      s_re[l] = (int8_t*)p;
      p += lv.g.nblk;
    }
    p = (char*)(((uintptr_t)p + 15) & ~(uintptr_t)15);
    s_ainv = (c.n0 * c.n0 <= K4_AINV_MAX) ? (const double*)p : c.Ainv;
  }
  __syncthreads();
  if (a.mode == 0) {
    // ú_0 = reg(A_0^{-1} f_0); u_0 = dec ú_0
    K4Lvl v0 = k4_lvl(D, P, 0, sm);
    const int n = v0.n, m = 2 * P - 1;
    const LevelDev& lv = c.lv[0];
    for (int e = tid; e < v0.len; e += NT4) {
      int x = e % n, y = (e / n) % n, z = (D == 3) ? e / (n * n) : 0;
      double f = 0.0;
      if (unk1(x, n) && unk1(y, n) && (D == 2 || unk1(z, n))) {
        f = cf.rhs_c * lv.gtab[x];
        f = f * lv.gtab[y];
        if (D == 3) f = f * lv.gtab[z];
      }
      v0.T[e] = f;
      v0.W[e] = 0.0;
    }
    __syncthreads();
    for (int I = tid; I < c.n0; I += NT4) {
      double acc = 0.0;
      for (int J = 0; J < c.n0; ++J) {
        int jx = J % m + 1, jy = (J / m) % m + 1, jz = (D == 3) ? J / (m * m) + 1 : 0;
        acc = fma(c.Ainv[(long long)I * c.n0 + J], v0.T[(jz * n + jy) * n + jx], acc);
      }
      int ix = I % m + 1, iy = (I / m) % m + 1, iz = (D == 3) ? I / (m * m) + 1 : 0;
      v0.W[(iz * n + iy) * n + ix] = acc;
    }
    __syncthreads();
    K4_BLOCKS(n, v0.len / n) {
      long long blk = k4_blk(lv, r, x);
      double val = x < n ? v0.W[r * n + x] : 0.0;
      double q = warp_encode(val, a.wu_out[0], lv.umant + blk * lv.ustride, lv.uexp + blk, lane, c.status);
      if (x < n) v0.U[r * n + x] = q;
    }
    __syncthreads();
    for (int e = tid; e < v0.len; e += NT4) c.usm[c.usm_off[0] + e] = v0.U[e];
    if (lc == 0) k4_to_global(D, n, v0.U, c.U[0], lv.g);
    return;
  }

  // ---- prologue: one round of coalesced loads (ú sections, A_0^{-1}, and in 2D
  //      the fine-level t_{lc+1} feeding the first restriction)
  for (int l = 0; l <= lce; ++l) {
    const LevelDev& lv = c.lv[l];
    const int nw = (int)(lv.g.nblk * lv.ustride);
    for (int i = tid; i < nw; i += NT4) s_uw[l][i] = lv.umant[i];
    for (int i = tid; i < (int)lv.g.nblk; i += NT4) s_ue[l][i] = lv.uexp[i];
  }
  if (s_ainv != c.Ainv)
    for (int i = tid; i < c.n0 * c.n0; i += NT4) ((double*)s_ainv)[i] = c.Ainv[i];
  const bool stage_fine = D == 2 && L > lc &&
                          (long long)c.lv[lc + 1].g.NX * c.lv[lc + 1].g.NY <= 4LL * lenc;
  if (stage_fine) {
    const Geom& gf = c.lv[lc + 1].g;
    const double* src = c.T[(lc + 1) & 1];
    const int nt = gf.NX * gf.NY;
    for (int i = tid; i < nt; i += NT4) S0[i] = src[i];
  }
  __syncthreads();

  if (L <= lc) {
    // ---- residual inside K4: u_L (persisted or P u_{L-1}), t_L = f_L - A_L u_L,
    //      r_L = enc(t_L)
    K4Lvl vL = k4_lvl(D, P, L, sm);
    if (a.first) {
      K4Lvl vp = k4_lvl(D, P, L - 1, sm);
      for (int e = tid; e < vp.len; e += NT4) vp.U[e] = c.usm[c.usm_off[L - 1] + e];
      __syncthreads();
      k4_P2<D, P>(cf, vL.n, vp.U, vL.U, nullptr, nullptr, S0);
    } else {
      for (int e = tid; e < vL.len; e += NT4) vL.U[e] = c.usm[c.usm_off[L] + e];
      __syncthreads();
    }
    const LevelDev& lv = c.lv[L];
    const int n = vL.n;
    k4_A<D, P>(cf, L, n, vL.U, S0, [&](int r, int x, double au) {
      int y = r % n, z = (D == 3) ? r / n : 0;
      double t = 0.0;
      if (x < n && unk1(x, n) && unk1(y, n) && (D == 2 || unk1(z, n))) {
        double f = cf.rhs_c * lv.gtab[x];
        f = f * lv.gtab[y];
        if (D == 3) f = f * lv.gtab[z];
        t = f - au;
      }
      long long blk = k4_blk(lv, r, x);
      double q = warp_encode(t, a.wr[L], s_rw[L] + blk * lv.rstride, s_re[L] + blk, lane, c.status);
      if (x < n) {
        vL.T[r * n + x] = t;
        vL.RQ[r * n + x] = q;
      }
    });
  } else {
    // ---- restriction from the grid level lc+1 (global t_{lc+1})
    K4Lvl vc = k4_lvl(D, P, lc, sm);
    const Geom& gf = c.lv[lc + 1].g;
    const LevelDev& lv = c.lv[lc];
    const int n = vc.n;
    const double* fine = stage_fine ? S0 : c.T[(lc + 1) & 1];
    double* rscr = stage_fine ? S0 + 4 * lenc : S0;  // 2D: t1 (2 lenc) after the staged fine level
    k4_R<D, P>(cf, gf.n, fine, gf.NX, (long long)gf.NX * gf.NY, rscr, [&](int r, int x, double t) {
      long long blk = k4_blk(lv, r, x);
      double q = warp_encode(t, a.wr[lc], s_rw[lc] + blk * lv.rstride, s_re[lc] + blk, lane, c.status);
      if (x < n) {
        vc.T[r * n + x] = t;
        vc.RQ[r * n + x] = q;
      }
    });
  }
  k4_stamp(stamp++);
  // ---- restriction sweep inside smem, r_l = enc(t_l)
  for (int l = lce - 1; l >= 0; --l) {
    K4Lvl vf = k4_lvl(D, P, l + 1, sm), vc = k4_lvl(D, P, l, sm);
    const LevelDev& lv = c.lv[l];
    const int n = vc.n;
    k4_R<D, P>(cf, vf.n, vf.T, vf.n, (long long)vf.n * vf.n, S0, [&](int r, int x, double t) {
      long long blk = k4_blk(lv, r, x);
      double q = warp_encode(t, a.wr[l], s_rw[l] + blk * lv.rstride, s_re[l] + blk, lane, c.status);
      if (x < n) {
        vc.T[r * n + x] = t;
        vc.RQ[r * n + x] = q;
      }
    });
  }
  k4_stamp(stamp++);
  // ---- norms ||t_l||_2 of the smem levels (grid levels: deferred, k_norms_all)
  for (int l = 0; l <= lce; ++l) {
    K4Lvl v = k4_lvl(D, P, l, sm);
    double sacc = 0.0;
    for (int e = tid; e < v.len; e += NT4) sacc = fma(v.T[e], v.T[e], sacc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sacc += __shfl_xor_sync(FULL, sacc, o);
    if (lane == 0) red[l * NW4 + threadIdx.y] = sacc;
  }
  // ---- coarse level (reading R5): ý_0 = enc(A_0^{-1} dec r_0);
  //      w_0 = dec ý_0; ú_0 = enc(dec ú_0 + dec ý_0); u_0 = dec ú_0
  {
    K4Lvl v0 = k4_lvl(D, P, 0, sm);
    const int n = v0.n, m = 2 * P - 1;
    for (int e = tid; e < v0.len; e += NT4) SB[e] = 0.0;
    __syncthreads();
    if (tid <= lce) {
      double sacc = 0.0;
      for (int i = 0; i < NW4; ++i) sacc += red[tid * NW4 + i];
      c.norms[(long long)a.row * c.levels + tid] = sqrt(sacc);
    }
    for (int I = tid; I < c.n0; I += NT4) {
      double acc = 0.0;
      for (int J = 0; J < c.n0; ++J) {
        int jx = J % m + 1, jy = (J / m) % m + 1, jz = (D == 3) ? J / (m * m) + 1 : 0;
        acc = fma(s_ainv[(long long)I * c.n0 + J], v0.RQ[(jz * n + jy) * n + jx], acc);
      }
      int ix = I % m + 1, iy = (I / m) % m + 1, iz = (D == 3) ? I / (m * m) + 1 : 0;
      SB[(iz * n + iy) * n + ix] = acc;
    }
    __syncthreads();
    const LevelDev& lv = c.lv[0];
    K4_BLOCKS(n, v0.len / n) {
      long long blk = k4_blk(lv, r, x);
      double y = x < n ? SB[r * n + x] : 0.0;
      double yq = warp_encode(y, a.wr[0], nullptr, nullptr, lane, c.status);
      uint32_t* uw = s_uw[0] + blk * lv.ustride;
      double uo = warp_decode(uw, s_ue[0][blk], a.wu_in[0], lane);
      double uq = warp_encode(uo + yq, a.wu_out[0], uw, s_ue[0] + blk, lane, c.status);
      if (x < n) {
        v0.W[r * n + x] = yq;
        v0.U[r * n + x] = uq;
      }
    }
    __syncthreads();
  }
  k4_stamp(stamp++);
  // ---- coarse-to-fine sweep, Chebyshev-Jacobi,
  //      correction and the next sweep's u_l, fused per level
  const int k = c.n_cheb;
  for (int l = 1; l <= lce; ++l) {
    K4Lvl vp = k4_lvl(D, P, l - 1, sm), v = k4_lvl(D, P, l, sm);
    const int n = v.n;
    const LevelDev& lv = c.lv[l];
    double* Y = v.T;    // t_l is dead: Chebyshev iterate
    double* PU = v.U;   // P u_{l-1} (new), then the emitted u_l
    k4_P2<D, P>(cf, n, vp.W, SZ, vp.U, PU, S0);  // z_l = P w_{l-1}; P u_{l-1}
    k4_stamp(stamp++);
    auto finalize = [&](int r, int x, double y) {
      // ý_l = enc_wr(y); w_l = z_l + dec ý; ú_l = enc(dec ú_l + dec ý); u_l = dec ú_l + P u_{l-1}
      long long blk = k4_blk(lv, r, x);
      double yq = warp_encode(y, a.wr[l], nullptr, nullptr, lane, c.status);
      uint32_t* uw = s_uw[l] + blk * lv.ustride;
      double uo = warp_decode(uw, s_ue[l][blk], a.wu_in[l], lane);
      double uq = warp_encode(uo + yq, a.wu_out[l], uw, s_ue[l] + blk, lane, c.status);
      if (x < n) {
        v.W[r * n + x] = SZ[r * n + x] + yq;
        PU[r * n + x] = uq + PU[r * n + x];
      }
    };
    // b = dec r_l - A z_l; d_1 = inv_theta (invD b); y_1 = d_1
    k4_A<D, P>(cf, l, n, SZ, S0, [&](int r, int x, double az) {
      double b = 0.0, d = 0.0;
      if (x < n) {
        b = v.RQ[r * n + x] - az;
        d = cf.inv_theta * (k4_invd_at(cf, D, P, l, n, r, x) * b);
      }
      if (k == 1) {
        finalize(r, x, d);
      } else if (x < n) {
        v.RQ[r * n + x] = b;
        SB[r * n + x] = d;
        Y[r * n + x] = d;
      }
    });
    k4_stamp(stamp++);
    for (int j = 2; j <= k; ++j) {
      // q = b - A y; d_j = fma(alpha_j, d_{j-1}, beta_j (invD q)); y_j = y_{j-1} + d_j
      k4_A<D, P>(cf, l, n, Y, S0, [&](int r, int x, double ay) {
        double y = 0.0;
        if (x < n) {
          double q = v.RQ[r * n + x] - ay;
          double d = fma(cf.cal[j - 1], SB[r * n + x], cf.cbe[j - 1] * (k4_invd_at(cf, D, P, l, n, r, x) * q));
          y = Y[r * n + x] + d;
          if (j < k) {
            SB[r * n + x] = d;
            Y[r * n + x] = y;
          }
        }
        if (j == k) finalize(r, x, y);
      });
      k4_stamp(stamp++);
    }
  }
  // ---- epilogue: sections back to global (one round of coalesced stores)
  for (int l = 0; l <= lce; ++l) {
    const LevelDev& lv = c.lv[l];
    const int nu = (int)(lv.g.nblk * lv.ustride), nr = (int)(lv.g.nblk * lv.rstride);
    for (int i = tid; i < nu; i += NT4) lv.umant[i] = s_uw[l][i];
    for (int i = tid; i < nr; i += NT4) lv.rmant[i] = s_rw[l][i];
    for (int i = tid; i < (int)lv.g.nblk; i += NT4) {
      lv.uexp[i] = s_ue[l][i];
      lv.rexp[i] = s_re[l][i];
    }
  }
  // ---- persist u_l; hand u_lc, w_lc to the grid levels above
  for (int l = 0; l <= lce; ++l) {
    K4Lvl v = k4_lvl(D, P, l, sm);
    for (int e = tid; e < v.len; e += NT4) c.usm[c.usm_off[l] + e] = v.U[e];
  }
  if (lce == lc) {
    K4Lvl v = k4_lvl(D, P, lc, sm);
    k4_to_global(D, v.n, v.U, c.U[lc & 1], c.lv[lc].g);
    k4_to_global(D, v.n, v.W, c.W[lc & 1], c.lv[lc].g);
  }
  __syncthreads();
  k4_stamp(stamp++);
}

void k4_debug(int on) { cudaMemcpyToSymbol(g_k4_debug, &on, sizeof(int)); }
void k4_stamps(unsigned long long* out) { cudaMemcpyFromSymbol(out, g_k4_stamps, sizeof(unsigned long long) * 64); }

// Deferred norms of the grid levels (end of the solve, off the critical path):
// one CTA per entry, fixed-order reduction.
__global__ void __launch_bounds__(256) k_norms_all(const DevCtx* __restrict__ cp, const NormEntry* __restrict__ en) {
  __shared__ double red[256];
  const DevCtx& c = *cp;
  NormEntry e = en[blockIdx.x];
  double s = 0.0;
  for (int i = threadIdx.x; i < e.count; i += 256) s += c.pbase[e.poff + i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) c.norms[(long long)e.row * c.levels + e.l] = sqrt(red[0]);
}

// ------------------------------------------------------- error norms -------
struct ErrTab {
  double qx[6], qw[6];
  double phi[6][4], dphi[6][4];
};
template <int D, int P>
__global__ void __launch_bounds__(256) k_errors(const double* __restrict__ U, Geom g, ErrTab et,
                                                double* __restrict__ partials) {
  constexpr int NQ = P + 3;
  const int nel = 1 << (g.l + 1);
  const long long nelt = (D == 3) ? (long long)nel * nel * nel : (long long)nel * nel;
  const double h = pow2(-(g.l + 1));
  const double pi = 3.141592653589793238462643383279502884;
  double e0 = 0.0, e1 = 0.0;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < nelt;
       e += (long long)gridDim.x * blockDim.x) {
    int ex = (int)(e % nel), ey = (int)((e / nel) % nel), ez = (D == 3) ? (int)(e / ((long long)nel * nel)) : 0;
    double loc[(P + 1) * (P + 1) * (D == 3 ? P + 1 : 1)];
    for (int c = 0; c < (D == 3 ? P + 1 : 1); ++c)
      for (int b = 0; b <= P; ++b)
        for (int a = 0; a <= P; ++a) {
          int ix = P * ex + a, iy = P * ey + b, iz = P * ez + c;
          double v = 0.0;
          if (ix < g.n && iy < g.n && (D == 2 || iz < g.n))
            v = U[((long long)(D == 3 ? iz : 0) * g.NY + iy) * g.NX + ix];
          loc[(c * (P + 1) + b) * (P + 1) + a] = v;
        }
    for (int qz = 0; qz < (D == 3 ? NQ : 1); ++qz)
      for (int qy = 0; qy < NQ; ++qy)
        for (int qx = 0; qx < NQ; ++qx) {
          double val = 0.0, gx = 0.0, gy = 0.0, gz = 0.0;
          for (int c = 0; c < (D == 3 ? P + 1 : 1); ++c)
            for (int b = 0; b <= P; ++b)
              for (int a = 0; a <= P; ++a) {
                double cz = D == 3 ? et.phi[qz][c] : 1.0, dcz = D == 3 ? et.dphi[qz][c] : 0.0;
                double co = loc[(c * (P + 1) + b) * (P + 1) + a];
                val += co * et.phi[qx][a] * et.phi[qy][b] * cz;
                gx += co * et.dphi[qx][a] * et.phi[qy][b] * cz;
                gy += co * et.phi[qx][a] * et.dphi[qy][b] * cz;
                gz += co * et.phi[qx][a] * et.phi[qy][b] * dcz;
              }
          gx /= h; gy /= h; gz /= h;
          double x = (ex + et.qx[qx]) * h, y = (ey + et.qx[qy]) * h, z = (ez + et.qx[qz]) * h;
          double sx = sin(pi * x), sy = sin(pi * y), sz = D == 3 ? sin(pi * z) : 1.0;
          double cx = cos(pi * x), cy = cos(pi * y), cz = D == 3 ? cos(pi * z) : 0.0;
          double u = sx * sy * sz;
          double ux = pi * cx * sy * sz, uy = pi * sx * cy * sz, uz = pi * sx * sy * cz;
          double wq = et.qw[qx] * et.qw[qy] * (D == 3 ? et.qw[qz] : 1.0);
          e0 += wq * (val - u) * (val - u);
          e1 += wq * ((gx - ux) * (gx - ux) + (gy - uy) * (gy - uy) + (D == 3 ? (gz - uz) * (gz - uz) : 0.0));
        }
  }
  __shared__ double r0[256], r1[256];
  r0[threadIdx.x] = e0;
  r1[threadIdx.x] = e1;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      r0[threadIdx.x] += r0[threadIdx.x + o];
      r1[threadIdx.x] += r1[threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    partials[2 * blockIdx.x] = r0[0];
    partials[2 * blockIdx.x + 1] = r1[0];
  }
}

// -------------------------------------------------------------- codec K1 --
__global__ void __launch_bounds__(256) k_bfp_encode(const double* __restrict__ x, long long nblk, int w,
                                                    uint32_t* __restrict__ mant, int8_t* __restrict__ exps,
                                                    int* status) {
  const int lane = threadIdx.x & 31;
  long long wg = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long b = wg; b < nblk; b += nw) {
    double v = __ldcs(x + b * 32 + lane);
    warp_encode(v, w, mant + b * w, exps + b, lane, status);
  }
}

__global__ void __launch_bounds__(256) k_bfp_decode(const uint32_t* __restrict__ mant,
                                                    const int8_t* __restrict__ exps, long long nblk, int w,
                                                    double* __restrict__ x) {
  const int lane = threadIdx.x & 31;
  long long wg = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long b = wg; b < nblk; b += nw) {
    double v = warp_decode(mant + b * w, exps[b], w, lane);
    __stcs(x + b * 32 + lane, v);
  }
}

// ============================================================ launchers ===
#define FMG_DISPATCH(dim, p, F)               \
  do {                                        \
    if (dim == 2 && p == 1) { F(2, 1); }      \
    else if (dim == 2 && p == 2) { F(2, 2); } \
    else if (dim == 2 && p == 3) { F(2, 3); } \
    else if (dim == 3 && p == 1) { F(3, 1); } \
    else if (dim == 3 && p == 2) { F(3, 2); } \
    else { F(3, 3); }                         \
  } while (0)

static int g_num_sms = 0;
static int num_sms() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (g_num_sms <= 0) g_num_sms = 148;
  }
  return g_num_sms;
}

int smem_bytes(int dim, int p) {
  int s = 0;
#define F(D, P) s = Plan<D, P>::SMEM
  FMG_DISPATCH(dim, p, F);
#undef F
  return s;
}

void set_kernel_attributes() {
#define SETA(D, P)                                                                                       \
  cudaFuncSetAttribute(k_op<D, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, Plan<D, P>::SMEM); \
  cudaFuncSetAttribute(k4_kernel<D, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, K4_MAX_SMEM);
  SETA(2, 1) SETA(2, 2) SETA(2, 3) SETA(3, 1) SETA(3, 2) SETA(3, 3)
#undef SETA
}

void tile_shape(int dim, int p, int* TY, int* TZ) {
#define F(D, P) do { *TY = TileCfg<D, P>::TY; *TZ = TileCfg<D, P>::TZ; } while (0)
  FMG_DISPATCH(dim, p, F);
#undef F
}

template <typename K, typename... Args>
static cudaError_t launch_pdl(K kernel, dim3 grid, int smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = dim3(32, NWARP);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

void launch_op(int dim, int p, cudaStream_t st, const void* devctx, const OpDesc& op, int tx, int ty, int tz) {
  const DevCtx* c = (const DevCtx*)devctx;
#define F(D, P) launch_pdl(k_op<D, P>, dim3(tx, ty, tz), Plan<D, P>::SMEM, st, c, op)
  FMG_DISPATCH(dim, p, F);
#undef F
}

int k4_smem_bytes(int dim, int p, int lc) { return k4_smem_doubles(dim, p, lc) * 8; }
int k4_ainv_staged(int n0) { return n0 * n0 <= K4_AINV_MAX; }

void launch_k4(int dim, int p, cudaStream_t st, const void* devctx, const K4Desc& a, int smem) {
  const DevCtx* c = (const DevCtx*)devctx;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(32, NW4);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
#define F(D, P) cudaLaunchKernelEx(&cfg, k4_kernel<D, P>, c, a)
  FMG_DISPATCH(dim, p, F);
#undef F
}

size_t devctx_size() { return sizeof(DevCtx); }
void set_devctx_pbase(void* host_buf, double* pbase) { ((DevCtx*)host_buf)->pbase = pbase; }
size_t op_size() { return sizeof(Op); }

void fill_devctx(void* host_buf, const DevCtxDesc& d) {
  DevCtx* c = (DevCtx*)host_buf;
  memset(c, 0, sizeof(DevCtx));
  for (int l = 0; l < d.levels; ++l) {
    LevelDev& lv = c->lv[l];
    lv.g = d.g[l];
    lv.umant = d.u[l].mant;
    lv.uexp = d.u[l].exps;
    lv.ustride = d.u[l].stride;
    lv.rmant = d.r[l].mant;
    lv.rexp = d.r[l].exps;
    lv.rstride = d.r[l].stride;
    lv.gtab = d.gtab[l];
    lv.tx = d.tiles[l][0];
    lv.ty = d.tiles[l][1];
    lv.tz = d.tiles[l][2];
    lv.part = d.part[l];
    lv.count = d.count ? d.count + l : nullptr;
  }
  for (int i = 0; i < 2; ++i) {
    c->U[i] = d.U[i];
    c->T[i] = d.T[i];
    c->W[i] = d.W[i];
    c->Y[i] = d.Y[i];
  }
  c->usm = d.usm;
  c->pbase = d.pbase;
  for (int l = 0; l < kMaxLev; ++l) c->usm_off[l] = d.usm_off[l];
  c->lc = d.lc;
  c->n_cheb = d.n_cheb;
  c->Z = d.Z;
  c->B = d.B;
  c->Dv = d.Dv;
  c->Ainv = d.Ainv;
  c->n0 = d.n0;
  c->norms = d.norms;
  c->levels = d.levels;
  c->n_ir = d.n_ir;
  c->status = d.status;
  c->cf = d.cf;
}

void pack_op(void* dst, const OpDesc& od) { memcpy(dst, &od, sizeof(Op)); }

void launch_norms_all(cudaStream_t st, const void* devctx, const NormEntry* entries_dev, int n) {
  if (n > 0) k_norms_all<<<n, 256, 0, st>>>((const DevCtx*)devctx, entries_dev);
}

void launch_errors(const Launch& L, const double* U, const Geom& g, double* partials, int* nparts) {
  ErrTab et;
  int nq = L.p + 3;
  for (int i = 0; i < nq; ++i) {
    double z = cos(3.141592653589793 * (i + 0.75) / (nq + 0.5)), pp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = 0.0;
      for (int j = 1; j <= nq; ++j) {
        double p2 = p1;
        p1 = p0;
        p0 = ((2.0 * j - 1.0) * z * p1 - (j - 1.0) * p2) / j;
      }
      pp = nq * (z * p0 - p1) / (z * z - 1.0);
      double dz = p0 / pp;
      z -= dz;
      if (fabs(dz) < 1e-16) break;
    }
    et.qx[i] = 0.5 * (1.0 - z);
    et.qw[i] = 1.0 / ((1.0 - z * z) * pp * pp);
    for (int a = 0; a <= L.p; ++a) {
      double val = 1.0, der = 0.0;
      for (int j = 0; j <= L.p; ++j) {
        if (j == a) continue;
        double fac = (L.p * et.qx[i] - j) / (double)(a - j), dfac = L.p / (double)(a - j);
        der = der * fac + val * dfac;
        val = val * fac;
      }
      et.phi[i][a] = val;
      et.dphi[i][a] = der;
    }
  }
  int blocks = num_sms() * 4;
  *nparts = blocks;
#define F(D, P) k_errors<D, P><<<blocks, 256, 0, L.st>>>(U, g, et, partials)
  FMG_DISPATCH(L.dim, L.p, F);
#undef F
}

void launch_bfp_encode(const double* x, long long n, int w, uint32_t* mant, int8_t* exps, int* status,
                       cudaStream_t st) {
  long long nblk = n / 32;
  long long want = (nblk + 7) / 8;
  int grid = (int)(want < (long long)num_sms() * 16 ? (want > 0 ? want : 1) : num_sms() * 16);
  k_bfp_encode<<<grid, 256, 0, st>>>(x, nblk, w, mant, exps, status);
}

void launch_bfp_decode(const uint32_t* mant, const int8_t* exps, long long n, int w, double* x, cudaStream_t st) {
  long long nblk = n / 32;
  long long want = (nblk + 7) / 8;
  int grid = (int)(want < (long long)num_sms() * 16 ? (want > 0 ? want : 1) : num_sms() * 16);
  k_bfp_decode<<<grid, 256, 0, st>>>(mant, exps, nblk, w, x);
}

}  // namespace fmg
