// fmg_fine3.cu -- 3D kernels of the FINEST level of each FMG level (DESIGN.md
// §4.3): the level where almost all of the work and all of the large FP64
// temporaries are.
//
// Three plane-marching kernels replace, at l = L, the six of fmg_march3.cu
// (prolong, residual, cfas1, Chebyshev steps) and drop every finest-size FP64
// array except one (t_L, which also holds b_L after the restriction sweep has
// consumed t_L) and, for Chebyshev degree 3, the direction d_2:
//
//   k_f3_residual  u_L = dec ú_L + P_L u_{L-1} is generated plane by plane on
//                  chip (the coarse u_{L-1} boxes arrive by TMA; prolongation
//                  x and y passes in shared memory, z pass from a ring of
//                  coarse planes), then t_L = f_L - A_L u_L, r_L = enc(t_L),
//                  ||t_L||^2 partials and t_L -> HBM for the restriction.
//                  No u_L array exists (Alg 3.2).
//   k_f3_cfas      z_L = P_L w_{L-1} generated the same way, b_L = dec r_L -
//                  A_L z_L -> HBM (in the t_L buffer).  No z_L array
//                  (Alg 3.1).
//   k_f3_cheb      Chebyshev step j = 2..k (k <= 3): y_{j-1} is recomputed
//                  from b (and d_2) on the staged boxes, A y_{j-1}; the last
//                  step encodes ý_L and applies the correction ú_L =
//                  enc(dec ú_L + dec ý_L).  At l = L
//                  neither w_L nor u_L is needed, so neither is written.
//
// Instruction economy (profiles/r2_summary.md): the node types of the y and
// z passes are warp- / CTA-uniform, so those passes are compile-time
// specialised on the type (switch), which turns every coefficient into a
// constant-bank operand and skips the taps that are structurally zero for
// interior node types (exact: every chain starts from +0, so fma(0, v, acc)
// = acc).  Section words are prefetched by cp.async several planes ahead.
//
// Every floating-point expression is the canonical tree of DESIGN.md §3
// with explicit fma() (-fmad=false): bit-identical to fmg_march3.cu and to
// the oracle.
#include <type_traits>

#include "fmg_device.cuh"

#ifndef F3_PF
#define F3_PF 2      // staging / section-word lookahead (planes)
#endif
// CTAs per SM the register budget is sized for (measured): P = 1 fits 4 (64
// registers; C3 -1.3 % against 3, -6 % for 3 against 2), P = 2 fits 3, P = 3
// needs ~128 registers (3 CTAs spill: C4 +18 %)
#ifndef F3_TPB_MINB
#define F3_TPB_MINB 4  // k_f3_tpb CTAs per SM the register budget is sized for
#endif
#ifndef F3_MINB_P1
#define F3_MINB_P1 4
#endif
#ifndef F3_MINB
#define F3_MINB(P) ((P) == 3 ? 2 : ((P) == 1 ? F3_MINB_P1 : 3))
#endif
#ifndef F3_MINB_CF
#define F3_MINB_CF(P) F3_MINB(P)  // k_f3_cfas
#endif
#ifndef F3_MINB_CH
#define F3_MINB_CH(P, J) F3_MINB(P)  // k_f3_cheb
#endif
#ifndef F3_MINB_RS
#define F3_MINB_RS(P) F3_MINB(P)  // k_f3_residual_s
#endif
#ifndef F3_MINB_RS32
#define F3_MINB_RS32(P) ((P) == 3 ? 3 : F3_MINB(P))  // the staged kernels in FP32 cFas (fewer registers)
#endif
#define F3_MINB_ST(P, T) (sizeof(T) == 4 ? F3_MINB_RS32(P) : F3_MINB_RS(P))

namespace fmg {

namespace {

constexpr int FW = 8;  // warps per CTA = output rows of the 32 x 8 tile

template <int P>
struct F3 {
  static constexpr int R = 2 * P + 1;          // stencil taps per direction
  static constexpr int NR = FW + 2 * P;        // staged box rows
  static constexpr int RS = 40;                // staged row stride (doubles; TMA box width)
  static constexpr int BOX = NR * RS;          // doubles per staged plane box
  static constexpr int SH = P & 1;             // TMA boxes start at an even column: consumers shift
  static constexpr int PF = F3_PF;             // staging lookahead (planes)
  static constexpr int NBF = PF + P + 1;       // staged fine-plane ring (cheb)
  static constexpr int NW = PF + P + 1;        // section-word ring (planes)
  // coarse boxes of the on-the-fly prolongation (fine box + halo -> coarse)
  static constexpr int CBX = P == 3 ? 28 : 24;
  static constexpr int CBY = P == 3 ? 14 : 10;
  static constexpr int CBOX = CBX * CBY;
  static constexpr int CBS = (CBOX + 15) & ~15;  // slot stride: TMA destinations are 128-byte aligned
  static constexpr int NCB = P + 1;            // raw coarse box ring (TMA)
  static constexpr int NCY = P + 1;            // xy-passed coarse plane ring
};

// Coefficients in the cFas working type T (double; float for FP32 cFas,
// reading R28: the FP64 constants rounded to float, as the oracle does).
template <class T>
struct CoefT {
  T Kc[3][7], Mc[3][7], Pw[6][4], invd[27], inv_theta, cal[8], cbe[8];
  double rhs_c;
};

__device__ __forceinline__ void mbar_wait_s(unsigned bar, unsigned parity) {  // bar: smem byte address
  asm volatile(
      "{\n.reg .pred P1;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// -------------------------------------------------------- A passes ------
// y pass at one output row of node type T (c = My a,
// d = Ky a, e = My b; s = d + e), zero taps of interior types skipped.
template <int P, int TY, class T>
__device__ __forceinline__ void ypass_t(const CoefT<T>& cf, const T* XA, const T* XB, int w, int lane, T& c, T& s) {
  constexpr int o0 = TY == 0 ? 0 : P - TY, o1 = TY == 0 ? 2 * P : 2 * P - TY;
  T cc = 0, dd = 0, ee = 0;
#pragma unroll
  for (int o = o0; o <= o1; ++o) {
    const T av = XA[(w + o) * 32 + lane], bv = XB[(w + o) * 32 + lane];
    cc = fma(cf.Mc[TY][o], av, cc);
    dd = fma(cf.Kc[TY][o], av, dd);
    ee = fma(cf.Mc[TY][o], bv, ee);
  }
  c = cc;
  s = dd + ee;
}
template <int P, class T>
__device__ __forceinline__ void ypass(const CoefT<T>& cf, int ty, const T* XA, const T* XB, int w, int lane, T& c,
                                      T& s) {
  if (P == 1 || ty == 0) ypass_t<P, 0>(cf, XA, XB, w, lane, c, s);
  else if (P == 2 || ty == 1) ypass_t<P, (P >= 2 ? 1 : 0)>(cf, XA, XB, w, lane, c, s);
  else ypass_t<P, (P >= 3 ? 2 : 0)>(cf, XA, XB, w, lane, c, s);
}
// z pass of node type TZ over the register rings (acc over Kz on c, then Mz on s)
template <int P, int TZ, class T>
__device__ __forceinline__ T zpass_t(const CoefT<T>& cf, const T* cr, const T* sr) {
  constexpr int o0 = TZ == 0 ? 0 : P - TZ, o1 = TZ == 0 ? 2 * P : 2 * P - TZ;
  T acc = 0;
#pragma unroll
  for (int o = o0; o <= o1; ++o) acc = fma(cf.Kc[TZ][o], cr[o], acc);
#pragma unroll
  for (int o = o0; o <= o1; ++o) acc = fma(cf.Mc[TZ][o], sr[o], acc);
  return acc;
}
template <int P, class T>
__device__ __forceinline__ T zpass(const CoefT<T>& cf, int tz, const T* cr, const T* sr) {
  if (P == 1 || tz == 0) return zpass_t<P, 0>(cf, cr, sr);
  if (P == 2 || tz == 1) return zpass_t<P, (P >= 2 ? 1 : 0)>(cf, cr, sr);
  return zpass_t<P, (P >= 3 ? 2 : 0)>(cf, cr, sr);
}

// x pass of the staged box rows of warp w: a = Mx u, b = Kx u (lane = output
// column x0 + lane; staged column c = fine x0 - P + c; `off` = TMA shift)
template <int P, class T, class S>
__device__ __forceinline__ void xpass(const S* box, int off, const T* km, const T* kk, T* XA, T* XB, int w, int lane) {
  constexpr int R = F3<P>::R, NR = F3<P>::NR, RS = F3<P>::RS;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int r = w + k * FW;
    if (r < NR) {
      const S* row = box + r * RS + off;
      T s = 0, t = 0;
#pragma unroll
      for (int o = 0; o < R; ++o) {
        const T v = (T)row[lane + o];  // (FP32 cFas from an FP64 staged box: exact, it holds float values)
        s = fma(km[o], v, s);
        t = fma(kk[o], v, t);
      }
      XA[r * 32 + lane] = s;
      XB[r * 32 + lane] = t;
    }
  }
}

// ------------------------------------------------------ tile geometry ----
struct F3Tile {
  int x0, y0, zs, ze, cta;
};
__device__ __forceinline__ F3Tile f3_tile(const F3Args& a) {
  F3Tile t;
  const int cta = blockIdx.x, tiles = a.nxb * a.nyb;
  const int q = cta % tiles, ch = cta / tiles;
  t.x0 = (q % a.nxb) * 32;
  t.y0 = (q / a.nxb) * FW;
  t.zs = a.zlo + ch * a.RC;
  t.ze = min(a.zhi, t.zs + a.RC);
  t.cta = cta;
  return t;
}

// Staged column of lane's halo element (lanes < 2P): left halo columns 0..P-1,
// right halo columns 32+P..32+2P-1; the own column is P + lane.
template <int P>
__device__ __forceinline__ int halo_col(int lane) {
  return lane < P ? lane : 32 + lane;
}

// ------------------------------------------------- section words ring ---
// Section words are copied by cp.async into a ring of per-plane slots, PF
// planes ahead.  Every lane owns one 4-byte source stream (a mantissa word or
// an aligned exponent word) that advances by a fixed byte step per plane
// (blocks per plane = NY nxb is a multiple of 4, so aligned exponent words
// advance linearly too); no per-plane index arithmetic.
struct WStream {
  const char* src;  // this lane's source at plane z0 (dereferenced only when valid)
  long long step;   // bytes per plane
  int dst;          // word offset in the slot
  bool on;          // this lane copies (row and block exist)
};

// Residual: box row fy, blocks xb-1, xb, xb+1 (3 w words: lane j < 3w) and
// the two aligned exponent words covering their exponents (lanes 3w, 3w+1).
// Record RW = 3 w + 2 words; `eoff` = byte offset of e(xb-1) in the pair.
__device__ __forceinline__ WStream wstream3(const uint32_t* mant, const int8_t* exps, int stride, int w, const Geom& g,
                                            int x0, int fy, int z0, int rec, bool rowon, int lane, int& eoff) {
  WStream s{};
  const int nxb = g.NX >> 5, xb = x0 >> 5;
  const long long bpp = (long long)g.NY * nxb;  // blocks per plane (multiple of 4)
  const long long b0 = ((long long)z0 * g.NY + fy) * nxb + xb;  // own block at plane z0
  const long long ea = (b0 - 1) & ~3LL;                         // (floor: also for negative z0)
  eoff = (int)((b0 - 1) - ea);
  if (lane < 3 * w) {
    const int k = lane / w, wd = lane - k * w;
    const int xbk = xb - 1 + k;
    s.on = rowon && xbk >= 0 && xbk < nxb;
    s.src = (const char*)(mant + (b0 - 1 + k) * stride + wd);
    s.step = bpp * stride * 4;
    s.dst = rec + lane;
  } else if (lane < 3 * w + 2) {
    s.on = rowon;
    s.src = (const char*)(exps + ea + 4 * (lane - 3 * w));
    s.step = bpp;
    s.dst = rec + lane;
  }
  return s;
}
// Own block of output row y: w words (lanes < w) and the aligned exponent
// word (lane w); record RW = w + 1 words, `eoff` = byte of e(xb) in it.
__device__ __forceinline__ WStream wstream1(const uint32_t* mant, const int8_t* exps, int stride, int w, const Geom& g,
                                            int x0, int y, int z0, int rec, bool rowon, int lane, int& eoff) {
  WStream s{};
  const long long bpp = (long long)g.NY * (g.NX >> 5);
  const long long b0 = ((long long)z0 * g.NY + y) * (g.NX >> 5) + (x0 >> 5);
  const long long ea = b0 & ~3LL;
  eoff = (int)(b0 - ea);
  if (lane < w) {
    s.on = rowon;
    s.src = (const char*)(mant + b0 * stride + lane);
    s.step = bpp * stride * 4;
    s.dst = rec + lane;
  } else if (lane == w) {
    s.on = rowon;
    s.src = (const char*)(exps + ea);
    s.step = bpp;
    s.dst = rec + lane;
  }
  return s;
}
__device__ __forceinline__ void wcopy(const WStream& s, unsigned slot_s, int plane_off) {  // slot: smem byte address
  if (s.on)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(slot_s + 4u * (unsigned)s.dst),
                 "l"(s.src + s.step * plane_off)
                 : "memory");
}
__device__ __forceinline__ int rec_e(const uint32_t* ew, int off) {  // byte `off` of the exponent word pair
  return (int)(int8_t)(ew[off >> 2] >> (8 * (off & 3)));
}
// r_L decode of the staged cFas step 1: compile-time width WR > 0 (the
// common top-level widths, warp_decode_w) or the runtime width.
template <int WR>
__device__ __forceinline__ double dec_rec(const uint32_t* rec, int E, int w, int lane) {
  if constexpr (WR > 0) return warp_decode_w<WR>(rec, E, lane);
  else return warp_decode(rec, E, w, lane);
}

// ------------------------------------------- on-the-fly prolongation ----
// Generates, plane by plane, v = P_l c_{l-1} on the staged box (32 + 2P) x
// (8 + 2P) (x pass over coarse taps, then y, then z; one fma
// chain per pass from +0; 0 at fine non-unknowns).  Coarse plane boxes CBX x
// CBY arrive by TMA into a ring of NCB slots; their x and y passes go to a
// ring of NCY xy-passed planes (rows and columns of the fine box), from which
// each fine plane takes its z pass.
//
// Thread mapping: the box's NR x BW elements are dealt out linearly (element
// e = tid + k NT), so every warp does the same work (no halo lanes); each
// element carries its packed smem offset, coarse tap offsets and weight rows.
// The x pass uses the same list with the row read as a coarse row (CBY <= NR).
template <int P>
struct Gen {
  static constexpr int BW = 32 + 2 * P, NE = F3<P>::NR * BW, KB = (NE + 32 * FW - 1) / (32 * FW);
  int off[KB];   // r RS + c; -1: inactive element
  int pk[KB];    // bxo | byo << 8 | rx << 16 | ry << 20 | (r < CBY) << 24   (coarse offsets from the box origin)
  int dk[KB];    // decode: record row offset | block << 10 | exponent byte << 12 | position << 16 | on << 24
  int zo[KB];    // output point of the tile (rows P..P+7, columns P..P+31): y NX + x in the plane; else -1
  int cx0, cy0;  // coarse box origin
  int cfirst;    // first coarse plane of the march (ring slots and barrier phases count from it)
  int clast;     // last coarse plane the march needs (no request beyond: no TMA left in flight)
  int cdone;     // next coarse plane to xy-pass
  int czoff;     // first allocated plane of the coarse array (TMA coordinates are window-relative)
};

// Element tables.  `rw` (record words per row, 0: no decode), `eoffr(r)`
// (exponent byte of block xb - 1 for box row r) describe the section records.
template <int P, class EO>
__device__ __forceinline__ void gen_init(Gen<P>& gn, const Geom& g, int x0, int y0, int rw, int wu, EO eoffr) {
  constexpr int NR = F3<P>::NR, RS = F3<P>::RS, CBY = F3<P>::CBY, BW = Gen<P>::BW;
  const int n = g.n, tid = threadIdx.y * 32 + threadIdx.x;
  gn.cx0 = (P * (max(x0 - P, 1) / (2 * P))) & ~1;
  gn.cy0 = P * (max(y0 - P, 1) / (2 * P));
#pragma unroll
  for (int k = 0; k < Gen<P>::KB; ++k) {
    const int e = tid + k * 32 * FW;
    gn.off[k] = -1;
    gn.pk[k] = 0;
    gn.dk[k] = 0;
    gn.zo[k] = -1;
    if (e < Gen<P>::NE) {
      const int r = e / BW, c = e - r * BW;
      const int fx = x0 - P + c, fy = y0 - P + r;
      const bool okx = unk1(fx, n), oky = unk1(fy, n);
      const int rx = okx ? fx % (2 * P) : 0, bxo = okx ? P * (fx / (2 * P)) - gn.cx0 : 0;
      const int ry = oky ? fy % (2 * P) : 0, byo = oky ? P * (fy / (2 * P)) - gn.cy0 : 0;
      gn.off[k] = r * RS + c;
      if (r >= P && r < P + FW && c >= P && c < P + 32 && fy < g.NY) gn.zo[k] = fy * g.NX + fx;
      // y pass reads PX[(byo + t) RS + c]: stored relative to the element's own offset
      gn.pk[k] = bxo | ((byo - r + 32) << 8) | (rx << 16) | (ry << 20) | ((r < CBY ? 1 : 0) << 24) |
                 ((okx ? 1 : 0) << 25) | ((oky ? 1 : 0) << 26);
      if (rw > 0 && okx && oky) {
        const int kb = c < P ? 0 : (c < 32 + P ? 1 : 2);
        gn.dk[k] = (r * rw) | (kb << 10) | ((eoffr(r) + kb) << 12) | ((fx & 31) << 16) | (1 << 24);
      }
    }
  }
}

// coarse plane index of the first tap of fine plane z (unknown z)
template <int P>
__device__ __forceinline__ int cbase(int z) {
  return P * (z / (2 * P));
}

// x and y passes of coarse plane c (raw box in `cb`) into the xy ring slot.
template <int P, class T>
__device__ __forceinline__ void gen_xy(const Gen<P>& gn, const T* pws, const double* cb, T* PX, T* yv) {
  constexpr int CBX = F3<P>::CBX, RS = F3<P>::RS;
#pragma unroll
  for (int k = 0; k < Gen<P>::KB; ++k) {
    const int pk = gn.pk[k];
    if (gn.off[k] >= 0 && (pk >> 24) & 1) {
      const int r = gn.off[k] / RS;  // (coarse row = box row index)
      T a = 0;
      if ((pk >> 25) & 1) {
        const T* wt = pws + ((pk >> 16) & 15) * (P + 1);
        const double* row = cb + r * CBX + (pk & 255);
#pragma unroll
        for (int t = 0; t <= P; ++t) a = fma(wt[t], (T)row[t], a);
      }
      PX[gn.off[k]] = a;
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < Gen<P>::KB; ++k) {
    const int pk = gn.pk[k];
    if (gn.off[k] >= 0) {
      T a = 0;
      if ((pk >> 26) & 1) {
        const T* wt = pws + ((pk >> 20) & 15) * (P + 1);
        const T* col = PX + gn.off[k] + (((pk >> 8) & 255) - 32) * RS;
#pragma unroll
        for (int t = 0; t <= P; ++t) a = fma(wt[t], col[t * RS], a);
      }
      yv[gn.off[k]] = a;
    }
  }
}

// Request the TMA box of coarse plane c (thread 0); slot and barrier phase
// count from the first plane of the march.
template <int P>
__device__ __forceinline__ void gen_request(const Gen<P>& gn, const CUtensorMap* tm, double* craw,
                                            unsigned long long* cbar, int c) {
  constexpr int NCB = F3<P>::NCB;
  if (c > gn.clast) return;
  const int k = (c - gn.cfirst) % NCB;
  fence_async_smem();
  tma_load_3d(craw + k * F3<P>::CBS, tm, gn.cx0, gn.cy0, c - gn.czoff, cbar + k, (unsigned)(F3<P>::CBOX * 8));
}
// Coarse planes of a march over fine input planes [z0, z0 + nin): the first
// and last unknown fine planes decide them (none: cfirst > clast).
template <int P>
__device__ __forceinline__ void gen_range(Gen<P>& gn, int z0, int nin, int n) {
  const int zf = max(z0, 1), zl = min(z0 + nin - 1, n - 1);
  gn.cfirst = P * (zf / (2 * P));
  gn.clast = zf <= zl ? P * (zl / (2 * P)) + P : gn.cfirst - 1;
  gn.cdone = gn.cfirst;
}

// Make the xy passes of every coarse plane <= cneed available.
template <int P, class T>
__device__ __forceinline__ void gen_advance(Gen<P>& gn, const T* pws, const CUtensorMap* tm, double* craw,
                                            unsigned long long* cbar, T* PX, T* yvring, int cneed) {
  constexpr int NCB = F3<P>::NCB, NCY = F3<P>::NCY, BOX = F3<P>::BOX;
  while (gn.cdone <= cneed) {
    const int c = gn.cdone, k = c - gn.cfirst;
    mbar_wait_s(smem_u32(cbar) + 8u * (unsigned)(k % NCB), (unsigned)(k / NCB) & 1u);
    gen_xy<P, T>(gn, pws, craw + (k % NCB) * F3<P>::CBS, PX, yvring + (c % NCY) * BOX);
    // (gen_xy synchronised after its x pass: the raw slot is free)
    if (threadIdx.x == 0 && threadIdx.y == 0) gen_request<P>(gn, tm, craw, cbar, c + NCB);
    gn.cdone = c + 1;
    __syncthreads();
  }
}

// Fine plane z into the box: z pass of the xy ring (0 at non-unknown planes),
// plus dec of the section record (residual, `rec` non-null).
template <int P, class T>
__device__ __forceinline__ void gen_z(const Gen<P>& gn, const CoefT<T>& cf, const T* yvring, int z, int n, T* box,
                                     const uint32_t* rec, int wu) {
  constexpr int NCY = F3<P>::NCY, BOX = F3<P>::BOX;
  const bool okz = unk1(z, n);
  const int rz = okz ? z % (2 * P) : 0, cb = okz ? cbase<P>(z) : 0;
  T pz[P + 1];
  const T* ys[P + 1];
#pragma unroll
  for (int t = 0; t <= P; ++t) {
    pz[t] = cf.Pw[rz][t];
    ys[t] = yvring + ((cb + t) % NCY) * BOX;
  }
#pragma unroll
  for (int k = 0; k < Gen<P>::KB; ++k) {
    const int o = gn.off[k];
    if (o >= 0) {
      T v = 0;
      if (okz) {
#pragma unroll
        for (int t = 0; t <= P; ++t) v = fma(pz[t], ys[t][o], v);
        const int dk = gn.dk[k];
        if (rec && (dk >> 24)) {
          const uint32_t* r0 = rec + (dk & 1023);
          const T dv = (T)point_decode(r0 + ((dk >> 10) & 3) * wu, rec_e(r0 + 3 * wu, (dk >> 12) & 15), wu,
                                       (dk >> 16) & 31);
          v = dv + v;  // u = dec ú + P u (the residual: T = double)
        }
      }
      box[o] = v;
    }
  }
}

}  // namespace

// ================================================================ kernels ==
// Shared-memory carve-up of the generating kernels (residual, cFas): raw
// coarse boxes (TMA, 128-byte aligned slots), xy-passed coarse planes, the
// generated box, the A x pass, the prolongation x pass, the P weight table,
// then the section-word ring and the barriers.
template <int P, class T>
struct GenSmem {
  double* craw;  // TMA boxes of the coarse FP64 array
  T *yvring, *box, *XA, *XB, *PX, *pws;
  uint32_t* wring;
  unsigned long long* cbar;
};
template <int P, class T>
__device__ __forceinline__ GenSmem<P, T> gen_smem(double* base, int ring_words) {
  using C = F3<P>;
  GenSmem<P, T> m;
  m.craw = base;
  m.yvring = (T*)(m.craw + C::NCB * C::CBS);
  m.box = m.yvring + C::NCY * C::BOX;
  m.XA = m.box + C::BOX;
  m.XB = m.XA + C::NR * 32;
  m.PX = m.XB + C::NR * 32;
  m.pws = m.PX + C::CBY * C::RS;
  m.wring = (uint32_t*)(m.pws + 2 * P * (P + 1));
  uintptr_t b = (uintptr_t)(m.wring + ring_words);
  m.cbar = (unsigned long long*)((b + 7) & ~(uintptr_t)7);
  return m;
}
template <int P, class T>
__host__ __device__ constexpr size_t gen_smem_bytes(int ring_words) {
  using C = F3<P>;
  return (size_t)C::NCB * C::CBS * 8 +
         ((size_t)C::NCY * C::BOX + C::BOX + 2 * C::NR * 32 + (size_t)C::CBY * C::RS + 2 * P * (P + 1)) * sizeof(T) +
         (size_t)ring_words * 4 + 8 + 8 * C::NCB;
}

// t_L = f_L - A_L u_L with u_L = dec ú_L + P u_{L-1} generated on chip;
// r_L = enc(t_L); t_L -> HBM; ||t_L||^2 partial per warp (Alg 3.2).
// ENC = false: r_L is encoded afterwards from t_L by k_f3_tpb<0> (thread per block).
template <int P, bool ENC>
__global__ void __launch_bounds__(32 * FW, F3_MINB(P)) k_f3_residual(const __grid_constant__ F3Args a,
                                                              const __grid_constant__ CoefT<double> cf) {
  using C = F3<P>;
  constexpr int R = C::R, NR = C::NR, NW = C::NW, PF = C::PF;
  extern __shared__ __align__(128) double fsm[];
  const int RW = 3 * a.wu + 2;  // record words per box row
  const GenSmem<P, double> m = gen_smem<P, double>(fsm, NW * NR * RW);
  const unsigned wring_s = smem_u32(m.wring);

  const int lane = threadIdx.x, w = threadIdx.y;
  const F3Tile tl = f3_tile(a);
  const Geom g = a.g;
  const int n = g.n;
  const int x = tl.x0 + lane, y = tl.y0 + w;
  const bool rowok = y < g.NY;
  const int tx = x % P, ty = y % P;
  double km[R], kk[R];
#pragma unroll
  for (int o = 0; o < R; ++o) {
    km[o] = cf.Mc[tx][o];
    kk[o] = cf.Kc[tx][o];
  }
  const double hl = pow2(-(a.l + 1));
  const double* __restrict__ gt = a.gtab;
  const bool uxy = unk1(x, n) && unk1(y, n);
  const double gxy = uxy ? (cf.rhs_c * gt[x]) * gt[y] : 0.0;
  const int z0 = tl.zs - P, nin = (tl.ze - tl.zs) + 2 * P;
  const int nxb = g.NX >> 5, xb = tl.x0 >> 5;
  Gen<P> gn;
  gen_init<P>(gn, g, tl.x0, tl.y0, RW, a.wu, [&](int r) {
    const long long b0 = ((long long)z0 * g.NY + (tl.y0 - P + r)) * nxb + xb;
    return (int)((b0 - 1) - ((b0 - 1) & ~3LL));
  });
  gen_range<P>(gn, z0, nin, n);
  gn.czoff = a.czoff;
  // section word streams of the warp's (up to) two box rows: only unknown
  // rows are decoded (the section and u are 0 elsewhere)
  WStream ws[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int r = w + k * FW, fy = tl.y0 - P + r;
    int eo;
    ws[k] = wstream3(a.umant, a.uexp, a.ustride, a.wu, g, tl.x0, fy, z0, r * RW, r < NR && unk1(fy, n), lane, eo);
  }
  // output pointers (advance one plane per output)
  const long long tplane = (long long)g.NY * g.NX;
  const long long bpp = (long long)g.NY * nxb;
  double* Tp = a.T + ((long long)tl.zs * g.NY + y) * g.NX + x;
  const long long blk0 = ((long long)tl.zs * g.NY + y) * nxb + xb;
  uint32_t* rmp = a.rmant + blk0 * a.rstride;
  int8_t* rep = a.rexp + blk0;

  {
    const int tid = w * 32 + lane;
    if (tid < 2 * P * (P + 1)) m.pws[tid] = cf.Pw[tid / (P + 1)][tid % (P + 1)];
  }
  if (threadIdx.x == 0 && threadIdx.y == 0) {
#pragma unroll
    for (int k = 0; k < C::NCB; ++k) mbar_init(m.cbar + k, 1);
    mbar_init_fence();
  }
  __syncthreads();
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x == 0 && threadIdx.y == 0)
    for (int k = 0; k < C::NCB; ++k) gen_request<P>(gn, a.tmc, m.craw, m.cbar, gn.cfirst + k);
  auto words = [&](int i, int slot) {  // words of input plane z0 + i into ring slot `slot`
    const int zz = z0 + i;
    if (zz >= 1 && zz <= n - 1) {
      const unsigned s = wring_s + (unsigned)(slot * NR * RW * 4);
      wcopy(ws[0], s, i);
      wcopy(ws[1], s, i);
    }
  };
  int wsl = 0;  // ring slot of input plane i
#pragma unroll
  for (int i = 0; i < PF; ++i) {
    if (i < nin) words(i, i);
    cpa_commit();
  }
  double cr[R], sr[R];
#pragma unroll
  for (int o = 0; o < R; ++o) cr[o] = sr[o] = 0.0;
  double ss = 0.0;
  int tzo = ((z0 % P) + P) % P;  // node type of plane z0 + i (= of output plane z0 + i - P)
  for (int i = 0; i < nin; ++i) {
    const int zi = z0 + i;
    const bool zu = zi >= 1 && zi <= n - 1;
    if (i + PF < nin) words(i + PF, wsl + PF >= NW ? wsl + PF - NW : wsl + PF);
    cpa_commit();
    if (zu) gen_advance<P>(gn, m.pws, a.tmc, m.craw, m.cbar, m.PX, m.yvring, cbase<P>(zi) + P);
    cpa_wait<PF>();
    __syncthreads();  // (the words of plane zi, from every thread)
    gen_z<P>(gn, cf, m.yvring, zi, n, m.box, zu ? m.wring + wsl * NR * RW : nullptr, a.wu);
    wsl = wsl + 1 == NW ? 0 : wsl + 1;
    __syncthreads();
    xpass<P>(m.box, 0, km, kk, m.XA, m.XB, w, lane);
    __syncthreads();
    double c, s;
    ypass<P>(cf, ty, m.XA, m.XB, w, lane, c, s);
#pragma unroll
    for (int o = 0; o < R - 1; ++o) {
      cr[o] = cr[o + 1];
      sr[o] = sr[o + 1];
    }
    cr[R - 1] = c;
    sr[R - 1] = s;
    if (i >= 2 * P) {
      const int z = zi - P;
      const double au = zpass<P>(cf, tzo, cr, sr) * hl;
      if (rowok) {
        const bool uz = unk1(z, n);
        const double gz = uz ? gt[z] : 0.0;
        const double t = (uxy && uz) ? gxy * gz - au : 0.0;  // (((C g(x)) g(y)) g(z)) - A u
        *Tp = t;
        ss = fma(t, t, ss);
        if (ENC) warp_encode(t, a.wr, rmp, rep, lane, a.status);
      }
      Tp += tplane;
      rmp += bpp * a.rstride;
      rep += bpp;
    }
    tzo = tzo + 1 == P ? 0 : tzo + 1;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(FULL, ss, o);
  if (lane == 0 && a.poff >= 0) a.pbase[a.poff + (long long)tl.cta * FW + w] = ss;
}

// b_L = dec r_L - A_L z_L with z_L = P w_{L-1} generated on chip -> B (the
// t_L buffer).  Chebyshev step 1 (cFas1 of fmg_march3.cu).
template <int P, class T>
__global__ void __launch_bounds__(32 * FW, F3_MINB_CF(P)) k_f3_cfas(const __grid_constant__ F3Args a,
                                                          const __grid_constant__ CoefT<T> cf) {
  using C = F3<P>;
  constexpr int R = C::R, NW = C::NW, PF = C::PF;
  extern __shared__ __align__(128) double fsm[];
  const int RW = a.wr + 1;
  const GenSmem<P, T> m = gen_smem<P, T>(fsm, NW * FW * RW);
  const unsigned wring_s = smem_u32(m.wring);

  const int lane = threadIdx.x, w = threadIdx.y;
  const F3Tile tl = f3_tile(a);
  const Geom g = a.g;
  const int n = g.n;
  const int x = tl.x0 + lane, y = tl.y0 + w;
  const bool rowok = y < g.NY;
  const int tx = x % P, ty = y % P;
  T km[R], kk[R];
#pragma unroll
  for (int o = 0; o < R; ++o) {
    km[o] = cf.Mc[tx][o];
    kk[o] = cf.Kc[tx][o];
  }
  const T hl = (T)pow2(-(a.l + 1));
  const int z0 = tl.zs - P, nin = (tl.ze - tl.zs) + 2 * P;
  Gen<P> gn;
  gen_init<P>(gn, g, tl.x0, tl.y0, 0, 0, [](int) { return 0; });
  gen_range<P>(gn, z0, nin, n);
  gn.czoff = a.czoff;
  // r_L words of the warp's output row, output planes zs, zs + 1, ...
  int eoff;
  const WStream ws = wstream1(a.rmant, a.rexp, a.rstride, a.wr, g, tl.x0, y, tl.zs, w * RW, rowok, lane, eoff);
  const long long tplane = (long long)g.NY * g.NX;
  double* Bp = a.T + ((long long)tl.zs * g.NY + y) * g.NX + x;
  const int nout = tl.ze - tl.zs;
  {
    const int tid = w * 32 + lane;
    if (tid < 2 * P * (P + 1)) m.pws[tid] = cf.Pw[tid / (P + 1)][tid % (P + 1)];
  }
  if (threadIdx.x == 0 && threadIdx.y == 0) {
#pragma unroll
    for (int k = 0; k < C::NCB; ++k) mbar_init(m.cbar + k, 1);
    mbar_init_fence();
  }
  __syncthreads();
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x == 0 && threadIdx.y == 0)
    for (int k = 0; k < C::NCB; ++k) gen_request<P>(gn, a.tmc, m.craw, m.cbar, gn.cfirst + k);
  // output plane j = 0..nout-1 (z = zs + j) is produced at iteration j + 2P;
  // its words go to ring slot j % NW, issued PF outputs ahead
#pragma unroll
  for (int j = 0; j < PF; ++j) {
    if (j < nout) wcopy(ws, wring_s + (unsigned)(j * FW * RW * 4), j);
    cpa_commit();
  }
  int osl = 0;  // ring slot of the next output plane
  T cr[R], sr[R];
#pragma unroll
  for (int o = 0; o < R; ++o) cr[o] = sr[o] = 0;
  int tzo = ((z0 % P) + P) % P;
  for (int i = 0; i < nin; ++i) {
    const int zi = z0 + i;
    const bool produce = i >= 2 * P;
    if (produce) {
      const int j = i - 2 * P + PF;
      if (j < nout) wcopy(ws, wring_s + (unsigned)((osl + PF >= NW ? osl + PF - NW : osl + PF) * FW * RW * 4), j);
    }
    cpa_commit();
    if (zi >= 1 && zi <= n - 1) gen_advance<P>(gn, m.pws, a.tmc, m.craw, m.cbar, m.PX, m.yvring, cbase<P>(zi) + P);
    gen_z<P>(gn, cf, m.yvring, zi, n, m.box, nullptr, 0);
    if (a.zout && zi >= tl.zs && zi < tl.ze) {  // z_l at the tile's points (levels below the finest)
      double* zp = a.Z + (long long)zi * tplane;
#pragma unroll
      for (int k = 0; k < Gen<P>::KB; ++k)
        if (gn.zo[k] >= 0) zp[gn.zo[k]] = (double)m.box[gn.off[k]];
    }
    cpa_wait<PF>();
    __syncthreads();
    xpass<P>(m.box, 0, km, kk, m.XA, m.XB, w, lane);
    __syncthreads();
    T c, s;
    ypass<P>(cf, ty, m.XA, m.XB, w, lane, c, s);
#pragma unroll
    for (int o = 0; o < R - 1; ++o) {
      cr[o] = cr[o + 1];
      sr[o] = sr[o + 1];
    }
    cr[R - 1] = c;
    sr[R - 1] = s;
    if (produce) {
      const T az = zpass<P>(cf, tzo, cr, sr) * hl;
      if (rowok) {
        const uint32_t* rec = m.wring + osl * FW * RW + w * RW;
        const double rv = warp_decode(rec, rec_e(rec + a.wr, eoff), a.wr, lane);
        *Bp = (double)((T)rv - az);  // b = dec r - A z (B lives in the t_L buffer)
      }
      Bp += tplane;
      osl = osl + 1 == NW ? 0 : osl + 1;
    }
    tzo = tzo + 1 == P ? 0 : tzo + 1;
  }
}

// Chebyshev step j = J in {2, 3} at l = L: the staged boxes
// are b (and d_2 for j = 3); y_{j-1} is recomputed on them (y_1 = inv_theta
// (invD b), y_2 = y_1 + d_2), A y_{j-1}, then q = b - A y, d_j = fma(al_j,
// d_{j-1}, be_j (invD q)), y_j = y_{j-1} + d_j.  A step below k stores d_j;
// the last one encodes ý_L and applies the correction.
// FIN (the last step with the thread-per-block finalisation):
// y_k goes to a.Dv (the host points it at the Y buffer) as FP64, and
// k_f3_tpb<1> then encodes ý, updates ú and writes w_l, u_l.
// FIN = 2 (the lean form's top level, no u_l / w_l): ý's mantissas (int8)
// and block exponents go to a.my / a.ey; k_f3_tpb<2> updates ú from them.
template <int P, int J, class T, int FIN, bool FS = false>
__global__ void __launch_bounds__(32 * FW, F3_MINB_CH(P, J)) k_f3_cheb(const __grid_constant__ F3Args a,
                                                          const __grid_constant__ CoefT<T> cf) {
  using C = F3<P>;
  constexpr int R = C::R, NR = C::NR, RS = C::RS, BOX = C::BOX, NBF = C::NBF, NW = C::NW, PF = C::PF;
  constexpr int NA = J >= 3 ? 2 : 1;  // staged arrays: b (+ d_2)
  // FS: FP32 cFas with float storage (b, d_2, y_k float arrays; float boxes
  // from x0 - 4, shift 4 - P, 128-byte aligned box slots), FIN = 1 or 0
  static_assert(!FS || (sizeof(T) == 4 && FIN < 2), "float storage: FP32 cFas, FIN 0 / 1");
  using S = typename std::conditional<FS, float, double>::type;
  constexpr int SHS = FS ? 4 - P : (P & 1);
  constexpr int BOXS = FS ? ((BOX + 31) & ~31) : BOX;
  extern __shared__ __align__(128) double fsm[];
  S* ring = (S*)fsm;                         // NBF x NA boxes
  T* yb = (T*)(fsm + NBF * NA * BOX);       // y_{j-1} on the current box
  T* XA = yb + BOX;
  T* XB = XA + NR * 32;
  T* ivd = XB + NR * 32;                     // invD factors: P node types x box
  double* aring = (double*)(ivd + P * BOX);  // NW x 2 x NT: z_l, P u_{l-1} at the output points (last step)
  const bool aux = !FIN && a.last && (a.wout || a.uout);
  uint32_t* wring = (uint32_t*)(aring + (aux ? NW * 2 * 32 * FW : 0));  // NW x FW x (w + 1) (last step: ú words)
  const int RW = a.wu + 1;
  unsigned long long* bars = (unsigned long long*)(wring + NW * FW * RW + 2);
  bars = (unsigned long long*)(((uintptr_t)bars + 7) & ~(uintptr_t)7);

  const int lane = threadIdx.x, w = threadIdx.y;
  const F3Tile tl = f3_tile(a);
  const Geom g = a.g;
  const int n = g.n;
  const int x = tl.x0 + lane, y = tl.y0 + w;
  const bool rowok = y < g.NY;
  const int tx = x % P, ty = y % P;
  T km[R], kk[R];
#pragma unroll
  for (int o = 0; o < R; ++o) {
    km[o] = cf.Mc[tx][o];
    kk[o] = cf.Kc[tx][o];
  }
  const T hl = (T)pow2(-(a.l + 1));
  const T al = cf.cal[J - 1], be = cf.cbe[J - 1], ith = cf.inv_theta;
  const int hc = halo_col<P>(lane);
  // invD factors of the thread's staged elements for every z node type
  // (RN(1/diag) 2^(l+1), 0 at non-unknowns; the z-unknown test is per plane)
  {
    const T isc = (T)pow2(a.l + 1);
    const int xh = lane < P ? tl.x0 - P + lane : tl.x0 + 32 + lane - P;
    const bool ux = unk1(x, n), uxh = lane < 2 * P && unk1(xh, n);
    const int txo = ux ? x % P : 0, txh = uxh ? xh % P : 0;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int r = w + k * FW, yy = tl.y0 - P + r;
      if (r < NR) {
        const bool uy = unk1(yy, n);
        const int tyy = uy ? yy % P : 0;
#pragma unroll
        for (int tz = 0; tz < P; ++tz) {
          const int tb = (tz * P + tyy) * P;
          ivd[tz * BOX + r * RS + P + lane] = (ux && uy) ? cf.invd[tb + txo] * isc : (T)0;
          if (lane < 2 * P) ivd[tz * BOX + r * RS + hc] = (uxh && uy) ? cf.invd[tb + txh] * isc : (T)0;
        }
      }
    }
  }
  const int z0 = tl.zs - P, nin = (tl.ze - tl.zs) + 2 * P;
  int eoff = 0;
  const WStream ws = wstream1(a.umant, a.uexp, a.ustride, a.wu, g, tl.x0, y, tl.zs, w * RW, rowok && a.last && !FIN,
                              lane, eoff);
  const long long tplane = (long long)g.NY * g.NX;
  const long long bpp = (long long)g.NY * (g.NX >> 5);
  S* Dp = (S*)a.Dv + ((long long)tl.zs * g.NY + y) * g.NX + x;
  const long long blk0 = ((long long)tl.zs * g.NY + y) * (g.NX >> 5) + (tl.x0 >> 5);
  uint32_t* ump = a.umant + blk0 * a.ustride;
  int8_t* uep = a.uexp + blk0;
  const long long ustep = bpp * a.ustride;
  const int nout = tl.ze - tl.zs;
  const unsigned ring_s = smem_u32(ring), bars_s = smem_u32(bars), wring_s = smem_u32(wring);
  const unsigned aring_s = smem_u32(aring);
  const int tid = w * 32 + lane;
  const long long pbase0 = ((long long)tl.zs * g.NY + y) * g.NX + x;  // output point, plane zs
  auto auxcopy = [&](int j, int slot) {  // z_l, P u_{l-1} of output plane zs + j -> aux ring slot
    if (aux && rowok) {
      const unsigned d = aring_s + (unsigned)(((slot * 2) * 32 * FW + tid) * 8);
      if (a.wout)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(a.Z + pbase0 + j * tplane) : "memory");
      if (a.uout)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d + 32 * FW * 8), "l"(a.PU + pbase0 + j * tplane)
                     : "memory");
    }
  };
  if (threadIdx.x == 0 && threadIdx.y == 0) {
#pragma unroll
    for (int k = 0; k < NBF; ++k) mbar_init(bars + k, 1);
    mbar_init_fence();
  }
  __syncthreads();
  pdl_wait();
  pdl_trigger();
  const int tmx = tl.x0 - P - SHS, tmy = tl.y0 - P;
  auto stage = [&](int i, int slot) {  // input plane z0 + i into ring slot `slot` (TMA, thread 0)
    if (threadIdx.x == 0 && threadIdx.y == 0) {
      const unsigned dst = ring_s + (unsigned)(slot * NA * BOXS * sizeof(S)), bar = bars_s + (unsigned)(slot * 8);
      fence_async_smem();
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"((unsigned)(NA * BOX * sizeof(S)))
                   : "memory");
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
          "[%5];" ::"r"(dst),
          "l"((unsigned long long)a.tmb), "r"(tmx), "r"(tmy), "r"(z0 + i - a.zoff), "r"(bar)
          : "memory");
      if (NA == 2)
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
            "%4}], [%5];" ::"r"(dst + (unsigned)(BOXS * sizeof(S))),
            "l"((unsigned long long)a.tmd), "r"(tmx), "r"(tmy), "r"(z0 + i - a.zoff), "r"(bar)
            : "memory");
    }
  };
  // ring slots: input plane i -> slot i % NBF; ú words of output plane j -> slot j % NW
#pragma unroll
  for (int i = 0; i < PF; ++i)
    if (i < nin) stage(i, i);
#pragma unroll
  for (int j = 0; j < PF; ++j) {
    if (j < nout) {
      wcopy(ws, wring_s + (unsigned)(j * FW * RW * 4), j);
      auxcopy(j, j);
    }
    cpa_commit();
  }
  T cr[R], sr[R];
#pragma unroll
  for (int o = 0; o < R; ++o) cr[o] = sr[o] = 0;
  int tz = ((z0 % P) + P) % P;   // node type of plane z0 + i (input; = output plane z0 + i - P)
  int isl = 0, osl = 0, oisl = NBF - P;  // slots: input plane i, ú words of the next output, input plane i - P
  unsigned par = 0;              // barrier phase of slot isl
  for (int i = 0; i < nin; ++i) {
    const int zi = z0 + i;
    const bool produce = i >= 2 * P;
    mbar_wait_s(bars_s + 8u * (unsigned)isl, par);
    cpa_wait<PF - 1>();
    __syncthreads();  // every thread is past iteration i - 1: slot (i + PF) % NBF is free
    if (i + PF < nin) stage(i + PF, isl + PF >= NBF ? isl + PF - NBF : isl + PF);
    if (produce) {
      const int j = i - 2 * P + PF;
      const int sl = osl + PF >= NW ? osl + PF - NW : osl + PF;
      if (j < nout) {
        wcopy(ws, wring_s + (unsigned)(sl * FW * RW * 4), j);
        auxcopy(j, sl);
      }
    }
    cpa_commit();
    // y_{j-1} on the thread's staged elements of plane zi
    {
      const S* bb = ring + isl * NA * BOXS + SHS;
      const T* iv = ivd + tz * BOX;
      const bool uz = zi >= 1 && zi <= n - 1;
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int r = w + k * FW;
        if (r < NR) {
          const int o = r * RS + P + lane;
          const T f = uz ? iv[o] : (T)0;
          T v = ith * (f * (T)bb[o]);
          if (J >= 3) v = v + (T)bb[BOXS + o];
          yb[o] = v;
          if (lane < 2 * P) {
            const int oh = r * RS + hc;
            const T fh = uz ? iv[oh] : (T)0;
            T vh = ith * (fh * (T)bb[oh]);
            if (J >= 3) vh = vh + (T)bb[BOXS + oh];
            yb[oh] = vh;
          }
        }
      }
    }
    __syncthreads();
    xpass<P>(yb, 0, km, kk, XA, XB, w, lane);
    __syncthreads();
    T c, s;
    ypass<P>(cf, ty, XA, XB, w, lane, c, s);
#pragma unroll
    for (int o = 0; o < R - 1; ++o) {
      cr[o] = cr[o + 1];
      sr[o] = sr[o + 1];
    }
    cr[R - 1] = c;
    sr[R - 1] = s;
    if (produce) {
      const int z = zi - P;
      const T ay = zpass<P>(cf, tz, cr, sr) * hl;
      const int o = (w + P) * RS + P + lane;
      const S* bo = ring + oisl * NA * BOXS + SHS + o;  // plane z, output point
      const T b = (T)bo[0];
      const T f = (z >= 1 && z <= n - 1) ? ivd[tz * BOX + o] : (T)0;
      T yprev = ith * (f * b);
      T dprev = yprev;
      if (J >= 3) {
        dprev = (T)bo[BOXS];
        yprev = yprev + dprev;
      }
      const T qq = b - ay;
      const T d = fma(al, dprev, be * (f * qq));
      const T yv = yprev + d;
      if (FIN == 1) {
        if (rowok) *Dp = (S)yv;  // y_k -> Y (k_f3_tpb<1> finalises)
      } else if (FIN == 2) {  // ý = enc_{w_r}(y_k) as mantissa + exponent (k_f3_tpb<2> finalises)
        long long mq = 0;
        int Eq = -128;
        warp_encode((double)yv, a.wr, nullptr, nullptr, lane, a.status, &mq, &Eq);
        if (rowok) {
          a.my[pbase0 + (long long)(z - tl.zs) * tplane] = (int8_t)mq;
          if (lane == 0) a.ey[uep - a.uexp] = (int8_t)Eq;
        }
      } else if (a.last) {
        const double yq = warp_encode((double)yv, a.wr, nullptr, nullptr, lane, a.status);
        if (rowok) {
          const double* ax = aring + osl * 2 * 32 * FW + tid;
          if (a.wout) a.W[pbase0 + (long long)(z - tl.zs) * tplane] = (double)((T)ax[0] + (T)yq);  // w_l = z_l + dec ý_l
          const uint32_t* rec = wring + osl * FW * RW + w * RW;
          const double uo = warp_decode(rec, rec_e(rec + a.wu, eoff), a.wu, lane);
          const double uq = warp_encode(uo + yq, a.wu_out, ump, uep, lane, a.status);
          if (a.uout) a.U[pbase0 + (long long)(z - tl.zs) * tplane] = uq + ax[32 * FW];  // u_l = dec ú_l + P u_{l-1}
        }
      } else if (rowok) {
        *Dp = (S)d;
      }
      Dp += tplane;
      ump += ustep;
      uep += bpp;
      osl = osl + 1 == NW ? 0 : osl + 1;
    }
    tz = tz + 1 == P ? 0 : tz + 1;
    oisl = oisl + 1 == NBF ? 0 : oisl + 1;
    if (++isl == NBF) {
      isl = 0;
      par ^= 1u;
    }
  }
}

// P u_{l-1} at the points of the 32 x 8 tile, marched along z (no halo): the
// P-u-only prolongation of the finest-level path (PU for the last Chebyshev
// step) and the level-push decode u_l = dec ú_l + P u_{l-1}.  Same coarse-box
// TMA ring and canonical x, y, z passes as the generating kernels (DESIGN.md
// §3.3), but one point per thread: warp w's x pass covers coarse rows w,
// w + 8 of the box, its y pass and z pass fine row y0 + w.  Replaces
// k_m3_prolong's per-point (p+1)^2 global loads by shared boxes.
// NA = 2 (the top level of the materialised form): the same for two coarse
// arrays at once, u_{l-1} -> PU and w_{l-1} -> a.out2 (z_l for k_f3_staged<P, 2>).
template <int P, int NA, class TW = double>
__global__ void __launch_bounds__(32 * FW, 4) k_f3_prolong(const __grid_constant__ F3Args a,
                                                            const __grid_constant__ CoefT<double> cf) {
  using C = F3<P>;
  constexpr int CBX = C::CBX, CBY = C::CBY, NCB = C::NCB, NCY = C::NCY, PF = C::PF, NW = C::NW;
  extern __shared__ __align__(128) double fsm[];
  double* craw = fsm;                         // NA x NCB coarse boxes (TMA)
  double* PX = craw + NA * NCB * C::CBS;      // NA x CBY x 32: x pass
  double* yv = PX + NA * CBY * 32;            // NA x NCY x FW x 32: xy-passed coarse planes at the tile
  uint32_t* wring = (uint32_t*)(yv + NA * NCY * FW * 32);  // NW x FW x (w + 1): ú words (decode mode)
  const int RW = a.wu + 1;
  unsigned long long* cbar = (unsigned long long*)(wring + NW * FW * RW + 2);
  cbar = (unsigned long long*)(((uintptr_t)cbar + 7) & ~(uintptr_t)7);  // NA x NCB
  const int lane = threadIdx.x, w = threadIdx.y;
  const F3Tile tl = f3_tile(a);
  const Geom g = a.g;
  const int n = g.n;
  const int x = tl.x0 + lane, y = tl.y0 + w;
  const bool rowok = y < g.NY;
  const bool okx = unk1(x, n), oky = unk1(y, n);
  Gen<P> gn;  // (only the coarse-box bookkeeping: origin, plane range, TMA ring)
  gn.cx0 = (P * (max(tl.x0 - P, 1) / (2 * P))) & ~1;
  gn.cy0 = P * (max(tl.y0 - P, 1) / (2 * P));
  gn.czoff = a.czoff;
  gen_range<P>(gn, tl.zs, tl.ze - tl.zs, n);
  const int bxo = okx ? P * (x / (2 * P)) - gn.cx0 : 0, rx = okx ? x % (2 * P) : 0;
  const int byo = oky ? P * (y / (2 * P)) - gn.cy0 : 0, ry = oky ? y % (2 * P) : 0;
  double pwx[P + 1], pwy[P + 1];
  TW pwxw[P + 1], pwyw[P + 1];  // (NA = 2, TW = float: P w_{l-1} in FP32 cFas, reading R28)
#pragma unroll
  for (int t = 0; t <= P; ++t) {
    pwx[t] = cf.Pw[rx][t];
    pwy[t] = cf.Pw[ry][t];
    pwxw[t] = (TW)pwx[t];
    pwyw[t] = (TW)pwy[t];
  }
  constexpr bool FW2 = NA == 2 && sizeof(TW) == 4;  // the second array in float
  const bool decode = NA == 1 && a.step == 1;  // (1: u_l = dec ú_l + P u_{l-1} -> U; 0: P u_{l-1} -> PU)
  int eoff = 0;
  const WStream ws = wstream1(a.umant, a.uexp, a.ustride, a.wu, g, tl.x0, y, tl.zs, w * RW, rowok && decode, lane,
                              eoff);
  const unsigned wring_s = smem_u32(wring);
  const long long tplane = (long long)g.NY * g.NX;
  const long long o0 = ((long long)tl.zs * g.NY + y) * g.NX + x;
  double* out = (decode ? a.U : a.PU) + o0;
  double* out2 = NA == 2 ? a.out2 + o0 : nullptr;
  float* out2f = NA == 2 ? (float*)a.out2 + o0 : nullptr;  // (FP32 cFas, float storage: z_l as float)
  const bool fs2 = FW2 && a.f32s;
  const CUtensorMap* tms[2] = {a.tmc, NA == 2 ? a.tmc2 : a.tmc};
  const int nout = tl.ze - tl.zs;
  if (threadIdx.x == 0 && threadIdx.y == 0) {
#pragma unroll
    for (int k = 0; k < NA * NCB; ++k) mbar_init(cbar + k, 1);
    mbar_init_fence();
  }
  __syncthreads();
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x == 0 && threadIdx.y == 0)
    for (int q = 0; q < NA; ++q)
      for (int k = 0; k < NCB; ++k)
        gen_request<P>(gn, tms[q], craw + q * NCB * C::CBS, cbar + q * NCB, gn.cfirst + k);
#pragma unroll
  for (int j = 0; j < PF; ++j) {
    if (j < nout) wcopy(ws, wring_s + (unsigned)(j * FW * RW * 4), j);
    cpa_commit();
  }
  int osl = 0;
  for (int j = 0; j < nout; ++j) {
    const int z = tl.zs + j;
    {
      const int sl = osl + PF >= NW ? osl + PF - NW : osl + PF;
      if (j + PF < nout) wcopy(ws, wring_s + (unsigned)(sl * FW * RW * 4), j + PF);
    }
    cpa_commit();
    const bool okz = unk1(z, n);
    if (okz) {
      const int cneed = cbase<P>(z) + P;
      while (gn.cdone <= cneed) {  // x and y passes of the next coarse plane
        const int c = gn.cdone, k = c - gn.cfirst;
#pragma unroll
        for (int q = 0; q < NA; ++q) {
          mbar_wait_s(smem_u32(cbar + q * NCB) + 8u * (unsigned)(k % NCB), (unsigned)(k / NCB) & 1u);
          const double* cb = craw + (q * NCB + k % NCB) * C::CBS;
#pragma unroll
          for (int r = 0; r < (CBY + FW - 1) / FW; ++r) {
            const int cr = w + r * FW;
            if (cr < CBY) {
              if (FW2 && q == 1) {
                TW acc = 0;
                if (okx) {
#pragma unroll
                  for (int t = 0; t <= P; ++t) acc = fma(pwxw[t], (TW)cb[cr * CBX + bxo + t], acc);
                }
                PX[(q * CBY + cr) * 32 + lane] = (double)acc;
              } else {
                double acc = 0.0;
                if (okx) {
#pragma unroll
                  for (int t = 0; t <= P; ++t) acc = fma(pwx[t], cb[cr * CBX + bxo + t], acc);
                }
                PX[(q * CBY + cr) * 32 + lane] = acc;
              }
            }
          }
        }
        __syncthreads();
        if (threadIdx.x == 0 && threadIdx.y == 0)
          for (int q = 0; q < NA; ++q) gen_request<P>(gn, tms[q], craw + q * NCB * C::CBS, cbar + q * NCB, c + NCB);
#pragma unroll
        for (int q = 0; q < NA; ++q) {
          if (FW2 && q == 1) {
            TW acc = 0;
            if (oky) {
#pragma unroll
              for (int t = 0; t <= P; ++t) acc = fma(pwyw[t], (TW)PX[(q * CBY + byo + t) * 32 + lane], acc);
            }
            yv[((q * NCY + c % NCY) * FW + w) * 32 + lane] = (double)acc;
          } else {
            double acc = 0.0;
            if (oky) {
#pragma unroll
              for (int t = 0; t <= P; ++t) acc = fma(pwy[t], PX[(q * CBY + byo + t) * 32 + lane], acc);
            }
            yv[((q * NCY + c % NCY) * FW + w) * 32 + lane] = acc;
          }
        }
        gn.cdone = c + 1;
        __syncthreads();
      }
    }
    double pu[NA];
#pragma unroll
    for (int q = 0; q < NA; ++q) {
      pu[q] = 0.0;
      if (okz) {
        const int rz = z % (2 * P), cb0 = cbase<P>(z);
        if (FW2 && q == 1) {
          TW acc = 0;
#pragma unroll
          for (int t = 0; t <= P; ++t)
            acc = fma((TW)cf.Pw[rz][t], (TW)yv[((q * NCY + (cb0 + t) % NCY) * FW + w) * 32 + lane], acc);
          pu[q] = (double)acc;
        } else {
#pragma unroll
          for (int t = 0; t <= P; ++t)
            pu[q] = fma(cf.Pw[rz][t], yv[((q * NCY + (cb0 + t) % NCY) * FW + w) * 32 + lane], pu[q]);
        }
      }
    }
    if (decode) {
      cpa_wait<PF>();
      __syncwarp();
      if (rowok) {
        const uint32_t* rec = wring + osl * FW * RW + w * RW;
        const double dv = warp_decode(rec, rec_e(rec + a.wu, eoff), a.wu, lane);
        *out = dv + pu[0];  // u_l = dec ú_l + P u_{l-1}
      }
    } else if (rowok) {
      *out = pu[0];
      if (NA == 2) {
        if (fs2) *out2f = (float)pu[NA - 1];
        else *out2 = pu[NA - 1];
      }
    }
    out += tplane;
    if (NA == 2) out2 += tplane, out2f += tplane;
    osl = osl + 1 == NW ? 0 : osl + 1;
  }
}

// k_f3_prolong with 32 x 16 tiles: each warp produces fine rows y0 + w and
// y0 + w + 8 (two independent chains in the y and z passes, half the barriers
// per point).  p = 1, 3 (the coarse box covers 16 fine rows there).  Same
// passes and order as k_f3_prolong.
template <int P, int NA, class TW = double>
__global__ void __launch_bounds__(32 * FW, 4) k_f3_prolong2(const __grid_constant__ F3Args a,
                                                             const __grid_constant__ CoefT<double> cf) {
  using C = F3<P>;
  constexpr int CBX = C::CBX, CBY = C::CBY, NCB = C::NCB, NCY = C::NCY, PF = C::PF, NW = C::NW, TH = 2 * FW;
  extern __shared__ __align__(128) double fsm[];
  double* craw = fsm;                          // NA x NCB coarse boxes (TMA)
  double* PX = craw + NA * NCB * C::CBS;       // NA x CBY x 32: x pass
  double* yv = PX + NA * CBY * 32;             // NA x NCY x TH x 32
  uint32_t* wring = (uint32_t*)(yv + NA * NCY * TH * 32);  // NW x TH x (w + 1): ú words (decode mode)
  const int RW = a.wu + 1;
  unsigned long long* cbar = (unsigned long long*)(wring + NW * TH * RW + 2);
  cbar = (unsigned long long*)(((uintptr_t)cbar + 7) & ~(uintptr_t)7);
  const int lane = threadIdx.x, w = threadIdx.y;
  const Geom g = a.g;
  const int n = g.n;
  // tile: 32 x 16 columns, z chunk of a.RC planes (a.nyb: tile rows of 16)
  F3Tile tl;
  {
    const int tiles = a.nxb * a.nyb, q = blockIdx.x % tiles, ch = blockIdx.x / tiles;
    tl.x0 = (q % a.nxb) * 32;
    tl.y0 = (q / a.nxb) * TH;
    tl.zs = a.zlo + ch * a.RC;
    tl.ze = min(a.zhi, tl.zs + a.RC);
    tl.cta = blockIdx.x;
  }
  const int x = tl.x0 + lane;
  const bool okx = unk1(x, n);
  Gen<P> gn;
  gn.cx0 = (P * (max(tl.x0 - P, 1) / (2 * P))) & ~1;
  gn.cy0 = P * (max(tl.y0 - P, 1) / (2 * P));
  gn.czoff = a.czoff;
  gen_range<P>(gn, tl.zs, tl.ze - tl.zs, n);
  const int bxo = okx ? P * (x / (2 * P)) - gn.cx0 : 0, rx = okx ? x % (2 * P) : 0;
  double pwx[P + 1];
  TW pwxw[P + 1];  // (NA = 2, TW = float: P w_{l-1} in FP32 cFas, reading R28)
#pragma unroll
  for (int t = 0; t <= P; ++t) {
    pwx[t] = cf.Pw[rx][t];
    pwxw[t] = (TW)pwx[t];
  }
  constexpr bool FW2 = NA == 2 && sizeof(TW) == 4;  // the second array in float
  int byo[2], ry[2];
  bool oky[2], rowok[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int y = tl.y0 + w + h * FW;
    rowok[h] = y < g.NY;
    oky[h] = unk1(y, n);
    byo[h] = oky[h] ? P * (y / (2 * P)) - gn.cy0 : 0;
    ry[h] = oky[h] ? y % (2 * P) : 0;
  }
  double pwy[2][P + 1];  // y-pass weights of the warp's two rows (registers, not per-tap constant loads)
  TW pwyw[2][P + 1];
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int t = 0; t <= P; ++t) {
      pwy[h][t] = cf.Pw[ry[h]][t];
      pwyw[h][t] = (TW)pwy[h][t];
    }
  const bool decode = NA == 1 && a.step == 1;
  int eoff[2] = {0, 0};
  const WStream ws0 = wstream1(a.umant, a.uexp, a.ustride, a.wu, g, tl.x0, tl.y0 + w, tl.zs, w * RW,
                               rowok[0] && decode, lane, eoff[0]);
  const WStream ws1 = wstream1(a.umant, a.uexp, a.ustride, a.wu, g, tl.x0, tl.y0 + w + FW, tl.zs, (w + FW) * RW,
                               rowok[1] && decode, lane, eoff[1]);
  const unsigned wring_s = smem_u32(wring);
  const long long tplane = (long long)g.NY * g.NX;
  const long long o0 = ((long long)tl.zs * g.NY + tl.y0 + w) * g.NX + x;
  double* out = (decode ? a.U : a.PU) + o0;
  double* out2 = NA == 2 ? a.out2 + o0 : nullptr;
  float* out2f = NA == 2 ? (float*)a.out2 + o0 : nullptr;  // (FP32 cFas, float storage: z_l as float)
  const bool fs2 = FW2 && a.f32s;
  const long long rs8 = (long long)FW * g.NX;  // the second row, 8 rows down
  const CUtensorMap* tms[2] = {a.tmc, NA == 2 ? a.tmc2 : a.tmc};
  const int nout = tl.ze - tl.zs;
  if (threadIdx.x == 0 && threadIdx.y == 0) {
#pragma unroll
    for (int k = 0; k < NA * NCB; ++k) mbar_init(cbar + k, 1);
    mbar_init_fence();
  }
  __syncthreads();
  pdl_wait();
  pdl_trigger();
  if (threadIdx.x == 0 && threadIdx.y == 0)
    for (int q = 0; q < NA; ++q)
      for (int k = 0; k < NCB; ++k)
        gen_request<P>(gn, tms[q], craw + q * NCB * C::CBS, cbar + q * NCB, gn.cfirst + k);
#pragma unroll
  for (int j = 0; j < PF; ++j) {
    if (j < nout) {
      wcopy(ws0, wring_s + (unsigned)(j * TH * RW * 4), j);
      wcopy(ws1, wring_s + (unsigned)(j * TH * RW * 4), j);
    }
    cpa_commit();
  }
  int osl = 0;
  for (int j = 0; j < nout; ++j) {
    const int z = tl.zs + j;
    {
      const int sl = osl + PF >= NW ? osl + PF - NW : osl + PF;
      if (j + PF < nout) {
        wcopy(ws0, wring_s + (unsigned)(sl * TH * RW * 4), j + PF);
        wcopy(ws1, wring_s + (unsigned)(sl * TH * RW * 4), j + PF);
      }
    }
    cpa_commit();
    const bool okz = unk1(z, n);
    if (okz) {
      const int cneed = cbase<P>(z) + P;
      while (gn.cdone <= cneed) {
        const int c = gn.cdone, k = c - gn.cfirst;
#pragma unroll
        for (int q = 0; q < NA; ++q) {
          mbar_wait_s(smem_u32(cbar + q * NCB) + 8u * (unsigned)(k % NCB), (unsigned)(k / NCB) & 1u);
          const double* cb = craw + (q * NCB + k % NCB) * C::CBS;
#pragma unroll
          for (int r = 0; r < (CBY + FW - 1) / FW; ++r) {
            const int cr = w + r * FW;
            if (cr < CBY) {
              if (FW2 && q == 1) {
                TW acc = 0;
                if (okx) {
#pragma unroll
                  for (int t = 0; t <= P; ++t) acc = fma(pwxw[t], (TW)cb[cr * CBX + bxo + t], acc);
                }
                PX[(q * CBY + cr) * 32 + lane] = (double)acc;
              } else {
                double acc = 0.0;
                if (okx) {
#pragma unroll
                  for (int t = 0; t <= P; ++t) acc = fma(pwx[t], cb[cr * CBX + bxo + t], acc);
                }
                PX[(q * CBY + cr) * 32 + lane] = acc;
              }
            }
          }
        }
        __syncthreads();
        if (threadIdx.x == 0 && threadIdx.y == 0)
          for (int q = 0; q < NA; ++q) gen_request<P>(gn, tms[q], craw + q * NCB * C::CBS, cbar + q * NCB, c + NCB);
#pragma unroll
        for (int q = 0; q < NA; ++q)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (FW2 && q == 1) {
              TW acc = 0;
              if (oky[h]) {
#pragma unroll
                for (int t = 0; t <= P; ++t) acc = fma(pwyw[h][t], (TW)PX[(q * CBY + byo[h] + t) * 32 + lane], acc);
              }
              yv[((q * NCY + c % NCY) * TH + w + h * FW) * 32 + lane] = (double)acc;
            } else {
              double acc = 0.0;
              if (oky[h]) {
#pragma unroll
                for (int t = 0; t <= P; ++t) acc = fma(pwy[h][t], PX[(q * CBY + byo[h] + t) * 32 + lane], acc);
              }
              yv[((q * NCY + c % NCY) * TH + w + h * FW) * 32 + lane] = acc;
            }
          }
        gn.cdone = c + 1;
        __syncthreads();
      }
    }
    double pu[NA][2];
    // z pass: per plane the P + 1 weights and the ring rows of the taps once
    // (shared by both arrays and both rows; constant offsets below)
    const int rz = okz ? z % (2 * P) : 0, cb0 = okz ? cbase<P>(z) : 0;
    double pz[P + 1];
    TW pzw[P + 1];
    const double* ys[P + 1];
#pragma unroll
    for (int t = 0; t <= P; ++t) {
      pz[t] = cf.Pw[rz][t];
      pzw[t] = (TW)pz[t];
      ys[t] = yv + (((cb0 + t) % NCY) * TH + w) * 32 + lane;
    }
#pragma unroll
    for (int q = 0; q < NA; ++q)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        pu[q][h] = 0.0;
        if (okz) {
          const int off = (q * NCY * TH + h * FW) * 32;
          if (FW2 && q == 1) {
            TW acc = 0;
#pragma unroll
            for (int t = 0; t <= P; ++t) acc = fma(pzw[t], (TW)ys[t][off], acc);
            pu[q][h] = (double)acc;
          } else {
#pragma unroll
            for (int t = 0; t <= P; ++t) pu[q][h] = fma(pz[t], ys[t][off], pu[q][h]);
          }
        }
      }
    if (decode) {
      cpa_wait<PF>();
      __syncwarp();
#pragma unroll
      for (int h = 0; h < 2; ++h)
        if (rowok[h]) {
          const uint32_t* rec = wring + osl * TH * RW + (w + h * FW) * RW;
          const double dv = warp_decode(rec, rec_e(rec + a.wu, eoff[h]), a.wu, lane);
          out[h * rs8] = dv + pu[0][h];  // u_l = dec ú_l + P u_{l-1}
        }
    } else {
#pragma unroll
      for (int h = 0; h < 2; ++h)
        if (rowok[h]) {
          out[h * rs8] = pu[0][h];
          if (NA == 2) {
            if (fs2) out2f[h * rs8] = (float)pu[NA - 1][h];
            else out2[h * rs8] = pu[NA - 1][h];
          }
        }
    }
    out += tplane;
    if (NA == 2) out2 += tplane, out2f += tplane;
    osl = osl + 1 == NW ? 0 : osl + 1;
  }
}

// Staged-input sweeps of the materialised form: the
// skeleton of k_f3_cheb (specialised y / z passes, incremental slots) over a
// TMA-staged FP64 input v, then per output point:
//   K = 0, 1: t_L = f_L - A_L u_L (v = u_L); t_L -> HBM; ||t_L||^2 partial per
//             warp; K = 0 also r_L = enc(t_L) (K = 1: k_f3_tpb<0> encodes);
//   K = 2:    b_L = dec r_L - A_L z_L (v = z_L = P w_{L-1}, materialised by
//             k_f3_prolong) -> the t_L buffer: cFas step 1 at the top level;
//             with a.yout also y_1 = inv_theta (invD b) -> a.yout;
//   K = 3, 4: Chebyshev step j = K - 1 from v = y_{j-1} (materialised by the
//             step before): b (and d_2 for j = 3) are read at the output
//             point only, d_j = fma(al_j, d_{j-1}, be_j (invD (b - A y_{j-1}))),
//             y_j = y_{j-1} + d_j -> a.yout, and d_2 -> a.Dv when j = 2 is
//             not the last step.  Same expressions as k_f3_cheb (which
//             recomputes y_{j-1} on its staged b / d_2 boxes instead).
template <int P, int K, class T = double, int WR = 0, bool FS = false>
__global__ void __launch_bounds__(32 * FW, F3_MINB_ST(P, T)) k_f3_staged(const __grid_constant__ F3Args a,
                                                                     const __grid_constant__ CoefT<T> cf) {
  static_assert(K >= 2 || sizeof(T) == 8, "the residual is FP64");
  using C = F3<P>;
  constexpr int R = C::R, NR = C::NR, RS = C::RS, BOX = C::BOX, NBF = C::NBF, PF = C::PF, NW = C::NW;
  constexpr int NX_ = K == 4 ? 2 : 1;  // point arrays of K = 3, 4: b (+ d_2)
  // FS: FP32 cFas with float storage (as k_f3_staged2): cFas step 1 only
  static_assert(!FS || (sizeof(T) == 4 && K == 2), "float storage: FP32 cFas step 1");
  using S = typename std::conditional<FS, float, double>::type;
  constexpr int SHS = FS ? 4 - P : (P & 1);
  constexpr int BOXS = FS ? ((BOX + 31) & ~31) : BOX;
  extern __shared__ __align__(128) double fsm[];
  S* ring = (S*)fsm;  // NBF boxes of v
  T* XA = (T*)(fsm + NBF * BOX);  // (T = float: FP32 cFas, reading R28)
  T* XB = XA + NR * 32;
  double* aring = fsm + NBF * BOX + 2 * NR * 32;  // (K >= 3) NW x NX_ x 256: b (+ d_2) at the output points
  uint32_t* wring = (uint32_t*)(aring + (K >= 3 ? NW * NX_ * 32 * FW : 0));  // (K = 2) NW x FW x (w_r + 1)
  const int wr_ = WR > 0 ? WR : a.wr;  // (K = 2: w_r(L, L), compile-time for the common widths)
  const int RW = wr_ + 1;
  unsigned long long* bars = (unsigned long long*)(wring + (K == 2 ? NW * FW * RW + 2 : 0));
  bars = (unsigned long long*)(((uintptr_t)bars + 7) & ~(uintptr_t)7);
  const int lane = threadIdx.x, w = threadIdx.y;
  const F3Tile tl = f3_tile(a);
  const Geom g = a.g;
  const int n = g.n;
  const int x = tl.x0 + lane, y = tl.y0 + w;
  const bool rowok = y < g.NY;
  const int tx = x % P, ty = y % P;
  T km[R], kk[R];
#pragma unroll
  for (int o = 0; o < R; ++o) {
    km[o] = cf.Mc[tx][o];
    kk[o] = cf.Kc[tx][o];
  }
  const T hl = (T)pow2(-(a.l + 1));
  const double* __restrict__ gt = a.gtab;
  const bool uxy = unk1(x, n) && unk1(y, n);
  const double gxy = K < 2 && uxy ? (cf.rhs_c * gt[x]) * gt[y] : 0.0;
  // invD at the output point per z node type (RN(1/diag) 2^(l+1), 0 at non-unknowns)
  T fv[P];
#pragma unroll
  for (int t = 0; t < P; ++t) fv[t] = uxy ? cf.invd[(t * P + ty) * P + tx] * (T)pow2(a.l + 1) : (T)0;
  const T al = cf.cal[K - 2 > 0 ? K - 2 : 0], be = cf.cbe[K - 2 > 0 ? K - 2 : 0], ith = cf.inv_theta;
  const int nxb = g.NX >> 5;
  const int z0 = tl.zs - P, nin = (tl.ze - tl.zs) + 2 * P;
  const long long tplane = (long long)g.NY * g.NX, bpp = (long long)g.NY * nxb;
  const long long pbase0 = ((long long)tl.zs * g.NY + y) * g.NX + x;
  double* Tp = a.T + pbase0;
  S* Bp = (S*)a.T + pbase0;  // (K = 2: b_l)
  S* Yo = a.yout ? (S*)a.yout + pbase0 : nullptr;
  double* Dp = a.Dv + pbase0;
  const long long blk0 = ((long long)tl.zs * g.NY + y) * nxb + (tl.x0 >> 5);
  uint32_t* rmp = a.rmant + blk0 * a.rstride;
  int8_t* rep = a.rexp + blk0;
  const long long rstep = bpp * a.rstride;
  const unsigned ring_s = smem_u32(ring), bars_s = smem_u32(bars), wring_s = smem_u32(wring);
  const unsigned aring_s = smem_u32(aring);
  const int tid = w * 32 + lane;
  const int nout = tl.ze - tl.zs;
  int eoff = 0;
  const WStream ws = wstream1(a.rmant, a.rexp, a.rstride, wr_, g, tl.x0, y, tl.zs, w * RW, K == 2 && rowok, lane,
                              eoff);
  auto pcopy = [&](int j, int slot) {  // (K >= 3) b (+ d_2) of output plane zs + j -> aux slot
    if (K >= 3 && rowok) {
      const unsigned d = aring_s + (unsigned)(((slot * NX_) * 32 * FW + tid) * 8);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(a.T + pbase0 + j * tplane) : "memory");
      if (K == 4)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d + 32 * FW * 8), "l"(a.Dv + pbase0 + j * tplane)
                     : "memory");
    }
  };
  if (threadIdx.x == 0 && threadIdx.y == 0) {
#pragma unroll
    for (int k = 0; k < NBF; ++k) mbar_init(bars + k, 1);
    mbar_init_fence();
  }
  __syncthreads();
  pdl_wait();
  pdl_trigger();
  const int tmx = tl.x0 - P - SHS, tmy = tl.y0 - P;
  auto stage = [&](int i, int slot) {  // plane z0 + i of v into ring slot `slot` (TMA, thread 0)
    if (threadIdx.x == 0 && threadIdx.y == 0) {
      const unsigned dst = ring_s + (unsigned)(slot * BOXS * sizeof(S)), bar = bars_s + (unsigned)(slot * 8);
      fence_async_smem();
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"((unsigned)(BOX * sizeof(S)))
                   : "memory");
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
          "[%5];" ::"r"(dst),
          "l"((unsigned long long)a.tmb), "r"(tmx), "r"(tmy), "r"(z0 + i - a.zoff), "r"(bar)
          : "memory");
    }
  };
#pragma unroll
  for (int i = 0; i < PF; ++i)
    if (i < nin) stage(i, i);
  if (K >= 2) {  // r_L words (K = 2) / point values (K >= 3) of output planes 0..PF-1 -> slots 0..PF-1
#pragma unroll
    for (int j = 0; j < PF; ++j) {
      if (j < nout) {
        if (K == 2) wcopy(ws, wring_s + (unsigned)(j * FW * RW * 4), j);
        else pcopy(j, j);
      }
      cpa_commit();
    }
  }
  T cr[R], sr[R];
#pragma unroll
  for (int o = 0; o < R; ++o) cr[o] = sr[o] = 0;
  double ss = 0.0;
  int tz = ((z0 % P) + P) % P;
  int isl = 0, osl = 0, oisl = NBF - P;  // slots: input plane i, words / points of the next output, input plane i - P
  unsigned par = 0;
  for (int i = 0; i < nin; ++i) {
    const int zi = z0 + i;
    const bool produce = i >= 2 * P;
    mbar_wait_s(bars_s + 8u * (unsigned)isl, par);
    if (K >= 2) cpa_wait<PF - 1>();
    __syncthreads();  // every thread is past iteration i - 1 (slot and XA/XB reuse)
    if (i + PF < nin) stage(i + PF, isl + PF >= NBF ? isl + PF - NBF : isl + PF);
    if (K >= 2) {
      if (produce) {
        const int j = i - 2 * P + PF;
        const int sl = osl + PF >= NW ? osl + PF - NW : osl + PF;
        if (j < nout) {
          if (K == 2) wcopy(ws, wring_s + (unsigned)(sl * FW * RW * 4), j);
          else pcopy(j, sl);
        }
      }
      cpa_commit();
    }
    xpass<P>(ring + isl * BOXS, SHS, km, kk, XA, XB, w, lane);
    __syncthreads();
    T c, s;
    ypass<P>(cf, ty, XA, XB, w, lane, c, s);
#pragma unroll
    for (int o = 0; o < R - 1; ++o) {
      cr[o] = cr[o + 1];
      sr[o] = sr[o + 1];
    }
    cr[R - 1] = c;
    sr[R - 1] = s;
    if (produce) {
      const int z = zi - P;
      const T av = zpass<P>(cf, tz, cr, sr) * hl;
      const bool uz = unk1(z, n);
      if (K >= 3) {
        if (rowok) {
          const double* ax = aring + osl * NX_ * 32 * FW + tid;
          const T b = (T)ax[0];
          T f = fv[0];  // (selected with constant indices: fv stays in registers)
#pragma unroll
          for (int t = 1; t < P; ++t) f = tz == t ? fv[t] : f;
          f = uz ? f : (T)0;
          const T yprev = (T)ring[oisl * BOXS + SHS + (w + P) * RS + P + lane];  // y_{j-1} at the point
          const T dprev = K == 4 ? (T)ax[32 * FW] : yprev;                        // d_{j-1} (d_1 = y_1)
          const T qq = b - av;
          const T d = fma(al, dprev, be * (f * qq));
          const T yv = yprev + d;
          *Yo = (S)yv;
          if (!a.last) *Dp = (double)d;
        }
        Yo += tplane;
        Dp += tplane;
        osl = osl + 1 == NW ? 0 : osl + 1;
      } else if (K == 2) {
        if (rowok) {
          const uint32_t* rec = wring + osl * FW * RW + w * RW;
          const double rv = dec_rec<WR>(rec, rec_e(rec + wr_, eoff), wr_, lane);
          const T b = (T)rv - av;  // b = dec r - A z (B lives in the t_L buffer)
          *Bp = (S)b;
          if (Yo) {
            T f = fv[0];
#pragma unroll
            for (int t = 1; t < P; ++t) f = tz == t ? fv[t] : f;
            *Yo = (S)(ith * ((uz ? f : (T)0) * b));  // y_1 = inv_theta (invD b)
          }
        }
        if (Yo) Yo += tplane;
        osl = osl + 1 == NW ? 0 : osl + 1;
      } else if (rowok) {
        const double gz = uz ? gt[z] : 0.0;
        const double t = (uxy && uz) ? gxy * gz - av : 0.0;  // (((C g(x)) g(y)) g(z)) - A u
        *Tp = t;
        ss = fma(t, t, ss);
        if (K == 0) warp_encode(t, a.wr, rmp, rep, lane, a.status);
      }
      Tp += tplane;
      Bp += tplane;
      rmp += rstep;
      rep += bpp;
    }
    tz = tz + 1 == P ? 0 : tz + 1;
    oisl = oisl + 1 == NBF ? 0 : oisl + 1;
    if (++isl == NBF) {
      isl = 0;
      par ^= 1u;
    }
  }
  if (K < 2) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(FULL, ss, o);
    if (lane == 0 && a.poff >= 0) a.pbase[a.poff + (long long)(a.ctaoff + tl.cta) * FW + w] = ss;
  }
}

// Two input planes per iteration: k_f3_staged with one
// barrier pair per two planes and twice the independent fma chains in the x,
// y and z passes (the single-plane kernel is latency bound: fixed-latency
// dependences and barrier waits).  Same expressions, same order per output.
template <int P>
struct F3S2 {
  static constexpr int PF = 2;              // planes staged ahead (one pair)
  static constexpr int NBF = P + 4;         // ring slots: pair being read, pair in flight, centre planes i - P
  static constexpr int NW = PF + 4;         // word / point slots per output
};
template <int P, int K, class T = double, int WR = 0, bool FS = false>
__global__ void __launch_bounds__(32 * FW, F3_MINB_ST(P, T)) k_f3_staged2(const __grid_constant__ F3Args a,
                                                                      const __grid_constant__ CoefT<T> cf) {
  static_assert(K >= 2 || sizeof(T) == 8, "the residual is FP64");
  using C = F3<P>;
  constexpr int R = C::R, NR = C::NR, RS = C::RS, BOX = C::BOX;
  constexpr int NBF = F3S2<P>::NBF, PF = F3S2<P>::PF, NW = F3S2<P>::NW;
  constexpr int NX_ = K == 4 ? 2 : 1;
  // FS: FP32 cFas with float storage: the staged input and
  // the point arrays (z_l, b, y_j, d_2) are float arrays over the same
  // buffers, float TMA boxes start at x0 - 4 (16-byte aligned), shift 4 - P
  static_assert(!FS || (sizeof(T) == 4 && K >= 2), "float storage: FP32 cFas only");
  using S = typename std::conditional<FS, float, double>::type;
  constexpr int SHS = FS ? 4 - P : (P & 1);
  constexpr int BOXS = FS ? ((BOX + 31) & ~31) : BOX;  // ring slot stride (TMA destinations 128-byte aligned)
  extern __shared__ __align__(128) double fsm[];
  S* ring = (S*)fsm;                      // NBF boxes of v
  T* XA = (T*)(fsm + NBF * BOX);          // 2 planes x NR x 32 (T = float: FP32 cFas, reading R28)
  T* XB = XA + 2 * NR * 32;
  S* aring = (S*)(fsm + NBF * BOX + 4 * NR * 32);  // (K >= 3) NW x NX_ x 256
  uint32_t* wring = (uint32_t*)(aring + (K >= 3 ? NW * NX_ * 32 * FW : 0));  // (K = 2) NW x FW x (w_r + 1)
  const int wr_ = WR > 0 ? WR : a.wr;  // (K = 2: w_r(L, L), compile-time for the common widths)
  const int RW = wr_ + 1;
  unsigned long long* bars = (unsigned long long*)(wring + (K == 2 ? NW * FW * RW + 2 : 0));
  bars = (unsigned long long*)(((uintptr_t)bars + 7) & ~(uintptr_t)7);
  const int lane = threadIdx.x, w = threadIdx.y;
  const F3Tile tl = f3_tile(a);
  const Geom g = a.g;
  const int n = g.n;
  const int x = tl.x0 + lane, y = tl.y0 + w;
  const bool rowok = y < g.NY;
  const int tx = x % P, ty = y % P;
  T km[R], kk[R];
#pragma unroll
  for (int o = 0; o < R; ++o) {
    km[o] = cf.Mc[tx][o];
    kk[o] = cf.Kc[tx][o];
  }
  const T hl = (T)pow2(-(a.l + 1));
  const double* __restrict__ gt = a.gtab;
  const bool uxy = unk1(x, n) && unk1(y, n);
  const double gxy = K < 2 && uxy ? (cf.rhs_c * gt[x]) * gt[y] : 0.0;
  T fv[P];
#pragma unroll
  for (int t = 0; t < P; ++t) fv[t] = uxy ? cf.invd[(t * P + ty) * P + tx] * (T)pow2(a.l + 1) : (T)0;
  const T al = cf.cal[K - 2 > 0 ? K - 2 : 0], be = cf.cbe[K - 2 > 0 ? K - 2 : 0], ith = cf.inv_theta;
  const int nxb = g.NX >> 5;
  const int z0 = tl.zs - P, nin = (tl.ze - tl.zs) + 2 * P;
  const long long tplane = (long long)g.NY * g.NX, bpp = (long long)g.NY * nxb;
  const long long pbase0 = ((long long)tl.zs * g.NY + y) * g.NX + x;
  double* Tp = a.T + pbase0;                               // (K < 2: t_L)
  S* Bp = (S*)a.T + pbase0;                                // (K = 2: b_l)
  S* Yo = a.yout ? (S*)a.yout + pbase0 : nullptr;
  S* Dp = (S*)a.Dv + pbase0;
  const S* Tsrc = (const S*)a.T + pbase0;
  const S* Dsrc = (const S*)a.Dv + pbase0;
  const long long blk0 = ((long long)tl.zs * g.NY + y) * nxb + (tl.x0 >> 5);
  uint32_t* rmp = a.rmant + blk0 * a.rstride;
  int8_t* rep = a.rexp + blk0;
  const long long rstep = bpp * a.rstride;
  const unsigned ring_s = smem_u32(ring), bars_s = smem_u32(bars), wring_s = smem_u32(wring);
  const unsigned aring_s = smem_u32(aring);
  const int tid = w * 32 + lane;
  const int nout = tl.ze - tl.zs;
  int eoff = 0;
  const WStream ws = wstream1(a.rmant, a.rexp, a.rstride, wr_, g, tl.x0, y, tl.zs, w * RW, K == 2 && rowok, lane,
                              eoff);
  auto pcopy = [&](int j, int slot) {
    if (K >= 3 && rowok) {
      constexpr unsigned SZ = sizeof(S);
      const unsigned d = aring_s + (unsigned)(((slot * NX_) * 32 * FW + tid) * SZ);
      asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(d), "l"(Tsrc + j * tplane), "n"(SZ) : "memory");
      if (K == 4)
        asm volatile("cp.async.ca.shared.global [%0], [%1], %2;\n" ::"r"(d + 32 * FW * SZ), "l"(Dsrc + j * tplane),
                     "n"(SZ)
                     : "memory");
    }
  };
  auto ocopy = [&](int j, int slot) {  // words (K = 2) / point values (K >= 3) of output plane zs + j
    if (j < nout) {
      if (K == 2) wcopy(ws, wring_s + (unsigned)(slot * FW * RW * 4), j);
      else if (K >= 3) pcopy(j, slot);
    }
  };
  if (threadIdx.x == 0 && threadIdx.y == 0) {
#pragma unroll
    for (int k = 0; k < NBF; ++k) mbar_init(bars + k, 1);
    mbar_init_fence();
  }
  __syncthreads();
  pdl_wait();
  pdl_trigger();
  const int tmx = tl.x0 - P - SHS, tmy = tl.y0 - P;
  auto stage = [&](int i, int slot) {
    if (threadIdx.x == 0 && threadIdx.y == 0) {
      const unsigned dst = ring_s + (unsigned)(slot * BOXS * sizeof(S)), bar = bars_s + (unsigned)(slot * 8);
      fence_async_smem();
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"((unsigned)(BOX * sizeof(S)))
                   : "memory");
      asm volatile(
          "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
          "[%5];" ::"r"(dst),
          "l"((unsigned long long)a.tmb), "r"(tmx), "r"(tmy), "r"(z0 + i - a.zoff), "r"(bar)
          : "memory");
    }
  };
#pragma unroll
  for (int i = 0; i < PF; ++i)
    if (i < nin) stage(i, i);
  if (K >= 2) {  // outputs 0, 1 -> slots 0, 1 (one group)
    ocopy(0, 0);
    ocopy(1, 1);
    cpa_commit();
  }
  T cr[R + 1], sr[R + 1];
#pragma unroll
  for (int o = 0; o <= R; ++o) cr[o] = sr[o] = 0;
  double ss = 0.0;
  int tz = ((z0 % P) + P) % P;           // node type of input plane i (= of output plane i - P)
  int isl = 0, osl = 0, oisl = NBF - P;  // slots: input plane i, words / points of output i - 2P, input plane i - P
  unsigned par = 0;                      // barrier phase of slot isl
  auto emit = [&](int z, T av, int tzo, int ois, int os) {  // the output at plane z
    const bool uz = unk1(z, n);
    if (K >= 3) {
      if (rowok) {
        const S* ax = aring + os * NX_ * 32 * FW + tid;
        const T b = (T)ax[0];
        T f = fv[0];
#pragma unroll
        for (int t = 1; t < P; ++t) f = tzo == t ? fv[t] : f;
        f = uz ? f : (T)0;
        const T yprev = (T)ring[ois * BOXS + SHS + (w + P) * RS + P + lane];
        const T dprev = K == 4 ? (T)ax[32 * FW] : yprev;
        const T qq = b - av;
        const T d = fma(al, dprev, be * (f * qq));
        const T yv = yprev + d;
        *Yo = (S)yv;
        if (!a.last) *Dp = (S)d;
      }
      Yo += tplane;
      Dp += tplane;
    } else if (K == 2) {
      if (rowok) {
        const uint32_t* rec = wring + os * FW * RW + w * RW;
        const double rv = dec_rec<WR>(rec, rec_e(rec + wr_, eoff), wr_, lane);
        const T b = (T)rv - av;
        *Bp = (S)b;
        if (Yo) {
          T f = fv[0];
#pragma unroll
          for (int t = 1; t < P; ++t) f = tzo == t ? fv[t] : f;
          *Yo = (S)(ith * ((uz ? f : (T)0) * b));
        }
      }
      if (Yo) Yo += tplane;
    } else if (rowok) {
      const double gz = uz ? gt[z] : 0.0;
      const double t = (uxy && uz) ? gxy * gz - av : 0.0;
      *Tp = t;
      ss = fma(t, t, ss);
      if (K == 0) warp_encode(t, a.wr, rmp, rep, lane, a.status);
    }
    Tp += tplane;
    Bp += tplane;
    rmp += rstep;
    rep += bpp;
  };
  for (int i = 0; i < nin; i += 2) {
    const bool two = i + 1 < nin;
    const int isl1 = isl + 1 == NBF ? 0 : isl + 1;
    const unsigned par1 = isl + 1 == NBF ? par ^ 1u : par;
    mbar_wait_s(bars_s + 8u * (unsigned)isl, par);
    if (two) mbar_wait_s(bars_s + 8u * (unsigned)isl1, par1);
    if (K >= 2) cpa_wait<0>();
    __syncthreads();  // every thread is past the previous pair (slots, XA/XB, output slots)
    {
      int s2 = isl + PF;
      s2 = s2 >= NBF ? s2 - NBF : s2;
      if (i + PF < nin) stage(i + PF, s2);
      if (i + PF + 1 < nin) stage(i + PF + 1, s2 + 1 == NBF ? 0 : s2 + 1);
    }
    if (K >= 2) {  // the outputs of the next pair (outputs start at i = 2P, even)
      if (i >= 2 * P) {
        const int j = i - 2 * P + PF;
        int sl = osl + PF;
        sl = sl >= NW ? sl - NW : sl;
        ocopy(j, sl);
        ocopy(j + 1, sl + 1 == NW ? 0 : sl + 1);
      }
      cpa_commit();
    }
    // x pass of both planes: rows w, w + 8 of each (four independent pairs of chains)
    {
      const S* b0 = ring + isl * BOXS + SHS;
      const S* b1 = ring + isl1 * BOXS + SHS;
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int r = w + k * FW;
        if (r < NR) {
          T s0 = 0, t0 = 0, s1 = 0, t1 = 0;
#pragma unroll
          for (int o = 0; o < R; ++o) {
            const T v0 = (T)b0[r * RS + lane + o];
            s0 = fma(km[o], v0, s0);
            t0 = fma(kk[o], v0, t0);
            if (two) {
              const T v1 = (T)b1[r * RS + lane + o];
              s1 = fma(km[o], v1, s1);
              t1 = fma(kk[o], v1, t1);
            }
          }
          XA[r * 32 + lane] = s0;
          XB[r * 32 + lane] = t0;
          XA[(NR + r) * 32 + lane] = s1;
          XB[(NR + r) * 32 + lane] = t1;
        }
      }
    }
    __syncthreads();
    T c0, s0, c1 = 0, s1 = 0;
    ypass<P>(cf, ty, XA, XB, w, lane, c0, s0);
    if (two) ypass<P>(cf, ty, XA + NR * 32, XB + NR * 32, w, lane, c1, s1);
#pragma unroll
    for (int o = 0; o < R - 1; ++o) {
      cr[o] = cr[o + 2];
      sr[o] = sr[o + 2];
    }
    cr[R - 1] = c0;
    sr[R - 1] = s0;
    cr[R] = c1;
    sr[R] = s1;
    // (ring: cr[k] = plane i + 1 - R + k; output of plane i uses cr[0..R-1], of plane i + 1 cr[1..R])
    const int tz1 = tz + 1 == P ? 0 : tz + 1;
    const int oisl1 = oisl + 1 == NBF ? 0 : oisl + 1;
    const int osl1 = osl + 1 == NW ? 0 : osl + 1;
    if (i >= 2 * P) {
      const T av0 = zpass<P>(cf, tz, cr, sr) * hl;
      if (two) {
        const T av1 = zpass<P>(cf, tz1, cr + 1, sr + 1) * hl;
        emit(z0 + i - P, av0, tz, oisl, osl);
        emit(z0 + i + 1 - P, av1, tz1, oisl1, osl1);
      } else {
        emit(z0 + i - P, av0, tz, oisl, osl);
      }
      osl = osl1 + 1 == NW ? 0 : osl1 + 1;
    } else if (two && i + 1 >= 2 * P) {
      const T av1 = zpass<P>(cf, tz1, cr + 1, sr + 1) * hl;
      emit(z0 + i + 1 - P, av1, tz1, oisl1, osl);
      osl = osl1;
    }
    tz = tz1 + 1 == P ? 0 : tz1 + 1;
    oisl = oisl1 + 1 == NBF ? 0 : oisl1 + 1;
    isl = isl1 + 1 == NBF ? 0 : isl1 + 1;
    par = (isl1 + 1 == NBF) ? par1 ^ 1u : par1;
  }
  if (K < 2) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(FULL, ss, o);
    if (lane == 0 && a.poff >= 0) a.pbase[a.poff + (long long)(a.ctaoff + tl.cta) * FW + w] = ss;
  }
}

// Thread-per-block epilogues: the BFP codec of the
// finest-level kernels' outputs moved out of the plane march, where the
// warp-cooperative codec (a block is one 32-point row) cost ~40 % of the last
// Chebyshev step's instructions.  A warp takes 32 consecutive blocks of the
// rank's planes [zlo, zhi): their doubles arrive by cp.async into a padded
// tile, one lane per block runs the codec (fmg_device.cuh tpb_*, the same
// arithmetic as warp_encode / warp_decode: reading R8), and the results leave
// through coalesced copies.
//   MODE 0: r_l = enc_{w_r}(t_l)                       (after k_f3_staged<P, 1>)
//   MODE 1: ý = enc_{w_r}(y_k) (values only), ú_l <- enc_{w_u'}(dec ú_l + ý),
//           w_l = z_l + ý (wout), u_l = ú_l + P u_{l-1} (uout)   (after k_f3_cheb<..., FIN>)
// Widths <= 32 (tpb_*).  T: the cFas arithmetic of w_l (FP32 cFas, R28).
constexpr int TP_WARPS = 4, TP_RS = 33, TP_WS = 33;
constexpr int tpb_smem_bytes() { return TP_WARPS * (32 * TP_RS * 8 + 32 * TP_WS * 4); }

// W, WR > 0: compile-time widths (tpb_*_w): MODE 1 without w_l with w_u = W,
// w_r = WR; MODE 0 with w_r = WR.  0: the runtime-width routines.
template <int MODE, class T, int W = 0, int WR = 0, bool FS = false>
__global__ void __launch_bounds__(TP_WARPS * 32, F3_TPB_MINB) k_f3_tpb(const __grid_constant__ F3Args a) {
  static_assert(!FS || (MODE == 1 && sizeof(T) == 4), "float storage: FP32 cFas, MODE 1");
  extern __shared__ __align__(16) double tsm[];
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  double* A = tsm + wp * 32 * TP_RS;  // t_l (MODE 0) / y_k -> ý -> dec ú_l + ý -> the new ú_l (MODE 1)
  uint32_t* wt = (uint32_t*)(tsm + TP_WARPS * 32 * TP_RS) + wp * 32 * TP_WS;
  const Geom g = a.g;
  const long long bpp = (long long)g.NY * (g.NX >> 5);
  const long long bfirst = (long long)a.zlo * bpp, nblk = (long long)(a.zhi - a.zlo) * bpp;
  const long long ntile = (nblk + 31) / 32;
  const long long wg = (long long)blockIdx.x * TP_WARPS + wp, nw = (long long)gridDim.x * TP_WARPS;
  const double* X = MODE == 1 ? a.Dv : a.T;
  const int wi = MODE >= 1 ? a.wu : 0, wo = MODE >= 1 ? a.wu_out : a.wr;
  uint32_t* mant = MODE >= 1 ? a.umant : a.rmant;
  int8_t* exps = MODE >= 1 ? a.uexp : a.rexp;
  const int stride = MODE >= 1 ? a.ustride : a.rstride;
  const unsigned mi = (unsigned)((0x100000000ULL + wi - 1) / (wi > 0 ? wi : 1));  // t / w for t < 2^16
  const unsigned mo = (unsigned)((0x100000000ULL + wo - 1) / wo);
  const double* __restrict__ Zr = a.Z;  // (read-only here)
  const double* __restrict__ Pr = a.PU;
  double* __restrict__ Wr = a.W;
  double* __restrict__ Ur = a.U;
  pdl_wait();
  pdl_trigger();
  bool bad = false;
  for (long long t = wg; t < ntile; t += nw) {
    const long long b0 = bfirst + t * 32;
    const int nb = (int)(nblk - t * 32 < 32 ? nblk - t * 32 : 32);
    if (MODE == 2) {  // ý from mantissas + exponents (k_f3_cheb FIN = 2), compile-time widths
      for (int o = lane; o < nb * wi; o += 32) {
        const int j = (int)__umulhi((unsigned)o, mi);
        cpa4(wt + j * TP_WS + (o - j * wi), mant + (b0 + j) * stride + (o - j * wi));
      }
      asm volatile("cp.async.commit_group;\n" ::: "memory");
      const int Eu = lane < nb ? (int)exps[b0 + lane] : -128;
      const int Ey = lane < nb ? (int)a.ey[b0 + lane] : -128;
      asm volatile("cp.async.wait_all;\n" ::: "memory");
      __syncwarp();
      if (lane < nb) {
        const int En = tpb_correct_m<(W > 0 ? W : 1), (WR > 0 ? WR : 1)>(a.my + (b0 + lane) * 32, Ey,
                                                                            wt + lane * TP_WS, Eu, wt + lane * TP_WS, bad);
        exps[b0 + lane] = (int8_t)En;
      }
      __syncwarp();
      for (int o = lane; o < nb * wo; o += 32) {
        const int j = (int)__umulhi((unsigned)o, mo);
        mant[(b0 + j) * stride + (o - j * wo)] = wt[j * TP_WS + (o - j * wo)];
      }
      __syncwarp();
      continue;
    }
    if constexpr (FS) {  // y_k stored as float (exact: it is a float value)
      const float* Xf = (const float*)a.Dv;
#pragma unroll 8
      for (int r = 0; r < 32; ++r) A[r * TP_RS + lane] = r < nb ? (double)__ldg(Xf + (b0 + r) * 32 + lane) : 0.0;
    } else {
#pragma unroll 8
      for (int r = 0; r < 32; ++r) cpa8(A + r * TP_RS + lane, X + (b0 + r) * 32 + lane, r < nb);
    }
    if (MODE == 1)
      for (int o = lane; o < nb * wi; o += 32) {
        const int j = (int)__umulhi((unsigned)o, mi);
        cpa4(wt + j * TP_WS + (o - j * wi), mant + (b0 + j) * stride + (o - j * wi));
      }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    const int Eu = MODE == 1 && lane < nb ? (int)exps[b0 + lane] : -128;
    const long long p0 = b0 * 32 + lane;
    double pv[MODE == 1 ? 32 : 1];  // P u_{l-1} of the tile, loaded now, used after the codec
    if (MODE == 1) {
#pragma unroll
      for (int r = 0; r < 32; ++r) pv[r] = a.uout && r < nb ? __ldg(Pr + p0 + r * 32) : 0.0;
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncwarp();
    double* row = A + lane * TP_RS;
    if (MODE == 0) {
      const int E = tpb_exponent(row, wo, bad);
      if (WR > 0) tpb_pack_w<(WR > 0 ? WR : 1)>(row, E, wt + lane * TP_WS, nullptr);
      else tpb_pack(row, E, wo, wt + lane * TP_WS, nullptr);
      if (lane < nb) exps[b0 + lane] = (int8_t)E;
    } else if (W > 0) {  // (no w_l; compile-time widths)
      const int En = tpb_correct_w<(W > 0 ? W : 1), (WR > 0 ? WR : 1)>(row, wt + lane * TP_WS, Eu, wt + lane * TP_WS, bad);
      if (lane < nb) exps[b0 + lane] = (int8_t)En;
    } else {
      const int Ey = tpb_exponent(row, a.wr, bad);  // ý = enc_{w_r}(y_k): values only (never stored)
      if (!a.wout) {  // (no w_l: ý, dec ú + ý and the new exponent's max in one pass)
        const unsigned long long mx = tpb_quant_add(row, Ey, a.wr, wt + lane * TP_WS, Eu, wi);
        const int En = tpb_exp_of_max(mx, wo, bad);
        tpb_pack(row, En, wo, wt + lane * TP_WS, row);
        if (lane < nb) exps[b0 + lane] = (int8_t)En;
        goto packed;
      }
      tpb_quant(row, Ey, a.wr);
      __syncwarp();
      if (a.wout) {  // w_l = z_l + dec ý_l (loads 8 rows deep)
#pragma unroll 1
        for (int r0 = 0; r0 < nb; r0 += 8) {
          double zv[8];
#pragma unroll
          for (int k = 0; k < 8; ++k)
            zv[k] = r0 + k < nb ? (FS ? (double)__ldg((const float*)Zr + p0 + (r0 + k) * 32) : __ldg(Zr + p0 + (r0 + k) * 32))
                                : 0.0;
#pragma unroll
          for (int k = 0; k < 8; ++k)
            if (r0 + k < nb) Wr[p0 + (r0 + k) * 32] = (double)((T)zv[k] + (T)A[(r0 + k) * TP_RS + lane]);
        }
        __syncwarp();
      }
      tpb_unpack_add(wt + lane * TP_WS, Eu, wi, row);  // dec ú_l + ý
      const int En = tpb_exponent(row, wo, bad);
      tpb_pack(row, En, wo, wt + lane * TP_WS, row);  // ú_l <- enc(dec ú_l + ý); row = its value
      if (lane < nb) exps[b0 + lane] = (int8_t)En;
    }
  packed:
    __syncwarp();
    for (int o = lane; o < nb * wo; o += 32) {
      const int j = (int)__umulhi((unsigned)o, mo);
      mant[(b0 + j) * stride + (o - j * wo)] = wt[j * TP_WS + (o - j * wo)];
    }
    if (MODE == 1 && a.uout) {  // u_l = dec ú_l + P u_{l-1}
#pragma unroll
      for (int r = 0; r < 32; ++r)
        if (r < nb) Ur[p0 + r * 32] = A[r * TP_RS + lane] + pv[r];
    }
    __syncwarp();
  }
  if (__any_sync(FULL, bad) && lane == 0) atomicOr(a.status, 1);
}

// ------------------------------------------------------------------ host --
template <int P>
static int smem_res(int wu) {
  return (int)gen_smem_bytes<P, double>(F3<P>::NW * F3<P>::NR * (3 * wu + 2)) + 16;
}
template <int P, class T>
static int smem_cfas(int wr) {
  return (int)gen_smem_bytes<P, T>(F3<P>::NW * FW * (wr + 1)) + 16;
}
template <int P, class T>
static int smem_cheb(int J, int wu, bool aux) {
  using C = F3<P>;
  const int NA = J >= 3 ? 2 : 1;
  const size_t d = (size_t)C::NBF * NA * C::BOX * 8 + (C::BOX + 2 * C::NR * 32 + (size_t)P * C::BOX) * sizeof(T) +
                   (aux ? (size_t)C::NW * 2 * 32 * FW * 8 : 0);
  const size_t wbytes = (size_t)C::NW * FW * (wu + 1) * 4 + 8;
  return (int)(d + wbytes + 8 + 8 * C::NBF + 16);
}

template <int P>
static int smem_staged2(int wr, int nx);
template <int P>
static int smem_staged(int wr, int nx);
// k_f3_staged (one plane per iteration) or k_f3_staged2 (two; F3Args::s2)
template <int P, int K, class T, int WR, bool FS = false>
static void staged_launch_w(cudaStream_t st, const F3Args& a, const CoefT<T>& ct, int wr, int nx) {
  if constexpr (FS) {  // (float storage; one plane per iteration for cFas step 1 only: the host requires s2 with csc)
    if constexpr (K == 2) {
      if (!a.s2) return f3_launch(k_f3_staged<P, K, T, WR, true>, a.nitems, smem_staged<P>(wr, nx), st, a, ct);
    }
    f3_launch(k_f3_staged2<P, K, T, WR, true>, a.nitems, smem_staged2<P>(wr, nx), st, a, ct);
  } else {
    if (a.s2) f3_launch(k_f3_staged2<P, K, T, WR>, a.nitems, smem_staged2<P>(wr, nx), st, a, ct);
    else f3_launch(k_f3_staged<P, K, T, WR>, a.nitems, smem_staged<P>(wr, nx), st, a, ct);
  }
}
// (K = 2: compile-time r_L widths 4, 5, 6 -- b_r = 4, k_r = 1 at the top
// three levels of every bench schedule; FMG_WR0=1 forces the runtime width)
template <int P, int K, class T = double>
static void staged_launch(cudaStream_t st, const F3Args& a, const CoefT<T>& ct, int wr, int nx) {
  if constexpr (sizeof(T) == 4 && K >= 2) {
    if (a.f32s) {  // FP32 cFas with float storage
      if constexpr (K == 2) {
        if (wr == 4) return staged_launch_w<P, K, T, 4, true>(st, a, ct, wr, nx);
        if (wr == 5) return staged_launch_w<P, K, T, 5, true>(st, a, ct, wr, nx);
        if (wr == 6) return staged_launch_w<P, K, T, 6, true>(st, a, ct, wr, nx);
      }
      return staged_launch_w<P, K, T, 0, true>(st, a, ct, wr, nx);
    }
  }
  if constexpr (K == 2) {
    const bool rt = getenv("FMG_WR0") && atoi(getenv("FMG_WR0")) != 0;  // (read at graph build)
    if (!rt && wr == 4) return staged_launch_w<P, K, T, 4>(st, a, ct, wr, nx);
    if (!rt && wr == 5) return staged_launch_w<P, K, T, 5>(st, a, ct, wr, nx);
    if (!rt && wr == 6) return staged_launch_w<P, K, T, 6>(st, a, ct, wr, nx);
  }
  staged_launch_w<P, K, T, 0>(st, a, ct, wr, nx);
}
template <int P>
static int smem_staged2(int wr, int nx) {
  using C = F3<P>;
  const size_t wb = wr > 0 ? (size_t)F3S2<P>::NW * FW * (wr + 1) * 4 + 8 : 0;
  const size_t xb = (size_t)F3S2<P>::NW * nx * 32 * FW * 8;
  return (int)(((size_t)F3S2<P>::NBF * C::BOX + 4 * C::NR * 32) * 8 + xb + wb + 8 * F3S2<P>::NBF + 16);
}
template <int P>
static int smem_staged(int wr, int nx) {  // (wr > 0: the r_L word ring of K = 2; nx: point arrays of K >= 3)
  using C = F3<P>;
  const size_t wb = wr > 0 ? (size_t)C::NW * FW * (wr + 1) * 4 + 8 : 0;
  const size_t xb = (size_t)C::NW * nx * 32 * FW * 8;
  return (int)(((size_t)C::NBF * C::BOX + 2 * C::NR * 32) * 8 + xb + wb + 8 * C::NBF + 16);
}
template <int P>
static int smem_prolong2(int wu, int na) {
  using C = F3<P>;
  const size_t d = ((size_t)C::NCB * C::CBS + C::CBY * 32 + (size_t)C::NCY * 2 * FW * 32) * na;
  return (int)(d * 8 + (size_t)C::NW * 2 * FW * (wu + 1) * 4 + 8 + 8 + 8 * C::NCB * na + 16);
}
template <int P>
static int smem_prolong(int wu, int na = 1);
// k_f3_prolong2 (32 x 16 tiles, p = 1, 3) or k_f3_prolong (32 x 8)
template <int P, int NA, class TW = double>
static void prolong_launch(cudaStream_t st, const F3Args& a, const CoefT<double>& ct) {
  if constexpr (P == 1 || P == 3) {
    if (a.pr2) {
      F3Args b = a;
      const int nch = a.nitems / (a.nxb * a.nyb);
      b.nyb = (a.g.NY + 2 * FW - 1) / (2 * FW);
      b.nitems = a.nxb * b.nyb * nch;
      f3_launch(k_f3_prolong2<P, NA, TW>, b.nitems, smem_prolong2<P>(a.wu, NA), st, b, ct);
      return;
    }
  }
  f3_launch(k_f3_prolong<P, NA, TW>, a.nitems, smem_prolong<P>(a.wu, NA), st, a, ct);
}
template <int P>
static int smem_prolong(int wu, int na) {
  using C = F3<P>;
  const size_t d = ((size_t)C::NCB * C::CBS + C::CBY * 32 + (size_t)C::NCY * FW * 32) * na;
  return (int)(d * 8 + (size_t)C::NW * FW * (wu + 1) * 4 + 8 + 8 + 8 * C::NCB * na + 16);
}

int fine3_box_dims(int p, int* cbx, int* cby, int* rs, int* nr) {
  switch (p) {
    case 1: *cbx = F3<1>::CBX; *cby = F3<1>::CBY; *rs = F3<1>::RS; *nr = F3<1>::NR; return 0;
    case 2: *cbx = F3<2>::CBX; *cby = F3<2>::CBY; *rs = F3<2>::RS; *nr = F3<2>::NR; return 0;
    case 3: *cbx = F3<3>::CBX; *cby = F3<3>::CBY; *rs = F3<3>::RS; *nr = F3<3>::NR; return 0;
    default: return -1;
  }
}

void fine3_set_attributes() {
  const int big = 200 * 1024;
#define FS2(P, K, W) \
  cudaFuncSetAttribute(k_f3_staged2<P, K, float, W, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, big); \
  if (K == 2) cudaFuncSetAttribute(k_f3_staged<P, 2, float, W, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, big); \
  if (K == 3 && W == 0) {                                                                              \
    cudaFuncSetAttribute(k_f3_cheb<P, 2, float, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, big); \
    cudaFuncSetAttribute(k_f3_cheb<P, 3, float, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, big); \
    cudaFuncSetAttribute(k_f3_cheb<P, 2, float, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, big); \
    cudaFuncSetAttribute(k_f3_cheb<P, 3, float, 0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, big); \
  }
#define W2(P, W)                                                                                           \
  cudaFuncSetAttribute(k_f3_staged<P, 2, double, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);  \
  cudaFuncSetAttribute(k_f3_staged2<P, 2, double, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, big); \
  cudaFuncSetAttribute(k_f3_staged<P, 2, float, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);   \
  cudaFuncSetAttribute(k_f3_staged2<P, 2, float, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
#define F(P)                                                                                        \
  cudaFuncSetAttribute(k_f3_residual<P, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);  \
  cudaFuncSetAttribute(k_f3_residual<P, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, big); \
  cudaFuncSetAttribute(k_f3_prolong<P, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);      \
  cudaFuncSetAttribute(k_f3_prolong<P, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);      \
  cudaFuncSetAttribute(k_f3_prolong2<P, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);     \
  cudaFuncSetAttribute(k_f3_prolong2<P, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);     \
  cudaFuncSetAttribute(k_f3_staged<P, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, big); \
  cudaFuncSetAttribute(k_f3_staged2<P, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, big); \
  cudaFuncSetAttribute(k_f3_staged2<P, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, big); \
  cudaFuncSetAttribute(k_f3_staged2<P, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, big); \
  cudaFuncSetAttribute(k_f3_staged2<P, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, big); \
  cudaFuncSetAttribute(k_f3_staged2<P, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, big); \
  cudaFuncSetAttribute(k_f3_staged<P, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, big); \
  cudaFuncSetAttribute(k_f3_staged<P, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, big); \
  cudaFuncSetAttribute(k_f3_staged<P, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, big); \
  cudaFuncSetAttribute(k_f3_staged<P, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, big); \
  cudaFuncSetAttribute(k_f3_cfas<P, double>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);    \
  cudaFuncSetAttribute(k_f3_cheb<P, 2, double, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, big); \
  cudaFuncSetAttribute(k_f3_cheb<P, 3, double, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, big); \
  cudaFuncSetAttribute(k_f3_cheb<P, 2, double, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, big); \
  cudaFuncSetAttribute(k_f3_cheb<P, 2, double, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, big); \
  cudaFuncSetAttribute(k_f3_cheb<P, 3, double, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, big); \
  cudaFuncSetAttribute(k_f3_cheb<P, 3, double, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, big); \
  cudaFuncSetAttribute(k_f3_cfas<P, float>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);     \
  cudaFuncSetAttribute(k_f3_cheb<P, 2, float, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, big); \
  cudaFuncSetAttribute(k_f3_cheb<P, 3, float, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, big); \
  cudaFuncSetAttribute(k_f3_cheb<P, 2, float, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, big); \
  cudaFuncSetAttribute(k_f3_cheb<P, 3, float, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, big); \
  cudaFuncSetAttribute(k_f3_prolong<P, 2, float>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);  \
  cudaFuncSetAttribute(k_f3_prolong2<P, 2, float>, cudaFuncAttributeMaxDynamicSharedMemorySize, big); \
  cudaFuncSetAttribute(k_f3_staged<P, 2, float>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);   \
  cudaFuncSetAttribute(k_f3_staged<P, 3, float>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);   \
  cudaFuncSetAttribute(k_f3_staged<P, 4, float>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);   \
  cudaFuncSetAttribute(k_f3_staged2<P, 2, float>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);  \
  W2(P, 4) W2(P, 5) W2(P, 6)                                                                          \
  FS2(P, 2, 0) FS2(P, 2, 4) FS2(P, 2, 5) FS2(P, 2, 6) FS2(P, 3, 0) FS2(P, 4, 0)                        \
  cudaFuncSetAttribute(k_f3_staged2<P, 3, float>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);  \
  cudaFuncSetAttribute(k_f3_staged2<P, 4, float>, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
  F(1) F(2) F(3)
#undef F
#undef W2
#undef FS2
#define TW(T_, W_, R_) \
  cudaFuncSetAttribute(k_f3_tpb<1, T_, W_, R_>, cudaFuncAttributeMaxDynamicSharedMemorySize, tpb_smem_bytes());
#define TWS(T_) TW(T_, 4, 4) TW(T_, 6, 4) TW(T_, 6, 5) TW(T_, 8, 5) TW(T_, 8, 6) TW(T_, 10, 5) TW(T_, 14, 6) TW(T_, 5, 4) TW(T_, 8, 4)
  TWS(double) TWS(float)
#undef TWS
#undef TW
#define TW(W_, R_) \
  cudaFuncSetAttribute(k_f3_tpb<1, float, W_, R_, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, tpb_smem_bytes());
  TW(4, 4) TW(6, 4) TW(6, 5) TW(8, 5) TW(8, 6) TW(10, 5) TW(14, 6) TW(5, 4) TW(8, 4) TW(0, 0)
#undef TW
  cudaFuncSetAttribute(k_f3_tpb<0, double, 0, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, tpb_smem_bytes());
#define TW(W_, R_) \
  cudaFuncSetAttribute(k_f3_tpb<2, double, W_, R_>, cudaFuncAttributeMaxDynamicSharedMemorySize, tpb_smem_bytes());
  TW(4, 4) TW(6, 4) TW(6, 5) TW(8, 5) TW(8, 6) TW(10, 5) TW(14, 6) TW(5, 4) TW(8, 4)
#undef TW
  cudaFuncSetAttribute(k_f3_tpb<0, double>, cudaFuncAttributeMaxDynamicSharedMemorySize, tpb_smem_bytes());
  cudaFuncSetAttribute(k_f3_tpb<1, double>, cudaFuncAttributeMaxDynamicSharedMemorySize, tpb_smem_bytes());
  cudaFuncSetAttribute(k_f3_tpb<1, float>, cudaFuncAttributeMaxDynamicSharedMemorySize, tpb_smem_bytes());
}

template <class T>
static CoefT<T> coefs_as(const Coefs& c) {  // (FP32: the FP64 constants rounded to float, reading R28)
  CoefT<T> t{};
  for (int i = 0; i < 3; ++i)
    for (int o = 0; o < 7; ++o) {
      t.Kc[i][o] = (T)c.Kc[i][o];
      t.Mc[i][o] = (T)c.Mc[i][o];
    }
  for (int r = 0; r < 6; ++r)
    for (int k = 0; k < 4; ++k) t.Pw[r][k] = (T)c.Pw[r][k];
  for (int i = 0; i < 27; ++i) t.invd[i] = (T)c.invd[i];
  t.inv_theta = (T)c.inv_theta;
  for (int j = 0; j < 8; ++j) {
    t.cal[j] = (T)c.cal[j];
    t.cbe[j] = (T)c.cbe[j];
  }
  t.rhs_c = c.rhs_c;
  return t;
}

static int g_f3_launches = 0;  // kernels issued by launch_fine3 since the last fine3_take_launches()
int fine3_take_launches() {
  const int n = g_f3_launches;
  g_f3_launches = 0;
  return n;
}
template <typename K, class CF>
static void f3_launch(K kernel, int nctas, int smem, cudaStream_t st, const F3Args& a, const CF& cf) {
  ++g_f3_launches;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(nctas);
  cfg.blockDim = dim3(32, FW);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, a, cf);
}

// thread-per-block epilogue over the rank's planes (PDL-chained like the march kernels)
template <int MODE, class T, int W = 0, int WR = 0, bool FS = false>
static void tpb_launch_w(cudaStream_t st, const F3Args& a);
// compile-time widths for the common cases (the top levels of the bench
// schedules), the runtime-width kernel otherwise
template <int MODE, class T, bool FS>
static void tpb_launch_fs(cudaStream_t st, const F3Args& a) {
  if constexpr (MODE == 0) {
    if (a.wr == 4) return tpb_launch_w<MODE, T, 0, 4>(st, a);
  } else if (MODE == 2 || (!a.wout && a.wu == a.wu_out)) {
#define TW(W_, R_) \
  if (a.wu == W_ && a.wr == R_) return tpb_launch_w<MODE, T, W_, R_, FS>(st, a);
    TW(4, 4) TW(6, 4) TW(6, 5) TW(8, 5) TW(8, 6) TW(10, 5) TW(14, 6) TW(5, 4) TW(8, 4)
#undef TW
  }
  if constexpr (MODE != 2) tpb_launch_w<MODE, T, 0, 0, FS>(st, a);  // (MODE 2 only for the listed widths: fine3_tpby_width)
}
template <int MODE, class T>
static void tpb_launch(cudaStream_t st, const F3Args& a) {
  if constexpr (MODE == 1 && sizeof(T) == 4) {
    if (a.f32s) return tpb_launch_fs<MODE, T, true>(st, a);  // (y_k, z_l stored as float)
  }
  tpb_launch_fs<MODE, T, false>(st, a);
}
template <int MODE, class T, int W, int WR, bool FS>
static void tpb_launch_w(cudaStream_t st, const F3Args& a) {
  const long long bpp = (long long)a.g.NY * (a.g.NX >> 5), nblk = (long long)(a.zhi - a.zlo) * bpp;
  const long long want = (nblk + 32 * TP_WARPS - 1) / (32 * TP_WARPS);
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int grid = (int)std::max(1LL, std::min(want, (long long)sms * 4));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(TP_WARPS * 32);
  cfg.dynamicSmemBytes = tpb_smem_bytes();
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  ++g_f3_launches;
  cudaLaunchKernelEx(&cfg, k_f3_tpb<MODE, T, W, WR, FS>, a);
}

template <int P, class T>
static void launch_cfas_cheb(int kind, cudaStream_t st, const F3Args& a, const CoefT<T>& ct) {
  const int n = a.nitems;
  const bool aux = a.last && (a.wout || a.uout);
  if (kind == 1) {
    f3_launch(k_f3_cfas<P, T>, n, smem_cfas<P, T>(a.wr), st, a, ct);
  } else if (a.last && a.tpby && sizeof(T) == 8) {  // lean top level: ý mantissas, then k_f3_tpb<2>
    if (a.step == 2) f3_launch(k_f3_cheb<P, 2, T, 2>, n, smem_cheb<P, T>(2, a.wu, false), st, a, ct);
    else f3_launch(k_f3_cheb<P, 3, T, 2>, n, smem_cheb<P, T>(3, a.wu, false), st, a, ct);
    tpb_launch<2, T>(st, a);
  } else if (a.last && a.tpb) {  // y_k -> Y, then the thread-per-block finalisation
    F3Args b = a;
    b.Dv = a.Yb;
    if (sizeof(T) == 4 && a.f32s) {  // (FP32 cFas, float storage)
      if (a.step == 2) f3_launch(k_f3_cheb<P, 2, T, 1, (sizeof(T) == 4)>, n, smem_cheb<P, T>(2, a.wu, false), st, b, ct);
      else f3_launch(k_f3_cheb<P, 3, T, 1, (sizeof(T) == 4)>, n, smem_cheb<P, T>(3, a.wu, false), st, b, ct);
    } else if (a.step == 2) {
      f3_launch(k_f3_cheb<P, 2, T, 1>, n, smem_cheb<P, T>(2, a.wu, false), st, b, ct);
    } else {
      f3_launch(k_f3_cheb<P, 3, T, 1>, n, smem_cheb<P, T>(3, a.wu, false), st, b, ct);
    }
    tpb_launch<1, T>(st, b);
  } else if (sizeof(T) == 4 && a.f32s && !a.last) {  // a step below the last (d_2 as float)
    if (a.step == 2) f3_launch(k_f3_cheb<P, 2, T, 0, (sizeof(T) == 4)>, n, smem_cheb<P, T>(2, a.wu, false), st, a, ct);
    else f3_launch(k_f3_cheb<P, 3, T, 0, (sizeof(T) == 4)>, n, smem_cheb<P, T>(3, a.wu, false), st, a, ct);
  } else if (a.step == 2) {
    f3_launch(k_f3_cheb<P, 2, T, 0>, n, smem_cheb<P, T>(2, a.wu, aux), st, a, ct);
  } else {
    f3_launch(k_f3_cheb<P, 3, T, 0>, n, smem_cheb<P, T>(3, a.wu, aux), st, a, ct);
  }
}

// widths k_f3_tpb<2> is compiled for (w_u = w_u', w_r <= 8: the int8 ý mantissas)
bool fine3_tpby_width(int wu, int wr) {
  return (wu == 4 && wr == 4) || (wu == 6 && wr == 4) || (wu == 6 && wr == 5) || (wu == 8 && wr == 5) ||
         (wu == 8 && wr == 6) || (wu == 10 && wr == 5) || (wu == 14 && wr == 6) || (wu == 5 && wr == 4) ||
         (wu == 8 && wr == 4);
}

// kind: 0 residual (u generated), 1 cfas (step 1), 2 Chebyshev step a.step (2 or 3), 3 prolongation,
// 4 residual (u staged);
// `fp32`: FP32 cFas (kinds 1, 2; reading R28)
void launch_fine3(int p, int kind, cudaStream_t st, const F3Args& a, const Coefs& cf, int fp32) {
  if (kind == 2 && a.cfs == 3) {  // staged Chebyshev step j from y_{j-1} (top level, materialised)
    F3Args b = a;
    const bool j2 = a.step == 2;
    b.tmb = j2 ? a.tmx1 : a.tmy;     // y_1 in X1 / y_2 in Y
    b.yout = j2 ? a.Yb : a.X1b;      // y_2 -> Y, y_3 -> X1
    auto run = [&](auto ct) {  // (CoefT<double>, or CoefT<float> for FP32 cFas: reading R28)
      using T = std::remove_reference_t<decltype(ct.inv_theta)>;
#define ST(PP)                                                                                              \
  if (j2) staged_launch<PP, 3, T>(st, b, ct, 0, 1);                      \
  else staged_launch<PP, 4, T>(st, b, ct, 0, 2);
      if (p == 1) {
        ST(1)
      } else if (p == 2) {
        ST(2)
      } else {
        ST(3)
      }
#undef ST
      if (a.last) {  // the thread-per-block finalisation from y_k
        F3Args t = a;
        t.Dv = b.yout;
        tpb_launch<1, T>(st, t);
      }
    };
    if (fp32) run(coefs_as<float>(cf));
    else run(coefs_as<double>(cf));
    return;
  }
  if (kind == 5 || (kind == 1 && a.cfs == 6)) {  // lean form in z chunks: u_L / z_L
    // materialised chunk by chunk in a.chk (a.chkrc planes + the 2P halo), then the staged kernel on it
    const CoefT<double> ct = coefs_as<double>(cf);
    const int n = a.g.n, P_ = p, rc = a.chkrc;
    const long long plane = (long long)a.g.NY * a.g.NX;
    const int tiles = a.nxb * a.nyb;
    int ci = 0;
    for (int za = a.zlo; za < a.zhi; za += rc, ++ci) {
      const int zb = std::min(a.zhi, za + rc), lo = std::max(0, za - P_), hi = std::min(n, zb + P_);
      F3Args g_ = a;  // generation: u_L = dec ú_L + P u_{L-1} (kind 5) / z_L = P w_{L-1} (cFas) over [lo, hi)
      g_.step = kind == 5 ? 1 : 0;
      g_.zlo = lo;
      g_.zhi = hi;
      g_.RC = hi - lo;
      g_.nitems = tiles;
      g_.U = a.chk - plane * lo;
      g_.PU = a.chk - plane * lo;
      F3Args s_ = a;  // the staged sweep over [za, zb)
      s_.zlo = za;
      s_.zhi = zb;
      s_.RC = zb - za;
      s_.nitems = tiles;
      s_.tmb = a.tmch;
      s_.zoff = lo;
      s_.ctaoff = ci * tiles;
      s_.yout = nullptr;
#define CH(PP)                                                                                   \
  prolong_launch<PP, 1>(st, g_, ct);                    \
  if (kind == 5) {                                                                               \
    if (a.tpb) staged_launch<PP, 1>(st, s_, ct, 0, 0);                                           \
    else staged_launch<PP, 0>(st, s_, ct, 0, 0);                                                 \
  } else {                                                                                       \
    staged_launch<PP, 2>(st, s_, ct, a.wr, 0);                                                   \
  }
      // (the planes past the level, up to zb + P, read as zero: the map's extent
      // is the buffer's, so clear them where the chunk ends at the level's end)
      if (zb + P_ > hi)
        cudaMemsetAsync(a.chk + (long long)(hi - lo) * plane, 0, sizeof(double) * plane * (zb + P_ - hi), st);
      if (p == 1) {
        CH(1)
      } else if (p == 2) {
        CH(2)
      } else {
        CH(3)
      }
#undef CH
    }
    if (kind == 5 && a.tpb) tpb_launch<0, double>(st, a);
    return;
  }
  if (kind == 4) {  // residual with u_L staged (materialised form)
    const CoefT<double> ct = coefs_as<double>(cf);
    if (a.tpb) {  // r_L encoded afterwards, thread per block
      if (p == 1) staged_launch<1, 1>(st, a, ct, 0, 0);
      else if (p == 2) staged_launch<2, 1>(st, a, ct, 0, 0);
      else staged_launch<3, 1>(st, a, ct, 0, 0);
      tpb_launch<0, double>(st, a);
      return;
    }
    if (p == 1) staged_launch<1, 0>(st, a, ct, 0, 0);
    else if (p == 2) staged_launch<2, 0>(st, a, ct, 0, 0);
    else staged_launch<3, 0>(st, a, ct, 0, 0);
    return;
  }
  if (kind == 3) {  // P u_{l-1} (step 0) or u_l = dec ú_l + P u_{l-1} (step 1) at the tile points
    const CoefT<double> ct = coefs_as<double>(cf);
    if (p == 1) prolong_launch<1, 1>(st, a, ct);
    else if (p == 2) prolong_launch<2, 1>(st, a, ct);
    else prolong_launch<3, 1>(st, a, ct);
    return;
  }
  if (kind == 0) {
    const CoefT<double> ct = coefs_as<double>(cf);
    if (a.tpb) {  // (lean form: r_L encoded afterwards from t_L, thread per block)
      if (p == 1) f3_launch(k_f3_residual<1, false>, a.nitems, smem_res<1>(a.wu), st, a, ct);
      else if (p == 2) f3_launch(k_f3_residual<2, false>, a.nitems, smem_res<2>(a.wu), st, a, ct);
      else f3_launch(k_f3_residual<3, false>, a.nitems, smem_res<3>(a.wu), st, a, ct);
      tpb_launch<0, double>(st, a);
      return;
    }
    if (p == 1) f3_launch(k_f3_residual<1, true>, a.nitems, smem_res<1>(a.wu), st, a, ct);
    else if (p == 2) f3_launch(k_f3_residual<2, true>, a.nitems, smem_res<2>(a.wu), st, a, ct);
    else f3_launch(k_f3_residual<3, true>, a.nitems, smem_res<3>(a.wu), st, a, ct);
    return;
  }
  if (kind == 1 && a.cfs && (!fp32 || a.cfs != 1)) {  // materialised: z_l = P w_{l-1} -> Y / Z, then b_l from staged z_l
    // (a.cfs == 2 / 5: P u_{l-1} -> PU in the same prolongation launch; FP32
    // cFas: P w_{l-1} and b_l, y_1 in float, reading R28)
    const CoefT<double> ct = coefs_as<double>(cf);
    const CoefT<float> ctf = coefs_as<float>(cf);
    F3Args b = a;
    b.step = 0;
    const bool below = a.cfs == 5;  // (z_l in the Z scratch: the last step's w_l = z_l + ý needs it)
    b.tmb = below ? a.tmz : a.tmy;
    const int na = a.cfs == 1 ? 1 : 2;
    b.yout = a.csc ? a.X1b : nullptr;  // y_1 for the staged Chebyshev steps
    if (na == 2) {
      b.tmc2 = a.tmc;     // w_{l-1} -> Y / Z
      b.out2 = below ? a.Z : a.Yb;
      b.tmc = a.tmcu;     // u_{l-1} -> PU
    } else {
      b.PU = a.Yb;
    }
#define PRO(PP)                                                                                          \
  if (fp32) {                                                                                            \
    prolong_launch<PP, 2, float>(st, b, ct);                                                             \
    staged_launch<PP, 2, float>(st, b, ctf, a.wr, 0);                                                    \
  } else {                                                                                               \
    if (na == 2) prolong_launch<PP, 2>(st, b, ct);                                                       \
    else prolong_launch<PP, 1>(st, b, ct);                                                               \
    staged_launch<PP, 2>(st, b, ct, a.wr, 0);                                                            \
  }
    if (p == 1) {
      PRO(1)
    } else if (p == 2) {
      PRO(2)
    } else {
      PRO(3)
    }
#undef PRO
    return;
  }
  if (fp32) {
    const CoefT<float> ct = coefs_as<float>(cf);
    if (p == 1) launch_cfas_cheb<1>(kind, st, a, ct);
    else if (p == 2) launch_cfas_cheb<2>(kind, st, a, ct);
    else launch_cfas_cheb<3>(kind, st, a, ct);
  } else {
    const CoefT<double> ct = coefs_as<double>(cf);
    if (p == 1) launch_cfas_cheb<1>(kind, st, a, ct);
    else if (p == 2) launch_cfas_cheb<2>(kind, st, a, ct);
    else launch_cfas_cheb<3>(kind, st, a, ct);
  }
}

}  // namespace fmg
