// fmg_march.cu -- 2D grid-level kernels of the compact-FMG hot path as
// row-marching warps.
//
// A warp owns one 32-entry block column (= one BFP block per row) and marches
// down a chunk of rows.  Input rows (the block plus its x halo) are staged in a
// per-warp shared ring by cp.async PF rows ahead; the x pass of the
// tensor-product operator reads the staged row, the y pass runs on a register
// ring of the last 2p+1 x-pass results, and the epilogue (residual, Chebyshev
// update, BFP encode / decode, correction) works on whole 32-entry rows with
// warp collectives.  Warps are independent (no __syncthreads): a CTA is just
// 8 warps of work items (block column, row chunk).
//
// Every expression follows the canonical evaluation order of DESIGN.md §3
// with explicit fma() (-fmad=false): results are bit-identical to the tile
// ops, the cluster kernel and the oracle.
//
// Paper: residual t_L = f_L - A_L u_L and r_L = enc(t_L) (Alg 3.2),
// restriction t_l = R t_{l+1}, r_l = enc(t_l), decode sweep
// u_l = dec ú_l + P u_{l-1}, cFas level step z_l = P w_{l-1},
// smoothing, ý encode, correction (Alg 3.1, Alg 3.3).
#include "fmg_device.cuh"

namespace fmg {

#ifndef FMG_MARCH_MINB
#define FMG_MARCH_MINB 3     // CTAs per SM the register budget is sized for
#endif
constexpr int MW = 8;        // warps per CTA
constexpr int MFW = MFUSED_WARPS;  // warps of the fused small-level kernel (k_m_fused)
constexpr int MNB = 8;       // staged rows per warp (ring; >= MPF + p + 1, >= 2p + 1)
constexpr int MPF = 4;       // rows staged ahead
constexpr int MSLOT = 80;    // doubles per staged row (>= 64 + 4p - 2 + 1)
constexpr int MGT = 72;      // residual: g_l(y') staged at row offset MGT (clear of the row box)

__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

struct MItem {
  int x0, ys, ye, item;
};
// work item `item`: (block column, row chunk)
__device__ __forceinline__ void m_item_at(const MArgs& a, int item, MItem& it) {
  const int xb = item % a.nxb, ch = item / a.nxb;
  it.x0 = xb * 32;
  it.ys = ch * a.RC;
  it.ye = min(a.NYo, it.ys + a.RC);
  it.item = item;
}
// work item of this warp in a one-op launch, or false if none
__device__ __forceinline__ bool m_item(const MArgs& a, MItem& it) {
  const int item = blockIdx.x * MW + threadIdx.y;
  if (item >= a.nitems) return false;
  m_item_at(a, item, it);
  return true;
}

// Stage row y of `src` (geometry g) into `dst`: dst[H + j] = src(x0 + j, y),
// dst[j] = src(x0 - H + j, y) and dst[H + 32 + j] = src(x0 + 32 + j, y) for
// j < H; zero outside the stored level.  cp.async (zero-filled when out of range).
__device__ __forceinline__ void stage_row(const double* __restrict__ src, const Geom& g, int x0, int y, int H,
                                          double* dst, int lane) {
  const bool rowok = y >= 0 && y < g.NY;
  const double* rp = src + (long long)(rowok ? y : 0) * g.NX;
  const int x = x0 + lane;
  const bool ok = rowok && x < g.NX;
  cpa8(dst + H + lane, ok ? rp + x : src, ok);
  if (lane < 2 * H) {
    const int xh = lane < H ? x0 - H + lane : x0 + 32 + (lane - H);
    const bool okh = rowok && xh >= 0 && xh < g.NX;
    cpa8(dst + (lane < H ? lane : 32 + lane), okh ? rp + xh : src, okh);
  }
}

// TMA variant of stage_row: one box of 32 + 2H doubles from (x0 - H, y), zero
// outside the level (the map's out-of-bounds fill); lane 0 issues it on the
// slot's barrier.
// The box starts at x0 - He, He = H rounded up to even (a TMA box must start
// on a 16-byte boundary), so the consumers read the slot shifted by H & 1.
__device__ __forceinline__ void stage_row_tma(const CUtensorMap* tm, int x0, int y, int H, double* slot,
                                              unsigned long long* bar, int lane) {
  if (lane == 0) {
    // (no proxy fence: the slot's previous generic reads were consumed MNB - MPF
    // rows ago behind __syncwarp; in-place writers fence themselves)
    const int He = H + (H & 1);
    tma_load_2d(slot, tm, x0 - He, y, bar, (unsigned)(32 + 2 * He) * 8u);
  }
}
// The warp's MNB staging barriers (after the rings in dynamic shared memory),
// initialised; nullptr when the launch does not stage through TMA.
__device__ __forceinline__ unsigned long long* m_bars(const MArgs& a, double* msm) {
  if (!a.tma) return nullptr;
  unsigned long long* b = (unsigned long long*)(msm + MW * MNB * MSLOT) + threadIdx.y * MNB;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < MNB; ++k) mbar_init(b + k, 1);
    mbar_init_fence();
  }
  __syncwarp();
  return b;
}

// P_l c at fine (x, y) from the coarse array (x, y passes); 0 at fine
// non-unknowns.  Direct (L1-cached) loads.
template <int P>
__device__ __forceinline__ double prolong_at(const Coefs& cf, const double* __restrict__ cA, const Geom& gc, int nf,
                                             int x, int y) {
  if (!unk1(x, nf) || !unk1(y, nf)) return 0.0;
  const int rx = x % (2 * P), bx = P * (x / (2 * P));
  const int ry = y % (2 * P), by = P * (y / (2 * P));
  double v[P + 1][P + 1];
#pragma unroll
  for (int t2 = 0; t2 <= P; ++t2)
#pragma unroll
    for (int t1 = 0; t1 <= P; ++t1) {
      const int cx = bx + t1, cy = by + t2;
      v[t2][t1] = (cx < gc.NX && cy < gc.NY) ? cA[(long long)cy * gc.NX + cx] : 0.0;
    }
  double accy = 0.0;
#pragma unroll
  for (int t2 = 0; t2 <= P; ++t2) {
    double accx = 0.0;
#pragma unroll
    for (int t1 = 0; t1 <= P; ++t1) accx = fma(cf.Pw[rx][t1], v[t2][t1], accx);
    accy = fma(cf.Pw[ry][t2], accx, accy);
  }
  return accy;
}

// warp_decode with the block's words already in registers (lane j holds word j
// and, for w > 32, word j + 32 in w1)
__device__ __forceinline__ double warp_decode_r(uint32_t my0, int E, int w, int lane, uint32_t my1 = 0u) {
  const int o = lane * w, j0 = o >> 5, s = o & 31;
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

__device__ __forceinline__ double invd2(const Coefs& cf, int P, int n, int x, int y) {
  return (unk1(x, n) && unk1(y, n)) ? cf.invd[(y % P) * P + x % P] : 0.0;
}

// Sum-factorised prolongation march (cFas1): P_l c at fine (X, y) is
//   accy = sum_t2 fma(Pw[ry][t2], accx(X, by + t2), accy),
//   accx(X, cy) = sum_t1 fma(Pw[rx][t1], c(bx + t1, cy), accx)
// (prolong_at's order exactly, so the values are bit-identical).  accx of a
// coarse row is computed once, for every fine column the warp needs, into a
// ring of P + 1 rows in shared memory; each fine row is then a (P + 1)-term
// y pass.  The coarse row segment is loaded once (one coalesced load per
// lane) and read through shuffles.
template <int P>
struct ProlongRing {
  static constexpr int NCR = 4;          // ring slots (>= P + 1 coarse rows by .. by + P live at once)
  static constexpr int XW = 32 + 2 * P;  // staged fine columns x0 - P .. x0 + 32 + P - 1
  static constexpr int SLOT = XW + 32;   // w x-pass (XW) then u x-pass (own columns)
  double* ring;                          // NCR * SLOT doubles (per warp)
  int next;                              // next coarse row to x-pass
  // accx of coarse row cy at fine column X (0 when X is not an unknown column)
  __device__ __forceinline__ static double xpass_at(const Coefs& cf, double cv, int cb0, int X, int nf) {
    const bool unk = unk1(X, nf);
    const int Xc = unk ? X : 1;
    const int rx = Xc % (2 * P), bx = P * (Xc / (2 * P));
    double acc = 0.0;
#pragma unroll
    for (int t1 = 0; t1 <= P; ++t1) {
      const double v = __shfl_sync(FULL, cv, (bx + t1 - cb0) & 31);
      acc = fma(cf.Pw[rx][t1], v, acc);
    }
    return unk ? acc : 0.0;
  }
  // x passes of coarse rows next .. need of W (staged columns), then of U
  // (own columns): each pass issues all its rows' loads before the first
  // shuffle (one exposed latency per pass, not per row)
  __device__ __forceinline__ void advance(const Coefs& cf, const double* __restrict__ W, const double* __restrict__ U,
                                          const Geom& gc, int nf, int x0, int need, int lane) {
    const int cb0 = P * ((x0 >= P ? x0 - P : 0) / (2 * P));  // first coarse column any unknown column needs
    const int cx = cb0 + lane;
    const int Xh = lane < P ? x0 - P + lane : x0 + 32 + (lane - P);
    const int jh = lane < P ? lane : 32 + lane;
#pragma unroll
    for (int pass = 0; pass < 2; ++pass) {  // w rows (staged columns), then u rows (own columns)
      const double* __restrict__ src = pass == 0 ? W : U;
      double cv[P + 1];
#pragma unroll
      for (int k = 0; k <= P; ++k) {
        const int cy = next + k;
        const bool ok = cy <= need && cy < gc.NY && cx < gc.NX;
        cv[k] = ok ? src[(long long)cy * gc.NX + cx] : 0.0;
      }
#pragma unroll
      for (int k = 0; k <= P; ++k) {
        const int cy = next + k;
        if (cy > need) break;  // (warp-uniform)
        double* r = ring + (cy & (NCR - 1)) * SLOT;
        if (pass == 0) {
          r[P + lane] = xpass_at(cf, cv[k], cb0, x0 + lane, nf);  // own column
          const double hv = xpass_at(cf, cv[k], cb0, Xh, nf);     // halo columns (lanes < 2P)
          if (lane < 2 * P) r[jh] = hv;
        } else {
          r[XW + lane] = xpass_at(cf, cv[k], cb0, x0 + lane, nf);
        }
      }
    }
    next = need + 1;
  }
  // y pass at fine row y for slot index j (0 .. XW-1), or the own column of U
  __device__ __forceinline__ double ypass(const Coefs& cf, int y, int j, int off) const {
    const int ry = y % (2 * P), by = P * (y / (2 * P));
    double acc = 0.0;
#pragma unroll
    for (int t2 = 0; t2 <= P; ++t2) acc = fma(cf.Pw[ry][t2], ring[((by + t2) & (NCR - 1)) * SLOT + off + j], acc);
    return acc;
  }
};

// The A march: input rows y' = ys-P .. ye+P-1 are staged
// (stage(y', slot), async or not), optionally transformed in place
// (xform(y', slot)), x-passed (a = Mx u, b = Kx u) into the register ring;
// out(y, Au, slot_of_row_y) runs for every output row y in [ys, ye).
template <int P, class Stage, class Xform, class Pre, class Out>
__device__ __forceinline__ void march_A(const Coefs& cf, int ys, int ye, int x, double* ring, Stage stage, Xform xform,
                                        Pre pre, Out out, unsigned long long* bars = nullptr) {
  constexpr int R = 2 * P + 1;
  const int lane = threadIdx.x;
  const int tx = x % P;
  double km[R], kk[R], ra[R], rb[R];
#pragma unroll
  for (int o = 0; o < R; ++o) {
    km[o] = cf.Mc[tx][o];
    kk[o] = cf.Kc[tx][o];
    ra[o] = 0.0;
    rb[o] = 0.0;
  }
  const int nin = (ye - ys) + 2 * P, y0 = ys - P;
  const int SH = bars ? (P & 1) : 0;  // TMA slots start one column early for odd P
  using AuxT = decltype(pre(0));
  if (ye - ys == 1) {
    // single output row: all 2P+1 input rows in flight at once, independent x passes
#pragma unroll
    for (int i = 0; i < R; ++i) stage(y0 + i, ring + i * MSLOT);
    cp_commit();
    const AuxT a1 = pre(ys);
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    if (bars) {
#pragma unroll
      for (int i = 0; i < R; ++i) mbar_wait(bars + i, 0);
    }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < R; ++i) xform(y0 + i, ring + i * MSLOT + SH);
#pragma unroll
    for (int i = 0; i < R; ++i) {
      const double* row = ring + i * MSLOT + SH;
      double s = 0.0, t = 0.0;
#pragma unroll
      for (int o = 0; o < R; ++o) {
        const double v = row[lane + o];
        s = fma(km[o], v, s);
        t = fma(kk[o], v, t);
      }
      ra[i] = s;
      rb[i] = t;
    }
    const int ty = ys % P;
    double d = 0.0, e = 0.0;
#pragma unroll
    for (int o = 0; o < R; ++o) {
      d = fma(cf.Kc[ty][o], ra[o], d);
      e = fma(cf.Mc[ty][o], rb[o], e);
    }
    out(ys, d + e, ring + P * MSLOT + SH, a1);
    __syncwarp();
    return;
  }
  AuxT cur{}, nxt{};
#pragma unroll
  for (int i = 0; i < MPF; ++i) {
    if (i < nin) stage(y0 + i, ring + (i % MNB) * MSLOT);
    cp_commit();
  }
  for (int i = 0; i < nin; ++i) {
    if (i + MPF < nin) stage(y0 + i + MPF, ring + ((i + MPF) % MNB) * MSLOT);
    cp_commit();
    // register prefetch of the per-row operands of the next output row
    if (i >= 2 * P - 1 && i + 1 < nin) nxt = pre(y0 + i + 1 - P);
    cp_wait<MPF>();
    if (bars) mbar_wait(bars + i % MNB, (unsigned)(i / MNB) & 1u);
    __syncwarp();
    double* row = ring + (i % MNB) * MSLOT + SH;
    xform(y0 + i, row);
    double s = 0.0, t = 0.0;
#pragma unroll
    for (int o = 0; o < R; ++o) {
      const double v = row[lane + o];
      s = fma(km[o], v, s);
      t = fma(kk[o], v, t);
    }
#pragma unroll
    for (int o = 0; o < R - 1; ++o) {
      ra[o] = ra[o + 1];
      rb[o] = rb[o + 1];
    }
    ra[R - 1] = s;
    rb[R - 1] = t;
    if (i >= 2 * P) {
      const int y = y0 + i - P;
      const int ty = y % P;
      double d = 0.0, e = 0.0;
#pragma unroll
      for (int o = 0; o < R; ++o) {
        d = fma(cf.Kc[ty][o], ra[o], d);
        e = fma(cf.Mc[ty][o], rb[o], e);
      }
      out(y, d + e, ring + ((i - P) % MNB) * MSLOT + SH, cur);
    }
    cur = nxt;
    __syncwarp();
  }
}

struct NoAux {};
struct RAux {  // r_l block words / exponent
  uint32_t w0, w1;
  int e;
};
struct CAux {  // Chebyshev operands of one output row
  double b, dv, z, pu;
  uint32_t w0, w1;
  int e;
};

// ------------------------------------------------------------ kernels --
// u_l = dec ú_l + P_l u_{l-1} (decode sweep S2)
template <int P>
__device__ __forceinline__ void m_decode_item(const MArgs& a, const Coefs& cf, const MItem& it, double* msm) {
  const MPtrs& c = a.p;
  const LevelDev& lv = a.lv;
  const LevelDev& lp = a.lo;
  const int lane = threadIdx.x, x = it.x0 + lane, nxb = lv.g.NX >> 5;
  for (int y = it.ys; y < it.ye; ++y) {
    const long long blk = (long long)y * nxb + (it.x0 >> 5);
    const double pu = a.l > 0 ? prolong_at<P>(cf, lp.U, lp.g, lv.g.n, x, y) : 0.0;
    const double dv = warp_decode(lv.umant + blk * lv.ustride, lv.uexp[blk], a.wu_in, lane);
    lv.U[(long long)y * lv.g.NX + x] = dv + pu;
  }
}
template <int P>
__global__ void __launch_bounds__(32 * MW, FMG_MARCH_MINB) k_m_decode(const DevCtx* __restrict__ cp, const __grid_constant__ MArgs a,
    const __grid_constant__ Coefs cf) {
  extern __shared__ __align__(128) double msm[];
  pdl_wait();
  pdl_trigger();
  MItem it;
  if (!m_item(a, it)) return;
  m_decode_item<P>(a, cf, it, msm);
}

// t_L = f_L - A_L u_L, r_L = enc(t_L), ||t_L||^2 partial
template <int P, bool TMA>
__device__ __forceinline__ void m_residual_item(const MArgs& a, const Coefs& cf, const MItem& it, double* msm) {
  const MPtrs& c = a.p;
  const LevelDev& lv = a.lv;
  const Geom g = lv.g;
  const int lane = threadIdx.x, x = it.x0 + lane, nxb = g.NX >> 5;
  double* ring = msm + threadIdx.y * (MNB * MSLOT);
  const double* __restrict__ U = lv.U;
  const double* __restrict__ gt = lv.gtab;
  const double gx = unk1(x, g.n) ? cf.rhs_c * gt[x] : 0.0;
  double ss = 0.0;
  unsigned long long* bars = TMA ? m_bars(a, msm) : nullptr;  // (compile-time path)
  march_A<P>(
      cf, it.ys, it.ye, x, ring,
      [&](int yy, double* slot) {
        if (bars) stage_row_tma(a.tm, it.x0, yy, P, slot, bars + (slot - ring) / MSLOT, lane);
        else stage_row(U, g, it.x0, yy, P, slot, lane);
        if (lane == 0) {
          const bool ok = yy >= 0 && yy < g.n;
          cpa8(slot + (TMA ? (P & 1) + MGT : 32 + 2 * P), ok ? gt + yy : gt, ok);  // g_l(y') for the RHS
        }
      },
      [&](int, double*) {}, [&](int) { return NoAux{}; },
      [&](int y, double au, const double* slot, const NoAux&) {
        const bool unk = unk1(x, g.n) && unk1(y, g.n);
        const double f = gx * slot[TMA ? MGT : 32 + 2 * P];  // ((C g(x)) g(y))
        const double t = unk ? f - au : 0.0;
        lv.T[(long long)y * g.NX + x] = t;
        ss = fma(t, t, ss);
        const long long blk = (long long)y * nxb + (it.x0 >> 5);
        warp_encode(t, a.wr, lv.rmant + blk * lv.rstride, lv.rexp + blk, lane, c.status);
      },
      bars);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(FULL, ss, o);
  if (lane == 0 && a.poff >= 0) c.pbase[a.poff + it.item] = ss;
}
template <int P, bool TMA>
__global__ void __launch_bounds__(32 * MW, FMG_MARCH_MINB) k_m_residual(const DevCtx* __restrict__ cp, const __grid_constant__ MArgs a,
    const __grid_constant__ Coefs cf) {
  extern __shared__ __align__(128) double msm[];
  pdl_wait();
  pdl_trigger();
  MItem it;
  if (!m_item(a, it)) return;
  m_residual_item<P, TMA>(a, cf, it, msm);
}

// t_l = R_{l+1} t_{l+1} (restricts t, not r: PAPER.md:742-744), r_l = enc(t_l).
// The warp owns 32 coarse columns; every coarse row consumes two fine rows.
template <int P, bool TMA>
__device__ __forceinline__ void m_restrict_item(const MArgs& a, const Coefs& cf, const MItem& it, double* msm) {
  constexpr int NS = 4 * P - 1, H = 2 * P - 1;
  const MPtrs& c = a.p;
  const LevelDev& lc_ = a.lv;
  const LevelDev& lf = a.lo;
  const Geom gc = lc_.g, gf = lf.g;
  const int lane = threadIdx.x, xc = it.x0 + lane, nxb = gc.NX >> 5;
  const int txc = xc % P;
  const int fxs = 2 * it.x0 - H;  // first staged fine column
  double* ring = msm + threadIdx.y * (MNB * MSLOT);
  const double* __restrict__ Tf = lf.T;
  double rw[NS], rv[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    rw[s] = cf.Rw[txc][s];
    rv[s] = 0.0;
  }
  // fine row f staged as columns fxs .. fxs + 64 + 2H - 1
  unsigned long long* bars = TMA ? m_bars(a, msm) : nullptr;  // (compile-time path)
  auto stage = [&](int fy, double* slot) {
    if (bars) {
      if (lane == 0) {
        tma_load_2d(slot, a.tm, fxs - 1, fy, bars + (slot - ring) / MSLOT, (unsigned)(64 + 2 * H + 2) * 8u);
      }
      return;
    }
    const bool rowok = fy >= 0 && fy < gf.NY;
    const double* rp = Tf + (long long)(rowok ? fy : 0) * gf.NX;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const int j = lane + 32 * k;
      if (j < 64 + 2 * H) {
        const int fx = fxs + j;
        const bool ok = rowok && fx >= 0 && fx < gf.NX;
        cpa8(slot + j, ok ? rp + fx : Tf, ok);
      }
    }
  };
  const int fy0 = 2 * it.ys - H, nin = 2 * (it.ye - it.ys) + 2 * H;
  double ss = 0.0;
#pragma unroll
  for (int i = 0; i < MPF; ++i) {
    if (i < nin) stage(fy0 + i, ring + (i % MNB) * MSLOT);
    cp_commit();
  }
  for (int i = 0; i < nin; ++i) {
    if (i + MPF < nin) stage(fy0 + i + MPF, ring + ((i + MPF) % MNB) * MSLOT);
    cp_commit();
    cp_wait<MPF>();
    if (bars) mbar_wait(bars + i % MNB, (unsigned)(i / MNB) & 1u);
    __syncwarp();
    const double* row = ring + (i % MNB) * MSLOT + (bars ? 1 : 0);  // (TMA box starts at fxs - 1: H is odd)
    double v = 0.0;
#pragma unroll
    for (int s = 0; s < NS; ++s) v = fma(rw[s], row[2 * lane + s], v);  // (t = +0 at fine non-unknowns)
#pragma unroll
    for (int s = 0; s < NS - 1; ++s) rv[s] = rv[s + 1];
    rv[NS - 1] = v;
    if (i >= NS - 1 && ((i - (NS - 1)) & 1) == 0) {
      const int yc = it.ys + (i - (NS - 1)) / 2;
      const int tyc = yc % P;
      double t = 0.0;
#pragma unroll
      for (int s = 0; s < NS; ++s) t = fma(cf.Rw[tyc][s], rv[s], t);
      t = (unk1(xc, gc.n) && unk1(yc, gc.n)) ? t : 0.0;
      lc_.T[(long long)yc * gc.NX + xc] = t;
      ss = fma(t, t, ss);
      const long long blk = (long long)yc * nxb + (it.x0 >> 5);
      if (!a.smode) warp_encode(t, a.wr, lc_.rmant + blk * lc_.rstride, lc_.rexp + blk, lane, c.status);
    }
    __syncwarp();
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(FULL, ss, o);
  if (lane == 0 && a.poff >= 0) c.pbase[a.poff + it.item] = ss;
}
template <int P, bool TMA>
__global__ void __launch_bounds__(32 * MW, FMG_MARCH_MINB) k_m_restrict(const DevCtx* __restrict__ cp, const __grid_constant__ MArgs a,
    const __grid_constant__ Coefs cf) {
  extern __shared__ __align__(128) double msm[];
  pdl_wait();
  pdl_trigger();
  MItem it;
  if (!m_item(a, it)) return;
  m_restrict_item<P, TMA>(a, cf, it, msm);
}

// ý_l = enc(y); w_l = z_l + dec ý_l (l < L); ú_l = enc(dec ú_l + dec ý_l);
// u_l = dec ú_l + P u_{l-1}
__device__ __forceinline__ void m_finalize(const MPtrs& c, const MArgs& a, const LevelDev& lv, long long idx,
                                           long long blk, double y, double zc, double pu, int lane) {
  const double yq = warp_encode(y, a.wr, nullptr, nullptr, lane, c.status);
  if (a.l < a.L) lv.W[idx] = zc + yq;
  uint32_t* uw = lv.umant + blk * lv.ustride;
  const double uo = warp_decode(uw, lv.uexp[blk], a.wu_in, lane);
  const double uq = warp_encode(uo + yq, a.wu_out, uw, lv.uexp + blk, lane, c.status);
  lv.U[idx] = uq + pu;
}

// m_finalize with the ú words / exponent and z, P u prefetched into registers
__device__ __forceinline__ void m_finalize_r(const MPtrs& c, const MArgs& a, const LevelDev& lv, long long idx,
                                             long long blk, double y, double zc, double pu, uint32_t w0, uint32_t w1,
                                             int e, int lane) {
  const double yq = warp_encode(y, a.wr, nullptr, nullptr, lane, c.status);
  if (a.l < a.L) lv.W[idx] = zc + yq;
  const double uo = warp_decode_r(w0, e, a.wu_in, lane, w1);
  const double uq = warp_encode(uo + yq, a.wu_out, lv.umant + blk * lv.ustride, lv.uexp + blk, lane, c.status);
  lv.U[idx] = uq + pu;
}

// Chebyshev step 1 with the prolongation fused:
// z_l = P w_{l-1} computed on the staged rows, b = dec r_l - A z_l;
// stores Z (l < L), PU = P u_{l-1}, B; k == 1 finalises directly.
template <int P, bool NU = false>
__device__ __forceinline__ void m_cfas1_item(const MArgs& a, const Coefs& cf, const MItem& it, double* msm) {
  const MPtrs& c = a.p;
  const LevelDev& lv = a.lv;
  const LevelDev& lp = a.lo;
  const Geom g = lv.g, gp = lp.g;
  const int lane = threadIdx.x, x = it.x0 + lane, nxb = g.NX >> 5;
  double* ring = msm + threadIdx.y * (MNB * MSLOT);
  const int xh = lane < P ? it.x0 - P + lane : it.x0 + 32 + (lane - P);  // halo column of lanes < 2P
  ProlongRing<P> pr;
  pr.ring = msm + blockDim.y * MNB * MSLOT + threadIdx.y * (ProlongRing<P>::NCR * ProlongRing<P>::SLOT);  // (after every warp's ring)
  pr.next = P * ((it.ys - P > 0 ? it.ys - P : 0) / (2 * P));
  const bool unkx = unk1(x, g.n), unkh = unk1(xh, g.n);
  march_A<P>(
      cf, it.ys, it.ye, x, ring,
      [&](int yy, double* slot) {
        // z row yy on the block columns and the x halo (0 outside the level),
        // P u_{l-1} at the own columns of the output rows
        const bool inrow = yy >= 0 && yy < g.NY;
        double zm = 0.0, zh = 0.0, pu = 0.0, yo = 0.0, yhv = 0.0;
        if (inrow && (!NU || a.l > 0)) {  // (warp-uniform; nu > 1 level 0: z_0 = 0, no coarser u)
          const int need = P * (yy / (2 * P)) + P;  // coarse rows by .. by + P
          if (pr.next <= need) {
            __syncwarp();  // the previous row's y passes are done with the slots about to be refilled
            pr.advance(cf, lp.W, lp.U, gp, g.n, it.x0, need, lane);
            __syncwarp();
          }
          const bool unky = unk1(yy, g.n);
          zm = (unkx && unky) ? pr.ypass(cf, yy, P + lane, 0) : 0.0;
          const int jh = lane < P ? lane : 32 + lane;
          zh = (unkh && unky && lane < 2 * P) ? pr.ypass(cf, yy, jh, 0) : 0.0;
          if (yy >= it.ys && yy < it.ye) pu = (unkx && unky) ? pr.ypass(cf, yy, lane, ProlongRing<P>::XW) : 0.0;
        }
        if constexpr (NU) {
          if (inrow && a.guess) {  // + dec ý of the previous cycle: A (z + ý) (reading R23)
            const long long blk = (long long)yy * nxb + (it.x0 >> 5);
            yo = warp_decode(lv.ymant + blk * lv.ystride, lv.yexp[blk], a.wr, lane);
            if (lane < 2 * P && xh >= 0 && xh < g.NX) {
              const long long hb = (long long)yy * nxb + (xh >> 5);
              yhv = point_decode(lv.ymant + hb * lv.ystride, lv.yexp[hb], a.wr, xh & 31);
            }
          }
        }
        slot[P + lane] = (NU && a.guess) ? zm + yo : zm;
        if (lane < 2 * P) slot[lane < P ? lane : 32 + lane] = (NU && a.guess) ? zh + yhv : zh;
        if (yy >= it.ys && yy < it.ye) {
          const long long idx = (long long)yy * g.NX + x;
          if (a.l < a.L) c.Z[idx] = zm;
          c.PU[idx] = pu;
          if (NU && a.guess) c.YO[idx] = yo;
        }
      },
      [&](int, double*) {},
      [&](int yn) {
        const long long blk = (long long)yn * nxb + (it.x0 >> 5);
        RAux r;
        r.w0 = lane < a.wr ? lv.rmant[blk * lv.rstride + lane] : 0u;
        r.w1 = lane + 32 < a.wr ? lv.rmant[blk * lv.rstride + lane + 32] : 0u;
        r.e = lv.rexp[blk];
        return r;
      },
      [&](int y, double az, const double* slot, const RAux& r) {
        const long long idx = (long long)y * g.NX + x, blk = (long long)y * nxb + (it.x0 >> 5);
        const double rv = warp_decode_r(r.w0, r.e, a.wr, lane, r.w1);
        // nu > 1, cycles >= 2: ((r - s) - A (z + ý)), s_L = 0 (reading R23)
        const double b = (NU && a.guess) ? (rv - (a.l < a.L ? lv.T[idx] : 0.0)) - az : rv - az;
        if (a.gs) {  // multicolour GS from y = 0: colour 0 gets y = 0 + invD (b - 0), others 0
          c.B[idx] = b;
          const bool c0 = x % (P + 1) == 0 && y % (P + 1) == 0;
          c.Y[1][idx] = c0 ? 0.0 + invd2(cf, P, g.n, x, y) * (b - 0.0) : 0.0;
        } else if (a.last) {  // k == 1: y = d_1 = inv_theta (invD b)
          const double d = cf.inv_theta * (invd2(cf, P, g.n, x, y) * b);
          m_finalize(c, a, lv, idx, blk, d, slot[P + lane], c.PU[idx], lane);
        } else {
          c.B[idx] = b;
        }
      });
}

// Multicolour Gauss-Seidel colour `a.step` (>= 1) in place on Y[1]: at the
// nodes of that colour y = y + invD (b - A y) (A on the current iterate; nodes
// of one colour are uncoupled, so in-place is exact); the last colour
// finalises every node of the row (oracle mc_gauss_seidel).
template <int P, bool TMA, bool NU = false>
__device__ __forceinline__ void m_gs_item(const MArgs& a, const Coefs& cf, const MItem& it, double* msm) {
  const MPtrs& c = a.p;
  const LevelDev& lv = a.lv;
  const Geom g = lv.g;
  const int lane = threadIdx.x, x = it.x0 + lane, nxb = g.NX >> 5;
  double* ring = msm + threadIdx.y * (MNB * MSLOT);
  double* __restrict__ Yv = c.Y[1];
  const int cx = a.step % (P + 1), cy = a.step / (P + 1);
  const bool colx = x % (P + 1) == cx;
  unsigned long long* bars = TMA ? m_bars(a, msm) : nullptr;  // (compile-time path)
  march_A<P>(
      cf, it.ys, it.ye, x, ring,
      [&](int yy, double* slot) {
        if (bars) stage_row_tma(a.tm, it.x0, yy, P, slot, bars + (slot - ring) / MSLOT, lane);
        else stage_row(Yv, g, it.x0, yy, P, slot, lane);
      },
      [&](int, double*) {},
      [&](int yn) {
        const long long idx = (long long)yn * g.NX + x, blk = (long long)yn * nxb + (it.x0 >> 5);
        CAux q{};
        q.b = c.B[idx];
        if (a.last) {
          q.z = a.l < a.L ? c.Z[idx] : 0.0;
          q.pu = c.PU[idx];
          q.w0 = lane < a.wu_in ? lv.umant[blk * lv.ustride + lane] : 0u;
          q.w1 = lane + 32 < a.wu_in ? lv.umant[blk * lv.ustride + lane + 32] : 0u;
          q.e = lv.uexp[blk];
        }
        return q;
      },
      [&](int y, double ay, const double* slot, const CAux& p) {
        const long long idx = (long long)y * g.NX + x, blk = (long long)y * nxb + (it.x0 >> 5);
        const bool mine = colx && y % (P + 1) == cy;
        const double yo = slot[P + lane];
        const double yv = mine ? yo + invd2(cf, P, g.n, x, y) * (p.b - ay) : yo;
        if (a.last) {
          if constexpr (NU) {  // nu > 1: ý_l + M_l(...), stored between cycles
            const double yt = a.guess ? c.YO[idx] + yv : yv;
            if (a.store) {
              const double yq = warp_encode(yt, a.wr, lv.ymant + blk * lv.ystride, lv.yexp + blk, lane, c.status);
              if (a.l < a.L) lv.W[idx] = p.z + yq;
            } else {
              m_finalize_r(c, a, lv, idx, blk, yt, p.z, p.pu, p.w0, p.w1, p.e, lane);
            }
          } else {
            m_finalize_r(c, a, lv, idx, blk, yv, p.z, p.pu, p.w0, p.w1, p.e, lane);
          }
        } else if (mine) {
          Yv[idx] = yv;
        }
      },
      bars);
}
template <int P, bool NU>
__global__ void __launch_bounds__(32 * MW, FMG_MARCH_MINB) k_m_cfas1(const DevCtx* __restrict__ cp, const __grid_constant__ MArgs a,
    const __grid_constant__ Coefs cf) {
  extern __shared__ __align__(128) double msm[];
  pdl_wait();
  pdl_trigger();
  MItem it;
  if (!m_item(a, it)) return;
  m_cfas1_item<P, NU>(a, cf, it, msm);
}

// Chebyshev step j >= 2: q = b - A y; d_j = fma(alpha_j, d_{j-1}, beta_j (invD q));
// y_j = y_{j-1} + d_j.  Step 2 stages b and forms
// y_1 = d_1 = inv_theta (invD b) in place; the last step finalises.
template <int P, bool TMA, bool NU = false>
__device__ __forceinline__ void m_cheb_item(const MArgs& a, const Coefs& cf, const MItem& it, double* msm) {
  const MPtrs& c = a.p;
  const LevelDev& lv = a.lv;
  const Geom g = lv.g;
  const int lane = threadIdx.x, x = it.x0 + lane, nxb = g.NX >> 5;
  const int j = a.step;
  double* ring = msm + threadIdx.y * (MNB * MSLOT);
  const double* __restrict__ src = (j == 2) ? c.B : c.Y[(j - 1) & 1];
  const int xh = lane < P ? it.x0 - P + lane : it.x0 + 32 + (lane - P);
  const double al = cf.cal[j - 1], be = cf.cbe[j - 1];
  unsigned long long* bars = TMA ? m_bars(a, msm) : nullptr;  // (compile-time path)
  march_A<P>(
      cf, it.ys, it.ye, x, ring,
      [&](int yy, double* slot) {
        if (bars) stage_row_tma(a.tm, it.x0, yy, P, slot, bars + (slot - ring) / MSLOT, lane);
        else stage_row(src, g, it.x0, yy, P, slot, lane);
      },
      [&](int yy, double* slot) {
        if (j != 2) return;
        // y_1 = inv_theta (invD b) on the lane's own staged entries
        slot[P + lane] = cf.inv_theta * (invd2(cf, P, g.n, x, yy) * slot[P + lane]);
        if (lane < 2 * P) {
          double& v = slot[lane < P ? lane : 32 + lane];
          v = cf.inv_theta * (invd2(cf, P, g.n, xh, yy) * v);
        }
        if (bars) fence_async_smem();  // these generic writes precede a later TMA refill of the slot
        __syncwarp();
      },
      [&](int yn) {
        const long long idx = (long long)yn * g.NX + x, blk = (long long)yn * nxb + (it.x0 >> 5);
        CAux q{};
        q.b = c.B[idx];
        if (j > 2) q.dv = c.Dv[idx];
        if (a.last) {
          q.z = a.l < a.L ? c.Z[idx] : 0.0;
          q.pu = c.PU[idx];
          q.w0 = lane < a.wu_in ? lv.umant[blk * lv.ustride + lane] : 0u;
          q.w1 = lane + 32 < a.wu_in ? lv.umant[blk * lv.ustride + lane + 32] : 0u;
          q.e = lv.uexp[blk];
        }
        return q;
      },
      [&](int y, double ay, const double* slot, const CAux& p) {
        const long long idx = (long long)y * g.NX + x, blk = (long long)y * nxb + (it.x0 >> 5);
        const double q = p.b - ay;
        const double yprev = slot[P + lane];
        const double dprev = (j == 2) ? yprev : p.dv;
        const double d = fma(al, dprev, be * (invd2(cf, P, g.n, x, y) * q));
        const double yv = yprev + d;
        if (a.last) {
          if constexpr (NU) {  // nu > 1: ý_l + M_l(...), stored between cycles
            const double yt = a.guess ? c.YO[idx] + yv : yv;
            if (a.store) {
              const double yq = warp_encode(yt, a.wr, lv.ymant + blk * lv.ystride, lv.yexp + blk, lane, c.status);
              if (a.l < a.L) lv.W[idx] = p.z + yq;
            } else {
              m_finalize_r(c, a, lv, idx, blk, yt, p.z, p.pu, p.w0, p.w1, p.e, lane);
            }
          } else {
            m_finalize_r(c, a, lv, idx, blk, yv, p.z, p.pu, p.w0, p.w1, p.e, lane);
          }
        } else {
          c.Y[j & 1][idx] = yv;
          c.Dv[idx] = d;
        }
      },
      bars);
}
template <int P, bool TMA, bool NU = false>
__global__ void __launch_bounds__(32 * MW, FMG_MARCH_MINB) k_m_cheb(const DevCtx* __restrict__ cp, const __grid_constant__ MArgs a,
    const __grid_constant__ Coefs cf) {
  extern __shared__ __align__(128) double msm[];
  pdl_wait();
  pdl_trigger();
  MItem it;
  if (!m_item(a, it)) return;
  m_cheb_item<P, TMA, NU>(a, cf, it, msm);
}

// Small 2D levels: a run of consecutive restriction / cFas
// step 1 / Chebyshev ops whose levels have at most MFW work items runs as ONE
// launch of one CTA, a warp per item and a CTA barrier between the ops, the
// same item code as the one-op kernels (bit-identical).  Removes the launch
// and grid-drain latency between the dependent small ops of a V-cycle.
template <int P>
__global__ void __launch_bounds__(32 * MFW, 1) k_m_fused(const DevCtx* __restrict__ cp, const __grid_constant__ MFused f,
                                                        const __grid_constant__ Coefs cf) {
  extern __shared__ __align__(128) double msm[];
  pdl_wait();
  pdl_trigger();
  for (int k = 0; k < f.n; ++k) {
    const MArgs& a = f.op[k];
    if ((int)threadIdx.y < a.nitems) {
      MItem it;
      m_item_at(a, threadIdx.y, it);
      if (a.type == OP_RESTRICT) m_restrict_item<P, false>(a, cf, it, msm);
      else if (a.type == OP_CFAS1) m_cfas1_item<P, false>(a, cf, it, msm);
      else m_cheb_item<P, false, false>(a, cf, it, msm);
    }
    __syncthreads();  // the op's outputs (global) are visible to the next op's warps (one CTA, one SM)
  }
}

// s sweep of nu > 1 cycles (Alg 3.1):
// q_l = A_l dec ý_l + s_l into W_l (s_l = 0 on the top level, 0 at fine
// non-unknowns); the restriction then forms s_{l-1} = R_l q_l.
template <int P>
__device__ __forceinline__ void m_sq_item(const MArgs& a, const Coefs& cf, const MItem& it, double* msm) {
  const LevelDev& lv = a.lv;
  const Geom g = lv.g;
  const int lane = threadIdx.x, x = it.x0 + lane, nxb = g.NX >> 5;
  double* ring = msm + threadIdx.y * (MNB * MSLOT);
  const int xh = lane < P ? it.x0 - P + lane : it.x0 + 32 + (lane - P);
  march_A<P>(
      cf, it.ys, it.ye, x, ring,
      [&](int yy, double* slot) {
        double vo = 0.0, vh = 0.0;
        if (yy >= 0 && yy < g.NY) {  // (warp-uniform)
          const long long blk = (long long)yy * nxb + (it.x0 >> 5);
          vo = warp_decode(lv.ymant + blk * lv.ystride, lv.yexp[blk], a.wr, lane);
          if (lane < 2 * P && xh >= 0 && xh < g.NX) {
            const long long hb = (long long)yy * nxb + (xh >> 5);
            vh = point_decode(lv.ymant + hb * lv.ystride, lv.yexp[hb], a.wr, xh & 31);
          }
        }
        slot[P + lane] = vo;
        if (lane < 2 * P) slot[lane < P ? lane : 32 + lane] = vh;
      },
      [&](int, double*) {}, [&](int) { return NoAux{}; },
      [&](int y, double ay, const double*, const NoAux&) {
        const long long idx = (long long)y * g.NX + x;
        const bool unk = unk1(x, g.n) && unk1(y, g.n);
        lv.W[idx] = unk ? ay + (a.smode ? 0.0 : lv.T[idx]) : 0.0;
      });
}
template <int P>
__global__ void __launch_bounds__(32 * MW, FMG_MARCH_MINB) k_m_sq(const DevCtx* __restrict__ cp, const __grid_constant__ MArgs a,
    const __grid_constant__ Coefs cf) {
  extern __shared__ __align__(128) double msm[];
  pdl_wait();
  pdl_trigger();
  MItem it;
  if (!m_item(a, it)) return;
  m_sq_item<P>(a, cf, it, msm);
}

// Level 0 of a nu > 1 cycle (one warp; oracle cfas_cycle): y_0 = A_0^{-1} b_0
// on the (2p-1)^d unknowns (b_0 = the bracket cFas1 stored in B), + dec ý_0 of
// the previous cycle (guess), ý_0 = enc_wr(y_0) stored, w_0 = dec ý_0; after
// the last cycle ú_0 = enc_wu(dec ú_0 + dec ý_0) and u_0 = dec ú_0.
template <int D, int P>
__global__ void __launch_bounds__(128) k_coarse_nu(const DevCtx* __restrict__ cp, const __grid_constant__ MArgs a) {
  pdl_wait();
  pdl_trigger();
  constexpr int m = 2 * P - 1, n0 = D == 3 ? m * m * m : m * m;
  __shared__ double sb[128], sy[128];
  const DevCtx& dc = *cp;
  const MPtrs& c = a.p;
  const LevelDev& lv = a.lv;
  const Geom g = lv.g;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nxb = g.NX >> 5;
  for (int J = tid; J < n0; J += 128) {
    const int jx = J % m + 1, jy = (J / m) % m + 1, jz = D == 3 ? J / (m * m) + 1 : 0;
    sb[J] = c.B[((long long)jz * g.NY + jy) * g.NX + jx];
  }
  __syncthreads();
  // y_0 = A_0^{-1} b_0: one unknown per thread, acc = fma(Ainv[I][J], b_J, acc)
  // over J ascending; the row's loads are independent of the
  // chain, so they are unrolled ahead of it
  for (int I = tid; I < n0; I += 128) {
    const double* Ai = dc.Ainv + (long long)I * n0;
    double s = 0.0;
#pragma unroll 8
    for (int J = 0; J < n0; ++J) s = fma(Ai[J], sb[J], s);
    sy[I] = s;
  }
  __syncthreads();
  // codec rows (warp-cooperative): ý_0, w_0 and the ú_0 correction
  const int nrows = (D == 3 ? g.NZ : 1) * g.NY;
  for (int row = wid; row < nrows; row += 4) {
    const int zr = D == 3 ? row / g.NY : 0, y = row - zr * g.NY, x = lane;
    double s = 0.0;
    if (unk1(x, g.n) && unk1(y, g.n) && (D == 2 || unk1(zr, g.n)))
      s = sy[((D == 3 ? zr - 1 : 0) * m + (y - 1)) * m + (x - 1)];
    const long long blk = (long long)row * nxb;
    if (a.guess) s = warp_decode(lv.ymant + blk * lv.ystride, lv.yexp[blk], a.wr, lane) + s;
    const double yq = warp_encode(s, a.wr, lv.ymant + blk * lv.ystride, lv.yexp + blk, lane, c.status);
    lv.W[(long long)row * g.NX + x] = yq;
    if (!a.store) {
      const double uo = warp_decode(lv.umant + blk * lv.ustride, lv.uexp[blk], a.wu_in, lane);
      const double uq = warp_encode(uo + yq, a.wu_out, lv.umant + blk * lv.ustride, lv.uexp + blk, lane, c.status);
      lv.U[(long long)row * g.NX + x] = uq;
    }
  }
}

template <int P, bool TMA, bool NU = false>
__global__ void __launch_bounds__(32 * MW, FMG_MARCH_MINB) k_m_gs(const DevCtx* __restrict__ cp, const __grid_constant__ MArgs a,
    const __grid_constant__ Coefs cf) {
  extern __shared__ __align__(128) double msm[];
  pdl_wait();
  pdl_trigger();
  MItem it;
  if (!m_item(a, it)) return;
  m_gs_item<P, TMA, NU>(a, cf, it, msm);
}

// ------------------------------------------------------------------ host --
int march_smem(bool tma) { return MW * MNB * MSLOT * 8 + (tma ? MW * MNB * 8 : 0); }
// cFas1: the rings plus the per-warp prolongation ring (ProlongRing)
static int march_smem_cfas1(int p) { return MW * MNB * MSLOT * 8 + MW * 4 * (64 + 2 * p) * 8; }
static int march_smem_fused(int p) { return MFW * MNB * MSLOT * 8 + MFW * 4 * (64 + 2 * p) * 8; }
int march_fused_warps() { return MFW; }
int march_warps() { return MW; }

#define M_DISPATCH(p, F)   \
  do {                     \
    if (p == 1) { F(1); }  \
    else if (p == 2) { F(2); } \
    else { F(3); }         \
  } while (0)

void march_set_attributes() {
#define F(P)                                                                                                   \
  cudaFuncSetAttribute(k_m_residual<P, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, march_smem(false)); \
  cudaFuncSetAttribute(k_m_residual<P, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, march_smem(true));   \
  cudaFuncSetAttribute(k_m_restrict<P, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, march_smem(false)); \
  cudaFuncSetAttribute(k_m_restrict<P, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, march_smem(true));   \
  cudaFuncSetAttribute(k_m_cfas1<P, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, march_smem_cfas1(P)); \
  cudaFuncSetAttribute(k_m_cfas1<P, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, march_smem_cfas1(P));  \
  cudaFuncSetAttribute(k_m_cheb<P, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, march_smem(false)); \
  cudaFuncSetAttribute(k_m_sq<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, march_smem(false));               \
  cudaFuncSetAttribute(k_m_gs<P, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, march_smem(false));   \
  cudaFuncSetAttribute(k_m_cheb<P, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, march_smem(false));     \
  cudaFuncSetAttribute(k_m_cheb<P, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, march_smem(true));       \
  cudaFuncSetAttribute(k_m_gs<P, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, march_smem(false));       \
  cudaFuncSetAttribute(k_m_gs<P, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, march_smem(true));       \
  cudaFuncSetAttribute(k_m_fused<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, march_smem_fused(P));
  F(1) F(2) F(3)
#undef F
}

template <typename K>
static void m_launch(K kernel, int nitems, int smem, cudaStream_t st, const DevCtx* c, const MArgs& a,
                     const Coefs& cf) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((nitems + MW - 1) / MW);
  cfg.blockDim = dim3(32, MW);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, c, a, cf);
}

void launch_march(int p, cudaStream_t st, const void* devctx, const MArgs& a, const Coefs& cf) {
  const DevCtx* c = (const DevCtx*)devctx;
  const bool t = a.tma != 0;
  const bool nu = a.guess || a.store;  // nu > 1 cycle kernels
  const int sm = march_smem(t);
#define TM(K, P) (t ? (void (*)(const DevCtx*, MArgs, Coefs))K<P, true> : (void (*)(const DevCtx*, MArgs, Coefs))K<P, false>)
#define F(P)                                                                                     \
  switch (a.type) {                                                                              \
    case OP_DECODE: m_launch(k_m_decode<P>, a.nitems, 0, st, c, a, cf); break;                   \
    case OP_RESIDUAL: m_launch(TM(k_m_residual, P), a.nitems, sm, st, c, a, cf); break;          \
    case OP_RESTRICT: m_launch(TM(k_m_restrict, P), a.nitems, sm, st, c, a, cf); break;          \
    case OP_CFAS1:                                                                               \
      if (nu) m_launch(k_m_cfas1<P, true>, a.nitems, march_smem_cfas1(P), st, c, a, cf);          \
      else m_launch(k_m_cfas1<P, false>, a.nitems, march_smem_cfas1(P), st, c, a, cf);            \
      break;                                                                                      \
    case OP_SQ: m_launch(k_m_sq<P>, a.nitems, march_smem(false), st, c, a, cf); break;           \
    case OP_GS:                                                                                  \
      if (nu) m_launch(k_m_gs<P, false, true>, a.nitems, march_smem(false), st, c, a, cf);        \
      else m_launch(TM(k_m_gs, P), a.nitems, sm, st, c, a, cf);                                   \
      break;                                                                                      \
    default:                                                                                     \
      if (nu) m_launch(k_m_cheb<P, false, true>, a.nitems, march_smem(false), st, c, a, cf);      \
      else m_launch(TM(k_m_cheb, P), a.nitems, sm, st, c, a, cf);                                 \
      break;                                                                                      \
  }
  M_DISPATCH(p, F);
#undef F
#undef TM
}

void launch_march_fused(int p, cudaStream_t st, const void* devctx, const MFused& f, const Coefs& cf) {
  const DevCtx* c = (const DevCtx*)devctx;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(32, MFW);
  cfg.dynamicSmemBytes = march_smem_fused(p);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (p == 1) cudaLaunchKernelEx(&cfg, k_m_fused<1>, c, f, cf);
  else if (p == 2) cudaLaunchKernelEx(&cfg, k_m_fused<2>, c, f, cf);
  else cudaLaunchKernelEx(&cfg, k_m_fused<3>, c, f, cf);
}

void launch_coarse_nu(int dim, int p, cudaStream_t st, const void* devctx, const MArgs& a) {
  const DevCtx* c = (const DevCtx*)devctx;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(128);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (dim == 2) {
    if (p == 1) cudaLaunchKernelEx(&cfg, k_coarse_nu<2, 1>, c, a);
    else if (p == 2) cudaLaunchKernelEx(&cfg, k_coarse_nu<2, 2>, c, a);
    else cudaLaunchKernelEx(&cfg, k_coarse_nu<2, 3>, c, a);
  } else {
    if (p == 1) cudaLaunchKernelEx(&cfg, k_coarse_nu<3, 1>, c, a);
    else if (p == 2) cudaLaunchKernelEx(&cfg, k_coarse_nu<3, 2>, c, a);
    else cudaLaunchKernelEx(&cfg, k_coarse_nu<3, 3>, c, a);
  }
}

}  // namespace fmg
