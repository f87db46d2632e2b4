// fmg_march3.cu -- 3D grid-level kernels of the compact-FMG hot path as
// plane-marching CTAs.
//
// A CTA (8 warps) owns an in-plane tile of 32 x 8 points -- warp w owns row
// y0 + w, i.e. one 32-entry BFP block per plane -- and marches along z over a
// chunk of planes.  Each input plane (the tile plus its x/y halo) is staged by
// cp.async a few planes ahead into a shared ring; the x pass and the y pass of
// the tensor-product operator go through shared memory, the z pass runs on a
// per-thread register ring of the last 2p+1 planes, so every input plane is
// loaded and x/y-passed once (no z halo recompute), and the epilogue works on
// whole BFP blocks with warp collectives.
//
// Every expression follows the canonical evaluation order of DESIGN.md §3 with
// explicit fma() (-fmad=false): results are bit-identical to the tile ops, the
// cluster kernel and the oracle.
//
// Paper: residual and r_L = enc(t_L) (Alg 3.2), restriction
// t_l = R t_{l+1}, decode sweep u_l = dec ú_l + P u_{l-1}
// (PAPER.md:733-735), cFas level step z_l = P w_{l-1}, smoothing, ý encode and
// correction (Alg 3.1, Alg 3.3).
#include "fmg_device.cuh"

namespace fmg {

#ifndef FMG_MARCH3_MINB
#define FMG_MARCH3_MINB 2    // CTAs per SM the register budget is sized for
#endif
constexpr int TW3 = 8;       // warps per CTA = tile rows
constexpr int PF3 = 3;       // planes staged ahead
constexpr int NB3 = 8;       // staged plane ring (>= PF3 + p + 2)
constexpr int RS3 = 40;      // staged row stride (doubles, >= 32 + 2p)

__device__ __forceinline__ void cp3_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp3_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(PF3) : "memory"); }

struct M3Item {
  int x0, y0, zs, ze, cta;
};
__device__ __forceinline__ void m3_item(const MArgs& a, M3Item& it) {
  const int cta = blockIdx.x;
  const int tiles = a.nxb * a.nyb;
  const int t = cta % tiles, ch = cta / tiles;
  it.x0 = (t % a.nxb) * 32;
  it.y0 = (t / a.nxb) * TW3;
  it.zs = a.zlo + ch * a.RC;  // (z-slab of this rank: planes [zlo, zhi))
  it.ze = min(a.zhi, it.zs + a.RC);
  it.cta = cta;
}

// Stage the (32 + 2H) x (TW3 + 2H) box of plane z (x from x0 - H, y from y0 - H)
// into `slot` (row stride RS3); zero outside the stored level.
__device__ __forceinline__ void stage_box(const double* __restrict__ src, const Geom& g, int x0, int y0, int z, int H,
                                          double* slot) {
  const int lane = threadIdx.x;
  const bool zok = z >= 0 && z < g.NZ;
  for (int r = threadIdx.y; r < TW3 + 2 * H; r += TW3) {
    const int y = y0 - H + r;
    const bool rowok = zok && y >= 0 && y < g.NY;
    const double* rp = src + ((long long)(rowok ? z : 0) * g.NY + (rowok ? y : 0)) * g.NX;
    double* dst = slot + r * RS3;
    const int x = x0 + lane;
    const bool ok = rowok && x < g.NX;
    cpa8(dst + H + lane, ok ? rp + x : src, ok);
    if (lane < 2 * H) {
      const int xh = lane < H ? x0 - H + lane : x0 + 32 + (lane - H);
      const bool okh = rowok && xh >= 0 && xh < g.NX;
      cpa8(dst + (lane < H ? lane : 32 + lane), okh ? rp + xh : src, okh);
    }
  }
}

// TMA variant of stage_box: one 40 x (TW3 + 2H) x 1 box from (x0 - He, y0 - H, z),
// He = H rounded up to even (16-byte box start), row stride RS3 = 40; the
// consumers read the slot shifted by H & 1; out-of-range elements zero-filled
// by the map.  Issued by thread (0, 0) on the slot's barrier.
__device__ __forceinline__ void stage_box_tma(const CUtensorMap* tm, int x0, int y0, int z, int H, double* slot,
                                              unsigned long long* bar) {
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    fence_async_smem();
    tma_load_3d(slot, tm, x0 - H - (H & 1), y0 - H, z, bar, (unsigned)(RS3 * (TW3 + 2 * H)) * 8u);
  }
}
// The CTA's NB3 staging barriers (after XB), initialised; nullptr without TMA.
__device__ __forceinline__ unsigned long long* m3_bars(const MArgs& a, double* after_xb) {
  if (!a.tma) return nullptr;
  unsigned long long* b = (unsigned long long*)after_xb;
  if (threadIdx.x == 0 && threadIdx.y == 0) {
#pragma unroll
    for (int k = 0; k < NB3; ++k) mbar_init(b + k, 1);
    mbar_init_fence();
  }
  __syncthreads();
  return b;
}

__device__ __forceinline__ double invd3(const Coefs& cf, int P, int n, int l, int x, int y, int z) {
  if (!unk1(x, n) || !unk1(y, n) || !unk1(z, n)) return 0.0;
  return cf.invd[((z % P) * P + y % P) * P + x % P] * pow2(l + 1);
}

// The A march: input planes z' = zs-P .. ze+P-1 are staged,
// optionally transformed in place (xform(z', slot), one point per thread of
// each staged row it loaded), x-passed (a = Mx u, b = Kx u) into shared memory,
// y-passed (c = My a, s = Ky a + My b) into the register ring; out(z, Au, slot
// of plane z, aux) runs for every output plane z in [zs, ze).
template <int P, class Stage, class Xform, class Pre, class Out>
__device__ __forceinline__ void march3_A(const Coefs& cf, const M3Item& it, int l, double* ring, double* XA,
                                         double* XB, Stage stage, Xform xform, Pre pre, Out out,
                                         unsigned long long* bars = nullptr) {
  constexpr int R = 2 * P + 1, NR = TW3 + 2 * P;
  const int lane = threadIdx.x, w = threadIdx.y;
  const int x = it.x0 + lane, y = it.y0 + w;
  const int tx = x % P, ty = y % P;
  const double hl = pow2(-(l + 1));
  double km[R], kk[R], cr[R], sr[R];
#pragma unroll
  for (int o = 0; o < R; ++o) {
    km[o] = cf.Mc[tx][o];
    kk[o] = cf.Kc[tx][o];
    cr[o] = 0.0;
    sr[o] = 0.0;
  }
  const int nin = (it.ze - it.zs) + 2 * P, z0 = it.zs - P;
  const int SH = bars ? (P & 1) : 0;  // TMA boxes start one column early for odd P
  using AuxT = decltype(pre(0));
  AuxT cur{}, nxt{};
#pragma unroll
  for (int i = 0; i < PF3; ++i) {
    if (i < nin) stage(z0 + i, ring + (i % NB3) * (NR * RS3));
    cp3_commit();
  }
  for (int i = 0; i < nin; ++i) {
    if (i + PF3 < nin) stage(z0 + i + PF3, ring + ((i + PF3) % NB3) * (NR * RS3));
    cp3_commit();
    if (i >= 2 * P - 1 && i + 1 < nin) nxt = pre(z0 + i + 1 - P);
    cp3_wait();
    if (bars) mbar_wait(bars + i % NB3, (unsigned)(i / NB3) & 1u);
    __syncthreads();
    double* slot = ring + (i % NB3) * (NR * RS3) + SH;
    xform(z0 + i, slot);
    // x pass of the NR staged rows (warp w: rows w, w + 8, ...)
    for (int r = w; r < NR; r += TW3) {
      const double* row = slot + r * RS3;
      double s = 0.0, t = 0.0;
#pragma unroll
      for (int o = 0; o < R; ++o) {
        const double v = row[lane + o];
        s = fma(km[o], v, s);
        t = fma(kk[o], v, t);
      }
      XA[r * 32 + lane] = s;
      XB[r * 32 + lane] = t;
    }
    __syncthreads();
    // y pass at the warp's row
    double c = 0.0, dd = 0.0, e = 0.0;
#pragma unroll
    for (int o = 0; o < R; ++o) {
      const double av = XA[(w + o) * 32 + lane], bv = XB[(w + o) * 32 + lane];
      c = fma(cf.Mc[ty][o], av, c);
      dd = fma(cf.Kc[ty][o], av, dd);
      e = fma(cf.Mc[ty][o], bv, e);
    }
#pragma unroll
    for (int o = 0; o < R - 1; ++o) {
      cr[o] = cr[o + 1];
      sr[o] = sr[o + 1];
    }
    cr[R - 1] = c;
    sr[R - 1] = dd + e;
    if (i >= 2 * P) {
      const int z = z0 + i - P, tz = z % P;
      double acc = 0.0;
#pragma unroll
      for (int o = 0; o < R; ++o) acc = fma(cf.Kc[tz][o], cr[o], acc);
#pragma unroll
      for (int o = 0; o < R; ++o) acc = fma(cf.Mc[tz][o], sr[o], acc);
      out(z, acc * hl, ring + ((i - P) % NB3) * (NR * RS3) + SH, cur);
    }
    cur = nxt;
  }
}

struct NoAux3 {};
struct RAux3 {
  uint32_t w0, w1;
  int e;
  double gz;
};
struct CAux3 {
  double b, dv, z, pu;
  uint32_t w0, w1;
  int e;
};

__device__ __forceinline__ double warp_decode_r3(uint32_t my0, int E, int w, int lane, uint32_t my1) {
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

template <int P>
__device__ __forceinline__ size_t m3_ring_doubles() {
  return (size_t)NB3 * (TW3 + 2 * P) * RS3;
}

// ------------------------------------------------------------ kernels --
// t_L = f_L - A_L u_L, r_L = enc(t_L), ||t_L||^2 partial
template <int P, bool TMA>
__global__ void __launch_bounds__(32 * TW3, FMG_MARCH3_MINB) k_m3_residual(const DevCtx* __restrict__ cp, const __grid_constant__ MArgs a,
                                                            const __grid_constant__ Coefs cf) {
  extern __shared__ __align__(128) double msm[];
  pdl_wait();
  pdl_trigger();
  M3Item it;
  m3_item(a, it);
  const MPtrs& c = a.p;
  const LevelDev& lv = a.lv;
  const Geom g = lv.g;
  const int lane = threadIdx.x, x = it.x0 + lane, y = it.y0 + threadIdx.y;
  const bool rowok = y < g.NY;
  double* ring = msm;
  double* XA = ring + m3_ring_doubles<P>();
  double* XB = XA + (TW3 + 2 * P) * 32;
  unsigned long long* bars = TMA ? m3_bars(a, XB + (TW3 + 2 * P) * 32) : nullptr;  // (compile-time path)
  const double* __restrict__ U = lv.U;
  const double* __restrict__ gt = lv.gtab;
  const double gxy = (unk1(x, g.n) && unk1(y, g.n)) ? (cf.rhs_c * gt[x]) * gt[y] : 0.0;
  const int nxb = g.NX >> 5;
  double ss = 0.0;
  march3_A<P>(
      cf, it, a.l, ring, XA, XB, [&](int zz, double* slot) {
        if (bars) stage_box_tma(a.tm, it.x0, it.y0, zz - a.zoff, P, slot, bars + (slot - ring) / ((TW3 + 2 * P) * RS3));
        else stage_box(U, g, it.x0, it.y0, zz, P, slot);
      },
      [&](int, double*) {},
      [&](int zn) {
        RAux3 r{};
        r.gz = (zn >= 0 && zn < g.n) ? gt[zn] : 0.0;
        return r;
      },
      [&](int z, double au, const double*, const RAux3& ax) {
        if (!rowok) return;
        const bool unk = unk1(x, g.n) && unk1(y, g.n) && unk1(z, g.n);
        const double t = unk ? gxy * ax.gz - au : 0.0;  // (((C g(x)) g(y)) g(z)) - A u
        const long long idx = ((long long)z * g.NY + y) * g.NX + x;
        lv.T[idx] = t;
        ss = fma(t, t, ss);
        const long long blk = ((long long)z * g.NY + y) * nxb + (it.x0 >> 5);
        warp_encode(t, a.wr, lv.rmant + blk * lv.rstride, lv.rexp + blk, lane, c.status);
      },
      bars);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(FULL, ss, o);
  if (lane == 0 && a.poff >= 0) c.pbase[a.poff + (long long)it.cta * TW3 + threadIdx.y] = ss;
}

// Chebyshev step 1: b = dec r_l - A z_l (z_l = P w_{l-1} staged
// by k_m3_prolong); stores B; k == 1 finalises.
__device__ __forceinline__ void m3_finalize(const MPtrs& c, const MArgs& a, const LevelDev& lv, long long idx,
                                            long long blk, double y, double zc, double pu, uint32_t w0, uint32_t w1,
                                            int e, int lane) {
  const double yq = warp_encode(y, a.wr, nullptr, nullptr, lane, c.status);
  if (a.l < a.L) lv.W[idx] = zc + yq;
  const double uo = warp_decode_r3(w0, e, a.wu_in, lane, w1);
  const double uq = warp_encode(uo + yq, a.wu_out, lv.umant + blk * lv.ustride, lv.uexp + blk, lane, c.status);
  lv.U[idx] = uq + pu;
}

template <int P, bool TMA, bool NU = false>
__global__ void __launch_bounds__(32 * TW3, FMG_MARCH3_MINB) k_m3_cfas1(const DevCtx* __restrict__ cp, const __grid_constant__ MArgs a,
                                                         const __grid_constant__ Coefs cf) {
  extern __shared__ __align__(128) double msm[];
  pdl_wait();
  pdl_trigger();
  M3Item it;
  m3_item(a, it);
  const MPtrs& c = a.p;
  const LevelDev& lv = a.lv;
  const Geom g = lv.g;
  const int lane = threadIdx.x, x = it.x0 + lane, y = it.y0 + threadIdx.y;
  const bool rowok = y < g.NY;
  double* ring = msm;
  double* XA = ring + m3_ring_doubles<P>();
  double* XB = XA + (TW3 + 2 * P) * 32;
  unsigned long long* bars = TMA ? m3_bars(a, XB + (TW3 + 2 * P) * 32) : nullptr;  // (compile-time path)
  const int nxb = g.NX >> 5;
  march3_A<P>(
      cf, it, a.l, ring, XA, XB, [&](int zz, double* slot) {
        if (bars) stage_box_tma(a.tm, it.x0, it.y0, zz - a.zoff, P, slot, bars + (slot - ring) / ((TW3 + 2 * P) * RS3));
        else stage_box(c.Z, g, it.x0, it.y0, zz, P, slot);
      },
      [&](int zz, double* slot) {
        if constexpr (NU) {
          if (!a.guess) return;
          // nu > 1: stage z + dec ý of the previous cycle (A (z + ý),
          // reading R23) on this thread's staged rows; keep dec ý of the output
          // points for the last Chebyshev step
          constexpr int NR = TW3 + 2 * P;
          const bool zok = zz >= 0 && zz < g.NZ;
          const int xh = lane < P ? it.x0 - P + lane : it.x0 + 32 + (lane - P);
          for (int r = threadIdx.y; r < NR; r += TW3) {
            const int yy = it.y0 - P + r;
            if (!zok || yy < 0 || yy >= g.NY) continue;  // (warp-uniform)
            const long long rb = ((long long)zz * g.NY + yy) * nxb;
            const double yo = warp_decode(lv.ymant + (rb + (it.x0 >> 5)) * lv.ystride, lv.yexp[rb + (it.x0 >> 5)],
                                          a.wr, lane);
            double* row = slot + r * RS3;
            row[P + lane] = row[P + lane] + yo;
            if (lane < 2 * P && xh >= 0 && xh < g.NX) {
              const long long hb = rb + (xh >> 5);
              double& v = row[lane < P ? lane : 32 + lane];
              v = v + point_decode(lv.ymant + hb * lv.ystride, lv.yexp[hb], a.wr, xh & 31);
            }
            if (zz >= it.zs && zz < it.ze && yy >= it.y0 && yy < it.y0 + TW3)
              c.YO[((long long)zz * g.NY + yy) * g.NX + x] = yo;
          }
          __syncthreads();
        }
      },
      [&](int zn) {
        CAux3 q{};
        if (rowok) {
          const long long blk = ((long long)zn * g.NY + y) * nxb + (it.x0 >> 5);
          q.w0 = lane < a.wr ? lv.rmant[blk * lv.rstride + lane] : 0u;
          q.w1 = lane + 32 < a.wr ? lv.rmant[blk * lv.rstride + lane + 32] : 0u;
          q.e = lv.rexp[blk];
          if (a.last) {
            const long long idx = ((long long)zn * g.NY + y) * g.NX + x;
            q.pu = c.PU[idx];
            const long long ub = blk;
            q.b = 0.0;
            q.dv = 0.0;
            (void)ub;
          }
        }
        return q;
      },
      [&](int z, double az, const double* slot, const CAux3& q) {
        if (!rowok) return;
        const long long idx = ((long long)z * g.NY + y) * g.NX + x;
        const long long blk = ((long long)z * g.NY + y) * nxb + (it.x0 >> 5);
        const double rv = warp_decode_r3(q.w0, q.e, a.wr, lane, q.w1);
        // nu > 1, cycles >= 2: ((r - s) - A (z + ý)), s_L = 0 (reading R23)
        const double b = (NU && a.guess) ? (rv - (a.l < a.L ? lv.T[idx] : 0.0)) - az : rv - az;
        if (a.gs) {  // multicolour GS from y = 0: colour 0 gets y = 0 + invD (b - 0), others 0
          c.B[idx] = b;
          const bool c0 = x % (P + 1) == 0 && y % (P + 1) == 0 && z % (P + 1) == 0;
          c.Y[1][idx] = c0 ? 0.0 + invd3(cf, P, g.n, a.l, x, y, z) * (b - 0.0) : 0.0;
        } else if (a.last) {  // k == 1: y = d_1 = inv_theta (invD b)
          const double d = cf.inv_theta * (invd3(cf, P, g.n, a.l, x, y, z) * b);
          const double zc = slot[(threadIdx.y + P) * RS3 + P + lane];
          uint32_t* uw = lv.umant + blk * lv.ustride;
          const uint32_t u0 = lane < a.wu_in ? uw[lane] : 0u, u1 = lane + 32 < a.wu_in ? uw[lane + 32] : 0u;
          m3_finalize(c, a, lv, idx, blk, d, zc, q.pu, u0, u1, lv.uexp[blk], lane);
        } else {
          c.B[idx] = b;
        }
      },
      bars);
}

// Chebyshev step j >= 2; step 2 stages b and forms
// y_1 = d_1 = inv_theta (invD b) in place; the last step finalises.
template <int P, bool TMA, bool NU = false>
__global__ void __launch_bounds__(32 * TW3, FMG_MARCH3_MINB) k_m3_cheb(const DevCtx* __restrict__ cp, const __grid_constant__ MArgs a,
                                                        const __grid_constant__ Coefs cf) {
  extern __shared__ __align__(128) double msm[];
  pdl_wait();
  pdl_trigger();
  M3Item it;
  m3_item(a, it);
  const MPtrs& c = a.p;
  const LevelDev& lv = a.lv;
  const Geom g = lv.g;
  const int lane = threadIdx.x, w = threadIdx.y, x = it.x0 + lane, y = it.y0 + w;
  const bool rowok = y < g.NY;
  double* ring = msm;
  double* XA = ring + m3_ring_doubles<P>();
  double* XB = XA + (TW3 + 2 * P) * 32;
  unsigned long long* bars = TMA ? m3_bars(a, XB + (TW3 + 2 * P) * 32) : nullptr;  // (compile-time path)
  const int nxb = g.NX >> 5;
  const int j = a.step;
  const double* __restrict__ src = (j == 2) ? c.B : c.Y[(j - 1) & 1];
  const double al = cf.cal[j - 1], be = cf.cbe[j - 1];
  constexpr int NR = TW3 + 2 * P;
  // invd3's factors hoisted (same values: invd[type] 2^(l+1), 0 at non-unknowns):
  // the thread's own / halo column and its staged rows are fixed for the march
  const double isc = pow2(a.l + 1);
  const int xh = lane < P ? it.x0 - P + lane : it.x0 + 32 + (lane - P);
  const bool ux = unk1(x, g.n), uxh = unk1(xh, g.n), uy = unk1(y, g.n);
  const int tx = ux ? x % P : 0, txh = uxh ? xh % P : 0, ty = uy ? y % P : 0;
  bool uyr[2];
  int tyr[2];
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int yy = it.y0 - P + w + k * TW3;
    uyr[k] = w + k * TW3 < NR && unk1(yy, g.n);
    tyr[k] = uyr[k] ? yy % P : 0;
  }
  march3_A<P>(
      cf, it, a.l, ring, XA, XB, [&](int zz, double* slot) {
        if (bars) stage_box_tma(a.tm, it.x0, it.y0, zz - a.zoff, P, slot, bars + (slot - ring) / ((TW3 + 2 * P) * RS3));
        else stage_box(src, g, it.x0, it.y0, zz, P, slot);
      },
      [&](int zz, double* slot) {
        if (j != 2) return;
        // y_1 = inv_theta (invD b) on the entries of this thread's staged rows
        const bool uz = unk1(zz, g.n);
        const int tz = uz ? zz % P : 0;
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int r = w + k * TW3;
          if (r >= NR) break;
          double* row = slot + r * RS3;
          const int tb = (tz * P + tyr[k]) * P;
          const double f = (ux && uyr[k] && uz) ? cf.invd[tb + tx] * isc : 0.0;
          row[P + lane] = cf.inv_theta * (f * row[P + lane]);
          if (lane < 2 * P) {
            const double fh = (uxh && uyr[k] && uz) ? cf.invd[tb + txh] * isc : 0.0;
            double& v = row[lane < P ? lane : 32 + lane];
            v = cf.inv_theta * (fh * v);
          }
        }
        __syncthreads();
      },
      [&](int zn) {
        CAux3 q{};
        if (rowok) {
          const long long idx = ((long long)zn * g.NY + y) * g.NX + x;
          const long long blk = ((long long)zn * g.NY + y) * nxb + (it.x0 >> 5);
          q.b = c.B[idx];
          if (j > 2) q.dv = c.Dv[idx];
          if (a.last) {
            q.z = a.l < a.L ? c.Z[idx] : 0.0;
            q.pu = c.PU[idx];
            q.w0 = lane < a.wu_in ? lv.umant[blk * lv.ustride + lane] : 0u;
            q.w1 = lane + 32 < a.wu_in ? lv.umant[blk * lv.ustride + lane + 32] : 0u;
            q.e = lv.uexp[blk];
          }
        }
        return q;
      },
      [&](int z, double ay, const double* slot, const CAux3& q) {
        if (!rowok) return;
        const long long idx = ((long long)z * g.NY + y) * g.NX + x;
        const long long blk = ((long long)z * g.NY + y) * nxb + (it.x0 >> 5);
        const double qq = q.b - ay;
        const double yprev = slot[(w + P) * RS3 + P + lane];
        const double dprev = (j == 2) ? yprev : q.dv;
        const bool uz = unk1(z, g.n);
        const double f = (ux && uy && uz) ? cf.invd[((uz ? z % P : 0) * P + ty) * P + tx] * isc : 0.0;
        const double d = fma(al, dprev, be * (f * qq));
        const double yv = yprev + d;
        if (a.last) {
          if constexpr (NU) {  // nu > 1: ý_l + M_l(...), stored between cycles
            const double yt = a.guess ? c.YO[idx] + yv : yv;
            if (a.store) {
              const double yqv = warp_encode(yt, a.wr, lv.ymant + blk * lv.ystride, lv.yexp + blk, lane, c.status);
              if (a.l < a.L) lv.W[idx] = q.z + yqv;
            } else {
              m3_finalize(c, a, lv, idx, blk, yt, q.z, q.pu, q.w0, q.w1, q.e, lane);
            }
          } else {
            m3_finalize(c, a, lv, idx, blk, yv, q.z, q.pu, q.w0, q.w1, q.e, lane);
          }
        } else {
          c.Y[j & 1][idx] = yv;
          c.Dv[idx] = d;
        }
      },
      bars);
}

// Multicolour Gauss-Seidel colour `a.step` (>= 1) in place on Y[1]
// (oracle mc_gauss_seidel): y = y + invD (b - A y) at the nodes
// of the colour, the last colour finalises every node.
template <int P, bool TMA, bool NU = false>
__global__ void __launch_bounds__(32 * TW3, FMG_MARCH3_MINB) k_m3_gs(const DevCtx* __restrict__ cp, const __grid_constant__ MArgs a,
                                                      const __grid_constant__ Coefs cf) {
  extern __shared__ __align__(128) double msm[];
  pdl_wait();
  pdl_trigger();
  M3Item it;
  m3_item(a, it);
  const MPtrs& c = a.p;
  const LevelDev& lv = a.lv;
  const Geom g = lv.g;
  const int lane = threadIdx.x, w = threadIdx.y, x = it.x0 + lane, y = it.y0 + w;
  const bool rowok = y < g.NY;
  double* ring = msm;
  double* XA = ring + m3_ring_doubles<P>();
  double* XB = XA + (TW3 + 2 * P) * 32;
  unsigned long long* bars = TMA ? m3_bars(a, XB + (TW3 + 2 * P) * 32) : nullptr;  // (compile-time path)
  const int nxb = g.NX >> 5;
  double* __restrict__ Yv = c.Y[1];
  const int cx = a.step % (P + 1), cy = (a.step / (P + 1)) % (P + 1), cz = a.step / ((P + 1) * (P + 1));
  const bool colxy = x % (P + 1) == cx && y % (P + 1) == cy;
  march3_A<P>(
      cf, it, a.l, ring, XA, XB, [&](int zz, double* slot) {
        if (bars) stage_box_tma(a.tm, it.x0, it.y0, zz - a.zoff, P, slot, bars + (slot - ring) / ((TW3 + 2 * P) * RS3));
        else stage_box(Yv, g, it.x0, it.y0, zz, P, slot);
      },
      [&](int, double*) {},
      [&](int zn) {
        CAux3 q{};
        if (rowok) {
          const long long idx = ((long long)zn * g.NY + y) * g.NX + x;
          const long long blk = ((long long)zn * g.NY + y) * nxb + (it.x0 >> 5);
          q.b = c.B[idx];
          if (a.last) {
            q.z = a.l < a.L ? c.Z[idx] : 0.0;
            q.pu = c.PU[idx];
            q.w0 = lane < a.wu_in ? lv.umant[blk * lv.ustride + lane] : 0u;
            q.w1 = lane + 32 < a.wu_in ? lv.umant[blk * lv.ustride + lane + 32] : 0u;
            q.e = lv.uexp[blk];
          }
        }
        return q;
      },
      [&](int z, double ay, const double* slot, const CAux3& q) {
        if (!rowok) return;
        const long long idx = ((long long)z * g.NY + y) * g.NX + x;
        const long long blk = ((long long)z * g.NY + y) * nxb + (it.x0 >> 5);
        const bool mine = colxy && z % (P + 1) == cz;
        const double yo = slot[(w + P) * RS3 + P + lane];
        const double yv = mine ? yo + invd3(cf, P, g.n, a.l, x, y, z) * (q.b - ay) : yo;
        if (a.last) {
          if constexpr (NU) {  // nu > 1: ý_l + M_l(...), stored between cycles
            const double yt = a.guess ? c.YO[idx] + yv : yv;
            if (a.store) {
              const double yqv = warp_encode(yt, a.wr, lv.ymant + blk * lv.ystride, lv.yexp + blk, lane, c.status);
              if (a.l < a.L) lv.W[idx] = q.z + yqv;
            } else {
              m3_finalize(c, a, lv, idx, blk, yt, q.z, q.pu, q.w0, q.w1, q.e, lane);
            }
          } else {
            m3_finalize(c, a, lv, idx, blk, yv, q.z, q.pu, q.w0, q.w1, q.e, lane);
          }
        } else if (mine) {
          Yv[idx] = yv;
        }
      },
      bars);
}

// Pointwise prolongation march: for each fine (x, y) the x/y
// passes of the coarse planes are kept in a register ring; fine plane z takes
// the z pass over coarse planes P floor(z/2p) .. + p.  mode 0 (decode):
// u_l = dec ú_l + P u_{l-1}; mode 1 (cFas): z_l = P w_{l-1} -> Z, P u_{l-1} -> PU.
template <int P>
__device__ __forceinline__ double pxy(const Coefs& cf, const double* __restrict__ cA, const Geom& gc, int rx, int bx,
                                      int ry, int by, int cz) {
  double v[P + 1][P + 1];
#pragma unroll
  for (int t2 = 0; t2 <= P; ++t2)
#pragma unroll
    for (int t1 = 0; t1 <= P; ++t1) {
      const int cx = bx + t1, cy = by + t2;
      v[t2][t1] = (cx < gc.NX && cy < gc.NY && cz >= 0 && cz < gc.NZ) ? cA[((long long)cz * gc.NY + cy) * gc.NX + cx]
                                                                       : 0.0;
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

template <int P>
__global__ void __launch_bounds__(32 * TW3) k_m3_prolong(const DevCtx* __restrict__ cp, const __grid_constant__ MArgs a,
                                                        const __grid_constant__ Coefs cf) {
  pdl_wait();
  pdl_trigger();
  M3Item it;
  m3_item(a, it);
  const MPtrs& c = a.p;
  const LevelDev& lv = a.lv;
  const LevelDev& lp = a.lo;
  const Geom g = lv.g, gp = lp.g;
  const int lane = threadIdx.x, x = it.x0 + lane, y = it.y0 + threadIdx.y;
  if (y >= g.NY) return;  // (no collectives across warps here)
  const int nxb = g.NX >> 5;
  const bool okxy = a.l > 0 && unk1(x, g.n) && unk1(y, g.n);
  const int rx = okxy ? x % (2 * P) : 0, bx = okxy ? P * (x / (2 * P)) : 0;
  const int ry = okxy ? y % (2 * P) : 0, by = okxy ? P * (y / (2 * P)) : 0;
  // register ring of the coarse planes cz0 .. cz0 + P for the two sources
  double wv[P + 1], uv[P + 1];
  int cz0 = -1000;
  for (int z = it.zs; z < it.ze; ++z) {
    const bool okz = okxy && unk1(z, g.n);
    const int rz = okz ? z % (2 * P) : 0, bz = okz ? P * (z / (2 * P)) : 0;
    if (okz && bz != cz0) {
      // consecutive windows bz .. bz + P share plane bz (= old bz + P): shift
      // it down and compute only the P new planes
      const int t0 = (bz == cz0 + P) ? 1 : 0;
      if (t0) {
        uv[0] = uv[P];
        if (a.type != OP_DECODE && !a.puonly) wv[0] = wv[P];
      }
#pragma unroll
      for (int t = 0; t <= P; ++t) {
        if (t < t0) continue;
        const int cz = bz + t;
        if (a.type == OP_DECODE || a.puonly) {
          uv[t] = pxy<P>(cf, lp.U, gp, rx, bx, ry, by, cz);
        } else {
          wv[t] = pxy<P>(cf, lp.W, gp, rx, bx, ry, by, cz);
          uv[t] = pxy<P>(cf, lp.U, gp, rx, bx, ry, by, cz);
        }
      }
      cz0 = bz;
    }
    double pu = 0.0, pw = 0.0;
    if (okz) {
#pragma unroll
      for (int t = 0; t <= P; ++t) {
        pu = fma(cf.Pw[rz][t], uv[t], pu);
        if (a.type != OP_DECODE && !a.puonly) pw = fma(cf.Pw[rz][t], wv[t], pw);
      }
    }
    const long long idx = ((long long)z * g.NY + y) * g.NX + x;
    if (a.type == OP_DECODE) {
      const long long blk = ((long long)z * g.NY + y) * nxb + (it.x0 >> 5);
      const double dv = warp_decode(lv.umant + blk * lv.ustride, lv.uexp[blk], a.wu_in, lane);
      lv.U[idx] = dv + pu;
    } else {
      if (!a.puonly) c.Z[idx] = pw;
      c.PU[idx] = pu;
    }
  }
}

// s sweep of nu > 1 cycles: q_l = A_l dec ý_l + s_l into W_l
// (s_l = 0 on the top level; 0 at non-unknowns); the staged boxes are the
// decoded ý (own columns by warp decode, halo columns by point decode).
template <int P>
__global__ void __launch_bounds__(32 * TW3, FMG_MARCH3_MINB) k_m3_sq(const DevCtx* __restrict__ cp, const __grid_constant__ MArgs a,
                                                      const __grid_constant__ Coefs cf) {
  extern __shared__ __align__(128) double msm[];
  pdl_wait();
  pdl_trigger();
  M3Item it;
  m3_item(a, it);
  const LevelDev& lv = a.lv;
  const Geom g = lv.g;
  const int lane = threadIdx.x, w = threadIdx.y, x = it.x0 + lane, y = it.y0 + w;
  const bool rowok = y < g.NY;
  double* ring = msm;
  double* XA = ring + m3_ring_doubles<P>();
  double* XB = XA + (TW3 + 2 * P) * 32;
  const int nxb = g.NX >> 5;
  constexpr int NR = TW3 + 2 * P;
  const int xh = lane < P ? it.x0 - P + lane : it.x0 + 32 + (lane - P);
  march3_A<P>(
      cf, it, a.l, ring, XA, XB,
      [&](int zz, double* slot) {
        const bool zok = zz >= 0 && zz < g.NZ;
        for (int r = threadIdx.y; r < NR; r += TW3) {
          const int yy = it.y0 - P + r;
          double vo = 0.0, vh = 0.0;
          if (zok && yy >= 0 && yy < g.NY) {  // (warp-uniform)
            const long long rb = ((long long)zz * g.NY + yy) * nxb;
            vo = warp_decode(lv.ymant + (rb + (it.x0 >> 5)) * lv.ystride, lv.yexp[rb + (it.x0 >> 5)], a.wr, lane);
            if (lane < 2 * P && xh >= 0 && xh < g.NX) {
              const long long hb = rb + (xh >> 5);
              vh = point_decode(lv.ymant + hb * lv.ystride, lv.yexp[hb], a.wr, xh & 31);
            }
          }
          double* row = slot + r * RS3;
          row[P + lane] = vo;
          if (lane < 2 * P) row[lane < P ? lane : 32 + lane] = vh;
        }
      },
      [&](int, double*) {}, [&](int) { return NoAux3{}; },
      [&](int z, double ay, const double*, const NoAux3&) {
        if (!rowok) return;
        const long long idx = ((long long)z * g.NY + y) * g.NX + x;
        const bool unk = unk1(x, g.n) && unk1(y, g.n) && unk1(z, g.n);
        lv.W[idx] = unk ? ay + (a.smode ? 0.0 : lv.T[idx]) : 0.0;
      });
}

// Restriction march: the CTA owns 32 x 8 coarse points; each
// fine plane box (64+4p-2 x 16+4p-2) is staged, x-passed to the coarse columns
// and y-passed to the coarse rows; the z pass runs on a register ring of the
// last 4p-1 fine planes (two new planes per coarse output plane).
#ifndef FMG_RPF3
#define FMG_RPF3 2
#endif
#ifndef FMG_RNB3
#define FMG_RNB3 3
#endif
constexpr int RPF3 = FMG_RPF3, RNB3 = FMG_RNB3, RRS3 = 80;  // planes staged ahead, ring slots, cp.async row stride
// TMA form (a.tma): the fine plane box starts at the even column 2 x0 - 2p and
// is 64 + 4p doubles wide (16-byte rows), so fine column fxs sits at index 1.
template <int P>
__host__ __device__ constexpr int rbox_w() { return 64 + 4 * P; }
template <int P>
__host__ __device__ constexpr int rbox_slot() {  // doubles per ring slot (128-byte multiple)
  return ((2 * TW3 + 2 * (2 * P - 1)) * rbox_w<P>() + 15) & ~15;
}
template <int P, bool TMA>
__global__ void __launch_bounds__(32 * TW3, FMG_MARCH3_MINB) k_m3_restrict(const DevCtx* __restrict__ cp, const __grid_constant__ MArgs a,
                                                            const __grid_constant__ Coefs cf) {
  extern __shared__ __align__(128) double msm[];
  constexpr int NS = 4 * P - 1, H = 2 * P - 1, FR = 2 * TW3 + 2 * H, FW = 64 + 2 * H;
  constexpr int SROW = TMA ? rbox_w<P>() : RRS3, SLOT = TMA ? rbox_slot<P>() : FR * RRS3, SX = TMA ? 1 : 0;
  double* ring = msm;                // RNB3 x SLOT
  double* XR = ring + RNB3 * SLOT;   // FR x 32
  unsigned long long* bars = (unsigned long long*)(XR + FR * 32);  // (TMA) RNB3
  if (TMA && threadIdx.x == 0 && threadIdx.y == 0) {
#pragma unroll
    for (int k = 0; k < RNB3; ++k) mbar_init(bars + k, 1);
    mbar_init_fence();
  }
  if (TMA) __syncthreads();
  pdl_wait();
  pdl_trigger();
  M3Item it;
  m3_item(a, it);
  const MPtrs& c = a.p;
  const LevelDev& lc_ = a.lv;
  const LevelDev& lf = a.lo;
  const Geom gc = lc_.g, gf = lf.g;
  const int lane = threadIdx.x, w = threadIdx.y, xc = it.x0 + lane, yc = it.y0 + w;
  const bool rowok = yc < gc.NY;
  const int txc = xc % P, tyc = yc % P;
  const int fxs = 2 * it.x0 - H, fys = 2 * it.y0 - H;
  const double* __restrict__ Tf = lf.T;
  const int nxb = gc.NX >> 5;
  double rw[NS], rv[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    rw[s] = cf.Rw[txc][s];
    rv[s] = 0.0;
  }
  auto stage = [&](int fz, int k) {  // fine plane fz into ring slot k
    double* slot = ring + k * SLOT;
    if (TMA) {
      if (threadIdx.x == 0 && threadIdx.y == 0) {
        fence_async_smem();
        tma_load_3d(slot, a.tm, fxs - SX, fys, fz - a.zoff, bars + k, (unsigned)(FR * SROW * 8));
      }
      return;
    }
    const bool zok = fz >= 0 && fz < gf.NZ;
    for (int r = w; r < FR; r += TW3) {
      const int fy = fys + r;
      const bool rok = zok && fy >= 0 && fy < gf.NY;
      const double* rp = Tf + ((long long)(rok ? fz : 0) * gf.NY + (rok ? fy : 0)) * gf.NX;
#pragma unroll
      for (int kk = 0; kk < 3; ++kk) {
        const int jx = lane + 32 * kk;
        if (jx < FW) {
          const int fx = fxs + jx;
          const bool ok = rok && fx >= 0 && fx < gf.NX;
          cpa8(slot + r * RRS3 + jx, ok ? rp + fx : Tf, ok);
        }
      }
    }
  };
  const int fz0 = 2 * it.zs - H, nin = 2 * (it.ze - it.zs) + 2 * H;
  double ss = 0.0;
#pragma unroll
  for (int i = 0; i < RPF3; ++i) {
    if (i < nin) stage(fz0 + i, i % RNB3);
    if (!TMA) cp3_commit();
  }
  for (int i = 0; i < nin; ++i) {
    if (i + RPF3 < nin) stage(fz0 + i + RPF3, (i + RPF3) % RNB3);
    if (TMA) {
      mbar_wait(bars + i % RNB3, (unsigned)(i / RNB3) & 1u);
    } else {
      cp3_commit();
      asm volatile("cp.async.wait_group %0;\n" ::"n"(RPF3) : "memory");
    }
    __syncthreads();
    const double* slot = ring + (i % RNB3) * SLOT + SX;
    for (int r = w; r < FR; r += TW3) {
      const double* row = slot + r * SROW;
      double v = 0.0;
      if (TMA) {
        // (slot index 1 + even + 2 lane + s: taps s = 1, 2 | 3, 4 | ... sit at
        // 16-byte aligned pairs -> one 128-bit load each, half the wavefronts of
        // the stride-2 double loads; same fma order)
        v = fma(rw[0], row[2 * lane], v);
#pragma unroll
        for (int k = 0; k < (NS - 1) / 2; ++k) {
          const double2 q = *reinterpret_cast<const double2*>(row + 2 * lane + 1 + 2 * k);
          v = fma(rw[1 + 2 * k], q.x, v);
          v = fma(rw[2 + 2 * k], q.y, v);
        }
      } else {
#pragma unroll
        for (int s = 0; s < NS; ++s) v = fma(rw[s], row[2 * lane + s], v);  // (t = +0 at fine non-unknowns)
      }
      XR[r * 32 + lane] = v;
    }
    __syncthreads();
    double yv = 0.0;
#pragma unroll
    for (int s = 0; s < NS; ++s) yv = fma(cf.Rw[tyc][s], XR[(2 * w + s) * 32 + lane], yv);
#pragma unroll
    for (int s = 0; s < NS - 1; ++s) rv[s] = rv[s + 1];
    rv[NS - 1] = yv;
    if (i >= NS - 1 && ((i - (NS - 1)) & 1) == 0 && rowok) {
      const int zc = it.zs + (i - (NS - 1)) / 2, tzc = zc % P;
      double t = 0.0;
#pragma unroll
      for (int s = 0; s < NS; ++s) t = fma(cf.Rw[tzc][s], rv[s], t);
      t = (unk1(xc, gc.n) && unk1(yc, gc.n) && unk1(zc, gc.n)) ? t : 0.0;
      const long long idx = ((long long)zc * gc.NY + yc) * gc.NX + xc;
      lc_.T[idx] = t;
      ss = fma(t, t, ss);
      const long long blk = ((long long)zc * gc.NY + yc) * nxb + (it.x0 >> 5);
      if (!a.smode) warp_encode(t, a.wr, lc_.rmant + blk * lc_.rstride, lc_.rexp + blk, lane, c.status);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(FULL, ss, o);
  if (lane == 0 && a.poff >= 0) c.pbase[a.poff + (long long)it.cta * TW3 + w] = ss;
}

// ------------------------------------------------------------------ host --
static int m3_smem_A(int p, bool tma = false) {
  return (int)(((size_t)NB3 * (TW3 + 2 * p) * RS3 + 2 * (TW3 + 2 * p) * 32) * 8 + (tma ? NB3 * 8 : 0));
}
static int m3_smem_R(int p, bool tma = false) {
  const int FR = 2 * TW3 + 2 * (2 * p - 1);
  const int slot = tma ? (p == 1 ? rbox_slot<1>() : p == 2 ? rbox_slot<2>() : rbox_slot<3>()) : FR * RRS3;
  return (RNB3 * slot + FR * 32) * 8 + (tma ? RNB3 * 8 : 0);
}
int march3_rows() { return TW3; }

void march3_set_attributes() {
#define F(P)                                                                                             \
  cudaFuncSetAttribute(k_m3_residual<P, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, m3_smem_A(P));      \
  cudaFuncSetAttribute(k_m3_residual<P, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, m3_smem_A(P, true)); \
  cudaFuncSetAttribute(k_m3_cfas1<P, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, m3_smem_A(P));         \
  cudaFuncSetAttribute(k_m3_cfas1<P, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, m3_smem_A(P, true));    \
  cudaFuncSetAttribute(k_m3_cheb<P, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, m3_smem_A(P));          \
  cudaFuncSetAttribute(k_m3_cheb<P, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, m3_smem_A(P, true));     \
  cudaFuncSetAttribute(k_m3_gs<P, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, m3_smem_A(P));            \
  cudaFuncSetAttribute(k_m3_cfas1<P, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, m3_smem_A(P));   \
  cudaFuncSetAttribute(k_m3_cheb<P, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, m3_smem_A(P));    \
  cudaFuncSetAttribute(k_m3_sq<P>, cudaFuncAttributeMaxDynamicSharedMemorySize, m3_smem_A(P));                  \
  cudaFuncSetAttribute(k_m3_gs<P, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, m3_smem_A(P));      \
  cudaFuncSetAttribute(k_m3_gs<P, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, m3_smem_A(P, true));       \
  cudaFuncSetAttribute(k_m3_restrict<P, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, m3_smem_R(P));      \
  cudaFuncSetAttribute(k_m3_restrict<P, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, m3_smem_R(P, true));
  F(1) F(2) F(3)
#undef F
}

template <typename K>
static void m3_launch(K kernel, int nctas, int smem, cudaStream_t st, const DevCtx* c, const MArgs& a,
                      const Coefs& cf) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(nctas);
  cfg.blockDim = dim3(32, TW3);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, c, a, cf);
}

void launch_march3(int p, cudaStream_t st, const void* devctx, const MArgs& a, const Coefs& cf) {
  const DevCtx* c = (const DevCtx*)devctx;
  const int n = a.nitems;
  const bool t = a.tma != 0;
  const bool nu = a.guess || a.store;  // nu > 1 cycle kernels
#define TM(K, P) (t ? (void (*)(const DevCtx*, MArgs, Coefs))K<P, true> : (void (*)(const DevCtx*, MArgs, Coefs))K<P, false>)
#define F(P)                                                                                  \
  switch (a.type) {                                                                           \
    case OP_DECODE:                                                                           \
    case OP_PROLONG: m3_launch(k_m3_prolong<P>, n, 0, st, c, a, cf); break;                   \
    case OP_RESIDUAL: m3_launch(TM(k_m3_residual, P), n, m3_smem_A(P, t), st, c, a, cf); break; \
    case OP_RESTRICT: m3_launch(TM(k_m3_restrict, P), n, m3_smem_R(P, t), st, c, a, cf); break; \
    case OP_CFAS1:                                                                            \
      if (nu) m3_launch(k_m3_cfas1<P, false, true>, n, m3_smem_A(P), st, c, a, cf);            \
      else m3_launch(TM(k_m3_cfas1, P), n, m3_smem_A(P, t), st, c, a, cf);                     \
      break;                                                                                   \
    case OP_SQ: m3_launch(k_m3_sq<P>, n, m3_smem_A(P), st, c, a, cf); break;                  \
    case OP_GS:                                                                               \
      if (nu) m3_launch(k_m3_gs<P, false, true>, n, m3_smem_A(P), st, c, a, cf);               \
      else m3_launch(TM(k_m3_gs, P), n, m3_smem_A(P, t), st, c, a, cf);                        \
      break;                                                                                   \
    default:                                                                                  \
      if (nu) m3_launch(k_m3_cheb<P, false, true>, n, m3_smem_A(P), st, c, a, cf);             \
      else m3_launch(TM(k_m3_cheb, P), n, m3_smem_A(P, t), st, c, a, cf);                      \
      break;                                                                                   \
  }
  if (p == 1) { F(1) } else if (p == 2) { F(2) } else { F(3) }
#undef F
#undef TM
}

}  // namespace fmg
