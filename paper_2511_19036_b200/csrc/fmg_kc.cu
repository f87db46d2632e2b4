// fmg_kc.cu -- the coarse-hierarchy cluster kernel ("KC") of the compact-FMG
// hot path.
//
// Levels 0..lc (the small ones, where a grid launch per step would cost more
// than the step itself) are run by ONE thread-block cluster (16 CTAs x 16
// warps when the device co-schedules it, else 8/4/2/1).  All their data --
// the FP64 level arrays u_l, t_l, w_l, the scratch arrays and the BFP sections
// ú_l, r_l -- live in the cluster's *distributed shared memory*: 32-entry block b
// of a level (= one BFP block) is owned by CTA b mod NC, which computes it
// ("owner computes"); stencil neighbours in other blocks are read from the
// owner CTA through DSMEM (mapa + generic loads).  Every step of the method is
// one *phase* separated by the hardware cluster barrier
// (barrier.cluster.arrive.release / wait.acquire), which here orders only
// shared-memory traffic: a phase costs a barrier and a DSMEM round trip
// instead of a kernel launch.  Global memory is touched only in the prologue
// (sections, and t_{lc+1} from the grid levels) and the epilogue (sections
// back, u_l / w_l for the grid levels, norm partials).  The small operators
// recompute their inner passes per output point (2D: one phase per A, R, P;
// 3D: the x/y passes of A and R go through a scratch phase).
//
// Every expression follows the canonical evaluation order of DESIGN.md §3 with
// explicit fma() (-fmad=false), so the results are bit-identical to the grid
// tile ops and to the oracle.
//
// Paper: fmgResidual restriction sweep (Alg 3.2), coarse solve
// (PAPER.md:640, 786), coarse-to-fine cFas sweep with nu = 1 (Alg 3.1
// PAPER.md:638-643, s = 0 by PAPER.md:809-812), correction (Alg 3.3)
// and, for FMG levels L <= lc, whole IR iterations.
#include <algorithm>
#include <cstdlib>
#include <new>

#include "fmg_device.cuh"

namespace fmg {

constexpr int KC_NW = 16;
constexpr int KC_NT = 32 * KC_NW;
constexpr int KC_SMEM_MAX = 176 * 1024;  // dynamic shared memory budget per CTA (static: ~46 KB)

__device__ __forceinline__ unsigned cl_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// generic address of the same shared-memory location in CTA `rank` of the cluster
template <class T>
__device__ __forceinline__ T* mapa(T* p, unsigned rank) {
  T* r;
  asm("mapa.u64 %0, %1, %2;" : "=l"(r) : "l"(p), "r"(rank));
  return r;
}

__device__ unsigned long long g_kc_stamps[256];
__device__ int g_kc_nstamp = 0;
// Cluster-wide phase barrier (release/acquire at cluster scope).
__device__ __noinline__ void kc_stamp() {  // debug phase stamps
  if (threadIdx.x == 0 && threadIdx.y == 0 && cl_rank() == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    int i = g_kc_nstamp;
    if (i < 256) g_kc_stamps[i] = t;
    g_kc_nstamp = i + 1;
  }
}
__device__ __forceinline__ void csync(bool dbg = false) {
  if (gridDim.x == 1) {  // one-CTA "cluster": all level data is local shared memory
    __syncthreads();
  } else {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  if (dbg) kc_stamp();
}

// Element access.  A distributed array is a per-CTA slab at the same shared
// offset in every CTA.  The 32-entry blocks of an index space (a level, or the
// 3D restriction staging box) are split into contiguous chunks of 2^lgc blocks
// (row-major: a CTA owns a band of rows, so most stencil neighbours are local);
// block b lives in CTA b >> lgc at slab block b & (2^lgc - 1).
// chunk = 2^lgc blocks, the smallest power of two >= ceil(nblk / NC)
__host__ __device__ __forceinline__ int kc_lgc(int nblk, int lg) {
  int per = (nblk + (1 << lg) - 1) >> lg, k = 0;
  while ((1 << k) < per) ++k;
  return k;
}

// stencil read of a distributed array (0 outside the index space)
struct DAcc {
  double* base;   // local slab
  Geom g;         // index space (NX, NY, NZ)
  int lgc;
  unsigned me;
  __device__ __forceinline__ double operator()(int x, int y, int z) const {
    if (x < 0 || x >= g.NX || y < 0 || y >= g.NY || z < 0 || z >= g.NZ) return 0.0;
    int idx = (z * g.NY + y) * g.NX + x;
    unsigned ow = (unsigned)(idx >> (5 + lgc));
    double* p = base + (idx & ((32 << lgc) - 1));
    return ow == me ? *p : *mapa(p, ow);
  }
  // pointer to the first entry of 32-entry block column xb of row (y, z), or null
  __device__ __forceinline__ const double* blk(int xb, int y, int z) const {
    if (xb < 0 || xb >= (g.NX >> 5) || y < 0 || y >= g.NY || z < 0 || z >= g.NZ) return nullptr;
    int idx = ((z * g.NY + y) * g.NX) + (xb << 5);
    unsigned ow = (unsigned)(idx >> (5 + lgc));
    double* p = base + (idx & ((32 << lgc) - 1));
    return ow == me ? p : mapa(p, ow);
  }
};
// stencil read of a global level array
struct GAcc {
  const double* p;
  Geom g;
  __device__ __forceinline__ double operator()(int x, int y, int z) const {
    if (x < 0 || x >= g.NX || y < 0 || y >= g.NY || z < 0 || z >= g.NZ) return 0.0;
    return p[((long long)z * g.NY + y) * g.NX + x];
  }
  __device__ __forceinline__ const double* blk(int xb, int y, int z) const {
    if (xb < 0 || xb >= (g.NX >> 5) || y < 0 || y >= g.NY || z < 0 || z >= g.NZ) return nullptr;
    return p + ((long long)z * g.NY + y) * g.NX + (xb << 5);
  }
};

constexpr int KC_ROWBUF = 320;  // per-warp staging tile (doubles): 7 rows x 40 (A) / 4 rows x 80 (R)

#define LANE ((int)threadIdx.x)
#define WID ((int)threadIdx.y)
#define SROW (kc_srow[threadIdx.y])
#define SROWR(r, j) (kc_srow[threadIdx.y][(r) * RSTR + (j)])
__shared__ double kc_srow[KC_NW][KC_ROWBUF];  // per-warp staging rows

// Out-of-line codec (one copy shared by every phase: KC is bound by
// instruction-cache misses, not by call overhead).
__device__ __noinline__ double kc_enc(double v, int w, uint32_t* words, int8_t* eptr, int* status) {
  return warp_encode(v, w, words, eptr, (int)threadIdx.x, status);
}
__device__ __noinline__ double kc_dec(const uint32_t* words, int E, int w) {
  return warp_decode(words, E, w, (int)threadIdx.x);
}

template <int D, int P>
struct Kc {
  const DevCtx& c;
  const KcLayout& ly;
  const KcDesc& a;
  const Coefs& cf;
  double* sd;          // this CTA's dynamic shared memory (as doubles)
  int NC, rank;
  bool dbg;            // debug phase stamps
  // (the object lives in shared memory; per-thread values come from threadIdx)

  __device__ int wu(int l, int L) const { return a.b_u + a.k_u * (L - l); }
  __device__ int wr(int l, int L) const { return a.b_r + a.k_r * (L - l); }
  // width of ú_l before the update of IR iteration `it` at FMG level L
  __device__ int wu_in(int l, int L, int it) const {
    if (it > 0) return wu(l, L);
    return l == L ? wu(L, L) : wu(l, L - 1);
  }
  __device__ DAcc acc(int off, const Geom& g) const {
    return DAcc{sd + off, g, kc_lgc((g.NX >> 5) * g.NY * g.NZ, ly.lg), (unsigned)rank};
  }
  // own element (of an index space with 2^lgc blocks per CTA)
  __device__ __forceinline__ double& own(int off, int lgc, long long idx) const {
    return sd[off + ((int)idx & ((32 << lgc) - 1))];
  }
  // owner-local section storage of block b of level l
  __device__ __forceinline__ int lblk(int l, long long b) const {
    return (int)b & ((1 << ly.lgc[l]) - 1);
  }
  __device__ __forceinline__ uint32_t* umw(int l, long long b) const {
    return (uint32_t*)sd + ly.um[l] + lblk(l, b) * c.lv[l].ustride;
  }
  __device__ __forceinline__ uint32_t* rmw(int l, long long b) const {
    return (uint32_t*)sd + ly.rm[l] + lblk(l, b) * c.lv[l].rstride;
  }
  __device__ __forceinline__ int8_t* uex(int l, long long b) const { return (int8_t*)sd + ly.ue[l] + lblk(l, b); }
  __device__ __forceinline__ int8_t* rex(int l, long long b) const { return (int8_t*)sd + ly.re[l] + lblk(l, b); }

  // ---- warp-level gathers: all loads of an item are issued before any use --
  // v[k] = a(xs + lane + 32 k, y, z) for lane + 32 k < W (else 0)
  template <int K, class U>
  __device__ __forceinline__ void gather(const U& a_, int xs, int W, int y, int z, double (&v)[K]) const {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      int j = LANE + 32 * k;
      v[k] = j < W ? a_(xs + j, y, z) : 0.0;
    }
  }
  // stage a gathered row into the warp's shared row buffer
  template <int K>
  __device__ __forceinline__ void stage(const double (&v)[K], int W) const {
    __syncwarp();
#pragma unroll
    for (int k = 0; k < K; ++k) {
      int j = LANE + 32 * k;
      if (j < W) SROW[j] = v[k];
    }
    __syncwarp();
  }
  // store a gathered row as row r (stride RSTR) of the warp's staging tile (no sync)
  template <int K, int RSTR>
  __device__ __forceinline__ void put(const double (&v)[K], int W, int r) const {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      int j = LANE + 32 * k;
      if (j < W) SROWR(r, j) = v[k];
    }
  }

  // ---- per-point operators, warp-level (canonical trees) ----
  // x0: first column of the warp's block; every LANE returns its column's value.
  // A, x and y passes at output row y, plane z: returns (2D) A u, or (3D) the
  // staged c = My Mx u and s = Ky Mx u + My Kx u (0 where x or y is not an unknown)
  template <class U>
  __device__ __noinline__ void Axy(U u, const Geom g, int x0, int y, int z, double& cv, double& sv) const {
    constexpr int R = 2 * P + 1, W = 32 + 2 * P;
    const int x = x0 + LANE, tx = x % P, ty = y % P;
    constexpr int RSTR = 40;
    double v[R][2];
#pragma unroll
    for (int r = 0; r < R; ++r) gather<2>(u, x0 - P, W, y - P + r, z, v[r]);
    // all rows staged at once; the R x passes are independent chains (ILP)
    __syncwarp();
#pragma unroll
    for (int r = 0; r < R; ++r) put<2, RSTR>(v[r], W, r);
    __syncwarp();
    double xs[R], xt[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      double s = 0.0, t = 0.0;
#pragma unroll
      for (int o = 0; o < R; ++o) {
        double val = SROWR(r, LANE + o);
        s = fma(cf.Mc[tx][o], val, s);
        t = fma(cf.Kc[tx][o], val, t);
      }
      xs[r] = s;
      xt[r] = t;
    }
    __syncwarp();
    double cc = 0.0, dd = 0.0, e = 0.0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const double s = xs[r], t = xt[r];
      if constexpr (D == 2) {
        dd = fma(cf.Kc[ty][r], s, dd);
        e = fma(cf.Mc[ty][r], t, e);
      } else {
        cc = fma(cf.Mc[ty][r], s, cc);
        dd = fma(cf.Kc[ty][r], s, dd);
        e = fma(cf.Mc[ty][r], t, e);
      }
    }
    const bool ok = unk1(x, g.n) && unk1(y, g.n);
    cv = ok ? (D == 2 ? dd + e : cc) : 0.0;
    sv = ok ? dd + e : 0.0;
  }
  // 3D z pass over the staged c, s (KS0, KS1), times h
  __device__ __noinline__ double A3z(const Geom g, int x, int y, int z) const {
    constexpr int R = 2 * P + 1;
    const DAcc C = acc(ly.KS0, g), S = acc(ly.KS1, g);
    double cz[R], sz[R];
#pragma unroll
    for (int o = 0; o < R; ++o) {
      cz[o] = C(x, y, z - P + o);
      sz[o] = S(x, y, z - P + o);
    }
    if (!unk1(x, g.n) || !unk1(y, g.n) || !unk1(z, g.n)) return 0.0;
    const int tz = z % P;
    double s = 0.0;
#pragma unroll
    for (int o = 0; o < R; ++o) s = fma(cf.Kc[tz][o], cz[o], s);
#pragma unroll
    for (int o = 0; o < R; ++o) s = fma(cf.Mc[tz][o], sz[o], s);
    return s * pow2(-(g.l + 1));
  }
  // (P_l coarse) at fine (x0 + LANE, y, z): x, y, z passes;
  // 0 at fine non-unknowns.  The coarse rows are gathered 32 columns wide.
  template <class U>
  __device__ __noinline__ double Pat(U cA, int nf, int x0, int y, int z) const {
    constexpr int NR = (D == 3) ? (P + 1) * (P + 1) : P + 1;
    const int x = x0 + LANE;
    const bool okx = unk1(x, nf);
    const int cxs = P * (x0 / (2 * P));
    const int rx = okx ? x % (2 * P) : 0, bx = okx ? P * (x / (2 * P)) : cxs;
    const bool oky = unk1(y, nf), okz = (D == 2) || unk1(z, nf);
    const int ry = oky ? y % (2 * P) : 0, by = oky ? P * (y / (2 * P)) : 0;
    const int rz = (D == 3 && okz) ? z % (2 * P) : 0, bz = (D == 3 && okz) ? P * (z / (2 * P)) : 0;
    double v[NR][1];
#pragma unroll
    for (int t3 = 0; t3 < (D == 3 ? P + 1 : 1); ++t3)
#pragma unroll
      for (int t2 = 0; t2 <= P; ++t2) gather<1>(cA, cxs, 32, by + t2, bz + t3, v[t3 * (P + 1) + t2]);
    double accz = 0.0, accy = 0.0;
#pragma unroll
    for (int t3 = 0; t3 < (D == 3 ? P + 1 : 1); ++t3) {
      accy = 0.0;
#pragma unroll
      for (int t2 = 0; t2 <= P; ++t2) {
        stage<1>(v[t3 * (P + 1) + t2], 32);
        double accx = 0.0;
#pragma unroll
        for (int t1 = 0; t1 <= P; ++t1) accx = fma(cf.Pw[rx][t1], SROW[bx - cxs + t1], accx);
        accy = fma(cf.Pw[ry][t2], accx, accy);
      }
      if (D == 3) accz = fma(cf.Pw[rz][t3], accy, accz);
    }
    if (!okx || !oky || !okz) return 0.0;
    return D == 2 ? accy : accz;
  }
  // R at coarse (x0c + LANE, yc) on fine plane fz: the x and y passes (2D: R t_f;
  // 3D: the staged y pass).  Fine rows are gathered in batches of RB.
  template <class U>
  __device__ __noinline__ double Rxy(U tf, const Geom gf, int nc, int x0c, int yc, int fz) const {
    constexpr int NS = 4 * P - 1, W = 64 + NS - 1, RB = 4, RSTR = 80;
    const int xc = x0c + LANE, txc = xc % P, tyc = yc % P;
    const int fxs = 2 * x0c - (2 * P - 1);
    double t = 0.0;
#pragma unroll
    for (int s0 = 0; s0 < NS; s0 += RB) {
      double v[RB][3];
#pragma unroll
      for (int r = 0; r < RB; ++r)
        if (s0 + r < NS) gather<3>(tf, fxs, W, 2 * yc - (2 * P - 1) + s0 + r, fz, v[r]);
      __syncwarp();
#pragma unroll
      for (int r = 0; r < RB; ++r)
        if (s0 + r < NS) put<3, 80>(v[r], W, r);
      __syncwarp();
      double xv[RB];
#pragma unroll
      for (int r = 0; r < RB; ++r) {
        xv[r] = 0.0;
        if (s0 + r >= NS) continue;
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          // (t is stored as +0 at fine non-unknowns: no mask needed)
          xv[r] = fma(cf.Rw[txc][s], SROWR(r, 2 * LANE + s), xv[r]);
        }
      }
#pragma unroll
      for (int r = 0; r < RB; ++r)
        if (s0 + r < NS) t = fma(cf.Rw[tyc][s0 + r], xv[r], t);
    }
    return (unk1(xc, nc) && unk1(yc, nc)) ? t : 0.0;
  }
  // 3D second half of R: z pass over the staged planes (KS0, geometry (NXc, NYc, NZf))
  __device__ __noinline__ double R3z(const Geom gc, int nzf, int xc, int yc, int zc) const {
    constexpr int NS = 4 * P - 1;
    Geom gs = gc;
    gs.NZ = nzf;
    const DAcc YV = acc(ly.KS0, gs);
    double v[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) v[s] = YV(xc, yc, 2 * zc - (2 * P - 1) + s);
    if (!unk1(xc, gc.n) || !unk1(yc, gc.n) || !unk1(zc, gc.n)) return 0.0;
    const int tzc = zc % P;
    double t = 0.0;
#pragma unroll
    for (int s = 0; s < NS; ++s) t = fma(cf.Rw[tzc][s], v[s], t);
    return t;
  }

  __device__ __forceinline__ double rhs(const LevelDev& lv, int x, int y, int z) const {
    double f = cf.rhs_c * lv.gtab[x];
    f = f * lv.gtab[y];
    if (D == 3) f = f * lv.gtab[z];
    return f;
  }
  __device__ __forceinline__ bool unk(const Geom& g, int x, int y, int z) const {
    return unk1(x, g.n) && unk1(y, g.n) && (D == 2 || unk1(z, g.n));
  }
  __device__ __forceinline__ double invd(const Geom& g, int x, int y, int z) const {
    if (!unk(g, x, y, z)) return 0.0;
    return cf.invd[((D == 3 ? z % P : 0) * P + y % P) * P + x % P] * pow2((g.l + 1) * (D - 2));
  }

  // ---- owned 32-entry blocks (one warp per block); warp-uniform loops ----
  // Blocks of a (NX, NY, nz) index space owned by this CTA (a contiguous chunk
  // of nbpc blocks); warp w takes the chunk's blocks w, w + 16, ...
  // body(x0, y, z, idx, b, nbpc) with x0 the block's first column.
  template <class F>
  __device__ __forceinline__ void blocks(const Geom& g, int nz, F body) const {
    const int nxb = g.NX >> 5;
    const int nb = nxb * g.NY * nz;
    const int lgc = kc_lgc(nb, ly.lg);
    const int b1 = min(nb, (rank + 1) << lgc);
    for (int b = (rank << lgc) + WID; b < b1; b += KC_NW) {
      int xb = b % nxb;
      int r = b / nxb;
      int y = r % g.NY, z = r / g.NY;
      body(xb * 32, y, z, (long long)(b * 32 + LANE), (long long)b, lgc);
    }
  }
  template <class F>
  __device__ __forceinline__ void blocks(const Geom& g, F body) const {
    blocks(g, g.NZ, body);
  }

  // per-warp norm partial of ||t_l||^2 into the shared table (flushed at the end)
  __device__ void norm_partial(double ss, int row, int l) const {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(FULL, ss, o);
    if (LANE == 0) sd[ly.part + ((row - a.row0) * (c.lc + 1) + l) * KC_NW + WID] = ss;
  }

  // A applied at the warp's block (2D: one phase; 3D: z pass over KS0/KS1 staged by ph_A3xy)
  __device__ __forceinline__ double Aat(int off, const Geom& g, int x0, int y, int z) const {
    if constexpr (D == 2) {
      double cv, sv;
      Axy(acc(off, g), g, x0, y, 0, cv, sv);
      return cv;
    } else {
      return A3z(g, x0 + LANE, y, z);
    }
  }

  // ---- phases ------------------------------------------------------------
  // u_L = dec ú_L + P_L u_{L-1} (decode sweep S2)
  __device__ __noinline__ void ph_decode(int L, int wd) const {
    const Geom& g = c.lv[L].g;
    const DAcc up = acc(ly.U[L - 1], c.lv[L - 1].g);
    blocks(g, [&](int x0, int y, int z, long long idx, long long b, int nb) {
      double pu = Pat(up, g.n, x0, y, z);
      double dv = kc_dec(umw(L, b), *uex(L, b), wd);
      own(ly.U[L], nb, idx) = dv + pu;
    });
  }
  // 3D scratch phase: KS0, KS1 = x/y passes of A on the array at `off`
  __device__ __noinline__ void ph_A3xy(int off, const Geom& g) const {
    const DAcc u = acc(off, g);
    blocks(g, [&](int x0, int y, int z, long long idx, long long, int nb) {
      double cv, sv;
      Axy(u, g, x0, y, z, cv, sv);
      own(ly.KS0, nb, idx) = cv;
      own(ly.KS1, nb, idx) = sv;
    });
  }
  // t_L = f_L - A_L u_L, r_L = enc(t_L)
  __device__ __noinline__ void ph_residual(int L, int row) const {
    const LevelDev& lv = c.lv[L];
    const int wrL = wr(L, L);
    double ss = 0.0;
    blocks(lv.g, [&](int x0, int y, int z, long long idx, long long b, int nb) {
      const int x = x0 + LANE;
      double au = Aat(ly.U[L], lv.g, x0, y, z);
      double t = unk(lv.g, x, y, z) ? rhs(lv, x, y, z) - au : 0.0;
      own(ly.T[L], nb, idx) = t;
      ss = fma(t, t, ss);
      double q = kc_enc(t, wrL, rmw(L, b), rex(L, b), c.status);
      if (L == 0) own(ly.RQ0, nb, idx) = q;
    });
    norm_partial(ss, row, L);
  }
  // fine t_{l+1}: global for l = lc (grid level lc+1), distributed otherwise
  template <class F>
  __device__ __forceinline__ void with_fine(int l, F f) const {
    if (l == c.lc) f(GAcc{c.lv[l + 1].T, c.lv[l + 1].g});
    else f(acc(ly.T[l + 1], c.lv[l + 1].g));
  }
  // 3D scratch phase of R: KS0 = y pass of the x pass of t_{l+1}, per fine plane
  __device__ __noinline__ void ph_R3xy(int l) const {
    const Geom& gc = c.lv[l].g;
    const Geom& gf = c.lv[l + 1].g;
    with_fine(l, [&](const auto& tf) {
      blocks(gc, gf.NZ, [&](int x0, int y, int fz, long long idx, long long, int nb) {
        own(ly.KS0, nb, idx) = Rxy(tf, gf, gc.n, x0, y, fz);
      });
    });
  }
  // t_l = R_{l+1} t_{l+1} (restricts t, not r: PAPER.md:742-744), r_l = enc(t_l)
  __device__ __noinline__ void ph_restrict(int l, int L, int row) const {
    const Geom& gc = c.lv[l].g;
    const Geom& gf = c.lv[l + 1].g;
    const int wrl = wr(l, L);
    double ss = 0.0;
    with_fine(l, [&](const auto& tf) {
      blocks(gc, [&](int x0, int y, int z, long long idx, long long b, int nb) {
        double t;
        if constexpr (D == 2) t = Rxy(tf, gf, gc.n, x0, y, 0);
        else t = R3z(gc, gf.NZ, x0 + LANE, y, z);
        own(ly.T[l], nb, idx) = t;
        ss = fma(t, t, ss);
        double q = kc_enc(t, wrl, rmw(l, b), rex(l, b), c.status);
        if (l == 0) own(ly.RQ0, nb, idx) = q;
      });
    });
    norm_partial(ss, row, l);
  }
  // unknown index of level 0 (x fastest among the (2p-1)^d unknowns)
  __device__ __forceinline__ int coarse_index(int x, int y, int z) const {
    const int m = 2 * P - 1;
    return ((D == 3 ? z - 1 : 0) * m + (y - 1)) * m + (x - 1);
  }
  // Initial coarse solve ú_0 = enc(A_0^{-1} f_0), u_0 = dec ú_0
  __device__ __noinline__ void ph_coarse_initial() const {
    const LevelDev& lv = c.lv[0];
    const int m = 2 * P - 1;
    blocks(lv.g, [&](int x0, int y, int z, long long idx, long long b, int nb) {
      const int x = x0 + LANE;
      double s = 0.0;
      if (unk(lv.g, x, y, z)) {
        const int I = coarse_index(x, y, z);
        for (int J = 0; J < c.n0; ++J) {
          int jx = J % m + 1, jy = (J / m) % m + 1, jz = (D == 3) ? J / (m * m) + 1 : 0;
          s = fma(c.Ainv[(long long)I * c.n0 + J], rhs(lv, jx, jy, jz), s);
        }
      }
      double q = kc_enc(s, wu(0, 0), umw(0, b), uex(0, b), c.status);
      own(ly.U[0], nb, idx) = q;
    });
  }
  // ý_0 = enc(A_0^{-1} dec r_0) (reading R5); w_0 = dec ý_0;
  // ú_0 = enc(dec ú_0 + dec ý_0); u_0 = dec ú_0.
  __device__ __noinline__ void ph_coarse(int L, int it, double* srq) const {
    const Geom& g = c.lv[0].g;
    const int m = 2 * P - 1;
    {  // every CTA gathers dec r_0 at the unknowns (one batched round of loads)
      const DAcc rq = acc(ly.RQ0, g);
      const int J = WID * 32 + LANE;
      if (J < c.n0) srq[J] = rq(J % m + 1, (J / m) % m + 1, (D == 3) ? J / (m * m) + 1 : 0);
      __syncthreads();
    }
    blocks(g, [&](int x0, int y, int z, long long idx, long long b, int nb) {
      const int x = x0 + LANE;
      double s = 0.0;
      if (unk(g, x, y, z)) {
        const double* Ai = c.Ainv + (long long)coarse_index(x, y, z) * c.n0;
#pragma unroll 9
        for (int J = 0; J < c.n0; ++J) s = fma(Ai[J], srq[J], s);
      }
      double yq = kc_enc(s, wr(0, L), nullptr, nullptr, c.status);
      double uo = kc_dec(umw(0, b), *uex(0, b), wu_in(0, L, it));
      double uq = kc_enc(uo + yq, wu(0, L), umw(0, b), uex(0, b), c.status);
      own(ly.W[0], nb, idx) = yq;
      own(ly.U[0], nb, idx) = uq;
    });
  }
  // z_l = P_l w_{l-1} and P_l u_{l-1} (for the emitted u_l)
  __device__ __noinline__ void ph_prolong(int l) const {
    const Geom& g = c.lv[l].g;
    const DAcc wp = acc(ly.W[l - 1], c.lv[l - 1].g), up = acc(ly.U[l - 1], c.lv[l - 1].g);
    blocks(g, [&](int x0, int y, int z, long long idx, long long, int nb) {
      own(ly.Z, nb, idx) = Pat(wp, g.n, x0, y, z);
      own(ly.PU, nb, idx) = Pat(up, g.n, x0, y, z);
    });
  }
  // ý_l = enc(y); w_l = z_l + dec ý_l; ú_l = enc(dec ú_l + dec ý_l); u_l = dec ú_l + P u_{l-1}
  __device__ __forceinline__ void finalize(int l, int L, int it, long long idx, long long b, int nb, double y) const {
    double yq = kc_enc(y, wr(l, L), nullptr, nullptr, c.status);
    if (l < L) own(ly.W[l], nb, idx) = own(ly.Z, nb, idx) + yq;
    double uo = kc_dec(umw(l, b), *uex(l, b), wu_in(l, L, it));
    double uq = kc_enc(uo + yq, wu(l, L), umw(l, b), uex(l, b), c.status);
    own(ly.U[l], nb, idx) = uq + own(ly.PU, nb, idx);
  }
  // Chebyshev step 1: b = dec r_l - A z_l; d_1 = y_1 = inv_theta (invD b)
  __device__ __noinline__ void ph_cheb1(int l, int L, int it) const {
    const Geom& g = c.lv[l].g;
    const int wrl = wr(l, L);
    const int k = c.n_cheb;
    blocks(g, [&](int x0, int y, int z, long long idx, long long b, int nb) {
      const int x = x0 + LANE;
      double az = Aat(ly.Z, g, x0, y, z);
      double rv = kc_dec(rmw(l, b), *rex(l, b), wrl);
      double bb = rv - az;
      double d = cf.inv_theta * (invd(g, x, y, z) * bb);
      if (c.smoother == 1) {  // multicolour GS from y = 0: colour 0 gets y = 0 + invD (b - 0)
        own(ly.B, nb, idx) = bb;
        const bool c0 = x % (P + 1) == 0 && y % (P + 1) == 0 && (D == 2 || z % (P + 1) == 0);
        own(ly.Y1, nb, idx) = c0 ? 0.0 + invd(g, x, y, z) * (bb - 0.0) : 0.0;
      } else if (k == 1) {
        finalize(l, L, it, idx, b, nb, d);
      } else {
        own(ly.B, nb, idx) = bb;
        own(ly.Y1, nb, idx) = d;
      }
    });
  }
  // step j >= 2: q = b - A y; d_j = fma(alpha_j, d_{j-1}, beta_j (invD q)); y_j = y_{j-1} + d_j
  __device__ __noinline__ void ph_chebj(int l, int L, int it, int j) const {
    const Geom& g = c.lv[l].g;
    const int k = c.n_cheb;
    const int yp = (j - 1) & 1 ? ly.Y1 : ly.Y0, yn = j & 1 ? ly.Y1 : ly.Y0;
    blocks(g, [&](int x0, int y, int z, long long idx, long long b, int nb) {
      const int x = x0 + LANE;
      double ay = Aat(yp, g, x0, y, z);
      double q = own(ly.B, nb, idx) - ay;
      double yprev = own(yp, nb, idx);
      double dprev = (j == 2) ? yprev : own(ly.Dv, nb, idx);
      double d = fma(cf.cal[j - 1], dprev, cf.cbe[j - 1] * (invd(g, x, y, z) * q));
      double yv = yprev + d;
      if (j == k) {
        finalize(l, L, it, idx, b, nb, yv);
      } else {
        own(yn, nb, idx) = yv;
        own(ly.Dv, nb, idx) = d;
      }
    });
  }

  // Multicolour Gauss-Seidel colour col >= 1 on Y1 in place (nodes of one colour
  // are uncoupled); the last colour finalises (oracle mc_gauss_seidel).
  __device__ __noinline__ void ph_gs(int l, int L, int it, int col, int ncol) const {
    const Geom& g = c.lv[l].g;
    const int cx = col % (P + 1), cy = (col / (P + 1)) % (P + 1), cz = col / ((P + 1) * (P + 1));
    blocks(g, [&](int x0, int y, int z, long long idx, long long b, int nb) {
      const int x = x0 + LANE;
      const double ay = Aat(ly.Y1, g, x0, y, z);
      const bool mine = x % (P + 1) == cx && y % (P + 1) == cy && (D == 2 || z % (P + 1) == cz);
      const double yo = own(ly.Y1, nb, idx);
      const double yv = mine ? yo + invd(g, x, y, z) * (own(ly.B, nb, idx) - ay) : yo;
      if (col == ncol - 1) finalize(l, L, it, idx, b, nb, yv);
      else if (mine) own(ly.Y1, nb, idx) = yv;
    });
  }

  // One IR iteration at FMG level L restricted to levels 0..min(L, lc)
  // (PAPER.md:791-798).  For L > lc the grid ops did the residual and the
  // restriction down to lc+1 and do the cFas levels above lc afterwards.
  __device__ __noinline__ void iteration(int L, int it, double* srq) const {
    const int lc = c.lc;
    const int top = L < lc ? L : lc;
    const int row = L * c.n_ir + it;
    if (L <= lc) {
      if (it == 0) {
        ph_decode(L, wu(L, L));
        csync(dbg);
      }
      if constexpr (D == 3) {
        ph_A3xy(ly.U[L], c.lv[L].g);
        csync(dbg);
      }
      ph_residual(L, row);
      csync(dbg);
    }
    for (int l = top - (L <= lc ? 1 : 0); l >= 0; --l) {
      if constexpr (D == 3) {
        ph_R3xy(l);
        csync(dbg);
      }
      ph_restrict(l, L, row);
      csync(dbg);
    }
    ph_coarse(L, it, srq);
    csync(dbg);
    for (int l = 1; l <= top; ++l) {
      ph_prolong(l);
      csync(dbg);
      if constexpr (D == 3) {
        ph_A3xy(ly.Z, c.lv[l].g);
        csync(dbg);
      }
      ph_cheb1(l, L, it);
      csync(dbg);
      if (c.smoother == 1) {
        const int ncol = D == 3 ? (P + 1) * (P + 1) * (P + 1) : (P + 1) * (P + 1);
        for (int col = 1; col < ncol; ++col) {
          if constexpr (D == 3) {
            ph_A3xy(ly.Y1, c.lv[l].g);
            csync(dbg);
          }
          ph_gs(l, L, it, col, ncol);
          csync(dbg);
        }
        continue;
      }
      for (int j = 2; j <= c.n_cheb; ++j) {
        if constexpr (D == 3) {
          ph_A3xy((j - 1) & 1 ? ly.Y1 : ly.Y0, c.lv[l].g);
          csync(dbg);
        }
        ph_chebj(l, L, it, j);
        csync(dbg);
      }
    }
  }

  // ---- prologue / epilogue (the only global-memory traffic) ---------------
  __device__ __noinline__ void load_sections(int top) const {
    const int tid = WID * 32 + LANE;
    for (int l = 0; l <= top; ++l) {
      const LevelDev& lv = c.lv[l];
      const int nb = (int)lv.g.nblk, nbpc = 1 << ly.lgc[l], b0 = rank * nbpc;
      const int nloc = max(0, min(nb, b0 + nbpc) - b0);
      const uint32_t* um = lv.umant + (long long)b0 * lv.ustride;
      const uint32_t* rm = lv.rmant + (long long)b0 * lv.rstride;
      for (int i = tid; i < nloc * lv.ustride; i += KC_NT) ((uint32_t*)sd)[ly.um[l] + i] = um[i];
      for (int i = tid; i < nloc * lv.rstride; i += KC_NT) ((uint32_t*)sd)[ly.rm[l] + i] = rm[i];
      for (int k = tid; k < nloc; k += KC_NT) {
        ((int8_t*)sd)[ly.ue[l] + k] = lv.uexp[b0 + k];
        ((int8_t*)sd)[ly.re[l] + k] = lv.rexp[b0 + k];
      }
    }
  }
  __device__ __noinline__ void store_back(int top, int nrows) const {
    const int tid = WID * 32 + LANE;
    for (int l = 0; l <= top; ++l) {
      const LevelDev& lv = c.lv[l];
      const int nb = (int)lv.g.nblk, nbpc = 1 << ly.lgc[l], b0 = rank * nbpc;
      const int nloc = max(0, min(nb, b0 + nbpc) - b0);
      uint32_t* um = lv.umant + (long long)b0 * lv.ustride;
      uint32_t* rm = lv.rmant + (long long)b0 * lv.rstride;
      for (int i = tid; i < nloc * lv.ustride; i += KC_NT) um[i] = ((uint32_t*)sd)[ly.um[l] + i];
      for (int i = tid; i < nloc * lv.rstride; i += KC_NT) rm[i] = ((uint32_t*)sd)[ly.rm[l] + i];
      for (int k = tid; k < nloc; k += KC_NT) {
        lv.uexp[b0 + k] = ((int8_t*)sd)[ly.ue[l] + k];
        lv.rexp[b0 + k] = ((int8_t*)sd)[ly.re[l] + k];
      }
      // u_l, w_l, t_l of the owned blocks (u_lc, w_lc feed the grid levels)
      const long long e0 = (long long)b0 * 32;
      for (int i = tid; i < nloc * 32; i += KC_NT) {
        lv.U[e0 + i] = sd[ly.U[l] + i];
        lv.W[e0 + i] = sd[ly.W[l] + i];
        lv.T[e0 + i] = sd[ly.T[l] + i];
      }
    }
    // norm partials: table [row - row0][l][warp] -> pbase[((row * levels) + l) * TW + gw]
    const int TW = NC * KC_NW;
    for (int i = tid; i < nrows * (c.lc + 1) * KC_NW; i += KC_NT) {
      int ww = i % KC_NW, l = (i / KC_NW) % (c.lc + 1), rr = i / (KC_NW * (c.lc + 1));
      int row = a.row0 + rr;
      if (l <= row / c.n_ir)  // levels 0..L of that row
        c.pbase[((long long)row * c.levels + l) * TW + rank * KC_NW + ww] = sd[ly.part + i];
    }
  }
};

#undef LANE
#undef WID
#undef SROW
#undef SROWR

template <int D, int P>
__global__ void __launch_bounds__(KC_NT, 1) kc_kernel(const DevCtx* __restrict__ cp, KcDesc a) {
  extern __shared__ __align__(16) double kc_dsm[];
  // The context (level descriptors, operator coefficients, layout) is copied
  // to shared memory once: the cluster barrier's acquire invalidates L1.
  __shared__ __align__(16) unsigned char sctx[sizeof(DevCtx)];
  __shared__ double srq[128];                // dec r_0 at the coarse unknowns (<= 125)
  pdl_wait();
  pdl_trigger();
  {
    const int4* src = (const int4*)cp;
    int4* dst = (int4*)sctx;
    for (int i = threadIdx.y * 32 + threadIdx.x; i < (int)(sizeof(DevCtx) / 16); i += KC_NT) dst[i] = src[i];
    __syncthreads();
  }
  const DevCtx& c = *(const DevCtx*)sctx;
  const KcLayout& ly = c.kc;
  const int NC = 1 << ly.lg;
  const bool dbg = a.debug != 0;
  if (dbg && threadIdx.x == 0 && threadIdx.y == 0 && cl_rank() == 0) g_kc_nstamp = 0;
  // The phase object lives in shared memory: its (non-inlined) phase functions
  // read their state with shared loads, never from the stack.
  __shared__ KcDesc sa;
  __shared__ __align__(16) unsigned char kbuf[sizeof(Kc<D, P>)];
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    sa = a;
    new (kbuf) Kc<D, P>{c, ly, sa, c.cf, kc_dsm, NC, (int)cl_rank(), dbg};
  }
  __syncthreads();
  Kc<D, P>& k = *reinterpret_cast<Kc<D, P>*>(kbuf);
  const int top = (a.mode == 0) ? a.Llast : c.lc;
  k.load_sections(top);
  csync(dbg);  // every CTA's slabs are loaded before any remote read
  if (a.mode == 0) {
    k.ph_coarse_initial();
    csync(dbg);
    for (int L = 1; L <= a.Llast; ++L) {
      const int iters = (L == a.Llast) ? a.iters_last : c.n_ir;
      for (int it = 0; it < iters; ++it) k.iteration(L, it, srq);
    }
  } else {
    k.iteration(a.L, a.it, srq);
  }
  // (the last phase ended with a cluster barrier: no remote reads follow)
  k.store_back(top, a.nrows);
}

// ------------------------------------------------------------------ host --
#define KC_DISPATCH(dim, p, F)                \
  do {                                        \
    if (dim == 2 && p == 1) { F(2, 1); }      \
    else if (dim == 2 && p == 2) { F(2, 2); } \
    else if (dim == 2 && p == 3) { F(2, 3); } \
    else if (dim == 3 && p == 1) { F(3, 1); } \
    else if (dim == 3 && p == 2) { F(3, 2); } \
    else { F(3, 3); }                         \
  } while (0)

template <int D, int P>
static bool kc_fits(int cs, int smem) {
  cudaFuncSetAttribute(kc_kernel<D, P>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(kc_kernel<D, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, KC_SMEM_MAX);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(cs);
  cfg.blockDim = dim3(32, KC_NW);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  cudaError_t e = cudaOccupancyMaxActiveClusters(&n, kc_kernel<D, P>, &cfg);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return n > 0;
}

// Shared-memory layout of KC for cluster size NC = 2^lg and levels 0..lc.
static int kc_layout(int lg, int lc, const Geom* g, const int* ust, const int* rst, int n_ir, KcLayout* ly) {
  const int NC = 1 << lg;
  memset(ly, 0, sizeof(*ly));
  ly->lg = lg;
  long long d = 0;  // doubles
  auto slab = [&](long long nblk) {
    long long o = d;
    d += (32LL << kc_lgc((int)nblk, lg));
    return (int)o;
  };
  for (int l = 0; l <= lc; ++l) ly->lgc[l] = kc_lgc((int)g[l].nblk, lg);
  for (int l = 0; l <= lc; ++l) {
    ly->U[l] = slab(g[l].nblk);
    ly->T[l] = slab(g[l].nblk);
    ly->W[l] = slab(g[l].nblk);
  }
  const long long nb = g[lc].nblk;
  ly->Z = slab(nb);
  ly->B = slab(nb);
  ly->Y0 = slab(nb);
  ly->Y1 = slab(nb);
  ly->Dv = slab(nb);
  ly->PU = slab(nb);
  ly->KS0 = slab(2 * nb);  // 3D restriction staging: (NXc, NYc, NZf) = twice level lc
  ly->KS1 = slab(nb);
  ly->RQ0 = slab(g[0].nblk);
  ly->part = (int)d;
  d += (long long)(lc > 0 ? lc : 1) * n_ir * (lc + 1) * KC_NW;
  long long words = 2 * d;
  for (int l = 0; l <= lc; ++l) {
    long long nloc = 1LL << ly->lgc[l];
    ly->um[l] = (int)words;
    words += nloc * ust[l];
    ly->rm[l] = (int)words;
    words += nloc * rst[l];
  }
  long long bytes = 4 * words;
  for (int l = 0; l <= lc; ++l) {
    long long nloc = 1LL << ly->lgc[l];
    ly->ue[l] = (int)bytes;
    bytes += nloc;
    ly->re[l] = (int)bytes;
    bytes += nloc;
  }
  bytes = (bytes + 15) / 16 * 16;
  ly->bytes = (int)bytes;
  return ly->bytes;
}

int kc_plan(int dim, int p, int Lmax, const Geom* g, const int* ust, const int* rst, int n_ir, int lc_cap,
            KcLayout* ly, int* lc_out, int* cs_out) {
  int forced = 0;
  if (const char* e = getenv("FMG_KC_CLUSTER")) forced = atoi(e);
  int bpw = 1;  // BFP blocks per KC warp at level lc (env FMG_KC_BPW; 2 measured slower on C2)
  if (const char* e = getenv("FMG_KC_BPW")) bpw = std::max(1, atoi(e));
  for (int lg = 4; lg >= 0; --lg) {
    const int cs = 1 << lg;
    if (forced && cs != forced) continue;
    // largest lc with at most one BFP block per KC warp whose layout fits
    int lc = 0;
    for (int l = 1; l <= std::min(Lmax, lc_cap); ++l) {
      if (g[l].nblk > (long long)cs * KC_NW * bpw) break;
      KcLayout t;
      if (kc_layout(lg, l, g, ust, rst, n_ir, &t) > KC_SMEM_MAX) break;
      lc = l;
    }
    int bytes = kc_layout(lg, lc, g, ust, rst, n_ir, ly);
    bool ok = false;
#define F(D, P) ok = kc_fits<D, P>(cs, bytes)
    KC_DISPATCH(dim, p, F);
#undef F
    if (ok) {
      *lc_out = lc;
      *cs_out = cs;
      return 0;
    }
  }
  return -1;
}

int kc_warps_per_cta() { return KC_NW; }

static int g_kc_debug_host = 0;
void kc_debug(int on) { g_kc_debug_host = on; }
int kc_stamps(unsigned long long* out) {
  int n = 0;
  cudaMemcpyFromSymbol(&n, g_kc_nstamp, sizeof(int));
  cudaMemcpyFromSymbol(out, g_kc_stamps, sizeof(unsigned long long) * 256);
  return n;
}

void launch_kc(int dim, int p, cudaStream_t st, const void* devctx, const KcDesc& a, int cluster, int smem) {
  const DevCtx* c = (const DevCtx*)devctx;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(cluster);
  cfg.blockDim = dim3(32, KC_NW);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cluster;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  KcDesc ad = a;
  ad.debug = g_kc_debug_host;
#define F(D, P) cudaLaunchKernelEx(&cfg, kc_kernel<D, P>, c, ad)
  KC_DISPATCH(dim, p, F);
#undef F
}

}  // namespace fmg
