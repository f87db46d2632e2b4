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
#include "fmg_device.cuh"

namespace fmg {

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
  double* out = c.lv[op.l].U;
  double* box = sm;  // DBX x DBY x DBZ
  if (op.l > 0) {
    double* cb = box + PL::DBX * PL::DBY * PL::DBZ;
    double* v1 = cb + PL::DCBX * PL::DCBY * PL::DCBZ;
    double* v2 = v1 + PL::DBX * PL::DCBY * PL::DCBZ;
    box_prolong<D, P, PL::DBX, PL::DBY, PL::DBZ, PL::DCBX, PL::DCBY, PL::DCBZ>(
        c.lv[op.l - 1].U, c.lv[op.l - 1].g, g.n, x0, y0, z0, c.cf, cb, v1, v2, box);
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
  box_async<D, P>(c.lv[op.L].U, g, x0, y0, z0, U);
  cpa_wait_sync();
  double* AB = R1;
  double* CS = R1 + 2 * PL::NAB;
  a_stages<D, P>(g, x0, y0, c.cf, U, AB, CS);
  const int lane = threadIdx.x;
  double* T = c.lv[op.L].T;
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
  const double* __restrict__ Tf = c.lv[op.l + 1].T;
  double* Tc = c.lv[op.l].T;
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
  if (op.l < op.L) c.lv[op.l].W[idx] = zc + yq;
  long long blk = idx >> 5;
  double uo = warp_decode(uw_s, lv.uexp[blk], op.wu_in, lane);
  double uq = warp_encode(uo + yq, op.wu_out, lv.umant + blk * lv.ustride, lv.uexp + blk, lane, c.status);
  c.lv[op.l].U[idx] = uq + pu;
}

// P_l u_{l-1} on the output tile (for the emitted u_l): coarse box issue
// (async) and the prolongation passes (after the wait).
template <int D, int P>
__device__ void tile_pu_issue(const DevCtx& c, int l, int x0, int y0, int z0, double* scratch) {
  using PL = Plan<D, P>;
  cbox_async<D, P, PL::DCBX, PL::DCBY, PL::DCBZ>(c.lv[l - 1].U, c.lv[l - 1].g, x0, y0, z0, scratch);
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
  cbox_async<D, P, PL::CBX, PL::CBY, PL::CBZ>(c.lv[op.l - 1].W, c.lv[op.l - 1].g, x0 - P, y0 - P, z0 - P, cb);
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

template <int D, int P, int T>
__device__ __forceinline__ void run_op(const DevCtx& c, const Op& op, const TileIdx& tile, double* sm) {
  if constexpr (T == OP_DECODE) tile_decode<D, P>(c, op, tile, sm);
  else if constexpr (T == OP_RESIDUAL) tile_residual<D, P>(c, op, tile, sm);
  else if constexpr (T == OP_RESTRICT) tile_restrict<D, P>(c, op, tile, sm);
  else if constexpr (T == OP_NORMS) op_norms(c, op, sm);
  else if constexpr (T == OP_CFAS1) tile_cfas1<D, P>(c, op, tile, sm);
  else tile_cheb<D, P>(c, op, tile, sm);
}

// Grid kernel: one CTA per tile of one operation; one kernel per operation
// type T, so a launch only pulls its own code into the instruction caches.
// The device context lives in global memory (uniform, L1-cached).
#ifndef FMG_KOP_MINB
#define FMG_KOP_MINB 4
#endif
template <int D, int P, int T>
__global__ void __launch_bounds__(NT, FMG_KOP_MINB) k_op(const DevCtx* __restrict__ cp, Op op) {
  extern __shared__ double sm[];
  pdl_wait();
  pdl_trigger();
  const DevCtx& c = *cp;
  TileIdx t{(int)blockIdx.x, (int)blockIdx.y, (int)blockIdx.z,
            (int)((blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x)};
  run_op<D, P, T>(c, op, t, sm);
}

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
  // squared norm: the host takes the root (after summing the z-slab partials of all ranks)
  if (threadIdx.x == 0) c.norms[(long long)e.row * c.levels + e.l] = red[0];
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

// Thread-per-block codec kernels (w <= 32): a warp stages 32 blocks (8 KB) in
// shared memory with cp.async, one lane per block encodes / decodes, and the
// packed words leave through a coalesced copy.
constexpr int TPB_RS = 33;        // row stride (doubles)
constexpr int TPB_WS = 33;        // packed row stride (words), >= w + 1
constexpr int TPB_WARPS = 4;
constexpr int TPB_SMEM = TPB_WARPS * (32 * TPB_RS * 8 + 32 * TPB_WS * 4);

__global__ void __launch_bounds__(TPB_WARPS * 32) k_bfp_encode_tpb(const double* __restrict__ x, long long nblk,
                                                                   int w, uint32_t* __restrict__ mant,
                                                                   int8_t* __restrict__ exps, int* status) {
  extern __shared__ __align__(16) unsigned char tpb_smem[];
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  double* tile = (double*)tpb_smem + wp * 32 * TPB_RS;
  uint32_t* wt = (uint32_t*)((double*)tpb_smem + TPB_WARPS * 32 * TPB_RS) + wp * 32 * TPB_WS;
  const unsigned magic = (unsigned)((0x100000000ULL + w - 1) / w);  // t / w for t < 2^16
  const long long ntile = (nblk + 31) / 32;
  const long long wg = (long long)blockIdx.x * TPB_WARPS + wp, nw = (long long)gridDim.x * TPB_WARPS;
  bool bad = false;
  for (long long t = wg; t < ntile; t += nw) {
    const long long b0 = t * 32;
    const int nb = (int)(nblk - b0 < 32 ? nblk - b0 : 32);
#pragma unroll 8
    for (int r = 0; r < 32; ++r) cpa8(tile + r * TPB_RS + lane, x + (b0 + r) * 32 + lane, r < nb);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncwarp();
    const double* row = tile + lane * TPB_RS;
    const int E = tpb_exponent(row, w, bad);
    tpb_pack(row, E, w, wt + lane * TPB_WS, nullptr);
    if (lane < nb) exps[b0 + lane] = (int8_t)E;
    __syncwarp();
    const int nwords = nb * w;
    uint32_t* dst = mant + b0 * w;
    for (int o = lane; o < nwords; o += 32) {
      const int j = (int)__umulhi((unsigned)o, magic);
      dst[o] = wt[j * TPB_WS + (o - j * w)];
    }
    __syncwarp();
  }
  if (__any_sync(FULL, bad) && lane == 0) atomicOr(status, 1);
}

__global__ void __launch_bounds__(TPB_WARPS * 32) k_bfp_decode_tpb(const uint32_t* __restrict__ mant,
                                                                   const int8_t* __restrict__ exps, long long nblk,
                                                                   int w, double* __restrict__ x) {
  extern __shared__ __align__(16) unsigned char tpb_smem[];
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  double* tile = (double*)tpb_smem + wp * 32 * TPB_RS;
  uint32_t* wt = (uint32_t*)((double*)tpb_smem + TPB_WARPS * 32 * TPB_RS) + wp * 32 * TPB_WS;
  const unsigned magic = (unsigned)((0x100000000ULL + w - 1) / w);
  const long long ntile = (nblk + 31) / 32;
  const long long wg = (long long)blockIdx.x * TPB_WARPS + wp, nw = (long long)gridDim.x * TPB_WARPS;
  for (long long t = wg; t < ntile; t += nw) {
    const long long b0 = t * 32;
    const int nb = (int)(nblk - b0 < 32 ? nblk - b0 : 32);
    const int nwords = nb * w;
    const uint32_t* src = mant + b0 * w;
    for (int o = lane; o < nwords; o += 32) {  // all copies in flight (LDGSTS)
      const int j = (int)__umulhi((unsigned)o, magic);
      cpa4(wt + j * TPB_WS + (o - j * w), src + o);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    const int E = lane < nb ? (int)exps[b0 + lane] : -128;
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncwarp();
    tpb_unpack(wt + lane * TPB_WS, E, w, tile + lane * TPB_RS);
    __syncwarp();
#pragma unroll 8
    for (int r = 0; r < 32; ++r)
      if (r < nb) __stcs(x + (b0 + r) * 32 + lane, tile[r * TPB_RS + lane]);
    __syncwarp();
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
#define SETA(D, P)                                                                                        \
  cudaFuncSetAttribute(k_op<D, P, OP_DECODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, Plan<D, P>::SMEM);   \
  cudaFuncSetAttribute(k_op<D, P, OP_RESIDUAL>, cudaFuncAttributeMaxDynamicSharedMemorySize, Plan<D, P>::SMEM); \
  cudaFuncSetAttribute(k_op<D, P, OP_RESTRICT>, cudaFuncAttributeMaxDynamicSharedMemorySize, Plan<D, P>::SMEM); \
  cudaFuncSetAttribute(k_op<D, P, OP_CFAS1>, cudaFuncAttributeMaxDynamicSharedMemorySize, Plan<D, P>::SMEM);    \
  cudaFuncSetAttribute(k_op<D, P, OP_CHEB>, cudaFuncAttributeMaxDynamicSharedMemorySize, Plan<D, P>::SMEM);
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
#define LT(D, P, T) launch_pdl(k_op<D, P, T>, dim3(tx, ty, tz), Plan<D, P>::SMEM, st, c, op)
#define F(D, P)                                            \
  do {                                                     \
    switch (op.type) {                                     \
      case OP_DECODE: LT(D, P, OP_DECODE); break;          \
      case OP_RESIDUAL: LT(D, P, OP_RESIDUAL); break;      \
      case OP_RESTRICT: LT(D, P, OP_RESTRICT); break;      \
      case OP_CFAS1: LT(D, P, OP_CFAS1); break;            \
      default: LT(D, P, OP_CHEB); break;                   \
    }                                                      \
  } while (0)
  FMG_DISPATCH(dim, p, F);
#undef F
#undef LT
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
    lv.U = d.Ul[l];
    lv.T = d.Tl[l];
    lv.W = d.Wl[l];
  }
  for (int i = 0; i < 2; ++i) c->Y[i] = d.Y[i];
  c->pbase = d.pbase;
  c->lc = d.lc;
  c->n_cheb = d.n_cheb;
  c->smoother = d.smoother;
  c->Z = d.Z;
  c->PU = d.PU;
  c->KS[0] = d.KS[0];
  c->KS[1] = d.KS[1];
  c->kc = d.kc;
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
  if (w <= 32) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_bfp_encode_tpb, cudaFuncAttributeMaxDynamicSharedMemorySize, TPB_SMEM);
      cudaFuncSetAttribute(k_bfp_decode_tpb, cudaFuncAttributeMaxDynamicSharedMemorySize, TPB_SMEM);
      attr = true;
    }
    long long want = (nblk + 32 * TPB_WARPS - 1) / (32 * TPB_WARPS);
    int grid = (int)(want < (long long)num_sms() * 3 ? (want > 0 ? want : 1) : num_sms() * 3);
    k_bfp_encode_tpb<<<grid, TPB_WARPS * 32, TPB_SMEM, st>>>(x, nblk, w, mant, exps, status);
    return;
  }
  long long want = (nblk + 7) / 8;
  int grid = (int)(want < (long long)num_sms() * 16 ? (want > 0 ? want : 1) : num_sms() * 16);
  k_bfp_encode<<<grid, 256, 0, st>>>(x, nblk, w, mant, exps, status);
}

void launch_bfp_decode(const uint32_t* mant, const int8_t* exps, long long n, int w, double* x, cudaStream_t st) {
  long long nblk = n / 32;
  if (w <= 32) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_bfp_encode_tpb, cudaFuncAttributeMaxDynamicSharedMemorySize, TPB_SMEM);
      cudaFuncSetAttribute(k_bfp_decode_tpb, cudaFuncAttributeMaxDynamicSharedMemorySize, TPB_SMEM);
      attr = true;
    }
    long long want = (nblk + 32 * TPB_WARPS - 1) / (32 * TPB_WARPS);
    int grid = (int)(want < (long long)num_sms() * 3 ? (want > 0 ? want : 1) : num_sms() * 3);
    k_bfp_decode_tpb<<<grid, TPB_WARPS * 32, TPB_SMEM, st>>>(mant, exps, nblk, w, x);
    return;
  }
  long long want = (nblk + 7) / 8;
  int grid = (int)(want < (long long)num_sms() * 16 ? (want > 0 ? want : 1) : num_sms() * 16);
  k_bfp_decode<<<grid, 256, 0, st>>>(mant, exps, nblk, w, x);
}

}  // namespace fmg
