// fmg_kernels.cu -- sm_100a kernels of the compact-FMG hot path.
//
// Every floating-point expression follows the canonical evaluation order of
// DESIGN.md §3 with explicit fma(); the file is compiled with -fmad=false so no
// other contraction happens.  Tensor-product operators are applied factor by
// factor (sum factorisation) on shared-memory tiles: x pass, then y, then z.
//
// Paper passages: BFP codec PAPER.md:1240-1274 with RNE; decode
// sweep / residual / truncate / restriction of fmgResidual (Alg 3.2,
// PAPER.md:713-748); cFas coarse-to-fine sweep (Alg 3.1, nu = 1
// so s = 0) fused with the correction (Alg 3.3).
#include <cstdint>
#include <cstdio>

#include "fmg_internal.h"

namespace fmg {

constexpr unsigned FULL = 0xffffffffu;
constexpr int NWARP = 8;  // warps per CTA of every tiled kernel

// Exact 2^k for k in [-1022, 1023].
__device__ __forceinline__ double pow2(int k) {
  return __longlong_as_double((long long)(k + 1023) << 52);
}

// ----------------------------------------------------------------- codec --
// Warp-cooperative decode: lane j returns entry j of the block whose `w` words
// start at `words`.  Must be called by all 32 lanes.
__device__ __forceinline__ double warp_decode(const uint32_t* __restrict__ words, int E, int w, int lane) {
  uint32_t my0 = lane < w ? __ldg(words + lane) : 0u;
  uint32_t my1 = 0u;
  if (w > 32) my1 = lane + 32 < w ? __ldg(words + lane + 32) : 0u;
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
  long long m = (long long)(field << (64 - w)) >> (64 - w);  // sign-extend w bits
  return (double)m * pow2(E - (w - 1));
}

// Warp-cooperative encode of one 32-entry block (R8); lane j holds
// entry j.  Writes the w words and the exponent (if `words` is non-null) and
// returns the quantised value m 2^(E-q) of this lane's entry.  Non-finite input
// or E > 127 sets *status (FMG_ERANGE) and stores a zero block.
__device__ __forceinline__ double warp_encode(double v, int w, uint32_t* __restrict__ words,
                                              int8_t* __restrict__ eptr, int lane, int* status) {
  unsigned long long bits = (unsigned long long)__double_as_longlong(v) & 0x7fffffffffffffffULL;
  bool bad = bits >= 0x7ff0000000000000ULL;
  unsigned hi = (unsigned)(bits >> 32), lo = (unsigned)bits;
  unsigned mh = __reduce_max_sync(FULL, hi);
  unsigned ml = __reduce_max_sync(FULL, hi == mh ? lo : 0u);
  bool err = __any_sync(FULL, bad);
  double mx = __longlong_as_double((long long)(((unsigned long long)mh << 32) | ml));
  int q = w - 1, E = -128;
  if (!err && mx != 0.0) {
    int E0 = ilogb(mx) + 1;
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
    m = (long long)rint(v * pow2(q - E));
  }
  if (words) {
    unsigned long long field = (unsigned long long)m & ((1ULL << w) - 1ULL);
    int o = lane * w;
    uint32_t mine0 = 0u, mine1 = 0u;
    for (int j = 0; j < w; ++j) {
      int s = o - 32 * j;
      uint32_t c = 0u;
      if (s > -w && s < 32) c = s >= 0 ? (uint32_t)(field << s) : (uint32_t)(field >> (-s));
      uint32_t word = __reduce_or_sync(FULL, c);
      if (j < 32) {
        if (lane == j) mine0 = word;
      } else if (lane == j - 32) {
        mine1 = word;
      }
    }
    if (lane < w) words[lane] = mine0;
    if (lane + 32 < w) words[lane + 32] = mine1;
    if (lane == 0) *eptr = (int8_t)E;
  }
  return E == -128 ? 0.0 : (double)m * pow2(E - q);
}

// --------------------------------------------------------------- tiles ----
template <int D, int P> struct TileCfg;
template <int P> struct TileCfg<2, P> { static constexpr int TY = 16, TZ = 1; };
template <> struct TileCfg<3, 1> { static constexpr int TY = 8, TZ = 4; };
template <> struct TileCfg<3, 2> { static constexpr int TY = 4, TZ = 4; };
template <> struct TileCfg<3, 3> { static constexpr int TY = 4, TZ = 4; };

// Shared-memory plan of the A-apply tile (output 32 x TY x TZ).
template <int D, int P> struct ATile {
  static constexpr int TY = TileCfg<D, P>::TY, TZ = TileCfg<D, P>::TZ;
  static constexpr int BX = 32 + 2 * P, BY = TY + 2 * P, BZ = (D == 3) ? TZ + 2 * P : 1;
  static constexpr int NU = BX * BY * BZ;          // input box
  static constexpr int NAB = 32 * BY * BZ;         // x-pass outputs a = Mx u, b = Kx u
  static constexpr int NCS = (D == 3) ? 32 * TY * BZ : 0;  // y-pass outputs c, s
  static constexpr int SMEM = (NU + 2 * NAB + 2 * NCS) * 8;
};

// Shared-memory plan of the restriction tile (coarse output 32 x TY x TZ).
template <int D, int P> struct RTile {
  static constexpr int TY = TileCfg<D, P>::TY, TZ = TileCfg<D, P>::TZ;
  static constexpr int FBY = 2 * TY + 4 * P - 3, FBZ = (D == 3) ? 2 * TZ + 4 * P - 3 : 1;
  static constexpr int NX = 32 * FBY * FBZ;         // x-pass outputs
  static constexpr int NYR = (D == 3) ? 32 * TY * FBZ : 0;  // y-pass outputs
  static constexpr int SMEM = (NX + NYR) * 8;
};

__device__ __forceinline__ bool unk1(int i, int n) { return i >= 1 && i <= n - 1; }

// Stages of A applied to the box around output tile (x0,y0,z0) of `src`
// (DESIGN.md §3.2): load u, x pass (a = Mx u, b = Kx u), y pass (3D: c = My a,
// s = Ky a + My b).  The last pass is done per output point by atile_final.
template <int D, int P>
__device__ void atile_stages(const double* __restrict__ src, const Geom& g, int x0, int y0, int z0,
                             const Coefs& cf, double* sm) {
  using T = ATile<D, P>;
  double* U = sm;
  double* A = U + T::NU;
  double* B = A + T::NAB;
  double* C = B + T::NAB;
  double* S = C + T::NCS;
  const int tid = threadIdx.y * 32 + threadIdx.x, nt = 32 * NWARP;
  for (int i = tid; i < T::NU; i += nt) {
    int bx = i % T::BX, r = i / T::BX, by = r % T::BY, bz = r / T::BY;
    int gx = x0 - P + bx, gy = y0 - P + by, gz = (D == 3) ? z0 - P + bz : 0;
    double v = 0.0;
    if (gx >= 0 && gx < g.NX && gy >= 0 && gy < g.NY && gz >= 0 && gz < g.NZ)
      v = src[((long long)gz * g.NY + gy) * g.NX + gx];
    U[i] = v;
  }
  __syncthreads();
  for (int i = tid; i < T::NAB; i += nt) {
    int lx = i & 31, r = i >> 5;
    int gx = x0 + lx;
    double a = 0.0, b = 0.0;
    if (unk1(gx, g.n)) {
      int tau = gx % P;
      const double* u = U + r * T::BX + lx;
#pragma unroll
      for (int o = 0; o <= 2 * P; ++o) {
        a = fma(cf.Mc[tau][o], u[o], a);
        b = fma(cf.Kc[tau][o], u[o], b);
      }
    }
    A[i] = a;
    B[i] = b;
  }
  __syncthreads();
  if constexpr (D == 3) {
    for (int i = tid; i < T::NCS; i += nt) {
      int lx = i & 31, r = i >> 5, ty = r % T::TY, bz = r / T::TY;
      int gy = y0 + ty;
      double c = 0.0, s = 0.0;
      if (unk1(gy, g.n)) {
        int tau = gy % P;
        const double* a = A + (bz * T::BY + ty) * 32 + lx;
        const double* b = B + (bz * T::BY + ty) * 32 + lx;
        double dd = 0.0, e = 0.0;
#pragma unroll
        for (int o = 0; o <= 2 * P; ++o) {
          c = fma(cf.Mc[tau][o], a[o * 32], c);
          dd = fma(cf.Kc[tau][o], a[o * 32], dd);
          e = fma(cf.Mc[tau][o], b[o * 32], e);
        }
        s = dd + e;
      }
      C[i] = c;
      S[i] = s;
    }
    __syncthreads();
  }
}

// Last pass of A at output (x0+lx, y0+ty, z0+tz): 2D  s = Ky a + My b;
// 3D  h * (Kz c + Mz s) as one fma chain.  0 at non-unknowns.
template <int D, int P>
__device__ __forceinline__ double atile_final(const double* sm, const Geom& g, int x0, int y0, int z0,
                                              int lx, int ty, int tz, const Coefs& cf) {
  using T = ATile<D, P>;
  const double* A = sm + T::NU;
  const double* B = A + T::NAB;
  const double* C = B + T::NAB;
  const double* S = C + T::NCS;
  int gx = x0 + lx, gy = y0 + ty, gz = z0 + tz;
  if (!unk1(gx, g.n) || !unk1(gy, g.n) || (D == 3 && !unk1(gz, g.n))) return 0.0;
  if constexpr (D == 2) {
    int tau = gy % P;
    double d = 0.0, e = 0.0;
#pragma unroll
    for (int o = 0; o <= 2 * P; ++o) {
      d = fma(cf.Kc[tau][o], A[(ty + o) * 32 + lx], d);
      e = fma(cf.Mc[tau][o], B[(ty + o) * 32 + lx], e);
    }
    return d + e;
  } else {
    int tau = gz % P;
    double acc = 0.0;
#pragma unroll
    for (int o = 0; o <= 2 * P; ++o) acc = fma(cf.Kc[tau][o], C[((tz + o) * T::TY + ty) * 32 + lx], acc);
#pragma unroll
    for (int o = 0; o <= 2 * P; ++o) acc = fma(cf.Mc[tau][o], S[((tz + o) * T::TY + ty) * 32 + lx], acc);
    return acc * pow2(-(g.l + 1));
  }
}

// Deterministic CTA sum of one double per thread -> partials[cta].
__device__ __forceinline__ void cta_sum(double v, double* out) {
  __shared__ double red[NWARP];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  if (threadIdx.x == 0) red[threadIdx.y] = v;
  __syncthreads();
  if (threadIdx.x == 0 && threadIdx.y == 0) {
    double s = 0.0;
    for (int i = 0; i < NWARP; ++i) s += red[i];
    *out = s;
  }
}

__device__ __forceinline__ long long cta_linear() {
  return ((long long)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
}

// ------------------------------------------------------- prolong/decode ----
// out_l = dec(section) + P_l coarse  (decode sweep PAPER.md:733-735 when both
// are given; z_l = P_l w_{l-1} with no section).  One warp per
// 32-entry x block; P evaluated per fine point in the canonical x, y, z order.
template <int D, int P>
__global__ void __launch_bounds__(256) k_prolong_decode(double* __restrict__ out, Geom gf,
                                                        const double* __restrict__ coarse, Geom gc,
                                                        const uint32_t* __restrict__ mant,
                                                        const int8_t* __restrict__ exps, int w, int stride,
                                                        Coefs cf) {
  const int lane = threadIdx.x;
  const int nxb = gf.NX >> 5;
  long long row = (long long)blockIdx.x * NWARP + threadIdx.y;
  if (row >= (long long)gf.NY * gf.NZ * nxb) return;
  int xb = (int)(row % nxb);
  long long yz = row / nxb;
  int y = (int)(yz % gf.NY), z = (int)(yz / gf.NY);
  int x = xb * 32 + lane;
  long long idx = ((long long)z * gf.NY + y) * gf.NX + x;
  double val = 0.0;
  bool unk = unk1(x, gf.n) && unk1(y, gf.n) && (D == 2 || unk1(z, gf.n));
  if (coarse != nullptr && unk) {
    const int nc = gc.n;
    int rx = x % (2 * P), bx = P * (x / (2 * P));
    int ry = y % (2 * P), by = P * (y / (2 * P));
    auto xpass = [&](int cy, int cz) -> double {  // v1 = Px v at (x, cy, cz)
      const double* row_ = coarse + ((long long)cz * gc.NY + cy) * gc.NX;
      double acc = 0.0;
#pragma unroll
      for (int t = 0; t <= P; ++t) {
        int cx = bx + t;
        double v = unk1(cx, nc) ? __ldg(row_ + cx) : 0.0;
        acc = fma(cf.Pw[rx][t], v, acc);
      }
      return acc;
    };
    auto ypass = [&](int cz) -> double {  // v2 = Py v1 at (x, y, cz)
      double acc = 0.0;
#pragma unroll
      for (int t = 0; t <= P; ++t) {
        int cy = by + t;
        double v = unk1(cy, nc) ? xpass(cy, cz) : 0.0;
        acc = fma(cf.Pw[ry][t], v, acc);
      }
      return acc;
    };
    if constexpr (D == 2) {
      val = ypass(0);
    } else {
      int rz = z % (2 * P), bz = P * (z / (2 * P));
      double acc = 0.0;
#pragma unroll
      for (int t = 0; t <= P; ++t) {
        int cz = bz + t;
        double v = unk1(cz, nc) ? ypass(cz) : 0.0;
        acc = fma(cf.Pw[rz][t], v, acc);
      }
      val = acc;
    }
  }
  if (mant != nullptr) {
    long long blk = idx >> 5;
    double dv = warp_decode(mant + blk * stride, exps[blk], w, lane);
    val = dv + val;
  }
  out[idx] = val;
}

// ---------------------------------------------------------- residual -------
// t_L = f_L - A_L u_L, r_L = enc(t_L), ||t_L||^2.
template <int D, int P>
__global__ void __launch_bounds__(256) k_residual(const double* __restrict__ U, double* __restrict__ T, Geom g,
                                                  const double* __restrict__ gtab, Sec r, int wr,
                                                  double* __restrict__ partials, Coefs cf, int* status) {
  extern __shared__ double sm[];
  using TT = ATile<D, P>;
  const int x0 = blockIdx.x * 32, y0 = blockIdx.y * TT::TY, z0 = blockIdx.z * TT::TZ;
  atile_stages<D, P>(U, g, x0, y0, z0, cf, sm);
  const int lane = threadIdx.x;
  double ss = 0.0;
  for (int row = threadIdx.y; row < TT::TY * TT::TZ; row += NWARP) {
    int ty = row % TT::TY, tz = row / TT::TY;
    int y = y0 + ty, z = z0 + tz;
    if (y >= g.NY || z >= g.NZ) continue;
    double au = atile_final<D, P>(sm, g, x0, y0, z0, lane, ty, tz, cf);
    int x = x0 + lane;
    bool unk = unk1(x, g.n) && unk1(y, g.n) && (D == 2 || unk1(z, g.n));
    double t = 0.0;
    if (unk) {
      double f = cf.rhs_c * __ldg(gtab + x);
      f = f * __ldg(gtab + y);
      if (D == 3) f = f * __ldg(gtab + z);
      t = f - au;
    }
    long long idx = ((long long)z * g.NY + y) * g.NX + x;
    T[idx] = t;
    ss = fma(t, t, ss);
    long long blk = idx >> 5;
    warp_encode(t, wr, r.mant + blk * r.stride, r.exps + blk, lane, status);
  }
  cta_sum(ss, partials + cta_linear());
}

// -------------------------------------------------------- restriction ------
// t_l = R_{l+1} t_{l+1} (restricts t, not r), r_l = enc(t_l).
template <int D, int P>
__global__ void __launch_bounds__(256) k_restrict(const double* __restrict__ Tf, Geom gf, double* __restrict__ Tc,
                                                  Geom gc, Sec r, int wr, double* __restrict__ partials,
                                                  Coefs cf, int* status) {
  extern __shared__ double sm[];
  using RT = RTile<D, P>;
  double* XR = sm;
  double* YR = sm + RT::NX;
  const int x0 = blockIdx.x * 32, y0 = blockIdx.y * RT::TY, z0 = blockIdx.z * RT::TZ;
  const int tid = threadIdx.y * 32 + threadIdx.x, nt = 32 * NWARP;
  const int nf = gf.n, nc = gc.n;
  for (int i = tid; i < RT::NX; i += nt) {
    int lx = i & 31, rr = i >> 5, by = rr % RT::FBY, bz = rr / RT::FBY;
    int fy = 2 * y0 - (2 * P - 1) + by;
    int fz = (D == 3) ? 2 * z0 - (2 * P - 1) + bz : 0;
    int cx = x0 + lx;
    double v = 0.0;
    if (unk1(cx, nc) && fy >= 0 && fy < gf.NY && fz >= 0 && fz < gf.NZ) {
      int tau = cx % P, fx0 = 2 * cx - (2 * P - 1);
      const double* rowp = Tf + ((long long)fz * gf.NY + fy) * gf.NX;
#pragma unroll
      for (int s = 0; s <= 4 * P - 2; ++s) {
        int fx = fx0 + s;
        double t = unk1(fx, nf) ? __ldg(rowp + fx) : 0.0;
        v = fma(cf.Rw[tau][s], t, v);
      }
    }
    XR[i] = v;
  }
  __syncthreads();
  if constexpr (D == 3) {
    for (int i = tid; i < RT::NYR; i += nt) {
      int lx = i & 31, rr = i >> 5, ty = rr % RT::TY, bz = rr / RT::TY;
      int cy = y0 + ty;
      double v = 0.0;
      if (unk1(cy, nc)) {
        int tau = cy % P;
        const double* xr = XR + (bz * RT::FBY + 2 * ty) * 32 + lx;
#pragma unroll
        for (int s = 0; s <= 4 * P - 2; ++s) v = fma(cf.Rw[tau][s], xr[s * 32], v);
      }
      YR[i] = v;
    }
    __syncthreads();
  }
  const int lane = threadIdx.x;
  double ss = 0.0;
  for (int row = threadIdx.y; row < RT::TY * RT::TZ; row += NWARP) {
    int ty = row % RT::TY, tz = row / RT::TY;
    int y = y0 + ty, z = z0 + tz, x = x0 + lane;
    if (y >= gc.NY || z >= gc.NZ) continue;
    double t = 0.0;
    if (unk1(x, nc) && unk1(y, nc) && (D == 2 || unk1(z, nc))) {
      if constexpr (D == 2) {
        int tau = y % P;
#pragma unroll
        for (int s = 0; s <= 4 * P - 2; ++s) t = fma(cf.Rw[tau][s], XR[(2 * ty + s) * 32 + lane], t);
      } else {
        int tau = z % P;
#pragma unroll
        for (int s = 0; s <= 4 * P - 2; ++s) t = fma(cf.Rw[tau][s], YR[((2 * tz + s) * RT::TY + ty) * 32 + lane], t);
      }
    }
    long long idx = ((long long)z * gc.NY + y) * gc.NX + x;
    Tc[idx] = t;
    ss = fma(t, t, ss);
    long long blk = idx >> 5;
    warp_encode(t, wr, r.mant + blk * r.stride, r.exps + blk, lane, status);
  }
  cta_sum(ss, partials + cta_linear());
}

// --------------------------------------------------------- coarse level ----
// mode 0: ú_0 = enc_{wu_out}(A_0^{-1} f_0)
// mode 1: ý_0 = enc_{wr}(A_0^{-1} dec r_0), W_0 = dec ý_0,
//         ú_0 <- enc_{wu_out}(dec_{wu_in} ú_0 + dec ý_0)
// Canonical mat-vec: acc = 0; acc = fma(Ainv[I][J], x_J, acc), J in unknown order.
template <int D, int P>
__global__ void __launch_bounds__(256) k_coarse(int mode, Geom g, const double* __restrict__ gtab,
                                                const double* __restrict__ Ainv, int n0, Sec u, int wu_in,
                                                int wu_out, Sec r, int wr, double* __restrict__ W0,
                                                Coefs cf, int* status) {
  constexpr int n = 2 * P, m = 2 * P - 1;
  constexpr int ROWS = (D == 3) ? n * n : n;
  __shared__ double X[ROWS * 32], Y[ROWS * 32];
  const int lane = threadIdx.x, tid = threadIdx.y * 32 + threadIdx.x;
  for (int row = threadIdx.y; row < ROWS; row += NWARP) {
    int y = row % n, z = row / n;
    double v;
    if (mode == 0) {
      bool unk = unk1(lane, n) && unk1(y, n) && (D == 2 || unk1(z, n));
      v = 0.0;
      if (unk) {
        v = cf.rhs_c * gtab[lane];
        v = v * gtab[y];
        if (D == 3) v = v * gtab[z];
      }
    } else {
      v = warp_decode(r.mant + (long long)row * r.stride, r.exps[row], wr, lane);
    }
    X[row * 32 + lane] = v;
    Y[row * 32 + lane] = 0.0;
  }
  __syncthreads();
  for (int I = tid; I < n0; I += 32 * NWARP) {
    double acc = 0.0;
    for (int J = 0; J < n0; ++J) {
      int jx = J % m + 1, jy = (J / m) % m + 1, jz = (D == 3) ? J / (m * m) + 1 : 0;
      acc = fma(Ainv[(long long)I * n0 + J], X[(jz * n + jy) * 32 + jx], acc);
    }
    int ix = I % m + 1, iy = (I / m) % m + 1, iz = (D == 3) ? I / (m * m) + 1 : 0;
    Y[(iz * n + iy) * 32 + ix] = acc;
  }
  __syncthreads();
  for (int row = threadIdx.y; row < ROWS; row += NWARP) {
    double y = Y[row * 32 + lane];
    uint32_t* uw = u.mant + (long long)row * u.stride;
    if (mode == 0) {
      warp_encode(y, wu_out, uw, u.exps + row, lane, status);
    } else {
      double yq = warp_encode(y, wr, nullptr, nullptr, lane, status);
      W0[row * 32 + lane] = yq;
      double uo = warp_decode(uw, u.exps[row], wu_in, lane);
      warp_encode(uo + yq, wu_out, uw, u.exps + row, lane, status);
    }
  }
}

// ------------------------------------------------------------ cFas level --
// Level l of the coarse-to-fine sweep with Chebyshev-Jacobi
// (DESIGN.md §3.5).  step 1: b = dec r_l - A_l z_l, d = inv_theta (invD b), y = d.
// step j >= 2: q = b - A y, d = fma(alpha_j, d, beta_j (invD q)), y = y + d.
// last step: ý = enc_{wr}(y); W_l = z_l + dec ý; ú_l <- enc_{wu_out}(dec ú_l + dec ý).
template <int D, int P>
__global__ void __launch_bounds__(256) k_cfas_step(Geom g, CfasArgs a, Coefs cf, int* status) {
  extern __shared__ double sm[];
  using TT = ATile<D, P>;
  const int x0 = blockIdx.x * 32, y0 = blockIdx.y * TT::TY, z0 = blockIdx.z * TT::TZ;
  atile_stages<D, P>(a.step == 1 ? a.Z : a.Yin, g, x0, y0, z0, cf, sm);
  const int lane = threadIdx.x;
  const double dsc = pow2((g.l + 1) * (D - 2));
  for (int row = threadIdx.y; row < TT::TY * TT::TZ; row += NWARP) {
    int ty = row % TT::TY, tz = row / TT::TY;
    int y = y0 + ty, z = z0 + tz, x = x0 + lane;
    if (y >= g.NY || z >= g.NZ) continue;
    double au = atile_final<D, P>(sm, g, x0, y0, z0, lane, ty, tz, cf);
    bool unk = unk1(x, g.n) && unk1(y, g.n) && (D == 2 || unk1(z, g.n));
    long long idx = ((long long)z * g.NY + y) * g.NX + x;
    long long blk = idx >> 5;
    double invD = 0.0;
    if (unk) invD = cf.invd[((D == 3 ? z % P : 0) * P + y % P) * P + x % P] * dsc;
    double d, yv, b = 0.0;
    if (a.step == 1) {
      double rv = warp_decode(a.r.mant + blk * a.r.stride, a.r.exps[blk], a.wr, lane);
      b = rv - au;
      d = cf.inv_theta * (invD * b);
      yv = d;
    } else {
      b = a.B[idx];
      double q = b - au;
      d = fma(cf.cal[a.step - 1], a.Dv[idx], cf.cbe[a.step - 1] * (invD * q));
      yv = a.Yin[idx] + d;
    }
    if (!a.last) {
      if (a.step == 1) a.B[idx] = b;
      a.Yout[idx] = yv;
      a.Dv[idx] = d;
    } else {
      double yq = warp_encode(yv, a.wr, nullptr, nullptr, lane, status);
      if (a.W) a.W[idx] = a.Z[idx] + yq;
      uint32_t* uw = a.u.mant + blk * a.u.stride;
      double uo = warp_decode(uw, a.u.exps[blk], a.wu_in, lane);
      warp_encode(uo + yq, a.wu_out, uw, a.u.exps + blk, lane, status);
    }
  }
}

// --------------------------------------------------------------- norms ----
struct NormArgs {
  long long offs[kMaxLev];
  int counts[kMaxLev];
  int nlev;
};
__global__ void k_norms(const double* __restrict__ partials, NormArgs na, double* __restrict__ out) {
  __shared__ double red[256];
  for (int l = 0; l < na.nlev; ++l) {
    double s = 0.0;
    for (int i = threadIdx.x; i < na.counts[l]; i += 256) s += partials[na.offs[l] + i];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
      if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
      __syncthreads();
    }
    if (threadIdx.x == 0) out[l] = sqrt(red[0]);
    __syncthreads();
  }
}

// ------------------------------------------------------- error norms -------
// Per element: tensor Gauss-Legendre (p+3)^d points; partial sums of
// (u_h - u)^2 and |grad(u_h - u)|^2 (R13).  Validation only.
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
#define FMG_DISPATCH(dim, p, F)                     \
  do {                                              \
    if (dim == 2 && p == 1) { F(2, 1); }            \
    else if (dim == 2 && p == 2) { F(2, 2); }       \
    else if (dim == 2 && p == 3) { F(2, 3); }       \
    else if (dim == 3 && p == 1) { F(3, 1); }       \
    else if (dim == 3 && p == 2) { F(3, 2); }       \
    else { F(3, 3); }                               \
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

void set_kernel_attributes() {
#define SETA(D, P)                                                                                    \
  cudaFuncSetAttribute(k_residual<D, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, ATile<D, P>::SMEM); \
  cudaFuncSetAttribute(k_cfas_step<D, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, ATile<D, P>::SMEM); \
  cudaFuncSetAttribute(k_restrict<D, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, RTile<D, P>::SMEM);
  SETA(2, 1) SETA(2, 2) SETA(2, 3) SETA(3, 1) SETA(3, 2) SETA(3, 3)
#undef SETA
}

static dim3 tile_grid(int dim, int p, const Geom& g) {
  int TY = 16, TZ = 1;
  if (dim == 3) {
    TY = (p == 1) ? 8 : 4;
    TZ = 4;
  }
  return dim3(g.NX / 32, (g.NY + TY - 1) / TY, (g.NZ + TZ - 1) / TZ);
}

int tile_count(int dim, int p, int kind, const Geom& g) {
  (void)kind;
  dim3 gr = tile_grid(dim, p, g);
  return gr.x * gr.y * gr.z;
}

void launch_prolong_decode(const Launch& L, double* out, const Geom& gf, const double* coarse, const Geom& gc,
                           const uint32_t* mant, const int8_t* exps, int w, int stride, const Coefs& cf) {
  long long rows = (long long)gf.NY * gf.NZ * (gf.NX / 32);
  dim3 grid((unsigned)((rows + NWARP - 1) / NWARP)), block(32, NWARP);
#define F(D, P) k_prolong_decode<D, P><<<grid, block, 0, L.st>>>(out, gf, coarse, gc, mant, exps, w, stride, cf)
  FMG_DISPATCH(L.dim, L.p, F);
#undef F
}

void launch_residual(const Launch& L, const double* U, double* T, const Geom& g, const double* gtab, Sec r,
                     int wr, double* partials, const Coefs& cf, int* status) {
  dim3 grid = tile_grid(L.dim, L.p, g), block(32, NWARP);
#define F(D, P) k_residual<D, P><<<grid, block, ATile<D, P>::SMEM, L.st>>>(U, T, g, gtab, r, wr, partials, cf, status)
  FMG_DISPATCH(L.dim, L.p, F);
#undef F
}

void launch_restrict(const Launch& L, const double* Tf, const Geom& gf, double* Tc, const Geom& gc, Sec r,
                     int wr, double* partials, const Coefs& cf, int* status) {
  dim3 grid = tile_grid(L.dim, L.p, gc), block(32, NWARP);
#define F(D, P) k_restrict<D, P><<<grid, block, RTile<D, P>::SMEM, L.st>>>(Tf, gf, Tc, gc, r, wr, partials, cf, status)
  FMG_DISPATCH(L.dim, L.p, F);
#undef F
}

void launch_coarse(const Launch& L, int mode, const Geom& g0, const double* gtab0, const double* Ainv, int n0,
                   Sec u, int wu_in, int wu_out, Sec r, int wr, double* W0, const Coefs& cf, int* status) {
  dim3 block(32, NWARP);
#define F(D, P) k_coarse<D, P><<<1, block, 0, L.st>>>(mode, g0, gtab0, Ainv, n0, u, wu_in, wu_out, r, wr, W0, cf, status)
  FMG_DISPATCH(L.dim, L.p, F);
#undef F
}

void launch_cfas_step(const Launch& L, const Geom& g, const CfasArgs& a, const Coefs& cf, int* status) {
  dim3 grid = tile_grid(L.dim, L.p, g), block(32, NWARP);
#define F(D, P) k_cfas_step<D, P><<<grid, block, ATile<D, P>::SMEM, L.st>>>(g, a, cf, status)
  FMG_DISPATCH(L.dim, L.p, F);
#undef F
}

void launch_norms(cudaStream_t st, const double* partials, const long long* offs, const int* counts, int nlev,
                  double* out) {
  NormArgs na;
  for (int l = 0; l < kMaxLev; ++l) {
    na.offs[l] = l < nlev ? offs[l] : 0;
    na.counts[l] = l < nlev ? counts[l] : 0;
  }
  na.nlev = nlev;
  k_norms<<<1, 256, 0, st>>>(partials, na, out);
}

void launch_errors(const Launch& L, const double* U, const Geom& g, double* partials, int* nparts) {
  // Gauss-Legendre nodes/weights on [0,1] (Newton on P_n) and Lagrange values.
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
