// fmg_kernels.cu -- sm_100a support kernels of the compact-FMG hot path:
// the deferred norm reduction, the error norms (K5), and the standalone BFP
// codec (K1, bfp_encode / bfp_decode, PAPER.md:1240-1274 with RNE
// PAPER.md:846).  The grid levels run in fmg_fine3.cu / fmg_march3.cu (3D)
// and fmg_march.cu (2D); the coarse levels in fmg_kc.cu.  (The round-1
// tile-box kernels `k_op` were retired in round 2.)
#include "fmg_device.cuh"

namespace fmg {

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

void set_kernel_attributes() {}

size_t devctx_size() { return sizeof(DevCtx); }
void set_devctx_pbase(void* host_buf, double* pbase) { ((DevCtx*)host_buf)->pbase = pbase; }

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
