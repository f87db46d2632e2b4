// fmg1d.cu -- the 1D B-spline compact FMG on the GPU (§8(f) row N4;
// include/fmg1d.h).
//
// One CTA solves one problem of the batch end to end: Alg 3.3 over the FMG
// levels, IR iterations of Alg 3.2 (fmgResidual) + Alg 3.1 (cFas, V(0,1) from
// zero) + the correction.  1D levels of the paper's sizes
// (n_L ~ 10^3 - 10^4 at the FP64-representable depths, reading R26) are far
// too small to spread over the GPU, so the batch dimension fills the 148 SMs
// and the whole solve is ONE launch; the phases inside are separated by
// group barriers (gsync), the working vectors stay in L1/L2.
//
// Arithmetic (reading R27, bit-identical to oracle/bspline1d.py): every row of
// a product is summed from 0.0 in ascending storage index; the encode / decode
// is the block codec of fmg_device.cuh (the same RNE BFP as fmg.h).  A sum
// started at +0.0 is never -0.0, so skipping the band terms outside 0..n-1
// (zero entries) changes nothing, and a lexicographic row skips the terms with
// j > i, which multiply the zero initial guess.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../include/fmg1d.h"
#include "fmg1d_internal.h"
#include "fmg_device.cuh"

namespace fmg1d {
using fmg::FULL;

// Threads per CTA: 256 for the multicolour sweep (every phase is parallel);
// 128 for the lexicographic one, whose sequential chain runs in one warp --
// smaller CTAs put 8 chains on an SM (measured: 64 threads / 16 chains is
// slower, the parallel phases become latency-bound).
// TP = threads per problem; a CTA of kCta<TP> threads holds kCta / TP problems
// (TP = 32: one warp per problem, all syncs are __syncwarp).
template <int TP>
constexpr int kCta = TP < 128 ? 128 : TP;
template <int TP>
constexpr int kMinBlocks = TP == 256 ? 4 : 8;

// barrier of one problem's thread group
template <int TP>
__device__ __forceinline__ void gsync(int grp) {
  if constexpr (TP == 32) {
    __syncwarp();
  } else if constexpr (TP == kCta<TP>) {
    __syncthreads();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(grp + 1), "r"(TP) : "memory");
  }
}

__device__ __forceinline__ double dec_at(const uint32_t* words, const int8_t* exps, int stride, int w, int i) {
  return fmg::point_decode(words + (long long)(i >> 5) * stride, exps[i >> 5], w, i & 31);
}

// Encode x[0..n) (zero-padded to the block boundary; x == nullptr: all zero)
// into a section of width w.  If zv != nullptr, wv[i] = zv[i] + (quantised x_i).
template <int NW1>
__device__ __forceinline__ void encode_level(int tid, const double* x, int n, int nblk, uint32_t* words, int stride,
                                             int8_t* exps, int w, const double* zv, double* wv, int* status) {
  const int lane = tid & 31, warp = tid >> 5;
  for (int blk = warp; blk < nblk; blk += NW1) {
    const int i = blk * 32 + lane;
    const double v = (x && i < n) ? x[i] : 0.0;
    const double q = fmg::warp_encode(v, w, words + (long long)blk * stride, exps + blk, lane, status);
    if (zv && i < n) wv[i] = zv[i] + q;
  }
}

template <int P, bool LEX, int TP>
__global__ void __launch_bounds__(kCta<TP>, kMinBlocks<TP>) k_fmg1d(const __grid_constant__ Args1 a) {
  constexpr int W = 2 * P + 1;
  constexpr int NT1 = TP, NW1 = NT1 / 32, GPC = kCta<TP> / TP;
  __shared__ __align__(16) double gsb_all[GPC][LEX ? 2 * 32 * (W + 1) : 1];  // lexicographic sweep staging
  __shared__ int wcur_all[GPC][kMaxLevels];  // current width of each u section
  const int grp = threadIdx.x / TP, tid = threadIdx.x % TP;
  const int b = blockIdx.x * GPC + grp;
  if (b >= a.batch) return;  // (whole groups only: no barrier is shared across groups)
  double* gsb = gsb_all[grp];
  int* wcur = wcur_all[grp];
  const int nL = a.nL, Lmax = a.levels - 1;
  const double* f = a.f + (long long)b * a.ftot;
  uint32_t* um = a.umant + (long long)b * a.mwords_u;
  uint32_t* rm = a.rmant + (long long)b * a.mwords_r;
  uint32_t* ym = a.ymant + (long long)b * a.mwords_r;
  int8_t* ue = a.uexp + (long long)b * a.eblk;
  int8_t* re = a.rexp + (long long)b * a.eblk;
  int8_t* ye = a.yexp + (long long)b * a.eblk;
  double* X0 = a.tmp + (long long)b * 8 * nL;
  double* X1 = X0 + nL;
  double* T0 = X0 + 2 * nL;
  double* T1 = X0 + 3 * nL;
  double* Z = X0 + 4 * nL;
  double* Bv = X0 + 5 * nL;
  double* Y = X0 + 6 * nL;
  double* D = X0 + 7 * nL;
  const int n0 = a.lv[0].n;
  auto wu = [&](int l, int L) { return a.b1 + (P + 1) * (L - l); };
  auto wr = [&](int l, int L) { return a.b2 + a.m * (L - l); };
  auto U = [&](int l) { return um + a.lv[l].uoff; };
  auto Rs = [&](int l) { return rm + a.lv[l].roff; };
  auto Ys = [&](int l) { return ym + a.lv[l].roff; };
  auto UE = [&](int l) { return ue + a.lv[l].eoff; };
  auto RE = [&](int l) { return re + a.lv[l].eoff; };
  auto YE = [&](int l) { return ye + a.lv[l].eoff; };

  // dense n0 x n0 product y = A0^-1 x (j ascending)
  auto coarse_mv = [&](const double* x, double* y) {
    for (int i = tid; i < n0; i += NT1) {
      double s = 0.0;
      for (int j = 0; j < n0; ++j) s = s + a.A0inv[(long long)i * n0 + j] * x[j];
      y[i] = s;
    }
  };
  // y = P_l x (ELL, k ascending); with dsec: y_i = dec(u_l)_i + (P_l x)_i
  auto prolong = [&](int l, const double* x, double* y, bool add_u) {
    const Level1& v = a.lv[l];
    const int nc = a.lv[l - 1].n;
    for (int i = tid; i < v.n; i += NT1) {
      double s = 0.0;
      const int c = v.c0[i];
      for (int k = 0; k < v.kp; ++k)
        if (c + k < nc) s = s + v.Pv[(long long)i * v.kp + k] * x[c + k];
      y[i] = add_u ? dec_at(U(l), UE(l), v.ustride, wcur[l], i) + s : s;
    }
  };
  // y = R_{l+1} x (transposed ELL, fine rows ascending), x on level l+1
  auto restrict_ = [&](int l, const double* x, double* y) {
    const Level1& v = a.lv[l + 1];
    const int n = a.lv[l].n, nf = v.n;
    for (int j = tid; j < n; j += NT1) {
      double s = 0.0;
      const int r = v.r0[j];
      for (int k = 0; k < v.kr; ++k)
        if (r + k < nf) s = s + v.Rv[(long long)j * v.kr + k] * x[r + k];
      y[j] = s;
    }
  };
  // (A_l x)_i, band terms ascending
  auto band_row = [&](const Level1& v, const double* x, int i) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < W; ++k) {
      const int j = i - P + k;
      if (j >= 0 && j < v.n) s = s + v.Ab[(long long)i * W + k] * x[j];
    }
    return s;
  };
  // standard form u_L = dec u_L + P_L(... dec u_0) into the returned buffer
  auto std_form = [&](int L) -> double* {
    for (int i = tid; i < n0; i += NT1) X0[i] = dec_at(U(0), UE(0), a.lv[0].ustride, wcur[0], i);
    gsync<TP>(grp);
    double *cur = X0, *nxt = X1;
    for (int l = 1; l <= L; ++l) {
      prolong(l, cur, nxt, true);
      gsync<TP>(grp);
      double* t = cur;
      cur = nxt;
      nxt = t;
    }
    return cur;
  };

  // ---- coarse-grid solve u_0 = A_0^-1 f_0
  if (tid < kMaxLevels) wcur[tid] = 0;
  coarse_mv(f + a.foff[0], X0);
  gsync<TP>(grp);
  encode_level<NW1>(tid, X0, n0, a.lv[0].nblk, U(0), a.lv[0].ustride, UE(0), wu(0, 0), nullptr, nullptr, a.status);
  if (tid == 0) wcur[0] = wu(0, 0);
  gsync<TP>(grp);

  for (int L = 1; L <= Lmax; ++L) {
    const Level1& vL = a.lv[L];
    // push level: u_L = 0
    encode_level<NW1>(tid, nullptr, vL.n, vL.nblk, U(L), vL.ustride, UE(L), wu(L, L), nullptr, nullptr, a.status);
    if (tid == 0) wcur[L] = wu(L, L);
    gsync<TP>(grp);
    for (int it = 0; it < a.N; ++it) {
      // ---- fmgResidual (Alg 3.2): t_L = f_L - A_L u_L; r_l = enc R..R t_L
      const double* uL = std_form(L);
      const double* fL = f + a.foff[L];
      for (int i = tid; i < vL.n; i += NT1) T0[i] = fL[i] - band_row(vL, uL, i);
      gsync<TP>(grp);
      encode_level<NW1>(tid, T0, vL.n, vL.nblk, Rs(L), vL.rstride, RE(L), wr(L, L), nullptr, nullptr, a.status);
      double *tc = T0, *tn = T1;
      for (int l = L - 1; l >= 0; --l) {
        restrict_(l, tc, tn);
        gsync<TP>(grp);
        encode_level<NW1>(tid, tn, a.lv[l].n, a.lv[l].nblk, Rs(l), a.lv[l].rstride, RE(l), wr(l, L), nullptr, nullptr,
                     a.status);
        double* t = tc;
        tc = tn;
        tn = t;
      }
      gsync<TP>(grp);
      // ---- cFas V(0,1) from zero (Alg 3.1): y_0 = A_0^-1 r_0, w = dec y_0
      for (int i = tid; i < n0; i += NT1) D[i] = dec_at(Rs(0), RE(0), a.lv[0].rstride, wr(0, L), i);
      gsync<TP>(grp);
      coarse_mv(D, Y);
      gsync<TP>(grp);
      double* Wv = X0;  // w_l (the std buffers are free now)
      for (int i = tid; i < n0; i += NT1) Z[i] = 0.0;
      gsync<TP>(grp);
      encode_level<NW1>(tid, Y, n0, a.lv[0].nblk, Ys(0), a.lv[0].rstride, YE(0), wr(0, L), Z, Wv, a.status);
      gsync<TP>(grp);
      for (int l = 1; l <= L; ++l) {
        const Level1& v = a.lv[l];
        // z = P_l w; b = dec r_l - A_l z; y = 0
        prolong(l, Wv, Z, false);
        gsync<TP>(grp);
        for (int i = tid; i < v.n; i += NT1) {
          Bv[i] = dec_at(Rs(l), RE(l), v.rstride, wr(l, L), i) - band_row(v, Z, i);
          Y[i] = 0.0;
        }
        gsync<TP>(grp);
        // one Gauss-Seidel sweep from zero
        if constexpr (LEX) {
          // The sequential chain runs in warp 0 over 32-row chunks: the warp
          // stages chunk c+32's b and band rows into shared memory with
          // cp.async (coalesced, behind the chain), lane j then holds row
          // c+j, every lane evaluates its own row against the shared window
          // y_{i-P..i-1}, and the shuffle from lane j yields y_{c+j}.  The
          // chain itself carries no global memory access.
          if (tid < 32) {
            const int lane = tid;
            double win[P];  // y_{i-P} .. y_{i-1}
#pragma unroll
            for (int k = 0; k < P; ++k) win[k] = 0.0;
            auto stage = [&](int c, int slot) {
              double* sb = gsb + slot * 32 * (W + 1);
              if (c < v.n) {
                const int cnt = min(32, v.n - c);
                fmg::cpa8(sb + lane, lane < cnt ? Bv + c + lane : Bv, lane < cnt);
                const double* src = v.Ab + (long long)c * W;
#pragma unroll
                for (int q = 0; q < W; ++q) {
                  const int t = lane + 32 * q;
                  fmg::cpa8(sb + 32 + t, t < cnt * W ? src + t : src, t < cnt * W);
                }
              }
              asm volatile("cp.async.commit_group;\n" ::: "memory");
            };
            stage(0, 0);
            int slot = 0;
            for (int c = 0; c < v.n; c += 32, slot ^= 1) {
              stage(c + 32, slot ^ 1);
              asm volatile("cp.async.wait_group 1;\n" ::: "memory");
              __syncwarp();
              const double* sb = gsb + slot * 32 * (W + 1);
              const double bq = sb[lane];
              double aq[P];
#pragma unroll
              for (int k = 0; k < P; ++k) aq[k] = sb[32 + lane * W + k];
              const double dq = sb[32 + lane * W + P];
              const int cnt = min(32, v.n - c);
              double ymine = 0.0;
              for (int j = 0; j < cnt; ++j) {
                double s = bq;
#pragma unroll
                for (int k = 0; k < P; ++k)
                  if (c + j - P + k >= 0) s = s - aq[k] * win[k];
                const double y = __shfl_sync(FULL, s / dq, j);
                if (lane == j) ymine = y;
#pragma unroll
                for (int k = 0; k < P - 1; ++k) win[k] = win[k + 1];
                win[P - 1] = y;
              }
              if (lane < cnt) Y[c + lane] = ymine;
              __syncwarp();  // the slot is restaged two chunks later
            }
            asm volatile("cp.async.wait_all;\n" ::: "memory");
          }
          gsync<TP>(grp);
        } else {
          for (int c = 0; c <= P; ++c) {
            for (int i = c + (P + 1) * tid; i < v.n; i += (P + 1) * NT1) {
              const double* ar = v.Ab + (long long)i * W;
              double s = Bv[i];
#pragma unroll
              for (int k = 0; k < W; ++k) {
                const int j = i - P + k;
                if (k != P && j >= 0 && j < v.n) s = s - ar[k] * Y[j];
              }
              Y[i] = s / ar[P];
            }
            gsync<TP>(grp);
          }
        }
        // y_l = enc y; w = z + dec y_l
        encode_level<NW1>(tid, Y, v.n, v.nblk, Ys(l), v.rstride, YE(l), wr(l, L), Z, Wv, a.status);
        gsync<TP>(grp);
      }
      // ---- correction u_l = enc(dec u_l + dec y_l) at w_u(l, L)
      {
        const int lane = tid & 31, warp = tid >> 5;
        for (int l = 0; l <= L; ++l) {
          const Level1& v = a.lv[l];
          for (int blk = warp; blk < v.nblk; blk += NW1) {
            const int i = blk * 32 + lane;
            double s = 0.0;
            if (i < v.n)
              s = dec_at(U(l), UE(l), v.ustride, wcur[l], i) + dec_at(Ys(l), YE(l), v.rstride, wr(l, L), i);
            fmg::warp_encode(s, wu(l, L), U(l) + (long long)blk * v.ustride, UE(l) + blk, lane, a.status);
          }
        }
        gsync<TP>(grp);
        if (tid <= L) wcur[tid] = wu(tid, L);
        gsync<TP>(grp);
      }
    }
  }
  // ---- the finest level's standard-form solution
  const double* u = std_form(Lmax);
  for (int i = tid; i < nL; i += NT1) a.sol[(long long)b * nL + i] = u[i];
}

}  // namespace fmg1d

using namespace fmg1d;

struct fmg1d_ctx {
  int p = 0, m = 0, levels = 0, batch = 0;
  int tp = 0;  // threads per problem
  fmg1d_schedule s{};
  cudaStream_t st = nullptr;
  std::vector<void*> allocs;
  Args1 a{};
  int n[kMaxLevels]{};
};

namespace {

void* dmalloc(fmg1d_ctx* c, size_t bytes) {
  void* p = nullptr;
  if (cudaMalloc(&p, bytes ? bytes : 16) != cudaSuccess) return nullptr;
  c->allocs.push_back(p);
  return p;
}
template <class T>
T* upload(fmg1d_ctx* c, const T* h, size_t count) {
  T* d = (T*)dmalloc(c, sizeof(T) * count);
  if (d && count && cudaMemcpy(d, h, sizeof(T) * count, cudaMemcpyHostToDevice) != cudaSuccess) return nullptr;
  return d;
}
void release(fmg1d_ctx* c) {
  for (void* p : c->allocs) cudaFree(p);
  c->allocs.clear();
}

}  // namespace

template <int P, bool LEX, int TP>
void launch_tp(fmg1d_ctx* c) {
  constexpr int GPC = kCta<TP> / TP;
  k_fmg1d<P, LEX, TP><<<(c->batch + GPC - 1) / GPC, kCta<TP>, 0, c->st>>>(c->a);
}
// Threads per problem: env FMG1D_TP in {32, 128, 256}
template <int P>
void launch(fmg1d_ctx* c) {
  const int tp = c->tp;
  if (c->a.smoother == FMG1D_LEX) {
    if (tp == 32) launch_tp<P, true, 32>(c);
    else launch_tp<P, true, 128>(c);
  } else {
    if (tp == 32) launch_tp<P, false, 32>(c);
    else launch_tp<P, false, 256>(c);
  }
}

extern "C" {

int fmg1d_create(int p, int m, int levels, const fmg1d_schedule* s, int batch, const double* const* Ab,
                 const double* const* Pv, const double* A0inv, void* stream, fmg1d_ctx** out) {
  if (!out) return FMG_EINVAL;
  *out = nullptr;
  if (!s || fmg1d_size(p, m, 0) < 1 || levels < 1 || levels > kMaxLevels || batch < 1) return FMG_EINVAL;
  if (s->N < 1 || s->b1 < 2 || s->b2 < 2 || (s->smoother != FMG1D_LEX && s->smoother != FMG1D_MCGS))
    return FMG_EINVAL;
  const int Lmax = levels - 1;
  if (s->b1 + (p + 1) * Lmax > 54 || s->b2 + m * Lmax > 54) return FMG_EINVAL;
  fmg1d_ctx* c = new fmg1d_ctx;
  c->p = p;
  c->m = m;
  c->levels = levels;
  c->batch = batch;
  c->s = *s;
  c->st = (cudaStream_t)stream;
  // threads per problem (measured): one warp for the
  // lexicographic sweep and for small problems (n_L <= 2048), a 256-thread CTA
  // for the multicolour sweep on large ones; FMG1D_TP = 32 / 128 / 256 forces it
  c->tp = (s->smoother == FMG1D_LEX || n_unknowns(p, m, levels - 1) <= 2048) ? 32 : 256;
  if (const char* e = getenv("FMG1D_TP")) c->tp = atoi(e) == 32 ? 32 : (s->smoother == FMG1D_LEX ? 128 : 256);
  Args1& a = c->a;
  a.batch = batch;
  a.p = p;
  a.m = m;
  a.levels = levels;
  a.N = s->N;
  a.b1 = s->b1;
  a.b2 = s->b2;
  a.smoother = s->smoother;
  const int W = 2 * p + 1;
  long long uw = 0, rw = 0, eb = 0, ft = 0;
  int rc = FMG_OK;
  for (int l = 0; l < levels && rc == FMG_OK; ++l) {
    const int n = n_unknowns(p, m, l);
    c->n[l] = n;
    Level1& v = a.lv[l];
    v.n = n;
    v.nblk = (n + 31) / 32;
    v.ustride = s->b1 + (p + 1) * (Lmax - l);
    v.rstride = s->b2 + m * (Lmax - l);
    v.uoff = uw;
    v.roff = rw;
    v.eoff = eb;
    uw += (long long)v.nblk * v.ustride;
    rw += (long long)v.nblk * v.rstride;
    eb += v.nblk;
    a.foff[l] = ft;
    ft += n;
    std::vector<double> ab((size_t)n * W);
    if (Ab && Ab[l]) memcpy(ab.data(), Ab[l], sizeof(double) * ab.size());
    else assemble_operator(p, m, l, ab.data());
    v.Ab = upload(c, ab.data(), ab.size());
    if (!v.Ab) rc = FMG_ENOMEM;
    if (l == 0) {
      std::vector<double> inv((size_t)n * n);
      if (A0inv) memcpy(inv.data(), A0inv, sizeof(double) * inv.size());
      else if (!invert(n, ab.data(), p, inv.data())) rc = FMG_EINVAL;
      a.A0inv = upload(c, inv.data(), inv.size());
      if (!a.A0inv) rc = FMG_ENOMEM;
      continue;
    }
    std::vector<int> c0, c1;
    structure(p, m, l, c0, c1);
    const int kp = ell_width(p, m, l), nc = c->n[l - 1];
    std::vector<double> pv((size_t)n * kp);
    if (Pv && Pv[l]) memcpy(pv.data(), Pv[l], sizeof(double) * pv.size());
    else assemble_prolongation(p, m, l, pv.data());
    // R_l = P_l^T: coarse j gathers the fine rows i with c0[i] <= j <= c1[i]
    std::vector<int> r0(nc, -1), r1(nc, -1);
    for (int i = 0; i < n; ++i)
      for (int j = c0[i]; j <= c1[i]; ++j) {
        if (r0[j] < 0) r0[j] = i;
        r1[j] = i;
      }
    int kr = 0;
    for (int j = 0; j < nc; ++j) kr = std::max(kr, r1[j] - r0[j] + 1);
    std::vector<double> rv((size_t)nc * kr, 0.0);
    for (int j = 0; j < nc; ++j)
      for (int i = r0[j]; i <= r1[j]; ++i) rv[(size_t)j * kr + (i - r0[j])] = pv[(size_t)i * kp + (j - c0[i])];
    v.kp = kp;
    v.kr = kr;
    v.Pv = upload(c, pv.data(), pv.size());
    v.c0 = upload(c, c0.data(), c0.size());
    v.Rv = upload(c, rv.data(), rv.size());
    v.r0 = upload(c, r0.data(), r0.size());
    if (!v.Pv || !v.c0 || !v.Rv || !v.r0) rc = FMG_ENOMEM;
  }
  if (rc == FMG_OK) {
    const int nL = c->n[Lmax];
    a.nL = nL;
    a.ftot = ft;
    a.mwords_u = uw;
    a.mwords_r = rw;
    a.eblk = eb;
    a.f = (const double*)dmalloc(c, sizeof(double) * batch * ft);
    a.umant = (uint32_t*)dmalloc(c, sizeof(uint32_t) * batch * uw);
    a.rmant = (uint32_t*)dmalloc(c, sizeof(uint32_t) * batch * rw);
    a.ymant = (uint32_t*)dmalloc(c, sizeof(uint32_t) * batch * rw);
    a.uexp = (int8_t*)dmalloc(c, batch * eb);
    a.rexp = (int8_t*)dmalloc(c, batch * eb);
    a.yexp = (int8_t*)dmalloc(c, batch * eb);
    a.tmp = (double*)dmalloc(c, sizeof(double) * batch * 8 * nL);
    a.sol = (double*)dmalloc(c, sizeof(double) * batch * nL);
    a.status = (int*)dmalloc(c, sizeof(int));
    if (!a.f || !a.umant || !a.rmant || !a.ymant || !a.uexp || !a.rexp || !a.yexp || !a.tmp || !a.sol || !a.status)
      rc = FMG_ENOMEM;
    else if (cudaMemset((void*)a.f, 0, sizeof(double) * batch * ft) != cudaSuccess ||
             cudaMemset(a.status, 0, sizeof(int)) != cudaSuccess ||
             cudaMemset(a.sol, 0, sizeof(double) * batch * nL) != cudaSuccess)
      rc = FMG_ECUDA;
  }
  if (rc == FMG_OK && cudaDeviceSynchronize() != cudaSuccess) rc = FMG_ECUDA;
  if (rc != FMG_OK) {
    release(c);
    delete c;
    return rc;
  }
  *out = c;
  return FMG_OK;
}

int fmg1d_destroy(fmg1d_ctx* c) {
  if (!c) return FMG_EINVAL;
  cudaStreamSynchronize(c->st);
  release(c);
  delete c;
  return FMG_OK;
}

int fmg1d_set_load(fmg1d_ctx* c, const double* const* f) {
  if (!c || !f) return FMG_EINVAL;
  for (int l = 0; l < c->levels; ++l) {
    if (!f[l]) return FMG_EINVAL;
    const size_t w = sizeof(double) * c->n[l];
    if (cudaMemcpy2DAsync((double*)c->a.f + c->a.foff[l], sizeof(double) * c->a.ftot, f[l], w, w, c->batch,
                          cudaMemcpyHostToDevice, c->st) != cudaSuccess)
      return FMG_ECUDA;
  }
  return FMG_OK;
}

int fmg1d_solve_async(fmg1d_ctx* c) {
  if (!c) return FMG_EINVAL;
  if (cudaMemsetAsync(c->a.status, 0, sizeof(int), c->st) != cudaSuccess) return FMG_ECUDA;
  switch (c->p) {
    case 1: launch<1>(c); break;
    case 2: launch<2>(c); break;
    case 3: launch<3>(c); break;
    case 4: launch<4>(c); break;
    case 5: launch<5>(c); break;
    case 6: launch<6>(c); break;
    default: launch<7>(c); break;
  }
  return cudaGetLastError() == cudaSuccess ? FMG_OK : FMG_ECUDA;
}

int fmg1d_sync(fmg1d_ctx* c) {
  if (!c) return FMG_EINVAL;
  if (cudaStreamSynchronize(c->st) != cudaSuccess) return FMG_ECUDA;
  int st = 0;
  if (cudaMemcpy(&st, c->a.status, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess) return FMG_ECUDA;
  return st ? FMG_ERANGE : FMG_OK;
}

int fmg1d_solve_host(fmg1d_ctx* c, const double* const* f, double* u) {
  if (!c || !f || !u) return FMG_EINVAL;
  int rc = fmg1d_set_load(c, f);
  if (rc == FMG_OK) rc = fmg1d_solve_async(c);
  if (rc != FMG_OK) return rc;
  if (cudaMemcpyAsync(u, c->a.sol, sizeof(double) * c->batch * c->a.nL, cudaMemcpyDeviceToHost, c->st) !=
      cudaSuccess)
    return FMG_ECUDA;
  return fmg1d_sync(c);
}

int fmg1d_solution(fmg1d_ctx* c, int b, double* u) {
  if (!c || !u || b < 0 || b >= c->batch) return FMG_EINVAL;
  if (cudaStreamSynchronize(c->st) != cudaSuccess) return FMG_ECUDA;
  return cudaMemcpy(u, c->a.sol + (long long)b * c->a.nL, sizeof(double) * c->a.nL, cudaMemcpyDeviceToHost) ==
                 cudaSuccess
             ? FMG_OK
             : FMG_ECUDA;
}

int fmg1d_solution_device(fmg1d_ctx* c, double** u) {
  if (!c || !u) return FMG_EINVAL;
  *u = c->a.sol;
  return FMG_OK;
}

int fmg1d_section(fmg1d_ctx* c, int which, int l, int b, uint32_t* mant, int8_t* exps, int* w) {
  if (!c || which < 0 || which > 2 || l < 0 || l >= c->levels || b < 0 || b >= c->batch || !mant || !exps || !w)
    return FMG_EINVAL;
  if (cudaStreamSynchronize(c->st) != cudaSuccess) return FMG_ECUDA;
  const Level1& v = c->a.lv[l];
  const int Lmax = c->levels - 1;
  const uint32_t* base;
  const int8_t* eb;
  int stride, width;
  if (which == 0) {
    base = c->a.umant + (long long)b * c->a.mwords_u + v.uoff;
    eb = c->a.uexp;
    stride = v.ustride;
    width = c->s.b1 + (c->p + 1) * (Lmax - l);
  } else {
    base = (which == 1 ? c->a.rmant : c->a.ymant) + (long long)b * c->a.mwords_r + v.roff;
    eb = which == 1 ? c->a.rexp : c->a.yexp;
    stride = v.rstride;
    width = c->s.b2 + c->m * (Lmax - l);
  }
  *w = width;
  if (cudaMemcpy2D(mant, sizeof(uint32_t) * width, base, sizeof(uint32_t) * stride, sizeof(uint32_t) * width, v.nblk,
                   cudaMemcpyDeviceToHost) != cudaSuccess)
    return FMG_ECUDA;
  if (cudaMemcpy(exps, eb + (long long)b * c->a.eblk + v.eoff, v.nblk, cudaMemcpyDeviceToHost) != cudaSuccess)
    return FMG_ECUDA;
  return FMG_OK;
}

}  // extern "C"
