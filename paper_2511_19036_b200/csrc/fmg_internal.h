// fmg_internal.h -- types shared by the host driver (fmg_api.cpp, fmg_tables.cpp)
// and the CUDA kernels (fmg_kernels.cu).  Product path only; nothing here is
// shared with oracle/.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace fmg {

constexpr int kMaxLev = 16;

// Geometry of one level.
struct Geom {
  int n;            // p 2^(l+1): stored nodes per dim (node 0 = boundary)
  int NX, NY, NZ;   // stored extents (NX = roundup(n, 32); NZ = 1 in 2D)
  long long size;   // NX*NY*NZ
  long long nblk;   // size / 32
  int l;            // level index
};

// Operator tables (correctly rounded doubles of exact rationals).
struct Coefs {
  double Kc[3][7];    // assembled 1D stiffness rows (reference, h-free) by node type, offsets -p..p
  double Mc[3][7];    // assembled 1D mass rows
  double Pw[6][4];    // prolongation weights [i mod 2p][t]
  double Rw[3][11];   // restriction weights [c mod p][s], fine j = 2c-(2p-1)+s
  double invd[27];    // 1/diag(Â) by node type (tz*p+ty)*p+tx
  double inv_theta;   // Chebyshev 1/theta
  double cal[8], cbe[8];  // Chebyshev alpha_j, beta_j (index j-1)
  double rhs_c;       // RN(dim pi^2)
};

// A BFP section stored with a fixed block stride (>= current width).
struct Sec {
  uint32_t* mant;
  int8_t* exps;
  int stride;
};

// Host-side table builders (fmg_tables.cpp).
void build_coefs(int dim, int p, double lambda_hi, double alpha, int cheb_degree, Coefs* c);
void build_rhs_table(int p, int l, double* g);       // g[0..n-1]
int coarse_count(int dim, int p);
int build_coarse_inverse(int dim, int p, double* Ainv);  // 0 on success

// Operation descriptors (mirrors the device Op).
enum { OP_DECODE = 0, OP_RESIDUAL, OP_RESTRICT, OP_NORMS, OP_CFAS1 = 6, OP_CHEB, OP_PROLONG, OP_GS, OP_SQ, OP_COARSE };
struct OpDesc {
  int type, l, L, step, last;
  int wr, wu_in, wu_out;
  int guess, store, smode;  // nu > 1 cycles: see MArgs
  int zout, wout, uout, puonly;  // finest-level kernels (F3Args) / P u_{l-1}-only prolongation (MArgs)
  int cfs;                       // finest-level cFas step 1 from a materialised z_L (F3Args::cfs)
  int row;
  long long poff;  // norm partials of this (FMG level, iteration, level): pbase + poff
};

// Device view of one level (also a member of the device context).
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
  double* U;       // decoded u_l = dec ú_l + P_l u_{l-1} (padded level layout)
  double* T;       // residual temporary t_l (nu > 1: s_l between cycles)
  double* W;       // w_l = z_l + dec ý_l (nu > 1 s sweep: q_l = A ý_l + s_l)
  uint32_t* ymant; // nu > 1: the correction ý_l kept across cycles (width w_r(l, L))
  int8_t* yexp;
  int ystride;
};

// Scratch and bookkeeping pointers of the march kernels.
struct MPtrs {
  double *Z, *B, *Y[2], *Dv, *PU;
  double* YO;      // nu > 1: dec ý_l of the previous cycle at the level being smoothed
  double* pbase;
  int* status;
};

// 2D row-march launch (fmg_march.cu): one warp per (32-column block, chunk of RC output rows).
struct MArgs {
  int type, l, L, step, last;
  int wr, wu_in, wu_out;
  int RC, nxb, nitems, NYo;  // rows (2D) / planes (3D) per chunk, block columns, work items (3D: CTAs), output rows
  int nyb, NZo;              // 3D: tile rows (of 8), output planes
  int zlo, zhi;              // 3D: the planes of this rank (z slab), [zlo, zhi)
  int gs;                    // smoother: multicolour Gauss-Seidel (cFas1 forms colour 0; OP_GS: colour `step`)
  // nu > 1 cycles (Alg 3.1, reading R23):
  int guess;                 // cFas1 / last step: ý of the previous cycle is the initial guess
  int store;                 // last step: store ý_l (not the last cycle), no correction
  int smode;                 // OP_RESTRICT: s sweep (no encode, no norm); OP_SQ: s_{l} = 0 (top level)
  int puonly;                // OP_PROLONG (3D): P u_{l-1} only (the finest-level cFas kernel generates z)
  // operands in the parameter space (no dependent global loads at kernel start)
  LevelDev lv;               // the output level l
  LevelDev lo;               // the other level: l-1 (decode, prolongation, cFas) or l+1 (restriction)
  MPtrs p;
  long long poff;            // norm partials (one per item) at pbase + poff, or -1
  // TMA map of the array this launch stages (2D rows / 3D plane boxes), or
  // none when the kernel stages nothing from global memory;
  // kept in device memory so the launch parameters stay small
  int tma;                   // 1: tm is valid and the kernel stages through it
  int zoff;                  // first plane of the staged array's allocation (z slabs keep a plane window; 0 otherwise)
  const CUtensorMap* tm;     // TMA map of the staged array, in device global memory
};

// Finest-level 3D kernels (fmg_fine3.cu): one launch of
// k_f3_residual / k_f3_cfas / k_f3_cheb at level l = L of FMG level L.
struct F3Args {
  Geom g;                    // level l
  int l, step, last;         // Chebyshev step (>= 2) and whether it is the last
  int wr, wu, wu_out;        // w_r(L, L), current and new w_u of ú_L
  int RC, nxb, nyb, nitems;  // planes per chunk, tile grid, CTAs
  int zlo, zhi;              // planes of this rank
  int zoff, czoff;           // first allocated plane of level l / l - 1 (TMA coordinates are window-relative)
  uint32_t* umant;
  int8_t* uexp;
  int ustride;
  uint32_t* rmant;
  int8_t* rexp;
  int rstride;
  const double* gtab;        // RHS table of level l
  double* T;                 // t_L (residual) / b_L (cFas and Chebyshev: the same buffer)
  double* Dv;                // Chebyshev direction d_2 (degree 3)
  double* pbase;             // norm partials
  long long poff;
  int* status;
  const CUtensorMap* tmc;    // coarse boxes of u_{L-1} (residual) / w_{L-1} (cFas), device copy
  const CUtensorMap* tmb;    // fine boxes of b_L (the t_L buffer)
  const CUtensorMap* tmd;    // fine boxes of d_2
  // levels below the finest and the materialised mode:
  double* Z;                 // cFas: z_l at the output points -> Z (zout)
  double* PU;                // last Chebyshev step: P u_{l-1} at the output points (uout)
  double* U;                 // last Chebyshev step: u_l = dec ú_l + P u_{l-1} -> U (uout)
  double* W;                 // last Chebyshev step: w_l = z_l + dec ý_l -> W (wout)
  int zout, wout, uout;
  int tpb;                   // thread-per-block epilogues (k_f3_tpb): r_L after the residual, the last step's codec
  double* Yb;                // (tpb) y_k of the last Chebyshev step, FP64, level window
  int cfs;                   // cFas step 1 from a materialised z_l (k_f3_staged<P, 2>): 1 top level, z_L in Yb;
                             // 2: also P u_{L-1} -> PU in the same prolongation launch; 5: below the top
                             // level, z_l -> the Z scratch and P u_{l-1} -> PU; 3 (Chebyshev item): staged step
  const CUtensorMap* tmy;    // fine boxes of Yb (cfs)
  const CUtensorMap* tmcu;   // coarse boxes of u_{L-1} (cfs == 2)
  const CUtensorMap* tmc2;   // (k_f3_prolong<P, 2>) second coarse array and its output
  double* out2;
  // staged Chebyshev steps (cfs == 3 on a Chebyshev item; k_f3_staged<P, 3 / 4>):
  // y_1 -> X1 (cFas step 1), y_2 -> Yb (step 2), y_3 -> X1 (step 3)
  double* X1b;
  const CUtensorMap* tmx1;   // fine boxes of X1b
  int csc;                   // (cFas step 1 with cfs) the Chebyshev steps are staged: write y_1
  const CUtensorMap* tmz;    // (cfs == 5, below the top level) fine boxes of the Z scratch
  double* yout;              // (k_f3_staged) where y_j goes
  int s2;                    // k_f3_staged2 (two input planes per iteration) instead of k_f3_staged
  int ctaoff;                // (k_f3_staged) first norm-partial CTA index of this launch (z chunks)
  int pr2;                   // k_f3_prolong2 (32 x 16 tiles) for p = 1, 3
  double* chk;               // lean form in z chunks: the chunk buffer (a.chkrc + 2P planes)
  int chkrc;
  const CUtensorMap* tmch;   // fine boxes of the chunk buffer
  int tpby;                  // lean top level: the last step stores ý as int8 mantissas + exponents (my, ey)
  int8_t* my;                //   per point (level window)
  int8_t* ey;                //   per block
  int f32s;                  // FP32 cFas with float storage at this level: z_l, b_l, y_j, d_2 are float arrays
};

// One deferred norm: ||t_l||_2 of norm row `row` from `count` partials at pbase + poff.
struct NormEntry {
  long long poff;
  int row, l, count, pad;
};

// KC (coarse-hierarchy cluster kernel, fmg_kc.cu) launch descriptor.
struct KcDesc {
  int mode;        // 0: coarse-grid solve, then FMG levels 1..Llast (<= lc) in full
                   // 1: the levels-0..lc part of IR iteration `it` at FMG level L > lc
  int L, it;       // mode 1
  int Llast;       // mode 0: last FMG level run inside (0: coarse solve only)
  int iters_last;  // mode 0: IR iterations at FMG level Llast
  int b_u, k_u, b_r, k_r;  // width law w_u = b_u + k_u (L - l), w_r = b_r + k_r (L - l)
  int row0, nrows;         // norm rows (L n_ir + it) written by this launch
  int debug;               // record phase timestamps (tools/kc_phases.py)
};

// KC distributed-shared-memory layout (same offsets in every CTA of the cluster):
// per-level slabs of u_l, t_l, w_l; scratch slabs; section storage of the owned
// blocks; the norm-partial table.  Double offsets unless noted.
struct KcLayout {
  int lg;  // log2(cluster size)
  int bytes;
  int U[kMaxLev], T[kMaxLev], W[kMaxLev];
  int Z, B, Y0, Y1, Dv, PU, KS0, KS1, RQ0;
  int part;
  int um[kMaxLev], rm[kMaxLev];  // uint32 word offsets
  int ue[kMaxLev], re[kMaxLev];  // byte offsets
  int lgc[kMaxLev];              // log2 of the blocks per CTA of each level
};

// Everything the device context needs.
struct DevCtxDesc {
  int levels, n_ir, n0;
  Geom g[kMaxLev];
  Sec u[kMaxLev], r[kMaxLev];
  const double* gtab[kMaxLev];
  int tiles[kMaxLev][3];
  double* part[kMaxLev];
  int* count;  // kMaxLev arrival counters (zeroed)
  double* pbase;
  double *Ul[kMaxLev], *Tl[kMaxLev], *Wl[kMaxLev];  // per-level u_l, t_l, w_l
  double *Y[2];
  double *Z, *B, *Dv, *PU;
  double *KS[2];   // (unused by the DSMEM KC; kept for layout compatibility)
  KcLayout kc;
  const double* Ainv;
  double* norms;
  int* status;
  int lc, n_cheb;
  int smoother;  // 0 Chebyshev, 1 multicolour Gauss-Seidel
  Coefs cf;
};

struct Launch {
  int dim, p;
  cudaStream_t st;
};

// Kernel side (fmg_kernels.cu).
void set_kernel_attributes();
size_t devctx_size();
void set_devctx_pbase(void* host_buf, double* pbase);
void fill_devctx(void* host_buf, const DevCtxDesc& d);
void march_set_attributes();
void launch_march(int p, cudaStream_t st, const void* devctx, const MArgs& a, const Coefs& cf);
// Small 2D levels: a run of up to MFUSED_OPS dependent ops in one launch (fmg_march.cu k_m_fused)
constexpr int MFUSED_WARPS = 16, MFUSED_OPS = 8;
struct MFused {
  MArgs op[MFUSED_OPS];
  int n;
};
void launch_march_fused(int p, cudaStream_t st, const void* devctx, const MFused& f, const Coefs& cf);
int march_fused_warps();
void march3_set_attributes();
int march3_rows();
void launch_march3(int p, cudaStream_t st, const void* devctx, const MArgs& a, const Coefs& cf);
void fine3_set_attributes();
int fine3_box_dims(int p, int* cbx, int* cby, int* rs, int* nr);
void launch_fine3(int p, int kind, cudaStream_t st, const F3Args& a, const Coefs& cf, int fp32);
bool fine3_tpby_width(int wu, int wr);
int fine3_take_launches();  // kernels launch_fine3 issued since the last call
void launch_coarse_nu(int dim, int p, cudaStream_t st, const void* devctx, const MArgs& a);  // nu > 1 level 0
int kc_plan(int dim, int p, int Lmax, const Geom* g, const int* ust, const int* rst, int n_ir, int lc_cap,
            KcLayout* ly, int* lc_out, int* cs_out);
int kc_warps_per_cta();
void launch_kc(int dim, int p, cudaStream_t st, const void* devctx, const KcDesc& a, int cluster, int smem);
void launch_norms_all(cudaStream_t st, const void* devctx, const NormEntry* entries_dev, int n);
void launch_errors(const Launch& L, const double* U, const Geom& g, double* partials, int* nparts);
void launch_bfp_encode(const double* x, long long n, int w, uint32_t* mant, int8_t* exps, int* status,
                       cudaStream_t st);
void launch_bfp_decode(const uint32_t* mant, const int8_t* exps, long long n, int w, double* x,
                       cudaStream_t st);
long long stream_work_bytes(long long n);
void launch_stream_encode(const double* x, long long n, int w, uint32_t* mant, int32_t* xexp, int64_t* xstart,
                          int32_t* nblocks, void* work, int* status, cudaStream_t st);
void launch_stream_decode(const uint32_t* mant, const int32_t* xexp, const int64_t* xstart, const int32_t* nblocks,
                          long long n, int w, double* x, cudaStream_t st);

}  // namespace fmg
