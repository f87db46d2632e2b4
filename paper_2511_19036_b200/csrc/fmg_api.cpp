// fmg_api.cpp -- C-ABI (include/fmg.h) and the FMG level driver (S11).
//
// The driver issues Alg 3.3 as a fixed sequence of kernel
// launches, captured once into a CUDA graph per context and replayed on every
// solve.  Per IR iteration at FMG level L:
//   fmgResidual: prolong/decode l = 0..L, fused residual + encode at L,
//                restriction + encode l = L-1..0, norm reduction;
//   cFas + correction: coarse kernel (exact solve, encode ý_0, W_0, ú_0 update),
//                then per l = 1..L: prolong W_{l-1}, k Chebyshev steps, the last
//                one fused with encode ý_l, W_l = z_l + dec ý_l and the ú_l update.
#include "../../include/fmg.h"

#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <vector>

#include <dlfcn.h>
#include <nccl.h>

#include "fmg_internal.h"

using namespace fmg;

namespace {
fmg_alloc_fn g_alloc = nullptr;
fmg_free_fn g_free = nullptr;
void* g_alloc_user = nullptr;
}  // namespace

struct fmg_ctx {
  int dim = 0, p = 0, levels = 0, Lmax = 0;
  fmg_schedule s{};
  cudaStream_t st = nullptr;      // user stream
  cudaStream_t cap = nullptr;     // private capture stream
  cudaStream_t cur = nullptr;     // stream launches are issued on
  Geom g[kMaxLev];
  Coefs cf{};
  Sec u[kMaxLev]{}, r[kMaxLev]{};
  Sec ysec[kMaxLev]{};            // nu > 1: the correction ý_l kept across cycles
  double* gtab[kMaxLev]{};
  int tiles[kMaxLev][3]{};
  double* Ainv = nullptr;
  int n0 = 0;
  double* buf[9]{};
  double* partials = nullptr;
  long long part_off[kMaxLev]{};
  double* norms_dev = nullptr;
  double* pbase = nullptr;         // deferred norm partials
  long long pbase_cap = 0;
  NormEntry* nent[2] = {nullptr, nullptr};  // deferred norm entries: [0] graph, [1] direct runs
  int nent_cap[2] = {0, 0};
  int nent_slot = 0;
  double* err_part = nullptr;
  int* status = nullptr;
  void* devctx = nullptr;         // DevCtx in device memory
  cudaGraphExec_t graph = nullptr;
  int solved_L = -1;
  int wu_cur[kMaxLev]{};
  int wu_graph[kMaxLev]{};        // section widths the captured solve graph leaves (restored on every replay)
  int lc = 0;                     // levels 0..lc run inside the cluster kernel KC
  int kc_cluster = 1;             // CTAs of the KC cluster
  KcLayout kcl{};                 // KC shared-memory layout
  int kc_tw = 16;                 // KC warps (cluster x warps per CTA): norm partials per level
  double* Ul[kMaxLev]{};          // per-level u_l, t_l, w_l (padded level layout)
  double* Tl[kMaxLev]{};
  double* Wl[kMaxLev]{};
  int mrc[kMaxLev]{}, mitems[kMaxLev]{};  // march rows / planes per chunk, work items (3D: CTAs) per level
  int mnyb[kMaxLev]{};
  // TMA maps of the staged arrays (march kernels): u_l rows /
  // boxes, fine t_{l} rows for the 2D restriction, and the Z, B, Y0, Y1
  // buffers with each level's geometry
  bool tma = false;
  CUtensorMap tmU[kMaxLev]{}, tmT[kMaxLev]{}, tmB[4][kMaxLev]{};
  // finest-level kernels (fmg_fine3.cu): coarse boxes of u_l / w_l, fine boxes
  // of t_l (= b_l) and of the Chebyshev direction
  CUtensorMap tmCU[kMaxLev]{}, tmCW[kMaxLev]{}, tmFB[kMaxLev]{}, tmFD[kMaxLev]{}, tmYB[kMaxLev]{}, tmX1[kMaxLev]{};
  CUtensorMap tmCH[kMaxLev]{};
  CUtensorMap* tm_dev = nullptr;  // device copy: [U | T | B0..B3 | CU | CW | FB | FD | YB | X1 | CH] x kMaxLev
  // 3D, one GPU, Chebyshev degree 2-3, nu = 1: level L of each FMG level runs
  // the finest-level kernels and keeps no u_L, z_L, P u_{L-1}, w_L or y arrays
  // (DESIGN.md §4.3); the level arrays of l = Lmax that remain are t (= b)
  // and, for degree 3, the direction d_2.  FMG_FINE3=0 selects the
  // level-by-level kernels everywhere.
  bool fine3 = false;
  // fine3, memory permitting: the finest level keeps u_L and P u_{L-1} arrays
  // too (the residual stages u_L instead of generating it).
  // FMG_F3MAT=0/1 forces the choice.
  bool f3mat = false;
  bool tpb = false;  // thread-per-block epilogues of the finest-level kernels (k_f3_tpb; needs f3mat's memory)
  bool cfs = false;  // top-level cFas step 1 from a materialised z_L (k_f3_prolong + k_f3_staged<P, 2>; in Y)
  bool csc = false;  // with cfs: the Chebyshev steps staged from the materialised y_{j-1} (X1, Y)
  long long tpb_min = 1LL << 16;  // levels of at least this many blocks take tpb / cfs (FMG_TPB_MIN_BLOCKS: tests)
  bool tpb0 = false;  // lean form: the generating residual's r_L encoded thread per block (k_f3_tpb<0>)
  bool tpby = false;  // lean form: the top level's last step stores ý as int8 mantissas (k_f3_tpb<2>)
  bool s2 = false;    // staged kernels two input planes per iteration (k_f3_staged2; FMG_S2)
  bool f32s = false;  // FP32 cFas with float storage of z_l, b_l, y_j, d_2 at the staged levels (FMG_F32S)
  bool chk = false;   // lean form in z chunks: u_L / z_L materialised chunk by chunk (FMG_CHK)
  int chk_rc = 0;     // planes per chunk
  double* chkbuf = nullptr;
  int8_t* my_base = nullptr;  // (tpby) finest-window points
  int8_t* ey_base = nullptr;  // (tpby) finest-window blocks
  int nccl_err = 0;               // an NCCL call of the last issue failed (reported by the solve)
  // z-slab decomposition (3D): this context computes planes
  // [zlo, zhi) of every grid level l > lc (full-size arrays; ghost planes are
  // exchanged before each stencil consumer, t_{lc+1} is gathered before KC)
  int G = 1, rank = 0;
  int zlo[kMaxLev]{}, zhi[kMaxLev]{};
  // allocated plane window [wlo, whi) of every level array and section: the
  // whole level, or on z slabs (levels > lc + 1) the rank's planes plus 2p
  // ghost planes each side (memory partitioned over the ranks).
  // Level pointers are shifted so that kernels index planes globally.
  int wlo[kMaxLev]{}, whi[kMaxLev]{};
  double* sbase[9]{};             // scratch allocations (buf[] are their level-0 views)
  std::vector<fmg_ctx*> sub;      // virtual slabs: G sub-contexts driven in lockstep (group handle)
  void* comm = nullptr;           // multi-GPU slabs: ncclComm_t (one rank per process)
  fmg_xfer_fn xfer = nullptr;     // host-staged slabs (fmg_create_hostx): the caller's transport
  void* xfer_user = nullptr;
  fmg_alloc_fn afn = nullptr;
  fmg_free_fn ffn = nullptr;
  void* auser = nullptr;
  std::vector<std::pair<void*, size_t>> allocs;
  // kernel timing
  int timing_cls = -1;
  std::vector<cudaEvent_t> ev;
  int ev_used = 0;
  long long launches = 0;
};

namespace {

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
PFN_cuTensorMapEncodeTiled_v12000 tma_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return fn;
}

// FP64 (esz = 8) or FP32 (esz = 4) tiled map over a [nz][ny][nx] array
// (rank 2 when nz == 0), box bx x by x 1, out-of-range elements zero-filled.
bool make_tmap(CUtensorMap* m, const void* base, long long nx, long long ny, long long nz, int bx, int by, int esz = 8) {
  PFN_cuTensorMapEncodeTiled_v12000 enc = tma_encoder();
  if (!enc || !base) return false;
  const cuuint32_t rank = nz > 0 ? 3 : 2;
  cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)ny, (cuuint64_t)(nz > 0 ? nz : 1)};
  cuuint64_t strides[2] = {(cuuint64_t)nx * esz, (cuuint64_t)nx * ny * esz};
  cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(m, esz == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, (void*)base, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

int wu(const fmg_ctx* c, int l, int L) { return c->s.b_u + c->s.k_u * (L - l); }
int wr(const fmg_ctx* c, int l, int L) { return c->s.b_r + c->s.k_r * (L - l); }

void* dalloc(fmg_ctx* c, size_t bytes) {
  if (bytes == 0) bytes = 16;
  void* ptr = nullptr;
  if (c->afn) {
    ptr = c->afn(bytes, c->auser);
  } else if (cudaMalloc(&ptr, bytes) != cudaSuccess) {
    ptr = nullptr;
  }
  if (ptr) c->allocs.emplace_back(ptr, bytes);
  return ptr;
}

void free_all(fmg_ctx* c) {
  for (auto& a : c->allocs) {
    if (c->ffn) c->ffn(a.first, a.second, c->auser);
    else cudaFree(a.first);
  }
  c->allocs.clear();
}

Launch L_(fmg_ctx* c) { return Launch{c->dim, c->p, c->cur}; }

// ---------------------------------------------------------------- schedule --
// A solve is a list of items: a grid launch of one tile op over all tiles of its
// level, or one launch of the coarse-hierarchy cluster kernel KC (levels
// 0..lc).  DESIGN.md §4.
struct Item {
  int kind;          // 0 grid op, 1 KC, 2 ghost-plane exchange / gather (z slabs), 3 finest-level op (fmg_fine3.cu)
  int f3kind;        // kind 3: 0 residual, 1 cFas step 1, 2 Chebyshev step op.step
  OpDesc op;         // grid item
  KcDesc kc;         // KC item
  int timed_cls;     // kernel-timing class of a grid item (-1: none)
  int xarr, xl, xdepth, xgather;  // exchange item: array, level, ghost depth, gather-all
};
enum { XA_U = 0, XA_T, XA_W, XA_Z, XA_B, XA_Y0, XA_Y1, XA_D, XA_SU };  // XA_SU: the ú section (BFP words + exponents)

struct Builder {
  fmg_ctx* c;
  std::vector<Item> items;
  std::vector<NormEntry> norms;
  long long ptot = 0;  // (set past the KC partial region by make_builder)
  // reserve partial slots for (row, level l) and record the deferred norm
  long long slot(int row, int l, long long items = -1) {
    int nt = c->dim == 2 ? c->mitems[l] : (int)((items >= 0 ? items : c->mitems[l]) * march3_rows());
    long long off = ptot;
    ptot += nt;
    NormEntry e{off, row, l, nt, 0};
    norms.push_back(e);
    return off;
  }
  void grid(const OpDesc& op, int cls = -1) {
    Item it{};
    it.kind = 0;
    it.op = op;
    it.timed_cls = cls;
    items.push_back(it);
  }
  // ghost planes of array `arr` at slab level l (l > lc) before a stencil consumer
  void xchg(int arr, int l, int depth, int gather = 0) {
    if (c->G <= 1 || l <= c->lc) return;
    Item it{};
    it.kind = 2;
    it.xarr = arr;
    it.xl = l;
    it.xdepth = depth;
    it.xgather = gather;
    it.timed_cls = -1;
    items.push_back(it);
  }
  void fine(int f3kind, const OpDesc& op, int cls = -1) {
    Item it{};
    it.kind = 3;
    it.f3kind = f3kind;
    it.op = op;
    it.timed_cls = cls;
    items.push_back(it);
  }
  void kc(const KcDesc& d) {
    Item it{};
    it.kind = 1;
    it.kc = d;
    it.timed_cls = -1;
    items.push_back(it);
  }
  // deferred norm of level l <= lc computed by KC: one partial per KC warp in
  // the KC region at the start of the partial buffer (fmg_kc.cu norm_partial)
  void kc_norm(int row, int l) {
    NormEntry e{((long long)row * c->levels + l) * c->kc_tw, row, l, c->kc_tw, 0};
    norms.push_back(e);
  }
};

Builder make_builder(fmg_ctx* c) {
  Builder b{c, {}, {}, 0};
  b.ptot = (long long)c->levels * c->s.n_ir * c->levels * c->kc_tw;
  return b;
}

KcDesc mkkc(fmg_ctx* c, int mode) {
  KcDesc d{};
  d.mode = mode;
  d.b_u = c->s.b_u;
  d.k_u = c->s.k_u;
  d.b_r = c->s.b_r;
  d.k_r = c->s.k_r;
  return d;
}

OpDesc mkop(int type, int l, int L) {
  OpDesc o{};
  o.type = type;
  o.l = l;
  o.L = L;
  o.poff = -1;
  return o;
}

// cFas at level l of FMG level L with the finest-level kernels (fmg_fine3.cu,
// DESIGN.md §4.3): [P u_{l-1} -> PU], z_l generated on chip -> b_l (+ z_l -> Z
// below the finest level), Chebyshev steps 2..k; the last one applies the
// correction and, below the finest level (or materialised), writes w_l and
// Levels of >= tpb_min blocks in the materialised form on one GPU: cFas step 1
// from a materialised z_l (k_f3_staged<P, 2>), and with FP32 cFas the float
// storage of the cFas arrays.
static bool level_cfs(const fmg_ctx* c, int l) {
  return c->cfs && (long long)(c->zhi[l] - c->zlo[l]) * c->g[l].NY * (c->g[l].NX / 32) >= c->tpb_min;
}

// u_l.  `xch`: z-slab ghost exchanges before each stencil consumer.
void add_fine3_level(Builder& b, int l, int L, bool fine, bool xch) {
  fmg_ctx* c = b.c;
  const int P = c->p, k = c->s.cheb_degree;
  const bool top = l == L, uout = !top || c->f3mat;
  // materialised form on one GPU, levels of >= 2^16 blocks: z_l = P w_{l-1}
  // materialised for cFas step 1 (in Y at the top level, in the Z scratch
  // below it, where the last step needs z_l again), P u_{l-1} in the same launch
  const bool cfs = level_cfs(c, l);
  if (uout && !cfs) {  // P u_{l-1} at the level's points (k_f3_prolong)
    if (xch) b.xchg(XA_U, l - 1, P);
    OpDesc q = mkop(OP_PROLONG, l, L);
    q.step = 0;
    b.fine(3, q);
  }
  if (xch) b.xchg(XA_W, l - 1, 2 * P);
  for (int step = 1; step <= k; ++step) {
    if (xch && step >= 2) b.xchg(XA_T, l, P);  // b_l (the t_l buffer)
    if (xch && step >= 3) b.xchg(XA_D, l, P);  // d_2
    OpDesc q = mkop(step == 1 ? OP_CFAS1 : OP_CHEB, l, L);
    q.step = step;
    q.last = step == k;
    q.wr = wr(c, l, L);
    q.wu_in = c->wu_cur[l];
    q.wu_out = wu(c, l, L);
    q.zout = step == 1 && !top;
    q.wout = q.last && !top;
    q.uout = q.last && uout;
    q.cfs = !cfs ? 0 : step == 1 ? (!top ? 5 : uout ? 2 : 1) : (c->csc ? 3 : 0);
    if (!cfs && step == 1 && top && c->chk && !c->f3mat && !c->s.cfas_fp32) q.cfs = 6;  // (lean, z chunks)
    b.fine(step == 1 ? 1 : 2, q, (fine && top) ? (step == k ? 5 : 1) : -1);
  }
}

// Grid-only fmgResidual (API paths): decode sweep, residual, restriction, norms.
void build_residual_grid(Builder& b, int L, int row) {
  fmg_ctx* c = b.c;
  const bool f3 = c->fine3 && L >= 1;  // u_L generated on chip: decode only l < L
  for (int l = 0; l <= (f3 ? L - 1 : L); ++l) {
    OpDesc o = mkop(OP_DECODE, l, L);
    o.wu_in = c->wu_cur[l];
    b.grid(o);
  }
  OpDesc o = mkop(OP_RESIDUAL, L, L);
  o.wr = wr(c, L, L);
  o.wu_in = c->wu_cur[L];
  o.row = row;
  o.poff = b.slot(row, L);
  if (f3) b.fine(0, o);
  else b.grid(o);
  for (int l = L - 1; l >= 0; --l) {
    OpDesc q = mkop(OP_RESTRICT, l, L);
    q.wr = wr(c, l, L);
    q.row = row;
    q.poff = b.slot(row, l);
    b.grid(q);
  }
}

int ncolours(const fmg_ctx* c) {
  const int q = c->p + 1;
  return c->dim == 3 ? q * q * q : q * q;
}

// One IR iteration at FMG level L: fmgResidual (Alg 3.2),
// cFas V(0,1) (Alg 3.1, nu = 1), correction.  Levels <= lc run inside KC.
// One IR iteration with nu > 1 compact V(0,1) cycles (Alg 3.1
// PAPER.md:633-661, reading R23; oracle orc_cfas_correct).  Chebyshev, one
// GPU, lc = 0: the grid kernels do every level >= 0 except the initial coarse solve.
void build_iteration_nu(Builder& b, int L, int it) {
  fmg_ctx* c = b.c;
  const bool fine = L == c->Lmax;
  const int row = L * c->s.n_ir + it;
  const int nu = c->s.nu, k = c->s.cheb_degree;
  // fmgResidual (Alg 3.2): t_L, r_L and the restriction sweep down to level 0
  {
    OpDesc o = mkop(OP_RESIDUAL, L, L);
    o.wr = wr(c, L, L);
    o.wu_in = c->wu_cur[L];
    o.row = row;
    o.poff = b.slot(row, L);
    if (c->fine3 && !c->f3mat && c->chk && L >= 1) {  // (lean, z chunks: one partial row of CTAs per chunk)
      b.norms.pop_back();
      b.ptot = o.poff;
      const int nch = (c->g[L].n + c->chk_rc - 1) / c->chk_rc;
      o.poff = b.slot(row, L, (long long)(c->g[L].NX / 32) * c->mnyb[L] * nch);
      b.fine(5, o, fine ? 0 : -1);
    } else if (c->fine3) {
      b.fine(c->f3mat ? 4 : 0, o, fine ? 0 : -1);  // u_L generated on chip / staged (fmg_fine3.cu)
    }
    else b.grid(o, fine ? 0 : -1);
  }
  for (int l = L - 1; l >= 0; --l) {
    OpDesc q = mkop(OP_RESTRICT, l, L);
    q.wr = wr(c, l, L);
    q.row = row;
    q.poff = b.slot(row, l);
    b.grid(q, (fine && l == L - 1) ? 3 : -1);
  }
  for (int cyc = 1; cyc <= nu; ++cyc) {
    const int guess = cyc > 1, store = cyc < nu;
    if (guess) {  // fine-to-coarse s sweep: q_{l+1} = A ý_{l+1} + s_{l+1} (into W), s_l = R q_{l+1} (into T)
      for (int l = L - 1; l >= 0; --l) {
        OpDesc q = mkop(OP_SQ, l + 1, L);
        q.wr = wr(c, l + 1, L);
        q.smode = (l + 1 == L);  // s_L = 0
        b.grid(q);
        OpDesc r = mkop(OP_RESTRICT, l, L);
        r.smode = 1;
        r.wr = wr(c, l, L);
        b.grid(r);
      }
    }
    {  // level 0: the bracket (cFas1 with z_0 = 0), then M_0 = A_0^{-1}, ý_0, w_0 (+ correction)
      if (c->dim == 3) b.grid(mkop(OP_PROLONG, 0, L));  // (3D: Z_0 = 0, P u_{-1} = 0)
      OpDesc q = mkop(OP_CFAS1, 0, L);
      q.step = 1;
      q.guess = guess;
      q.store = 1;  // (selects the nu kernel: level 0 has no coarser level to prolongate from)
      q.wr = wr(c, 0, L);
      b.grid(q);
      OpDesc cc = mkop(OP_COARSE, 0, L);
      cc.guess = guess;
      cc.store = store;
      cc.wr = wr(c, 0, L);
      cc.wu_in = c->wu_cur[0];
      cc.wu_out = wu(c, 0, L);
      b.grid(cc);
    }
    const bool gs = c->s.smoother == 1;
    const int nsteps = gs ? ncolours(c) : k;  // GS: colour 0 in cFas1, then colours 1 .. (p+1)^d - 1
    for (int l = 1; l <= L; ++l) {
      if (c->fine3) {  // z_l generated on chip (fmg_fine3.cu); w_l, u_l materialised below the finest level
        add_fine3_level(b, l, L, fine, false);
        continue;
      }
      if (c->dim == 3) b.grid(mkop(OP_PROLONG, l, L));  // z_l = P w_{l-1}, P u_{l-1}
      for (int step = 1; step <= nsteps; ++step) {
        OpDesc q = mkop(step == 1 ? OP_CFAS1 : (gs ? OP_GS : OP_CHEB), l, L);
        q.step = gs ? step - 1 : step;
        q.last = step == nsteps;
        q.guess = guess;
        q.store = store;
        q.wr = wr(c, l, L);
        q.wu_in = c->wu_cur[l];
        q.wu_out = wu(c, l, L);
        b.grid(q, (fine && l == L && !store) ? (step == nsteps ? 5 : 1) : -1);
      }
    }
  }
  for (int l = 0; l <= L; ++l) c->wu_cur[l] = wu(c, l, L);
}

void build_iteration(Builder& b, int L, int it) {
  fmg_ctx* c = b.c;
  // nu > 1, or KC kept for the initial coarse solve only (one GPU, lc = 0):
  // every level of the iteration is a grid op, level 0 through cFas1 +
  // k_coarse_nu (with nu = 1 its one cycle has guess = store = 0, i.e. the
  // plain V(0,1) cycle of Alg 3.1)
  if (c->s.nu > 1 || (c->lc == 0 && c->G == 1)) {
    build_iteration_nu(b, L, it);
    return;
  }
  const int lc = c->lc;
  const bool fine = L == c->Lmax;
  const int row = L * c->s.n_ir + it;
  const int P = c->p;
  if (L > lc) {
    OpDesc o = mkop(OP_RESIDUAL, L, L);
    o.wr = wr(c, L, L);
    o.wu_in = c->wu_cur[L];
    o.row = row;
    o.poff = b.slot(row, L);
    if (c->fine3 && !c->f3mat) {  // u_L generated on chip from ú_L (BFP ghost planes) and u_{L-1} (fmg_fine3.cu)
      b.xchg(XA_SU, L, P);
      b.xchg(XA_U, L - 1, 2 * P);
      b.fine(0, o, fine ? 0 : -1);
    } else {
      b.xchg(XA_U, L, P);
      if (c->fine3) b.fine(4, o, fine ? 0 : -1);
      else b.grid(o, fine ? 0 : -1);
    }
    for (int l = L - 1; l > lc; --l) {
      b.xchg(XA_T, l + 1, 2 * P - 1);
      OpDesc q = mkop(OP_RESTRICT, l, L);
      q.wr = wr(c, l, L);
      q.row = row;
      q.poff = b.slot(row, l);
      b.grid(q, (fine && l == L - 1) ? 3 : -1);
    }
  }
  // levels 0..lc: KC (restriction tail, coarse solve, cFas + correction);
  // with z slabs every rank runs it on the gathered t_{lc+1} (replicated)
  if (L > lc) b.xchg(XA_T, lc + 1, 0, 1);
  KcDesc d = mkkc(c, 1);
  d.L = L;
  d.it = it;
  d.row0 = row;
  d.nrows = 1;
  b.kc(d);
  for (int l = 0; l <= lc; ++l) {
    b.kc_norm(row, l);
    c->wu_cur[l] = wu(c, l, L);
  }
  const int k = c->s.cheb_degree;
  for (int l = lc + 1; l <= L; ++l) {
    if (c->fine3) {  // z_l generated on chip; b_l in the t_l buffer (fmg_fine3.cu)
      add_fine3_level(b, l, L, fine, true);
      c->wu_cur[l] = wu(c, l, L);
      continue;
    }
    if (c->dim == 3) {  // z_l = P w_{l-1}, P u_{l-1} (fmg_march3.cu k_m3_prolong)
      b.xchg(XA_W, l - 1, P);
      b.xchg(XA_U, l - 1, P);
      OpDesc q = mkop(OP_PROLONG, l, L);
      b.grid(q);
      b.xchg(XA_Z, l, P);
    }
    const bool gs = c->s.smoother == 1;
    const int nsteps = gs ? ncolours(c) : k;  // GS: colour 0 in cFas1, then colours 1 .. (p+1)^d - 1
    for (int step = 1; step <= nsteps; ++step) {
      if (step >= 2) b.xchg(gs ? XA_Y1 : (step == 2 ? XA_B : ((step - 1) & 1 ? XA_Y1 : XA_Y0)), l, P);
      OpDesc q = mkop(step == 1 ? OP_CFAS1 : (gs ? OP_GS : OP_CHEB), l, L);
      q.step = gs ? step - 1 : step;
      q.last = step == nsteps;
      q.wr = wr(c, l, L);
      q.wu_in = c->wu_cur[l];
      q.wu_out = wu(c, l, L);
      b.grid(q, (fine && l == L) ? (step == nsteps ? 5 : 1) : -1);
    }
    c->wu_cur[l] = wu(c, l, L);
  }
}

// Alg 3.3 up to FMG level Lstop (iters_last IR iterations there).  One KC
// launch runs the coarse-grid solve and every FMG level L <= lc in full.
void build_solve(Builder& b, int Lstop, int iters_last) {
  fmg_ctx* c = b.c;
  const int lc = c->lc;
  for (int l = 0; l <= c->Lmax; ++l) c->wu_cur[l] = wu(c, l, l);
  KcDesc d = mkkc(c, 0);
  d.Llast = std::min(Lstop, lc);
  d.iters_last = (Lstop <= lc) ? iters_last : c->s.n_ir;
  d.row0 = c->s.n_ir;  // (L = 1, it = 0)
  d.nrows = d.Llast >= 1 ? (d.Llast - 1) * c->s.n_ir + d.iters_last : 0;
  b.kc(d);  // coarse-grid solve PAPER.md:786, FMG levels 1..min(Lstop, lc)
  c->wu_cur[0] = wu(c, 0, 0);
  for (int L = 1; L <= d.Llast; ++L) {
    c->wu_cur[L] = wu(c, L, L);
    int iters = (L == d.Llast) ? d.iters_last : c->s.n_ir;
    for (int it = 0; it < iters; ++it) {
      for (int l = 0; l <= L; ++l) {
        b.kc_norm(L * c->s.n_ir + it, l);
        c->wu_cur[l] = wu(c, l, L);
      }
    }
  }
  for (int L = lc + 1; L <= Lstop; ++L) {
    // push level PAPER.md:788: ú_L = 0 (zeroed at solve start); the widening of
    // ú_{0..L-1} is value-preserving and happens at the next encode.
    c->wu_cur[L] = wu(c, L, L);
    // u_L = dec ú_L + P u_{L-1} = P u_{L-1} for the first residual
    if (c->fine3 && !c->f3mat) {
      // u_{L-1} = dec ú_{L-1} + P u_{L-2}: a grid level L-1 was the finest
      // level of FMG level L-1, whose kernels keep no u array (fmg_fine3.cu);
      // the cluster kernel writes u_l of its levels <= lc itself
      if (L - 1 > lc) {
        b.xchg(XA_U, L - 2, c->p);
        OpDesc o = mkop(OP_DECODE, L - 1, L - 1);
        o.wu_in = c->wu_cur[L - 1];
        o.step = 1;
        b.fine(3, o, -1);  // (L - 1 > lc >= 0: a coarser level exists)
      }
    } else {
      b.xchg(XA_U, L - 1, c->p);
      OpDesc o = mkop(OP_DECODE, L, L);
      o.wu_in = c->wu_cur[L];
      if (c->fine3) {  // (materialised: u_L = P u_{L-1}, ú_L = 0)
        o.step = 1;
        b.fine(3, o, (L == c->Lmax) ? 2 : -1);
      } else {
        b.grid(o, (L == c->Lmax) ? 2 : -1);
      }
    }
    int iters = (L == Lstop) ? iters_last : c->s.n_ir;
    for (int it = 0; it < iters; ++it) build_iteration(b, L, it);
  }
}

void mark(fmg_ctx* c, int cls) {
  if (c->timing_cls == 4) cls = 4;  // class 4: every launch
  if (c->timing_cls == 1 && cls == 5) cls = 1;  // class 1 covers every fine cFas step
  if (c->timing_cls != cls || cls < 0) return;
  if (c->ev_used >= (int)c->ev.size()) return;
  cudaEventRecordWithFlags(c->ev[c->ev_used++], c->cur, cudaEventRecordExternal);
}


// Size the partial / norm-entry buffers for a built item list (before capture).
int prepare(fmg_ctx* c, const Builder& b, int slot) {
  c->nent_slot = slot;
  bool dirty = false;
  if (b.ptot > c->pbase_cap) {
    c->pbase = (double*)dalloc(c, sizeof(double) * b.ptot);
    if (!c->pbase) return FMG_ENOMEM;
    c->pbase_cap = b.ptot;
    dirty = true;
  }
  if ((int)b.norms.size() > c->nent_cap[slot]) {
    c->nent[slot] = (NormEntry*)dalloc(c, sizeof(NormEntry) * b.norms.size());
    if (!c->nent[slot]) return FMG_ENOMEM;
    c->nent_cap[slot] = (int)b.norms.size();
  }
  if (!b.norms.empty())
    cudaMemcpy(c->nent[slot], b.norms.data(), sizeof(NormEntry) * b.norms.size(), cudaMemcpyHostToDevice);
  if (dirty) {
    // the device context carries pbase
    std::vector<char> host(devctx_size());
    cudaMemcpy(host.data(), c->devctx, host.size(), cudaMemcpyDeviceToHost);
    set_devctx_pbase(host.data(), c->pbase);
    cudaMemcpy(c->devctx, host.data(), host.size(), cudaMemcpyHostToDevice);
  }
  return FMG_OK;
}

// Host copy of the device view of level l (mirrors fill_devctx).
LevelDev level_dev(const fmg_ctx* c, int l) {
  LevelDev v{};
  v.g = c->g[l];
  v.umant = c->u[l].mant;
  v.uexp = c->u[l].exps;
  v.ustride = c->u[l].stride;
  v.rmant = c->r[l].mant;
  v.rexp = c->r[l].exps;
  v.rstride = c->r[l].stride;
  v.gtab = c->gtab[l];
  v.U = c->Ul[l];
  v.T = c->Tl[l];
  v.W = c->Wl[l];
  v.ymant = c->ysec[l].mant;
  v.yexp = c->ysec[l].exps;
  v.ystride = c->ysec[l].stride;
  return v;
}

// Scratch buffer i as seen by level l: shifted so that level-l planes index
// globally inside the level's window (z slabs; identity otherwise).
double* sview(const fmg_ctx* c, int i, int l) {
  return c->sbase[i] ? c->sbase[i] - (long long)c->g[l].NX * c->g[l].NY * c->wlo[l] : c->buf[i];
}

// March-kernel arguments of a grid op.
MArgs march_args(const fmg_ctx* c, const OpDesc& o) {
  MArgs m{};
  m.type = o.type;
  m.l = o.l;
  m.L = o.L;
  m.step = o.step;
  m.last = o.last;
  m.wr = o.wr;
  m.wu_in = o.wu_in;
  m.wu_out = o.wu_out;
  m.RC = c->mrc[o.l];
  m.nxb = c->g[o.l].NX / 32;
  m.nitems = c->mitems[o.l];
  m.NYo = c->g[o.l].NY;
  m.nyb = c->mnyb[o.l];
  m.NZo = c->g[o.l].NZ;
  m.zlo = c->zlo[o.l];
  m.zhi = c->zhi[o.l];
  m.gs = c->s.smoother;
  m.poff = o.poff;
  m.lv = level_dev(c, o.l);
  const int lo = o.type == OP_RESTRICT ? o.l + 1 : o.l - 1;
  if (lo >= 0 && lo <= c->Lmax) m.lo = level_dev(c, lo);
  m.p = MPtrs{sview(c, 0, o.l), sview(c, 1, o.l), {sview(c, 2, o.l), sview(c, 3, o.l)}, sview(c, 4, o.l), sview(c, 5, o.l),
              c->buf[8], c->pbase, c->status};
  m.zoff = c->wlo[o.l];
  m.guess = o.guess;
  m.store = o.store;
  m.puonly = o.puonly;
  m.smode = o.smode;
  if (o.type == OP_RESTRICT && o.smode) m.lo.T = c->Wl[o.l + 1];  // s sweep: restrict q_{l+1} (in W)
  if (c->tma) {
    const int l = o.l;
    const CUtensorMap* U = c->tm_dev, *T = U + kMaxLev, *B = T + kMaxLev;  // device copies
    switch (o.type) {
      case OP_RESIDUAL: m.tm = U + l; break;
      case OP_RESTRICT: m.tm = T + l + 1; break;
      case OP_CFAS1: if (c->dim == 3) m.tm = B + l; break;
      case OP_GS: m.tm = B + 3 * kMaxLev + l; break;
      case OP_CHEB: m.tm = B + (o.step == 2 ? 1 : 2 + ((o.step - 1) & 1)) * kMaxLev + l; break;
      default: break;
    }
    m.tma = (o.type == OP_RESIDUAL || o.type == OP_GS || o.type == OP_CHEB || (o.type == OP_RESTRICT && !o.smode) ||
             (o.type == OP_CFAS1 && c->dim == 3)) ? 1 : 0;
    if (o.type == OP_RESTRICT && c->dim == 3) m.zoff = c->wlo[l + 1];  // (the staged array is t_{l+1})
  }
  return m;
}

// Arguments of a finest-level op (fmg_fine3.cu).
F3Args fine3_args(const fmg_ctx* c, const Item& it) {
  const OpDesc& o = it.op;
  const int l = o.l;
  F3Args a{};
  a.g = c->g[l];
  a.l = l;
  a.step = o.step;
  a.last = o.last;
  a.wr = o.wr;
  a.wu = o.wu_in;
  a.wu_out = o.wu_out;
  a.RC = c->mrc[l];
  a.nxb = c->g[l].NX / 32;
  a.nyb = c->mnyb[l];
  a.nitems = c->mitems[l];
  a.zlo = c->zlo[l];
  a.zhi = c->zhi[l];
  a.umant = c->u[l].mant;
  a.uexp = c->u[l].exps;
  a.ustride = c->u[l].stride;
  a.rmant = c->r[l].mant;
  a.rexp = c->r[l].exps;
  a.rstride = c->r[l].stride;
  a.gtab = c->gtab[l];
  a.T = c->Tl[l];
  a.Dv = sview(c, 4, l);
  a.Z = sview(c, 0, l);
  a.PU = sview(c, 5, l);
  a.U = c->Ul[l];
  a.W = c->Wl[l];
  a.zout = o.zout;
  a.wout = o.wout;
  a.uout = o.uout;
  // (levels of >= 2^16 blocks: below that the extra launch costs more than the
  // warp-cooperative codec it replaces)
  // (the residual's r_L encode needs no extra array: the lean form takes it too)
  a.tpb = (c->tpb ? (it.f3kind == 2 || it.f3kind == 4) : ((it.f3kind == 0 || it.f3kind == 5) && c->tpb0)) && a.wu <= 32 &&
          a.wu_out <= 32 && a.wr <= 32 && (long long)(a.zhi - a.zlo) * a.g.NY * a.nxb >= c->tpb_min;
  a.Yb = sview(c, 2, l);
  {
    const long long plane = (long long)c->g[l].NX * c->g[l].NY;
    a.my = c->my_base ? c->my_base - plane * c->wlo[l] : nullptr;
    a.ey = c->ey_base ? c->ey_base - plane / 32 * c->wlo[l] : nullptr;
    a.tpby = c->tpby && it.f3kind == 2 && o.last && !o.wout && !o.uout && o.wu_in == o.wu_out && o.wr <= 8 &&
             fine3_tpby_width(o.wu_in, o.wr) && (long long)(a.zhi - a.zlo) * a.g.NY * a.nxb >= c->tpb_min;
  }
  a.cfs = (it.f3kind == 1 || it.f3kind == 2) ? o.cfs : 0;
  // (the staged levels: cFas step 1 from a materialised z_l, add_fine3_level)
  a.f32s = c->f32s && (it.f3kind == 1 || it.f3kind == 2) && level_cfs(c, l);
  a.csc = c->csc;
  a.X1b = sview(c, 3, l);
  a.tmx1 = c->tm_dev + 11 * kMaxLev + l;
  a.tmz = c->tm_dev + 2 * kMaxLev + l;  // (fine boxes of the Z scratch, levels < Lmax)
  a.s2 = c->s2;
  a.pr2 = !(getenv("FMG_PR2") && atoi(getenv("FMG_PR2")) == 0);
  a.chk = c->chkbuf;
  a.chkrc = c->chk_rc;
  a.tmch = c->tm_dev + 12 * kMaxLev + l;
  a.tmy = c->tm_dev + 10 * kMaxLev + l;
  if (l >= 1) a.tmcu = c->tm_dev + 6 * kMaxLev + (l - 1);
  a.zoff = c->wlo[l];
  a.czoff = l >= 1 ? c->wlo[l - 1] : 0;
  a.pbase = c->pbase;
  a.poff = o.poff;
  a.status = c->status;
  const CUtensorMap* base = c->tm_dev;
  if (l >= 1) a.tmc = base + (it.f3kind == 0 || it.f3kind == 3 || it.f3kind == 5 ? 6 : 7) * kMaxLev + (l - 1);
  a.tmb = base + (it.f3kind == 4 ? 0 : 8) * kMaxLev + l;  // (kind 4: the u_l boxes)
  a.tmd = base + 9 * kMaxLev + l;
  return a;
}

// Launch one op / KC item of the list on c->cur.
void issue_item(fmg_ctx* c, const Item& it) {
  if (it.kind == 3) {
    mark(c, it.timed_cls);
    fine3_take_launches();
    launch_fine3(c->p, it.f3kind, c->cur, fine3_args(c, it), c->cf, c->s.cfas_fp32);
    mark(c, it.timed_cls);
    c->launches += fine3_take_launches();  // (an item can be several kernels: tpb epilogues, z chunks)
    return;
  }
  if (it.kind == 1) {
    mark(c, -2);
    launch_kc(c->dim, c->p, c->cur, c->devctx, it.kc, c->kc_cluster, c->kcl.bytes);
    mark(c, -2);
  } else {
    mark(c, it.timed_cls);
    {
      const MArgs m = march_args(c, it.op);
      if (it.op.type == OP_COARSE) launch_coarse_nu(c->dim, c->p, c->cur, c->devctx, m);
      else if (c->dim == 2) launch_march(c->p, c->cur, c->devctx, m, c->cf);
      else launch_march3(c->p, c->cur, c->devctx, m, c->cf);
    }
    mark(c, it.timed_cls);
  }
  c->launches++;
}

// FP64 level array of an exchange item
double* xarray(fmg_ctx* c, int arr, int l) {
  switch (arr) {
    case XA_U: return c->Ul[l];
    case XA_T: return c->Tl[l];
    case XA_W: return c->Wl[l];
    case XA_Z: return sview(c, 0, l);
    case XA_B: return sview(c, 1, l);
    case XA_Y0: return sview(c, 2, l);
    case XA_D: return sview(c, 4, l);
    default: return sview(c, 3, l);
  }
}
// The raw buffers an exchange item moves, as (globally indexed base, bytes per
// plane): one FP64 array, or a section's mantissa words and exponents (the
// compressed ghost planes of the finest-level kernels).
struct XBuf {
  char* base;
  size_t plane;
};
int xbufs(fmg_ctx* c, int arr, int l, XBuf* out) {
  const Geom& g = c->g[l];
  if (arr == XA_SU) {
    const size_t bpp = (size_t)(g.NX / 32) * g.NY;
    out[0] = {(char*)c->u[l].mant, bpp * c->u[l].stride * sizeof(uint32_t)};
    out[1] = {(char*)c->u[l].exps, bpp};
    return 2;
  }
  out[0] = {(char*)xarray(c, arr, l), (size_t)g.NX * g.NY * sizeof(double)};
  return 1;
}

// ---- exchange plan (shared by virtual slabs and NCCL ranks) ----------------
// Rank r of G equal slabs of NZ planes: the plane runs it receives (ghost
// planes [zlo-h, zlo) and [zhi, zhi+h), or every foreign plane for a gather)
// from their owners, and the runs of its own planes the other ranks receive
// from it.  Both sides list a pair's runs in increasing z, so NCCL
// send/recv pairs match.
struct XPiece {
  int peer, z0, z1, send;
};
std::vector<XPiece> slab_plan(int NZ, int G, int r, int h, int gather) {
  std::vector<XPiece> out;
  const int slab = NZ / G;
  auto ghost = [&](int s, int k, int& a, int& b) {  // k = 0 low, 1 high ghost run of rank s
    const int zlo = s * slab, zhi = (s + 1) * slab;
    if (gather) {
      a = k == 0 ? 0 : zhi;
      b = k == 0 ? zlo : NZ;
    } else {
      a = k == 0 ? std::max(0, zlo - h) : zhi;
      b = k == 0 ? zlo : std::min(NZ, zhi + h);
    }
  };
  for (int s = 0; s < G; ++s) {
    if (s == r) continue;
    // receive from owner s: my ghost runs within s's planes
    for (int k = 0; k < 2; ++k) {
      int a, b;
      ghost(r, k, a, b);
      a = std::max(a, s * slab);
      b = std::min(b, (s + 1) * slab);
      if (a < b) out.push_back({s, a, b, 0});
    }
    // send to s: s's ghost runs within my planes
    for (int k = 0; k < 2; ++k) {
      int a, b;
      ghost(s, k, a, b);
      a = std::max(a, r * slab);
      b = std::min(b, (r + 1) * slab);
      if (a < b) out.push_back({s, a, b, 1});
    }
  }
  return out;
}

struct NcclApi {
  bool ok = false;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
};

// NCCL is resolved at run time (the torch-bundled libnccl.so.2 is normally
// already loaded; FMG_NCCL_LIB names another copy), so libfmg.so carries no
// link-time NCCL dependency.
NcclApi& nccl() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h && getenv("FMG_NCCL_LIB")) h = dlopen(getenv("FMG_NCCL_LIB"), RTLD_NOW | RTLD_GLOBAL);
  if (!h) return api;
  api.getUniqueId = (decltype(api.getUniqueId))dlsym(h, "ncclGetUniqueId");
  api.commInitRank = (decltype(api.commInitRank))dlsym(h, "ncclCommInitRank");
  api.commDestroy = (decltype(api.commDestroy))dlsym(h, "ncclCommDestroy");
  api.send = (decltype(api.send))dlsym(h, "ncclSend");
  api.recv = (decltype(api.recv))dlsym(h, "ncclRecv");
  api.allGather = (decltype(api.allGather))dlsym(h, "ncclAllGather");
  api.allReduce = (decltype(api.allReduce))dlsym(h, "ncclAllReduce");
  api.groupStart = (decltype(api.groupStart))dlsym(h, "ncclGroupStart");
  api.groupEnd = (decltype(api.groupEnd))dlsym(h, "ncclGroupEnd");
  api.ok = api.getUniqueId && api.commInitRank && api.commDestroy && api.send && api.recv && api.allGather &&
           api.allReduce && api.groupStart && api.groupEnd;
  return api;
}

// Multi-GPU slabs: the same plan as grouped NCCL point-to-point transfers over
// NVLink (a gather is an in-place all-gather), on the context stream (captured
// into the solve graph).
int nccl_exchange(fmg_ctx* c, const Item& it) {
  NcclApi& N = nccl();
  const int l = it.xl;
  const Geom& g = c->g[l];
  ncclComm_t comm = (ncclComm_t)c->comm;
  XBuf xb[2];
  const int nb = xbufs(c, it.xarr, l, xb);
  if (it.xgather) {  // (FP64 t of level lc + 1: full arrays)
    const size_t plane = xb[0].plane;
    const size_t cnt = plane * (size_t)(g.NZ / c->G);
    if (N.allGather(xb[0].base + (size_t)c->zlo[l] * plane, xb[0].base, cnt, ncclUint8, comm, c->cur) != ncclSuccess)
      return FMG_ENCCL;
    return FMG_OK;
  }
  if (N.groupStart() != ncclSuccess) return FMG_ENCCL;
  bool ok = true;
  for (const XPiece& q : slab_plan(g.NZ, c->G, c->rank, it.xdepth, 0)) {
    for (int k = 0; k < nb; ++k) {
      char* p = xb[k].base + (size_t)q.z0 * xb[k].plane;
      const size_t cnt = xb[k].plane * (size_t)(q.z1 - q.z0);
      ok &= (q.send ? N.send(p, cnt, ncclUint8, q.peer, comm, c->cur)
                    : N.recv(p, cnt, ncclUint8, q.peer, comm, c->cur)) == ncclSuccess;
    }
  }
  ok &= N.groupEnd() == ncclSuccess;
  return ok ? FMG_OK : FMG_ENCCL;
}

// Virtual z slabs: fill the ghost planes (or, for a gather, every foreign plane)
// of each sub-context from the sub-context that owns them (D2D copies on the
// group's stream; the owners computed those planes in the previous item).
void group_exchange(fmg_ctx* grp, const Item& it) {
  const int G = (int)grp->sub.size(), l = it.xl;
  const Geom& g = grp->sub[0]->g[l];
  for (int r = 0; r < G; ++r) {
    fmg_ctx* dst = grp->sub[r];
    for (const XPiece& q : slab_plan(g.NZ, G, r, it.xdepth, it.xgather)) {
      if (q.send) continue;  // (the receiving side performs each copy)
      XBuf xd[2], xs[2];
      const int nb = xbufs(dst, it.xarr, l, xd);
      xbufs(grp->sub[q.peer], it.xarr, l, xs);
      for (int k = 0; k < nb; ++k)
        cudaMemcpyAsync(xd[k].base + (size_t)q.z0 * xd[k].plane, xs[k].base + (size_t)q.z0 * xs[k].plane,
                        xd[k].plane * (q.z1 - q.z0), cudaMemcpyDeviceToDevice, dst->cur);
    }
  }
}

// Host-staged slabs (fmg_create_hostx): the same plan, each piece copied
// through host memory and delivered by the caller's transport.
int host_exchange(fmg_ctx* c, const Item& it) {
  const int l = it.xl;
  const Geom& g = c->g[l];
  XBuf xb[2];
  const int nb = xbufs(c, it.xarr, l, xb);
  if (cudaStreamSynchronize(c->cur) != cudaSuccess) return FMG_ECUDA;
  std::vector<std::vector<char>> stage;
  std::vector<int> peer, send;
  std::vector<void*> buf;
  std::vector<int64_t> bytes;
  std::vector<char*> dev;
  for (const XPiece& q : slab_plan(g.NZ, c->G, c->rank, it.xgather ? 0 : it.xdepth, it.xgather)) {
    for (int k = 0; k < nb; ++k) {
      char* d = xb[k].base + (size_t)q.z0 * xb[k].plane;
      const size_t n = xb[k].plane * (size_t)(q.z1 - q.z0);
      stage.emplace_back(n);
      if (q.send && cudaMemcpy(stage.back().data(), d, n, cudaMemcpyDeviceToHost) != cudaSuccess) return FMG_ECUDA;
      peer.push_back(q.peer);
      send.push_back(q.send);
      bytes.push_back((int64_t)n);
      dev.push_back(d);
    }
  }
  for (auto& v : stage) buf.push_back(v.data());
  if (!buf.empty() && c->xfer(c->xfer_user, (int)buf.size(), peer.data(), send.data(), buf.data(), bytes.data()) != 0)
    return FMG_ENCCL;
  for (size_t i = 0; i < buf.size(); ++i)
    if (!send[i] && cudaMemcpy(dev[i], buf[i], (size_t)bytes[i], cudaMemcpyHostToDevice) != cudaSuccess) return FMG_ECUDA;
  return FMG_OK;
}

// A grid item k_m_fused can take (2D, one GPU, Chebyshev, nu = 1, untimed): a
// restriction / cFas step 1 / Chebyshev step whose level has at most
// march_fused_warps() work items.  FMG_FUSE2=0 disables the fusion.
static bool fusible(const fmg_ctx* c, const Item& it) {
  if (it.kind != 0 || it.timed_cls >= 0 || c->dim != 2 || c->tma || c->s.smoother != 0 || c->timing_cls == 4)
    return false;
  const OpDesc& o = it.op;
  if (o.guess || o.store || o.smode) return false;
  if (o.type != OP_RESTRICT && o.type != OP_CFAS1 && o.type != OP_CHEB) return false;
  return c->mitems[o.l] <= march_fused_warps();
}

// Issue every item on c->cur (inside a capture or directly), then the deferred norms.
void issue(fmg_ctx* c, const Builder& b) {
  const bool fuse2 = getenv("FMG_FUSE2") && atoi(getenv("FMG_FUSE2")) != 0;  // (read at every capture; off until measured)
  // FMG_SYNC_DEBUG=1 (direct runs only): synchronise after every launch and
  // report the first failing item.
  const bool dbg = c->cur == c->st && getenv("FMG_SYNC_DEBUG") != nullptr;
  if (dbg) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) fprintf(stderr, "[fmg] pending CUDA error before issue: %s\n", cudaGetErrorString(e));
  }
  for (size_t ii = 0; ii < b.items.size(); ++ii) {
    const Item& it = b.items[ii];
    if (it.kind == 2) {  // ghost planes: NCCL ranks (single-rank contexts have none)
      if (c->comm && nccl_exchange(c, it) != FMG_OK) c->nccl_err = 1;
      if (c->xfer && host_exchange(c, it) != FMG_OK) c->nccl_err = 1;
      continue;
    }
    if (fuse2 && !dbg && fusible(c, it)) {  // a run of dependent small 2D ops: one launch
      size_t jj = ii;
      MFused f{};
      while (jj < b.items.size() && f.n < MFUSED_OPS && fusible(c, b.items[jj])) f.op[f.n++] = march_args(c, b.items[jj++].op);
      if (f.n >= 2) {
        launch_march_fused(c->p, c->cur, c->devctx, f, c->cf);
        c->launches++;
        ii = jj - 1;
        continue;
      }
    }
    issue_item(c, it);
    if (dbg) {
      cudaError_t e = cudaStreamSynchronize(c->cur);
      if (e == cudaSuccess) e = cudaGetLastError();
      if (e != cudaSuccess) {
        fprintf(stderr, "[fmg] CUDA error in item kind=%d type=%d l=%d L=%d: %s\n", it.kind, it.op.type, it.op.l,
                it.kind ? it.kc.L : it.op.L, cudaGetErrorString(e));
        return;
      }
    }
  }
  launch_norms_all(c->cur, c->devctx, c->nent[c->nent_slot], (int)b.norms.size());
  c->launches++;
}

// Group (virtual slabs): every item on every sub-context in rank order, the
// exchanges in between, all on one stream (no cross-launch waiting).
void issue_group(fmg_ctx* grp, const Builder& b) {
  for (const Item& it : b.items) {
    if (it.kind == 2) {
      group_exchange(grp, it);
      continue;
    }
    for (fmg_ctx* s : grp->sub) issue_item(s, it);
  }
  for (fmg_ctx* s : grp->sub) {
    launch_norms_all(s->cur, s->devctx, s->nent[s->nent_slot], (int)b.norms.size());
    s->launches++;
  }
}

void zero_sections(fmg_ctx* c) {
  for (int l = 0; l <= c->Lmax; ++l) {
    const long long bpp = (long long)(c->g[l].NX / 32) * c->g[l].NY, b0 = bpp * c->wlo[l];
    const long long nb = bpp * (c->whi[l] - c->wlo[l]);
    cudaMemsetAsync(c->u[l].mant + b0 * c->u[l].stride, 0, sizeof(uint32_t) * nb * c->u[l].stride, c->cur);
    cudaMemsetAsync(c->u[l].exps + b0, 0x80, nb, c->cur);
  }
  cudaMemsetAsync(c->norms_dev, 0, sizeof(double) * c->levels * c->s.n_ir * c->levels, c->cur);
}

int cuda_err(cudaError_t e) {
  if (e == cudaSuccess) return FMG_OK;
  if (e == cudaErrorMemoryAllocation) return FMG_ENOMEM;
  return FMG_ECUDA;
}

int sync_check(fmg_ctx* c) {
  cudaError_t e = cudaStreamSynchronize(c->st);
  if (e != cudaSuccess) return cuda_err(e);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_err(e);
  int st = 0;
  e = cudaMemcpy(&st, c->status, sizeof(int), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_err(e);
  if (st) {
    cudaMemset(c->status, 0, sizeof(int));
    return FMG_ERANGE;
  }
  return FMG_OK;
}

// Run a freshly built item list directly on the user stream (no graph).
int run_direct(fmg_ctx* c, Builder& b) {
  c->cur = c->st;
  int save = c->timing_cls;
  long long save_l = c->launches;
  c->timing_cls = -1;
  cudaStreamSynchronize(c->st);
  int prc = prepare(c, b, 1);
  if (prc) return prc;
  c->nccl_err = 0;
  issue(c, b);
  c->timing_cls = save;
  c->launches = save_l;
  if (c->nccl_err) return FMG_ENCCL;
  return sync_check(c);
}

}  // namespace

namespace fmg {
void kc_debug(int on);
int kc_stamps(unsigned long long* out);
}

extern "C" {

/* debug: phase timestamps (globaltimer ns, CTA 0 after every cluster barrier)
 * of the last KC launch; returns the stamp count when `stamps` is non-null. */
int fmg_debug_kc(int on, unsigned long long* stamps) {
  if (stamps) {
    cudaDeviceSynchronize();
    return fmg::kc_stamps(stamps);
  }
  fmg::kc_debug(on);
  return 0;
}

int fmg_set_allocator(fmg_alloc_fn alloc, fmg_free_fn free_fn, void* user) {
  if ((alloc == nullptr) != (free_fn == nullptr)) return FMG_EINVAL;
  g_alloc = alloc;
  g_free = free_fn;
  g_alloc_user = user;
  return FMG_OK;
}

static int check_args(int dim, int p, int levels, const fmg_schedule* s) {
  if ((dim != 2 && dim != 3) || p < 1 || p > 3 || levels < 1 || levels > kMaxLev) return FMG_EINVAL;
  if (s->b_u < 2 || s->b_r < 2 || s->k_u < 0 || s->k_r < 0 || s->n_ir < 1 || s->cheb_degree < 1 ||
      s->cheb_degree > 8 || !(s->lambda_hi > 0) || !(s->alpha > 1) || s->smoother < 0 || s->smoother > 1 ||
      s->nu < 0 || s->nu > 8)
    return FMG_EINVAL;
  // nu > 1 on the GPU: Chebyshev of degree >= 2 or multicolour GS; one GPU (no z slabs)
  if (s->nu > 1 && s->smoother == 0 && s->cheb_degree < 2) return FMG_EINVAL;
  // FP32 cFas (reading R28): the finest-level kernels' Chebyshev path only
  if (s->cfas_fp32 && (dim != 3 || s->smoother != 0 || s->nu > 1 || s->cheb_degree < 2 || s->cheb_degree > 3))
    return FMG_EINVAL;
  const int Lmax = levels - 1;
  if (s->b_u + s->k_u * Lmax > 54 || s->b_r + s->k_r * Lmax > 54) return FMG_EINVAL;
  return FMG_OK;
}

static int create_impl(int dim, int p, int levels, const fmg_schedule* s, void* stream, int G, int rank,
                       fmg_ctx** out) {
  if (!out || !s) return FMG_EINVAL;
  *out = nullptr;
  if (check_args(dim, p, levels, s)) return FMG_EINVAL;
  int Lmax = levels - 1;
  fmg_ctx* c = new fmg_ctx();
  c->dim = dim; c->p = p; c->levels = levels; c->Lmax = Lmax; c->s = *s;
  c->G = G;
  c->rank = rank;
  c->st = (cudaStream_t)stream;
  c->afn = g_alloc; c->ffn = g_free; c->auser = g_alloc_user;
  if (cudaStreamCreateWithFlags(&c->cap, cudaStreamNonBlocking) != cudaSuccess) { delete c; return FMG_ECUDA; }
  set_kernel_attributes();
  march_set_attributes();
  march3_set_attributes();
  fine3_set_attributes();
  if (s->nu > 1 && G > 1) {  // (nu > 1: single GPU this round)
    fmg_destroy(c);
    return FMG_EINVAL;
  }
  if (getenv("FMG_SYNC_DEBUG")) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) fprintf(stderr, "[fmg] set_kernel_attributes: %s\n", cudaGetErrorString(e));
  }
  build_coefs(dim, p, s->lambda_hi, s->alpha, s->cheb_degree, &c->cf);
  const int TY = dim == 3 ? 8 : 16, TZ = dim == 3 ? 4 : 1;  // (tile counts of the norm-partial table)
  int rc = FMG_OK;
  long long tot_parts = 0;
  DevCtxDesc dd{};
  for (int l = 0; l <= Lmax; ++l) {
    Geom& g = c->g[l];
    g.l = l;
    g.n = p << (l + 1);
    g.NX = ((g.n + 31) / 32) * 32;
    g.NY = g.n;
    g.NZ = dim == 3 ? g.n : 1;
    g.size = (long long)g.NX * g.NY * g.NZ;
    g.nblk = g.size / 32;
    c->tiles[l][0] = g.NX / 32;
    c->tiles[l][1] = (g.NY + TY - 1) / TY;
    c->tiles[l][2] = (g.NZ + TZ - 1) / TZ;
    int nt = c->tiles[l][0] * c->tiles[l][1] * c->tiles[l][2];
    c->u[l].stride = wu(c, l, Lmax);
    c->r[l].stride = wr(c, l, Lmax);
    c->gtab[l] = (double*)dalloc(c, sizeof(double) * g.n);
    if (!c->gtab[l]) { rc = FMG_ENOMEM; break; }
    std::vector<double> gt(g.n);
    build_rhs_table(p, l, gt.data());
    cudaMemcpy(c->gtab[l], gt.data(), sizeof(double) * g.n, cudaMemcpyHostToDevice);
    c->part_off[l] = tot_parts;
    tot_parts += nt;
    int nxb = g.NX / 32;
    if (dim == 2) {
      // 2D row march: ~3600 warps of work (148 SMs x 24 warps) per full level
      long long want = 148LL * 24;
      int rc = (int)(((long long)g.NY * nxb + want - 1) / want);
      rc = std::max(1, std::min(rc, g.NY));
      c->mrc[l] = rc;
      c->mitems[l] = nxb * ((g.NY + rc - 1) / rc);
    }  // (3D march geometry: after the KC plan, per z slab)
  }
  // KC (one thread-block cluster, fmg_kc.cu) owns levels 0..lc: the largest
  // prefix with <= 2 BFP blocks per KC warp whose data fits the cluster's
  // distributed shared memory (env FMG_LC caps lc, FMG_KC_CLUSTER forces NC).
  if (rc == FMG_OK) {
    int lc_cap = Lmax;
    if (const char* e = getenv("FMG_LC")) lc_cap = std::min(lc_cap, atoi(e));
    if (s->nu > 1) lc_cap = 0;  // nu > 1: KC runs the initial coarse solve only; the grid kernels do the rest
    int ust[kMaxLev], rst[kMaxLev];
    for (int l = 0; l <= Lmax; ++l) {
      ust[l] = c->u[l].stride;
      rst[l] = c->r[l].stride;
    }
    if (kc_plan(dim, p, Lmax, c->g, ust, rst, s->n_ir, lc_cap, &c->kcl, &c->lc, &c->kc_cluster)) rc = FMG_ECUDA;
    // Measured (profiles/r1e_summary.md): KC beats the
    // PDL-chained grid kernels only when it runs the whole FMG in one launch
    // (lc = Lmax, e.g. C1). Otherwise, on one GPU, its levels 1..lc go to the
    // grid path and KC keeps the coarse solve (C2 -6 %, C3 -1.3 %, C4 flat).
    // Slab contexts keep the plan: their grid levels need NZ % G == 0.
    // FMG_LC overrides.
    else if (!getenv("FMG_LC") && G == 1 && c->lc > 0 && c->lc < Lmax) {
      if (kc_plan(dim, p, Lmax, c->g, ust, rst, s->n_ir, 0, &c->kcl, &c->lc, &c->kc_cluster)) rc = FMG_ECUDA;
    }
    c->kc_tw = c->kc_cluster * kc_warps_per_cta();
  }
  // z slabs: rank r owns planes [r NZ/G, (r+1) NZ/G) of every grid level l > lc
  for (int l = 0; l <= Lmax && rc == FMG_OK; ++l) {
    const Geom& g = c->g[l];
    if (G > 1 && l > c->lc) {
      if (dim != 3 || g.NZ % G != 0) rc = FMG_EINVAL;
      c->zlo[l] = rank * (g.NZ / G);
      c->zhi[l] = (rank + 1) * (g.NZ / G);
    } else {
      c->zlo[l] = 0;
      c->zhi[l] = g.NZ;
    }
    if (dim == 3) {
      // 3D plane march: CTAs of 32 x 8 columns over this rank's planes, the
      // planes in nch z chunks of rcz.  Measured (tools/ab_env.py, FMG_NCHL;
      // DESIGN.md §4.3): large p = 1 levels gain from ~10 waves of the staged
      // kernels' CTAs (C3 finest 2 -> 6 chunks: -0.47 ms), small levels whose
      // chunks would be shorter than the 2p halo planes from one wave of long
      // chunks (C4 levels 3, 4: -1.8 ms); the rest keeps ~4 waves of 2 CTAs
      // per SM.  FMG_NCH forces the count (0: the round-1 rule everywhere).
      const int nxb = g.NX / 32, nz = c->zhi[l] - c->zlo[l];
      int nyb = (g.NY + march3_rows() - 1) / march3_rows();
      int tiles = nxb * nyb;
      const char* ev = getenv("FMG_NCH");
      const int fz = ev ? atoi(ev) : -1;
      const int nch0 = std::min(nz, (148 * 2 * 4 + tiles - 1) / tiles);
      // (the march3 kernels' per-tile partial table holds nxb (NY/8) (NZ/4) slots, 8 per CTA)
      const int nchmax = std::max(nch0, std::min(nz, (c->tiles[l][1] * c->tiles[l][2]) / (8 * nyb)));
      int nch = nch0;
      if (fz > 0) {
        nch = fz;
      } else if (fz < 0) {
        const int slots = 148 * (p == 1 ? 4 : p == 2 ? 3 : 2);  // staged kernels' CTAs per SM
        const int rk0 = (nz + nch0 - 1) / nch0;
        if (2 * tiles >= slots) {
          if (p == 1) nch = std::max(nch0, std::min((10 * slots + tiles - 1) / tiles, nz / 8));
        } else if (rk0 < 2 * p) {
          nch = std::max(1, std::min(nz, slots / tiles));
        }
      }
      if (const char* el = getenv("FMG_NCHL")) {  // per-level override "l:n,l:n" (tools/ab_env.py)
        for (const char* q = el; *q;) {
          int ll = 0, nn = 0, used = 0;
          if (sscanf(q, "%d:%d%n", &ll, &nn, &used) != 2) break;
          if (ll == l && nn > 0) nch = nn;
          q += used;
          if (*q == ',') ++q;
        }
      }
      nch = std::max(1, std::min({nch, nz, nchmax}));
      int rcz = (nz + nch - 1) / nch;
      nch = (nz + rcz - 1) / rcz;
      c->mnyb[l] = nyb;
      c->mrc[l] = rcz;
      c->mitems[l] = tiles * nch;
    }
  }
  // Plane windows (memory partition of z slabs) and the compact sections.
  for (int l = 0; l <= Lmax && rc == FMG_OK; ++l) {
    const Geom& g = c->g[l];
    const bool part = G > 1 && l > c->lc + 1;  // (level lc + 1: gathered in full for KC)
    c->wlo[l] = part ? std::max(0, c->zlo[l] - 2 * p) : 0;
    c->whi[l] = part ? std::min(g.NZ, c->zhi[l] + 2 * p) : g.NZ;
    const long long bpp = (long long)(g.NX / 32) * g.NY, nb = bpp * (c->whi[l] - c->wlo[l]), b0 = bpp * c->wlo[l];
    auto sec = [&](Sec& q, int stride) {
      q.stride = stride;
      uint32_t* m = (uint32_t*)dalloc(c, sizeof(uint32_t) * nb * stride);
      int8_t* e = (int8_t*)dalloc(c, nb + 16);  // (+16: aligned 4-byte exponent reads, fmg_fine3.cu)
      if (!m || !e) return false;
      q.mant = m - b0 * stride;  // (global block indexing)
      q.exps = e - b0;
      return true;
    };
    if (!sec(c->u[l], wu(c, l, Lmax)) || !sec(c->r[l], wr(c, l, Lmax)) ||
        (s->nu > 1 && !sec(c->ysec[l], wr(c, l, Lmax))))
      rc = FMG_ENOMEM;
  }
  // Finest-level kernels (fmg_fine3.cu): 3D, Chebyshev
  // degree 2-3, nu = 1, a grid level above the cluster kernel's, b_u <= 10
  // (the residual's three-block section records fit one warp).
  {
    const char* e = getenv("FMG_FINE3");
    c->fine3 = rc == FMG_OK && dim == 3 && s->nu <= 1 && s->smoother == 0 &&
               (s->cheb_degree == 2 || s->cheb_degree == 3) && Lmax > c->lc && s->b_u <= 10 && !(e && atoi(e) == 0);
  }
  if (rc == FMG_OK && s->cfas_fp32 && !c->fine3) rc = FMG_EINVAL;  // (FP32 cFas runs in the finest-level kernels)
  // FP64 workspace.  Level arrays u_l, t_l, w_l (padded level layout); the
  // scratch Z, B, Y[2], PU of the level-by-level kernels and the Chebyshev
  // direction Dv, each used by one level at a time.  With fine3 the finest
  // level keeps only t (which also holds b) and, for degree 3, Dv: its u, w
  // and the scratch of levels < Lmax are one level smaller.
  if (c->fine3) {
    // materialise u_L and P u_{L-1} when the two extra finest-size arrays fit
    // comfortably (half the device memory with everything else): faster for
    // Q3 and Q1 (the residual stages u_L; profiles/r2_summary.md); the lean
    // form is what makes C5's per-GPU share fit
    const char* e = getenv("FMG_F3MAT");
    size_t freeb = 0, totalb = 0;
    cudaMemGetInfo(&freeb, &totalb);
    double need = 0.0;
    for (int l = 0; l <= Lmax; ++l)
      need += 8.0 * (double)c->g[l].NX * c->g[l].NY * (c->whi[l] - c->wlo[l]) * (l == Lmax ? 5.0 : 3.0);
    c->f3mat = e ? atoi(e) != 0 : need < 0.5 * (double)totalb;
    // thread-per-block epilogues (fmg_fine3.cu k_f3_tpb): one more finest-size
    // array (y_k of the last Chebyshev step), with the materialised form;
    // measured faster (profiles/r2_summary.md).  FMG_TPB=0 disables.
    const char* et = getenv("FMG_TPB");
    const double ytop = 8.0 * (double)c->g[Lmax].NX * c->g[Lmax].NY * (c->whi[Lmax] - c->wlo[Lmax]);
    // (with room for X1 of the staged Chebyshev steps too: two more arrays)
    c->tpb = c->f3mat && (et ? atoi(et) != 0 : (e != nullptr || need + 2.0 * ytop < 0.5 * (double)totalb));
    // z_L = P w_{L-1} materialised in Y for the top level's cFas step 1 (one
    // GPU: its ghost planes would need an exchange).  FMG_CFS=0 disables.
    const char* ec = getenv("FMG_CFS");
    // FP32 cFas too (P w_{l-1}, b_l and y_j in float; FMG_CFS32=0 keeps its
    // generating kernels for the A/B)
    const char* e32 = getenv("FMG_CFS32");
    c->cfs = c->tpb && c->G == 1 && !(s->cfas_fp32 && e32 && atoi(e32) == 0) && !(ec && atoi(ec) == 0);
    // ... and the Chebyshev steps from materialised y_1, y_2 (one more
    // finest-size array X1; k_f3_staged<P, 3 / 4>): measured faster for
    // p = 3 (C4 145.2 -> 136.4 ms), flat for p = 1 (C3 20.35 / 20.49 ms), so
    // the default is p = 3; FMG_CSC=0/1 forces it.
    if (const char* em = getenv("FMG_TPB_MIN_BLOCKS")) c->tpb_min = atoll(em);
    // two input planes per iteration in the staged kernels: C4 126.9 -> 120.4 ms,
    // C3 flat (18.84 / 18.87), so the default is p = 3; FMG_S2=0/1 forces it
    c->s2 = p == 3;
    if (const char* e2 = getenv("FMG_S2")) c->s2 = atoi(e2) != 0;
    c->tpb0 = !(et && atoi(et) == 0);
    const char* es = getenv("FMG_CSC");
    c->csc = c->cfs && (es ? atoi(es) != 0 : p == 3);
    // FP32 cFas with the staged Chebyshev steps: z_l, b_l, y_j and d_2 stored
    // as float (half the bytes of the staged kernels, which are HBM-bound in
    // FP32: profiles/r2b_summary.md).  FMG_F32S=0 keeps FP64 storage.
    const char* efs = getenv("FMG_F32S");
    c->f32s = s->cfas_fp32 && c->cfs && (!c->csc || c->s2) && !(efs && atoi(efs) == 0);
  }
  for (int l = 0; l <= Lmax && rc == FMG_OK; ++l) {
    const long long plane = (long long)c->g[l].NX * c->g[l].NY, off = plane * c->wlo[l];
    const size_t bytes = sizeof(double) * plane * (c->whi[l] - c->wlo[l]);
    const bool top = c->fine3 && l == Lmax;
    auto arr = [&](double*& a) {
      double* q = (double*)dalloc(c, bytes);
      if (q) cudaMemset(q, 0, bytes);
      a = q ? q - off : nullptr;  // (global plane indexing)
      return q != nullptr;
    };
    if (!arr(c->Tl[l]) || ((!top || c->f3mat) && !arr(c->Ul[l])) || (!top && !arr(c->Wl[l]))) rc = FMG_ENOMEM;
  }
  {
    // scratch: each buffer serves one level at a time with that level's
    // window, so it is sized for the largest window it serves
    auto win = [&](int l) { return (size_t)c->g[l].NX * c->g[l].NY * (c->whi[l] - c->wlo[l]); };
    size_t scratch = 0;
    for (int l = 0; l <= (c->fine3 ? Lmax - 1 : Lmax); ++l) scratch = std::max(scratch, win(l));
    const bool dv = !c->fine3 || s->cheb_degree >= 3;
    // (fine3: every level's cFas runs the finest-level kernels, whose b_l
    // lives in the t_l buffer and whose y_{j-1} is recomputed: no B, Y scratch)
    for (int i = 0; i < 6 && rc == FMG_OK; ++i) {
      size_t n = i == 4 ? (dv ? win(Lmax) : 2) : ((i >= 1 && i <= 3) && c->fine3 ? 2 : scratch);
      if (i == 1 && c->fine3) n = win(0);  // (level 0's bracket b_0: cFas1 + k_coarse_nu)
      if (i == 5 && c->f3mat) n = win(Lmax);  // (P u_{L-1} at the finest level)
      if (i == 2 && c->tpb) n = win(Lmax);    // (y_k of the last Chebyshev step, k_f3_tpb)
      if (i == 3 && c->csc) n = win(Lmax);    // (X1: y_1, y_3 of the staged Chebyshev steps)
      const size_t bytes = sizeof(double) * n;
      c->buf[i] = (double*)dalloc(c, bytes);
      c->sbase[i] = c->buf[i];
      if (!c->buf[i]) rc = FMG_ENOMEM;
      else cudaMemset(c->buf[i], 0, bytes);
    }
  }
  // lean form: ý of the top level's last step as int8 mantissas + exponents
  // (1 byte per point) when that fits, for the thread-per-block correction
  // (k_f3_tpb<2>).  FMG_TPBY=0 disables.
  if (rc == FMG_OK && c->fine3 && !c->f3mat && !(getenv("FMG_TPBY") && atoi(getenv("FMG_TPBY")) == 0)) {
    const size_t pts = (size_t)c->g[Lmax].NX * c->g[Lmax].NY * (c->whi[Lmax] - c->wlo[Lmax]);
    size_t freeb = 0, totalb = 0;
    cudaMemGetInfo(&freeb, &totalb);
    if (freeb > pts + pts / 32 + ((size_t)4 << 30)) {
      c->my_base = (int8_t*)dalloc(c, pts + 64);
      c->ey_base = (int8_t*)dalloc(c, pts / 32 + 64);
      c->tpby = c->my_base && c->ey_base;
    }
  }
  // lean form on one GPU: the finest level's u_L (residual) and z_L (cFas
  // step 1) materialised in z chunks of chk_rc planes (+ the 2p halo) for the
  // staged kernels, instead of generated on every staged box (FMG_CHK=0:
  // generating kernels).  The buffer takes at most a quarter of the free memory
  // and 8 GB.
  if (rc == FMG_OK && c->fine3 && !c->f3mat && c->G == 1 && s->smoother == 0 &&
      !(getenv("FMG_CHK") && atoi(getenv("FMG_CHK")) == 0)) {
    const long long plane = (long long)c->g[Lmax].NX * c->g[Lmax].NY;
    size_t freeb = 0, totalb = 0;
    cudaMemGetInfo(&freeb, &totalb);
    const double budget = std::min((double)freeb / 4.0, 8.0 * (1 << 30));
    long long rcz = (long long)(budget / (8.0 * plane)) - 2 * p;
    if (const char* er = getenv("FMG_CHK_PLANES")) rcz = atoll(er);
    rcz = std::min<long long>(rcz, c->g[Lmax].n);
    if (rcz >= 8) {
      c->chkbuf = (double*)dalloc(c, sizeof(double) * plane * (rcz + 2 * p));
      if (c->chkbuf) {
        c->chk = true;
        c->chk_rc = (int)rcz;
      }
    }
  }
  if (rc == FMG_OK && s->nu > 1) {  // YO: dec ý of the previous cycle at the level being smoothed
    c->buf[8] = (double*)dalloc(c, sizeof(double) * c->g[Lmax].size);
    if (!c->buf[8]) rc = FMG_ENOMEM;
    else cudaMemset(c->buf[8], 0, sizeof(double) * c->g[Lmax].size);
  }
  for (int i = 6; i < 8 && rc == FMG_OK; ++i) {
    c->buf[i] = (double*)dalloc(c, sizeof(double) * 2 * c->g[c->lc].size);
    if (!c->buf[i]) rc = FMG_ENOMEM;
  }
  // TMA maps of the staged arrays (grid levels).  Measured: 3D
  // plane boxes gain 7-8 % (C3, C4) over per-lane cp.async, 2D rows of 36-40
  // doubles lose 0.4 % (C2), so the default is TMA in 3D only; FMG_TMA=1 forces
  // it in 2D too, FMG_TMA=0 turns it off.
  {
    const char* e = getenv("FMG_TMA");
    const int want = e ? atoi(e) : -1;
    c->tma = want == 1 || (want < 0 && dim == 3);
  }
  // (3D with the finest-level kernels: the maps are built with FMG_TMA=0 too;
  // k_f3_staged reads u_l through them, the march kernels go by c->tma)
  for (int l = 0; l <= Lmax && rc == FMG_OK && (c->tma || (dim == 3 && c->fine3)); ++l) {
    const Geom& g = c->g[l];
    bool ok = true;
    if (dim == 2) {
      // boxes start on 16-byte boundaries: halo rounded up to even (fmg_march.cu)
      const int pe = p + (p & 1);
      ok &= make_tmap(&c->tmU[l], c->Ul[l], g.NX, g.NY, 0, 32 + 2 * pe, 1);
      ok &= make_tmap(&c->tmT[l], c->Tl[l], g.NX, g.NY, 0, 64 + 4 * p, 1);
      for (int i = 0; i < 4; ++i) ok &= make_tmap(&c->tmB[i][l], c->buf[i], g.NX, g.NY, 0, 32 + 2 * pe, 1);
    } else if (c->fine3 && l == Lmax) {  // (fine3: the scratch is one level smaller; u only if materialised)
      if (c->f3mat)
        ok &= make_tmap(&c->tmU[l], c->Ul[l] + (long long)g.NX * g.NY * c->wlo[l], g.NX, g.NY, c->whi[l] - c->wlo[l],
                        40, 8 + 2 * p);
    } else {
      // maps over the level's plane window (TMA coordinates z - wlo)
      const long long off = (long long)g.NX * g.NY * c->wlo[l];
      const int nz = c->whi[l] - c->wlo[l];
      ok &= make_tmap(&c->tmU[l], c->Ul[l] + off, g.NX, g.NY, nz, 40, 8 + 2 * p);
      for (int i = 0; i < 4; ++i)
        if (!(c->fine3 && i >= 1))
          ok &= make_tmap(&c->tmB[i][l], c->sbase[i], g.NX, g.NY, nz, 40, 8 + 2 * p);
    }
    if (!ok) rc = FMG_ECUDA;
  }
  // 3D restriction (k_m3_restrict, TMA form): fine-plane boxes of t_l, l >= 1,
  // 64 + 4p wide from an even column, 16 + 4p - 2 rows
  for (int l = 1; l <= Lmax && rc == FMG_OK && c->tma && dim == 3; ++l) {
    const Geom& g = c->g[l];
    const long long off = (long long)g.NX * g.NY * c->wlo[l];
    if (!make_tmap(&c->tmT[l], c->Tl[l] + off, g.NX, g.NY, c->whi[l] - c->wlo[l], 64 + 4 * p, 16 + 4 * p - 2))
      rc = FMG_ECUDA;
  }
  // finest-level kernels: coarse boxes of u_l, w_l (l < Lmax), fine boxes of
  // t_l and of Dv (levels >= 1)
  for (int l = 0; l <= Lmax && rc == FMG_OK && c->fine3; ++l) {
    const Geom& g = c->g[l];
    int cbx = 0, cby = 0, rs = 0, nr = 0;
    fine3_box_dims(p, &cbx, &cby, &rs, &nr);
    bool ok = true;
    const long long off = (long long)g.NX * g.NY * c->wlo[l];
    const int nz = c->whi[l] - c->wlo[l];
    if (l < Lmax) {
      ok &= make_tmap(&c->tmCU[l], c->Ul[l] + off, g.NX, g.NY, nz, cbx, cby);
      ok &= make_tmap(&c->tmCW[l], c->Wl[l] + off, g.NX, g.NY, nz, cbx, cby);
    }
    if (l >= 1) {
      const int ef = c->f32s && level_cfs(c, l) ? 4 : 8;  // (float storage of b, d_2 at the staged levels)
      ok &= make_tmap(&c->tmFB[l], c->Tl[l] + off, g.NX, g.NY, nz, rs, nr, ef);
      if (s->cheb_degree >= 3) ok &= make_tmap(&c->tmFD[l], c->sbase[4], g.NX, g.NY, nz, rs, nr, ef);
      const int es = c->f32s ? 4 : 8;  // (float storage: float boxes of Y, X1 and the Z scratch)
      if (c->cfs) ok &= make_tmap(&c->tmYB[l], c->sbase[2], g.NX, g.NY, nz, rs, nr, es);
      if (c->csc) ok &= make_tmap(&c->tmX1[l], c->sbase[3], g.NX, g.NY, nz, rs, nr, es);
      if (c->f32s && l < Lmax) ok &= make_tmap(&c->tmB[0][l], c->sbase[0], g.NX, g.NY, nz, rs, nr, 4);
      if (c->chk) ok &= make_tmap(&c->tmCH[l], c->chkbuf, g.NX, g.NY, std::min<long long>(g.NZ, c->chk_rc + 2 * p), rs, nr);
    }
    if (!ok) rc = FMG_ECUDA;
  }
  if (rc == FMG_OK && (c->tma || c->fine3)) {
    std::vector<CUtensorMap> all(13 * kMaxLev);
    for (int l = 0; l < kMaxLev; ++l) {
      all[l] = c->tmU[l];
      all[kMaxLev + l] = c->tmT[l];
      for (int i = 0; i < 4; ++i) all[(2 + i) * kMaxLev + l] = c->tmB[i][l];
      all[6 * kMaxLev + l] = c->tmCU[l];
      all[7 * kMaxLev + l] = c->tmCW[l];
      all[8 * kMaxLev + l] = c->tmFB[l];
      all[9 * kMaxLev + l] = c->tmFD[l];
      all[10 * kMaxLev + l] = c->tmYB[l];
      all[11 * kMaxLev + l] = c->tmX1[l];
      all[12 * kMaxLev + l] = c->tmCH[l];
    }
    c->tm_dev = (CUtensorMap*)dalloc(c, sizeof(CUtensorMap) * all.size());  // (256-byte aligned)
    if (!c->tm_dev) rc = FMG_ENOMEM;
    else cudaMemcpy(c->tm_dev, all.data(), sizeof(CUtensorMap) * all.size(), cudaMemcpyHostToDevice);
  }
  if (rc == FMG_OK) {
    c->n0 = coarse_count(dim, p);
    std::vector<double> Ai((size_t)c->n0 * c->n0);
    if (build_coarse_inverse(dim, p, Ai.data())) rc = FMG_EINVAL;
    c->Ainv = (double*)dalloc(c, sizeof(double) * Ai.size());
    c->partials = (double*)dalloc(c, sizeof(double) * tot_parts);
    c->norms_dev = (double*)dalloc(c, sizeof(double) * levels * s->n_ir * levels);
    // error partials (2 per CTA of k_errors) and, on NCCL ranks, the norm log all-reduce
    c->err_part = (double*)dalloc(c, sizeof(double) * std::max<size_t>(2 * 148 * 16, (size_t)levels * levels * s->n_ir));
    c->status = (int*)dalloc(c, sizeof(int));
    int* counters = (int*)dalloc(c, sizeof(int) * kMaxLev);
    if (counters) cudaMemset(counters, 0, sizeof(int) * kMaxLev);
    dd.count = counters;
    c->devctx = dalloc(c, devctx_size());
    if (!c->Ainv || !c->partials || !c->norms_dev || !c->err_part || !c->status || !c->devctx)
      rc = FMG_ENOMEM;
    else {
      cudaMemcpy(c->Ainv, Ai.data(), sizeof(double) * Ai.size(), cudaMemcpyHostToDevice);
      cudaMemset(c->status, 0, sizeof(int));
      cudaMemset(c->norms_dev, 0, sizeof(double) * levels * s->n_ir * levels);
      dd.levels = levels;
      dd.n_ir = s->n_ir;
      dd.n0 = c->n0;
      for (int l = 0; l <= Lmax; ++l) {
        dd.g[l] = c->g[l];
        dd.u[l] = c->u[l];
        dd.r[l] = c->r[l];
        dd.gtab[l] = c->gtab[l];
        for (int k = 0; k < 3; ++k) dd.tiles[l][k] = c->tiles[l][k];
        dd.part[l] = c->partials + c->part_off[l];
        dd.Ul[l] = c->Ul[l];
        dd.Tl[l] = c->Tl[l];
        dd.Wl[l] = c->Wl[l];
      }
      dd.Z = c->buf[0];
      dd.B = c->buf[1];
      dd.Y[0] = c->buf[2];
      dd.Y[1] = c->buf[3];
      dd.Dv = c->buf[4];
      dd.PU = c->buf[5];
      dd.KS[0] = c->buf[6];
      dd.KS[1] = c->buf[7];
      dd.kc = c->kcl;
      dd.lc = c->lc;
      dd.n_cheb = s->cheb_degree;
      dd.smoother = s->smoother;
      dd.Ainv = c->Ainv;
      dd.norms = c->norms_dev;
      dd.status = c->status;
      dd.cf = c->cf;
      std::vector<char> host(devctx_size());
      fill_devctx(host.data(), dd);
      cudaMemcpy(c->devctx, host.data(), host.size(), cudaMemcpyHostToDevice);
    }
  }
  if (rc == FMG_OK) rc = cuda_err(cudaDeviceSynchronize());
  if (getenv("FMG_SYNC_DEBUG")) {
    cudaError_t e = cudaGetLastError();
    fprintf(stderr, "[fmg] create: rc=%d last=%s lc=%d kc_cluster=%d\n", rc, cudaGetErrorString(e), c->lc,
            c->kc_cluster);
  }
  if (rc != FMG_OK) {
    fmg_destroy(c);
    return rc;
  }
  *out = c;
  return FMG_OK;
}

int fmg_create(int dim, int p, int levels, const fmg_schedule* s, void* stream, fmg_ctx** out) {
  return create_impl(dim, p, levels, s, stream, 1, 0, out);
}

int fmg_nccl_unique_id(void* id) {
  if (!id) return FMG_EINVAL;
  NcclApi& N = nccl();
  if (!N.ok) return FMG_ENCCL;
  ncclUniqueId u;
  if (N.getUniqueId(&u) != ncclSuccess) return FMG_ENCCL;
  std::memcpy(id, &u, sizeof(u));
  return FMG_OK;
}

int fmg_create_dist(int dim, int p, int levels, const fmg_schedule* s, int nranks, int rank, const void* id,
                    void* stream, fmg_ctx** out) {
  if (!out || !id || dim != 3 || nranks < 1 || rank < 0 || rank >= nranks) return FMG_EINVAL;
  NcclApi& N = nccl();
  if (!N.ok) return FMG_ENCCL;
  int rc = create_impl(dim, p, levels, s, stream, nranks, rank, out);
  if (rc) return rc;
  ncclUniqueId u;
  std::memcpy(&u, id, sizeof(u));
  ncclComm_t comm = nullptr;
  if (N.commInitRank(&comm, nranks, u, rank) != ncclSuccess) {
    fmg_destroy(*out);
    *out = nullptr;
    return FMG_ENCCL;
  }
  (*out)->comm = comm;
  return FMG_OK;
}

int fmg_create_hostx(int dim, int p, int levels, const fmg_schedule* s, int nranks, int rank, fmg_xfer_fn fn,
                     void* user, void* stream, fmg_ctx** out) {
  if (!out || !fn || dim != 3 || nranks < 1 || rank < 0 || rank >= nranks) return FMG_EINVAL;
  int rc = create_impl(dim, p, levels, s, stream, nranks, rank, out);
  if (rc) return rc;
  (*out)->xfer = fn;
  (*out)->xfer_user = user;
  return FMG_OK;
}

int fmg_slab_plan(int nz, int nslabs, int rank, int depth, int gather, int* out, int cap) {
  if (nz < 1 || nslabs < 1 || nz % nslabs != 0 || rank < 0 || rank >= nslabs || depth < 0) return -FMG_EINVAL;
  std::vector<XPiece> v = slab_plan(nz, nslabs, rank, depth, gather);
  if (out)
    for (int i = 0; i < (int)v.size() && i < cap; ++i) {
      out[4 * i] = v[i].peer;
      out[4 * i + 1] = v[i].z0;
      out[4 * i + 2] = v[i].z1;
      out[4 * i + 3] = v[i].send;
    }
  return (int)v.size();
}

int fmg_create_slabs(int dim, int p, int levels, const fmg_schedule* s, int nslabs, void* stream, fmg_ctx** out) {
  if (!out || !s || dim != 3 || nslabs < 1 || nslabs > 64) return FMG_EINVAL;
  *out = nullptr;
  fmg_ctx* grp = new fmg_ctx();
  grp->dim = dim; grp->p = p; grp->levels = levels; grp->Lmax = levels - 1; grp->s = *s;
  grp->st = (cudaStream_t)stream;
  grp->G = nslabs;
  if (cudaStreamCreateWithFlags(&grp->cap, cudaStreamNonBlocking) != cudaSuccess) { delete grp; return FMG_ECUDA; }
  for (int r = 0; r < nslabs; ++r) {
    fmg_ctx* sc = nullptr;
    int rc = create_impl(dim, p, levels, s, stream, nslabs, r, &sc);
    if (rc != FMG_OK) {
      fmg_destroy(grp);
      return rc;
    }
    grp->sub.push_back(sc);
  }
  grp->lc = grp->sub[0]->lc;
  *out = grp;
  return FMG_OK;
}

// Group (virtual slabs) solve: the item list is built once (identical for all
// ranks: equal slabs) and issued to every sub-context in lockstep.
static int group_solve(fmg_ctx* grp, int Lstop, int iters_last, bool graph) {
  fmg_ctx* s0 = grp->sub[0];
  Builder b = make_builder(s0);
  build_solve(b, Lstop, iters_last);
  for (fmg_ctx* s : grp->sub) {
    std::memcpy(s->wu_cur, s0->wu_cur, sizeof(s->wu_cur));
    s->solved_L = Lstop;
    s->launches = 0;
    int prc = prepare(s, b, graph ? 0 : 1);
    if (prc) return prc;
  }
  grp->solved_L = Lstop;
  if (graph) {
    if (!grp->graph) {
      for (fmg_ctx* s : grp->sub) s->cur = grp->cap;
      cudaError_t e = cudaStreamBeginCapture(grp->cap, cudaStreamCaptureModeThreadLocal);
      if (e != cudaSuccess) return cuda_err(e);
      for (fmg_ctx* s : grp->sub) zero_sections(s);
      issue_group(grp, b);
      cudaGraph_t gr;
      e = cudaStreamEndCapture(grp->cap, &gr);
      if (e != cudaSuccess) return cuda_err(e);
      e = cudaGraphInstantiate(&grp->graph, gr, 0);
      cudaGraphDestroy(gr);
      if (e != cudaSuccess) { grp->graph = nullptr; return cuda_err(e); }
    }
    cudaError_t e = cudaGraphLaunch(grp->graph, grp->st);
    return cuda_err(e);
  }
  cudaStreamSynchronize(grp->st);
  for (fmg_ctx* s : grp->sub) {
    s->cur = grp->st;
    zero_sections(s);
  }
  issue_group(grp, b);
  return FMG_OK;
}

static int group_check(fmg_ctx* grp) {
  for (fmg_ctx* s : grp->sub) {
    int rc = sync_check(s);
    if (rc) return rc;
  }
  return FMG_OK;
}

int fmg_solve_async(fmg_ctx* c) {
  if (!c) return FMG_EINVAL;
  if (!c->sub.empty()) return group_solve(c, c->Lmax, c->s.n_ir, true);
  if (c->xfer) return fmg_solve_upto(c, c->Lmax, c->s.n_ir);  // (host transport: no graph)
  if (!c->graph) {
    Builder b = make_builder(c);
    c->launches = 0;
    c->ev_used = 0;
    build_solve(b, c->Lmax, c->s.n_ir);
    int prc = prepare(c, b, 0);
    if (prc) return prc;
    c->cur = c->cap;
    cudaError_t e = cudaStreamBeginCapture(c->cap, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) return cuda_err(e);
    zero_sections(c);
    c->nccl_err = 0;
    issue(c, b);
    cudaGraph_t gr;
    e = cudaStreamEndCapture(c->cap, &gr);
    if (e != cudaSuccess) return cuda_err(e);
    if (c->nccl_err) return FMG_ENCCL;
    e = cudaGraphInstantiate(&c->graph, gr, 0);
    cudaGraphDestroy(gr);
    if (e != cudaSuccess) { c->graph = nullptr; return cuda_err(e); }
    std::memcpy(c->wu_graph, c->wu_cur, sizeof(c->wu_graph));
  }
  cudaError_t e = cudaGraphLaunch(c->graph, c->st);
  if (e != cudaSuccess) return cuda_err(e);
  // a replay leaves the sections at the widths of the captured build, whatever
  // fmg_solve_upto ran in between (wu_cur went stale on replay)
  std::memcpy(c->wu_cur, c->wu_graph, sizeof(c->wu_cur));
  c->solved_L = c->Lmax;
  return FMG_OK;
}

int fmg_solve(fmg_ctx* c) {
  int rc = fmg_solve_async(c);
  if (rc) return rc;
  if (!c->sub.empty()) return group_check(c);
  return sync_check(c);
}

int fmg_solve_upto(fmg_ctx* c, int Lstop, int iters_last) {
  if (!c || Lstop < 0 || Lstop > c->Lmax || iters_last < 0) return FMG_EINVAL;
  if (!c->sub.empty()) {
    int rc = group_solve(c, Lstop, iters_last, false);
    if (rc) return rc;
    return group_check(c);
  }
  Builder b = make_builder(c);
  c->cur = c->st;
  cudaStreamSynchronize(c->st);
  zero_sections(c);
  build_solve(b, Lstop, iters_last);
  c->solved_L = Lstop;
  return run_direct(c, b);
}

// Squared norms ||t_l||^2 of the log (device holds sums of squares; z-slab
// levels l > lc of a group are summed over the slabs, KC levels are replicated).
static int norms_sq(fmg_ctx* c, double* host) {
  const size_t n = (size_t)c->levels * c->s.n_ir * c->levels;
  if (c->sub.empty()) {
    cudaError_t e = cudaStreamSynchronize(c->st);
    if (e != cudaSuccess) return cuda_err(e);
    e = cudaMemcpy(host, c->norms_dev, sizeof(double) * n, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess && c->xfer) {  // host transport: exchange the partial vectors, sum in rank order
      for (size_t i = 0; i < n; ++i)
        if ((int)(i % c->levels) <= c->lc && c->rank != 0) host[i] = 0.0;
      std::vector<std::vector<double>> all(c->G, std::vector<double>(n));
      all[c->rank].assign(host, host + n);
      std::vector<int> peer, send;
      std::vector<void*> buf;
      std::vector<int64_t> bytes;
      for (int r = 0; r < c->G; ++r) {
        if (r == c->rank) continue;
        peer.push_back(r); send.push_back(1); buf.push_back(all[c->rank].data()); bytes.push_back((int64_t)(8 * n));
        peer.push_back(r); send.push_back(0); buf.push_back(all[r].data()); bytes.push_back((int64_t)(8 * n));
      }
      if (!buf.empty() && c->xfer(c->xfer_user, (int)buf.size(), peer.data(), send.data(), buf.data(), bytes.data()))
        return FMG_ENCCL;
      for (size_t i = 0; i < n; ++i) {
        double t = 0.0;
        for (int r = 0; r < c->G; ++r) t += all[r][i];
        host[i] = t;
      }
      return FMG_OK;
    }
    if (e != cudaSuccess || !c->comm) return cuda_err(e);
    // NCCL ranks: sum the slab partials of levels > lc (KC levels from rank 0)
    for (size_t i = 0; i < n; ++i)
      if ((int)(i % c->levels) <= c->lc && c->rank != 0) host[i] = 0.0;
    e = cudaMemcpyAsync(c->err_part, host, sizeof(double) * n, cudaMemcpyHostToDevice, c->st);
    if (e != cudaSuccess) return cuda_err(e);
    e = cudaStreamSynchronize(c->st);  // (pageable source: the copy has completed before the all-reduce)
    if (e != cudaSuccess) return cuda_err(e);
    if (nccl().allReduce(c->err_part, c->err_part, n, ncclDouble, ncclSum, (ncclComm_t)c->comm, c->st) != ncclSuccess)
      return FMG_ENCCL;
    e = cudaStreamSynchronize(c->st);
    if (e != cudaSuccess) return cuda_err(e);
    return cuda_err(cudaMemcpy(host, c->err_part, sizeof(double) * n, cudaMemcpyDeviceToHost));
  }
  std::vector<double> tmp(n);
  for (size_t i = 0; i < n; ++i) host[i] = 0.0;
  for (size_t r = 0; r < c->sub.size(); ++r) {
    int rc = norms_sq(c->sub[r], tmp.data());
    if (rc) return rc;
    for (size_t i = 0; i < n; ++i) {
      const int l = (int)(i % c->levels);
      if (l > c->lc || r == 0) host[i] += tmp[i];
    }
  }
  return FMG_OK;
}

int fmg_norms(fmg_ctx* c, double* host) {
  if (!c || !host) return FMG_EINVAL;
  int rc = norms_sq(c, host);
  if (rc) return rc;
  for (size_t i = 0; i < (size_t)c->levels * c->s.n_ir * c->levels; ++i) host[i] = std::sqrt(host[i]);
  return FMG_OK;
}

int fmg_residual(fmg_ctx* c, double* host_norms) {
  if (!c || !c->sub.empty() || c->comm || c->xfer) return FMG_EINVAL;  // (slab groups / ranks: solve / norms / sections only)
  if (c->solved_L < 0) return FMG_ESTATE;
  int L = c->solved_L;
  if (L < 1) return FMG_ESTATE;
  // Runs into norm row (L*n_ir) and restores the log afterwards.
  std::vector<double> keep(c->levels);
  double* row = c->norms_dev + ((size_t)L * c->s.n_ir) * c->levels;
  cudaStreamSynchronize(c->st);
  cudaMemcpy(keep.data(), row, sizeof(double) * c->levels, cudaMemcpyDeviceToHost);
  Builder b = make_builder(c);
  build_residual_grid(b, L, L * c->s.n_ir);
  int rc = run_direct(c, b);
  if (rc) return rc;
  if (host_norms) {
    std::vector<double> tmp(c->levels, 0.0);
    cudaMemcpy(tmp.data(), row, sizeof(double) * c->levels, cudaMemcpyDeviceToHost);
    for (int l = 0; l < c->levels; ++l) host_norms[l] = l <= L ? std::sqrt(tmp[l]) : 0.0;
  }
  cudaMemcpy(row, keep.data(), sizeof(double) * c->levels, cudaMemcpyHostToDevice);
  return FMG_OK;
}

// û_L into the level-L u array (decode ops for l = 0..L, materialised).
static int decode_solution(fmg_ctx* c, int* which) {
  int L = c->solved_L;
  if (!c->Ul[L]) {  // fine3: the finest level has no u array until a solution is asked for
    const size_t bytes = sizeof(double) * c->g[L].size;
    c->Ul[L] = (double*)dalloc(c, bytes);
    if (!c->Ul[L]) return FMG_ENOMEM;
    cudaMemset(c->Ul[L], 0, bytes);
  }
  Builder b = make_builder(c);
  for (int l = 0; l <= L; ++l) {
    OpDesc o = mkop(OP_DECODE, l, L);
    o.wu_in = c->wu_cur[l];
    b.grid(o);
  }
  *which = L;
  return run_direct(c, b);
}

int fmg_get_solution(fmg_ctx* c, double* dst_dev) {
  if (!c || !dst_dev) return FMG_EINVAL;
  if (!c->sub.empty() || c->comm || c->xfer) return FMG_EINVAL;  // (slab ranks hold only their planes)
  if (c->solved_L < 0) return FMG_ESTATE;
  int which = 0;
  int rc = decode_solution(c, &which);
  if (rc) return rc;
  cudaMemcpyAsync(dst_dev, c->Ul[which], sizeof(double) * c->g[c->solved_L].size, cudaMemcpyDeviceToDevice,
                  c->st);
  return sync_check(c);
}

int fmg_errors(fmg_ctx* c, double* err3) {
  if (!c || !err3) return FMG_EINVAL;
  if (!c->sub.empty() || c->comm || c->xfer) return FMG_EINVAL;  // (slab ranks hold only their planes)
  if (c->solved_L < 0) return FMG_ESTATE;
  int which = 0;
  int rc = decode_solution(c, &which);
  if (rc) return rc;
  int np = 0;
  c->cur = c->st;
  launch_errors(L_(c), c->Ul[which], c->g[c->solved_L], c->err_part, &np);
  rc = sync_check(c);
  if (rc) return rc;
  std::vector<double> h(2 * np);
  cudaMemcpy(h.data(), c->err_part, sizeof(double) * 2 * np, cudaMemcpyDeviceToHost);
  double e0 = 0.0, e1 = 0.0;
  for (int i = 0; i < np; ++i) { e0 += h[2 * i]; e1 += h[2 * i + 1]; }
  double hh = std::ldexp(1.0, -(c->solved_L + 1));
  double vol = c->dim == 3 ? hh * hh * hh : hh * hh;
  e0 *= vol; e1 *= vol;
  double nL2 = std::ldexp(1.0, -c->dim), nH1 = c->dim * M_PI * M_PI * std::ldexp(1.0, -c->dim);
  err3[0] = std::sqrt(e0 / nL2);
  err3[1] = std::sqrt(e1 / nH1);
  err3[2] = std::sqrt((e0 + e1) / (nL2 + nH1));
  return FMG_OK;
}

int fmg_get_section(fmg_ctx* c, int which, int level, uint32_t* mant, int8_t* exps, int* width) {
  if (!c || which < 0 || which > 1 || level < 0 || level > c->Lmax || !width) return FMG_EINVAL;
  if (c->solved_L < 0) return FMG_ESTATE;
  if (!c->sub.empty()) {
    // assemble: every slab's planes [zlo, zhi) from its owner (KC levels from rank 0)
    fmg_ctx* s0 = c->sub[0];
    int rc = fmg_get_section(s0, which, level, mant, exps, width);
    if (rc || level <= c->lc) return rc;
    const Geom& g = s0->g[level];
    const long long bpp = (long long)(g.NX / 32) * g.NY;  // blocks per plane
    const int w = *width;
    std::vector<uint32_t> m2(mant ? (size_t)g.nblk * w : 0);
    std::vector<int8_t> e2(exps ? (size_t)g.nblk : 0);
    for (size_t r = 1; r < c->sub.size(); ++r) {
      fmg_ctx* sr = c->sub[r];
      rc = fmg_get_section(sr, which, level, mant ? m2.data() : nullptr, exps ? e2.data() : nullptr, width);
      if (rc) return rc;
      const long long b0 = sr->zlo[level] * bpp, b1 = sr->zhi[level] * bpp;
      if (mant) std::memcpy(mant + b0 * w, m2.data() + b0 * w, sizeof(uint32_t) * (b1 - b0) * w);
      if (exps) std::memcpy(exps + b0, e2.data() + b0, (size_t)(b1 - b0));
    }
    return FMG_OK;
  }
  const Geom& g = c->g[level];
  const Sec& s = which == 0 ? c->u[level] : c->r[level];
  int w = which == 0 ? c->wu_cur[level] : wr(c, level, c->solved_L);
  *width = w;
  cudaError_t e = cudaStreamSynchronize(c->st);
  if (e != cudaSuccess) return cuda_err(e);
  // the allocated plane window (the whole level unless partitioned over z slabs)
  const long long bpp = (long long)(g.NX / 32) * g.NY, b0 = bpp * c->wlo[level], nb = bpp * (c->whi[level] - c->wlo[level]);
  if (mant) {
    std::vector<uint32_t> tmp((size_t)nb * s.stride);
    e = cudaMemcpy(tmp.data(), s.mant + b0 * s.stride, sizeof(uint32_t) * tmp.size(), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_err(e);
    for (long long b = 0; b < nb; ++b) std::memcpy(mant + (b0 + b) * w, tmp.data() + b * s.stride, sizeof(uint32_t) * w);
  }
  if (exps) {
    e = cudaMemcpy(exps + b0, s.exps + b0, nb, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_err(e);
  }
  return FMG_OK;
}

int fmg_info(fmg_ctx* c, double* info) {
  if (!c || !info) return FMG_EINVAL;
  if (!c->sub.empty()) {
    int rc = fmg_info(c->sub[0], info);
    double launches = 0.0;
    for (fmg_ctx* s : c->sub) launches += (double)s->launches;
    info[9] = launches;
    return rc;
  }
  const Geom& g = c->g[c->Lmax];
  info[0] = c->dim; info[1] = c->p; info[2] = c->levels;
  info[3] = g.NX; info[4] = g.NY; info[5] = g.NZ;
  info[6] = std::pow((double)(g.n - 1), c->dim);
  // stored bits at the finest FMG level: mantissas + exponents of u and r sections
  double bits = 0.0, bytes_solve = 0.0;
  for (int l = 0; l <= c->Lmax; ++l)
    bits += (double)c->g[l].size * (wu(c, l, c->Lmax) + wr(c, l, c->Lmax)) + 2.0 * 8 * c->g[l].nblk;
  info[7] = bits;
  // algorithmic bytes: per IR iteration at FMG level L every
  // stored u and r section is read once and written once.
  for (int L = 1; L <= c->Lmax; ++L) {
    double sweep = 0.0;
    for (int l = 0; l <= L; ++l)
      sweep += 2.0 * ((double)c->g[l].size * (wu(c, l, L) + wr(c, l, L)) / 8.0 + 2.0 * c->g[l].nblk);
    bytes_solve += c->s.n_ir * sweep;
  }
  info[8] = bytes_solve;
  info[9] = (double)c->launches;
  return FMG_OK;
}

// Storage accounting (§8(f) row N3).  Host only.
int fmg_memory_model(int dim, int p, int levels, const fmg_schedule* s, double* out, int cap) {
  if (!s || !out || cap < FMG_MEM_COUNT) return FMG_EINVAL;
  if (check_args(dim, p, levels, s)) return FMG_EINVAL;
  const int L = levels - 1;
  const double two_d = std::pow(2.0, dim), cst = two_d / (two_d - 1.0);
  double nL = 0.0, um = 0.0, rm = 0.0, ue = 0.0, re = 0.0, ub = 0.0, rb = 0.0, ef = 0.0, es = 0.0;
  double tmp62 = 0.0, tmp63 = 0.0, fp64 = 0.0, sec = 0.0;
  for (int l = 0; l <= L; ++l) {
    const int n = p << (l + 1);                       // nodes per side incl. the two boundary nodes - 1
    const double N = std::pow((double)(n - 1), dim);  // unknowns (interior nodes), reading R2
    const long long NX = ((n + 31) / 32) * 32;
    const double stored = (double)NX * n * (dim == 3 ? n : 1);  // padded x rows
    const int wul = s->b_u + s->k_u * (L - l), wrl = s->b_r + s->k_r * (L - l);
    um += stored * wul;
    rm += stored * wrl;
    ue += N * wul;  // Eq 6.1 summand over unknowns
    re += N * wrl;
    ef += 2.0 * 8.0 * stored / 32.0;             // one int8 exponent per 32-entry block, u and r
    es += (double)(wul + wrl) * (32.0 + 64.0);   // <= w (exponent, block start) pairs per section
    // Eq 6.2 / 6.3: only delta(M_l) ~ (w(M_l) - 1) n_l^((d-1)/d) entries of a
    // temporary live at once when streaming lexicographically;
    // w(A) = 2p + 1 nodes per direction for Q_p, a_L = k L + b bits
    const double delta = 2.0 * p * std::pow((double)(n - 1), dim - 1);
    const int aL = s->b_u + s->k_u * L;
    tmp62 += 2.0 * aL * delta;                  // u and t at a_L bits (Eq 6.2)
    tmp63 += (double)(s->k_u * l + s->b_u) * delta;  // z, progressive (Eq 6.3)
    // this implementation's FP64 arrays (create_impl): u_l, t_l, w_l per level;
    // scratch Z, B, Y[2], PU and the Chebyshev direction Dv.  With the
    // finest-level kernels (3D, Chebyshev degree 2-3, nu = 1)
    // level L keeps only t_L (lean form), the scratch is Z and PU one level
    // smaller, and Dv exists for degree 3 only.
    const bool f3 = dim == 3 && s->nu <= 1 && s->smoother == 0 && (s->cheb_degree == 2 || s->cheb_degree == 3) && L >= 1;
    fp64 += (f3 && l == L ? 1.0 : 3.0) * 8.0 * stored;
    if (f3 && l == L - 1) fp64 += 2.0 * 8.0 * stored;  // Z, PU scratch (the lean form, FMG_F3MAT=0)
    if (f3 && l == 0) fp64 += 8.0 * stored;           // B of level 0's bracket
    sec += 4.0 * (double)(NX * n * (dim == 3 ? n : 1) / 32) * (wul + wrl) + 2.0 * stored / 32.0;
    if (l == L) {
      nL = N;
      if (!f3) fp64 += 6.0 * 8.0 * stored;      // finest-size Z, B, Y[2], Dv, PU
      else if (s->cheb_degree >= 3) fp64 += 8.0 * stored;  // Dv
    }
  }
  ub = (cst * s->b_u + cst / (two_d - 1.0) * s->k_u) * nL;
  rb = (cst * s->b_r + cst / (two_d - 1.0) * s->k_r) * nL;
  const double v[FMG_MEM_COUNT] = {nL, um, rm, ue, ub, re, rb, ef, es, tmp62, tmp63, fp64, sec};
  for (int i = 0; i < FMG_MEM_COUNT; ++i) out[i] = v[i];
  return FMG_OK;
}

int64_t fmg_device_bytes(fmg_ctx* c) {
  if (!c) return -FMG_EINVAL;
  int64_t b = 0;
  for (auto& a : c->allocs) b += (int64_t)a.second;
  for (fmg_ctx* sub : c->sub) b += fmg_device_bytes(sub);
  return b;
}

int fmg_enable_kernel_timing(fmg_ctx* c, int cls) {
  if (!c || cls < -1 || cls > 5) return FMG_EINVAL;
  if (c->graph) {
    cudaGraphExecDestroy(c->graph);
    c->graph = nullptr;
  }
  for (auto e : c->ev) cudaEventDestroy(e);
  c->ev.clear();
  c->timing_cls = cls;
  if (cls >= 0) {
    int per = (cls == 1) ? c->s.cheb_degree : 1;
    int n = 2 * c->s.n_ir * per;
    if (cls == 4) n = 2 * 20000;
    for (int i = 0; i < n; ++i) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      c->ev.push_back(e);
    }
  }
  return FMG_OK;
}

int fmg_kernel_times(fmg_ctx* c, float* ms, int cap) {
  if (!c || !ms) return -FMG_EINVAL;
  cudaError_t e = cudaStreamSynchronize(c->st);
  if (e != cudaSuccess) return -cuda_err(e);
  int n = 0;
  for (int i = 0; i + 1 < c->ev_used && n < cap; i += 2) {
    float t = 0.f;
    cudaEventElapsedTime(&t, c->ev[i], c->ev[i + 1]);
    ms[n++] = t;
  }
  return n;
}

int fmg_kernel_time(fmg_ctx* c, double* total_ms, int* launches) {
  if (!c || !total_ms || !launches) return FMG_EINVAL;
  cudaError_t e = cudaStreamSynchronize(c->st);
  if (e != cudaSuccess) return cuda_err(e);
  double tot = 0.0;
  int n = 0;
  for (int i = 0; i + 1 < c->ev_used; i += 2) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, c->ev[i], c->ev[i + 1]) == cudaSuccess) {
      tot += ms;
      n++;
    }
  }
  *total_ms = tot;
  *launches = n;
  return FMG_OK;
}

int64_t fmg_rhs_size(fmg_ctx* c) {
  if (!c) return -1;
  int64_t n = 0;
  for (int l = 0; l <= c->Lmax; ++l) n += c->g[l].n;
  return n;
}

int fmg_set_rhs(fmg_ctx* c, const double* host) {
  if (!c || !host) return FMG_EINVAL;
  int64_t off = 0;
  for (int l = 0; l <= c->Lmax; ++l) {
    cudaError_t e = cudaMemcpyAsync(c->gtab[l], host + off, sizeof(double) * c->g[l].n, cudaMemcpyHostToDevice, c->st);
    if (e != cudaSuccess) return cuda_err(e);
    off += c->g[l].n;
  }
  return FMG_OK;
}

int fmg_get_rhs(fmg_ctx* c, double* host) {
  if (!c || !host) return FMG_EINVAL;
  cudaError_t e = cudaStreamSynchronize(c->st);
  if (e != cudaSuccess) return cuda_err(e);
  int64_t off = 0;
  for (int l = 0; l <= c->Lmax; ++l) {
    e = cudaMemcpy(host + off, c->gtab[l], sizeof(double) * c->g[l].n, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_err(e);
    off += c->g[l].n;
  }
  return FMG_OK;
}

int64_t fmg_export_solution(fmg_ctx* c, void* host, int64_t cap) {
  if (!c) return -FMG_EINVAL;
  // every level's allocated window of ú (mantissa words, then exponents)
  auto nblocks = [&](int l) { return (int64_t)(c->g[l].NX / 32) * c->g[l].NY * (c->whi[l] - c->wlo[l]); };
  int64_t need = 0;
  for (int l = 0; l <= c->Lmax; ++l) need += nblocks(l) * (4 * c->u[l].stride + 1);
  if (!host || cap < need) return need;
  char* dst = (char*)host;
  for (int l = 0; l <= c->Lmax; ++l) {
    const int64_t b0 = (int64_t)(c->g[l].NX / 32) * c->g[l].NY * c->wlo[l], nb = nblocks(l);
    size_t mb = sizeof(uint32_t) * nb * c->u[l].stride;
    cudaError_t e = cudaMemcpyAsync(dst, c->u[l].mant + b0 * c->u[l].stride, mb, cudaMemcpyDeviceToHost, c->st);
    if (e != cudaSuccess) return -cuda_err(e);
    dst += mb;
    e = cudaMemcpyAsync(dst, c->u[l].exps + b0, nb, cudaMemcpyDeviceToHost, c->st);
    if (e != cudaSuccess) return -cuda_err(e);
    dst += nb;
  }
  return need;
}

void fmg_destroy(fmg_ctx* c) {
  if (!c) return;
  cudaDeviceSynchronize();
  for (fmg_ctx* s : c->sub) fmg_destroy(s);
  c->sub.clear();
  if (c->comm) nccl().commDestroy((ncclComm_t)c->comm);
  if (c->graph) cudaGraphExecDestroy(c->graph);
  for (auto e : c->ev) cudaEventDestroy(e);
  free_all(c);
  if (c->cap) cudaStreamDestroy(c->cap);
  delete c;
}

const char* fmg_strerror(int code) {
  switch (code) {
    case FMG_OK: return "ok";
    case FMG_EINVAL: return "invalid argument";
    case FMG_ERANGE: return "BFP exponent out of range or non-finite value";
    case FMG_ENOMEM: return "device allocation failed";
    case FMG_ECUDA: return "CUDA runtime error";
    case FMG_ESTATE: return "call out of order";
    case FMG_ENCCL: return "NCCL unavailable or failed";
    default: return "unknown error";
  }
}

// ------------------------------------------------------------ codec API --
static int* g_codec_status = nullptr;

int bfp_encode(const double* x, int64_t n, int width, uint32_t* mant, int8_t* exps, void* stream) {
  if (width < 2 || width > 54 || n < 0 || (n % 32) != 0 || (n > 0 && (!x || !mant || !exps))) return FMG_EINVAL;
  if (n == 0) return FMG_OK;
  if (!g_codec_status) {
    if (cudaMalloc(&g_codec_status, sizeof(int)) != cudaSuccess) return FMG_ENOMEM;
    cudaMemset(g_codec_status, 0, sizeof(int));
  }
  launch_bfp_encode(x, n, width, mant, exps, g_codec_status, (cudaStream_t)stream);
  return cuda_err(cudaGetLastError());
}

int bfp_decode(const uint32_t* mant, const int8_t* exps, int64_t n, int width, double* x, void* stream) {
  if (width < 2 || width > 54 || n < 0 || (n % 32) != 0 || (n > 0 && (!x || !mant || !exps))) return FMG_EINVAL;
  if (n == 0) return FMG_OK;
  launch_bfp_decode(mant, exps, n, width, x, (cudaStream_t)stream);
  return cuda_err(cudaGetLastError());
}

int64_t bfp_stream_work_bytes(int64_t n) {
  if (n < 0 || (n % 32) != 0) return -FMG_EINVAL;
  return (int64_t)stream_work_bytes(n);
}

int bfp_stream_encode(const double* x, int64_t n, int width, uint32_t* mant, int32_t* xexp, int64_t* xstart,
                      int32_t* nblocks, void* work, void* stream) {
  if (width < 2 || width > 54 || n < 0 || (n % 32) != 0 || !nblocks) return FMG_EINVAL;
  if (n > 0 && (!x || !mant || !xexp || !xstart || !work)) return FMG_EINVAL;
  if (n == 0) return cuda_err(cudaMemsetAsync(nblocks, 0, sizeof(int32_t), (cudaStream_t)stream));
  if (!g_codec_status) {
    if (cudaMalloc(&g_codec_status, sizeof(int)) != cudaSuccess) return FMG_ENOMEM;
    cudaMemset(g_codec_status, 0, sizeof(int));
  }
  launch_stream_encode(x, n, width, mant, xexp, xstart, nblocks, work, g_codec_status, (cudaStream_t)stream);
  return cuda_err(cudaGetLastError());
}

int bfp_stream_decode(const uint32_t* mant, const int32_t* xexp, const int64_t* xstart, const int32_t* nblocks,
                      int64_t n, int width, double* x, void* stream) {
  if (width < 2 || width > 54 || n < 0 || (n % 32) != 0) return FMG_EINVAL;
  if (n == 0) return FMG_OK;
  if (!mant || !xexp || !xstart || !nblocks || !x) return FMG_EINVAL;
  launch_stream_decode(mant, xexp, xstart, nblocks, n, width, x, (cudaStream_t)stream);
  return cuda_err(cudaGetLastError());
}

int bfp_status(void* stream) {
  cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_err(e);
  if (!g_codec_status) return FMG_OK;
  int st = 0;
  cudaMemcpy(&st, g_codec_status, sizeof(int), cudaMemcpyDeviceToHost);
  if (st) {
    cudaMemset(g_codec_status, 0, sizeof(int));
    return FMG_ERANGE;
  }
  return FMG_OK;
}

}  // extern "C"
