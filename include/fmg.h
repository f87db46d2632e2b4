/*
 * fmg.h -- C-ABI of libfmg.so: the B200 compact full multigrid hot path of
 * arXiv 2511.19036 ("compact FMG": solution, residual and correction stored as
 * multilevel compact sections in block floating point at regressive widths).
 *
 * Problem (eq:pde-poisson PAPER.md:1418-1424):
 *   -Δu = f on (0,1)^dim, u = 0 on the boundary, Lagrange Q_p elements on the
 *   uniform dyadic hierarchy; level l has element size h_l = 2^-(l+1) and
 *   n_l = p 2^(l+1) nodes per dimension excluding the far boundary; f is the
 *   load vector of the manufactured solution u = prod_k sin(pi x_k).
 *
 * Storage layout of a level: x fastest, stored extent
 *   NX = roundup(n_l, 32), NY = n_l, NZ = n_l (3D) or 1 (2D); node index 0 is the
 *   (zero) boundary; entries at non-unknowns (index 0, x >= n_l) are 0.
 *
 * BFP format (rounding PAPER.md:846, R8):
 *   blocks of 32 consecutive x entries; one int8 exponent E per block;
 *   w-bit two's-complement mantissas (sign bit included),
 *   value = m 2^(E-(w-1)); entry j of a block occupies bits [j w, j w + w) of
 *   the block's bit stream, stream bit k = bit (k mod 32) of word k/32, so a
 *   block is exactly w uint32 words.  E = -128 marks an all-zero block.
 *   Encode: q = w-1, E0 = ilogb(max|x|)+1, E = E0+1 if RNE(max|x| 2^(q-E0)) = 2^q
 *   else E0, E < -127 saturates to -127, E > 127 -> FMG_ERANGE; m = RNE(x 2^(q-E)).
 *
 * Threading / streams: every call is issued on the context's stream (or the
 * `stream` argument); calls documented "synchronous" wait for completion.
 * All pointers are owned by the caller unless stated otherwise.
 * Errors: every function returns FMG_OK (0) or one of the codes below.
 */
#ifndef FMG_H
#define FMG_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FMG_OK 0
#define FMG_EINVAL 1  /* bad argument (dim, p, levels, width outside [2,54], n % 32) */
#define FMG_ERANGE 2  /* BFP exponent > 127 or non-finite value met by an encode */
#define FMG_ENOMEM 3  /* device allocation failed */
#define FMG_ECUDA 4   /* CUDA runtime error */
#define FMG_ESTATE 5  /* call out of order (e.g. residual before any solve) */
#define FMG_ENCCL 6   /* NCCL not loadable or an NCCL call failed (multi-GPU slabs) */

/* Bit-width schedule (tab:precisions PAPER.md:820-841).
 *   w_u(l,L) = b_u + k_u (L-l)   solution sections  (b1 of Table 3, k_u = p+1)
 *   w_r(l,L) = b_r + k_r (L-l)   residual / correction sections (b2, k_r = m = 1)
 * n_ir: IR iterations N per FMG level (Alg 3.3).
 * cheb_degree, lambda_hi, alpha: Chebyshev-Jacobi smoother of degree k on
 * [lambda_hi/alpha, lambda_hi] for D^-1 A (reading R4). */
typedef struct {
  int b_u, k_u;
  int b_r, k_r;
  int n_ir;
  int cheb_degree;
  double lambda_hi;
  double alpha;
  int smoother; /* 0: Chebyshev-Jacobi of degree cheb_degree (R4);
                   1: one multicolour Gauss-Seidel sweep, (p+1)^d colours
                   (the paper's smoother family PAPER.md:1624) */
  int nu;       /* compact V(0,1) cycles per IR iteration (Alg 3.1 PAPER.md:
                   633-661).  0 or 1: the method of Alg 3.3.
                   2..8: the nonzero-guess cycles of reading R23, on one GPU
                   (2D and 3D) with the Chebyshev smoother of degree >= 2 or
                   multicolour Gauss-Seidel; fmg_create returns FMG_EINVAL for
                   nu > 8, Chebyshev degree 1 with nu > 1, and z slabs with nu > 1. */
  int cfas_fp32; /* 1: cFas in FP32 (tab:precisions PAPER.md:820-841 bounds the
                   cFas working precision by L + b_r <= 15 bits at the
                   configurations; reading R28): z, b, the Chebyshev
                   iterates and w in float with the FP64 constants rounded to
                   float.  The coarse solve, the correction and the residual
                   stay FP64.  3D with the Chebyshev smoother of degree 2-3 and
                   nu = 1 only (else FMG_EINVAL).  0: everything FP64. */
} fmg_schedule;

typedef struct fmg_ctx fmg_ctx;

/* Device allocator hook (e.g. torch's caching allocator).  alloc returns a
 * device pointer of at least `bytes` or NULL; free releases it.  Applies to
 * contexts created afterwards.  Pass NULLs to restore cudaMalloc/cudaFree. */
typedef void* (*fmg_alloc_fn)(size_t bytes, void* user);
typedef void (*fmg_free_fn)(void* ptr, size_t bytes, void* user);
int fmg_set_allocator(fmg_alloc_fn alloc, fmg_free_fn free_fn, void* user);

/* Create a solver context on the current CUDA device.
 *   dim in {2,3}; p in {1,2,3}; levels >= 1 (solver levels 0..levels-1, finest
 *   element size 2^-levels; reading R3); s: schedule (copied);
 *   stream: cudaStream_t the context runs on (NULL = legacy default stream).
 * Allocates every section and workspace (owned by the context) and uploads the
 * operator / RHS tables.  Errors: FMG_EINVAL (any width w_u(0,L), w_r(0,L) > 54
 * or < 2, bad dim/p/levels/schedule), FMG_ENOMEM, FMG_ECUDA. */
int fmg_create(int dim, int p, int levels, const fmg_schedule* s, void* stream, fmg_ctx** out);

/* z-slab decomposition emulated on ONE device: a
 * group of `nslabs` sub-contexts (3D only), each computing the planes
 * [r NZ_l/G, (r+1) NZ_l/G) of every grid level l > lc, with the ghost planes
 * each stencil consumer needs copied from the owning sub-context (device to
 * device, on the group stream) and t_{lc+1} gathered before the replicated
 * coarse-hierarchy kernel.  The same exchange plan a multi-GPU run performs
 * over NVLink; its results are bit-identical to fmg_create (decomposition
 * invariance).  Supports fmg_solve / fmg_solve_async / fmg_solve_upto /
 * fmg_norms / fmg_get_section / fmg_info / fmg_destroy (others: FMG_EINVAL).
 * Errors: FMG_EINVAL (dim != 3, a slab level with NZ_l % nslabs != 0), as
 * fmg_create otherwise. */
int fmg_create_slabs(int dim, int p, int levels, const fmg_schedule* s, int nslabs, void* stream,
                     fmg_ctx** out);

/* Multi-GPU z slabs: one process per GPU, rank `rank` of `nranks` (3D only).
 * Same decomposition and exchange plan as fmg_create_slabs; ghost planes move
 * by grouped ncclSend/ncclRecv over NVLink and t_{lc+1} by an in-place
 * ncclAllGather, all on the context stream inside the solve graph.  `id` is a
 * 128-byte ncclUniqueId from fmg_nccl_unique_id on rank 0, broadcast by the
 * caller (e.g. torch.distributed); collective over the ranks.  NCCL is
 * resolved at run time (libnccl.so.2 already loaded, or FMG_NCCL_LIB).  After
 * a solve each rank's sections hold its own planes of the grid levels;
 * fmg_norms all-reduces the slab partials.  Errors: FMG_ENCCL, as
 * fmg_create_slabs otherwise. */
int fmg_nccl_unique_id(void* id);
int fmg_create_dist(int dim, int p, int levels, const fmg_schedule* s, int nranks, int rank, const void* id,
                    void* stream, fmg_ctx** out);

/* z slabs with a HOST-STAGED transport (one process per rank; ranks may share
 * a device): the same decomposition, exchange plan and memory partition as
 * fmg_create_dist, but every exchange is handed to the caller.  At each
 * exchange the library synchronises the stream, copies the send pieces
 * device -> host, calls
 *     fn(user, n, peer[], send[], buf[], bytes[])
 * with all n pieces of the exchange (send[i] = 1: buf[i] holds bytes[i] to
 * deliver to rank peer[i]; 0: receive bytes[i] from peer[i] into buf[i]),
 * and copies the received pieces host -> device.  fn must complete every
 * piece before returning (e.g. torch.distributed isend/irecv over gloo, then
 * wait) and return 0, else the solve fails with FMG_ENCCL.  Pieces are listed
 * in the order of fmg_slab_plan.  Solves run directly on `stream` (no graph:
 * the callback runs between kernels); fmg_norms sums the slab partials
 * through fn as well.  The buffers are library-owned and valid only during
 * the call.  Errors: as fmg_create_slabs. */
typedef int (*fmg_xfer_fn)(void* user, int n, const int* peer, const int* send, void* const* buf,
                           const int64_t* bytes);
int fmg_create_hostx(int dim, int p, int levels, const fmg_schedule* s, int nranks, int rank, fmg_xfer_fn fn,
                     void* user, void* stream, fmg_ctx** out);

/* Host-only helper (no device work): the ghost-plane exchange plan of rank
 * `rank` of `nslabs` equal slabs of `nz` planes for halo depth `depth` (or a
 * gather of every foreign plane): up to `cap` pieces of 4 ints {peer, z0, z1,
 * send} (planes [z0, z1) sent to / received from peer) into `out`; returns
 * the piece count, or -FMG_EINVAL. */
int fmg_slab_plan(int nz, int nslabs, int rank, int depth, int gather, int* out, int cap);

/* Alg 3.3 from scratch: coarse solve, then for L = 1..levels-1
 * push a level and run N x {fmgResidual, cFas V(0,1), correction}.  Enqueues one
 * CUDA graph on the context stream and returns without waiting (asynchronous).
 * Deterministic: repeated solves are bit-identical. */
int fmg_solve_async(fmg_ctx* c);

/* fmg_solve_async + wait + device error check (synchronous).
 * Errors: FMG_ERANGE if any encode saw a non-finite value or exponent > 127. */
int fmg_solve(fmg_ctx* c);

/* Partial solve for parity tests: stops after `iters_last` IR iterations of FMG
 * level Lstop (0 <= Lstop < levels).  Synchronous. */
int fmg_solve_upto(fmg_ctx* c, int Lstop, int iters_last);

/* Norm log of the last solve: norms[(L*n_ir + it)*levels + l] = ||t_l||_2 after
 * the residual of IR iteration `it` at FMG level L (entries l > L are 0).
 * `host` holds levels*n_ir*levels doubles.  Synchronous. */
int fmg_norms(fmg_ctx* c, double* host);

/* Alg 3.2 fmgResidual on the current compact solution at the
 * finest FMG level reached; leaves r_l sections on the device and writes
 * ||t_l||_2, l = 0..L, to `host_norms` (levels doubles, l > L zero).
 * FMG_ESTATE before any solve.  Synchronous. */
int fmg_residual(fmg_ctx* c, double* host_norms);

/* Decoded standard representation û_L (eq:compact-to-standard PAPER.md:186) of
 * the finest FMG level reached, written to the caller's device buffer `dst`
 * in the stored layout of level L (NX*NY*NZ doubles).  Synchronous. */
int fmg_get_solution(fmg_ctx* c, double* dst_dev);

/* Relative L2, H1-semi and H1 errors of û_L against u = prod sin(pi x_k)
 * (tensor Gauss-Legendre, p+3 points per dim per element; R13).
 * err3: host, 3 doubles.  Synchronous. */
int fmg_errors(fmg_ctx* c, double* err3);

/* Copy a compact section to the host in the dense BFP layout above.
 *   which: 0 = solution ú_l, 1 = residual r_l.  mant: nblk*width words (may be
 *   NULL to query width), exps: nblk bytes (may be NULL), width: out.  Synchronous. */
int fmg_get_section(fmg_ctx* c, int which, int level, uint32_t* mant, int8_t* exps, int* width);

/* Geometry / accounting of the context.  info[0..9] = dim, p, levels, NX, NY, NZ
 * of the finest level, unknowns of the finest level, stored section bits of the
 * finest FMG level (mantissas + exponents, u and r), algorithmic bytes of one
 * full solve, number of kernel launches per solve. */
int fmg_info(fmg_ctx* c, double* info10);

/* Storage accounting (§8(f) row N3; Eq 6.1-6.3,
 * DESIGN.md §2).  Host only, no device work.  For a solve whose finest FMG
 * level is L = levels - 1, writes FMG_MEM_COUNT doubles into out (cap >=
 * FMG_MEM_COUNT; n_l = unknowns of level l, reading R2):
 *   0  n_L
 *   1  mantissa bits of u_0..u_L as stored (padded x rows, w_u(l,L) bits)
 *   2  mantissa bits of r_0..r_L as stored
 *   3  Eq 6.1 sum for u: sum_l (k_u (L-l) + b_u) n_l
 *   4  Eq 6.1 bound for u: (2^d/(2^d-1) b_u + 2^d/(2^d-1)^2 k_u) n_L
 *   5  Eq 6.1 sum for r      6  Eq 6.1 bound for r
 *   7  exponent bits with fixed 32-entry blocks (u and r, as stored)
 *   8  exponent bits with streaming exponents (N3): <= w (32 + 64) per section
 *   9  Eq 6.2 model: u and t as streaming windows of delta(A_l) entries at a_L bits
 *  10  Eq 6.3 model: z as progressive-precision streaming windows
 *  11  bytes of FP64 temporaries this implementation allocates (full arrays:
 *      u_l, t_l, w_l per level plus six finest-size arrays; KC scratch excluded)
 *  12  bytes of section storage this implementation allocates
 * Errors: FMG_EINVAL (as fmg_create, or cap too small). */
#define FMG_MEM_COUNT 13
int fmg_memory_model(int dim, int p, int levels, const fmg_schedule* s, double* out, int cap);
/* Device bytes a context (and its slabs) holds; negative FMG error code on NULL. */
int64_t fmg_device_bytes(fmg_ctx* c);

/* Kernel-time instrumentation for bench.py: when enabled before the first
 * solve, the captured graph brackets every launch of kernel class `cls`
 * (0 = fine residual, 1 = every fine cFas smoothing step, 2 = prolong/decode,
 * 3 = restriction, 4 = every launch, 5 = last (finalising) fine cFas step) with CUDA events; fmg_kernel_time returns the summed device
 * time (ms) and launch count of the last solve (synchronous). */
int fmg_enable_kernel_timing(fmg_ctx* c, int cls);
int fmg_kernel_time(fmg_ctx* c, double* total_ms, int* launches);
/* Class 4 brackets every launch; fmg_kernel_times returns the per-launch
 * device times (ms, launch order) of the last solve into ms[cap]; returns the
 * count (synchronous). */
int fmg_kernel_times(fmg_ctx* c, float* ms, int cap);

/* Separable right-hand side f_l(i,j,k) = ((C g_l(i)) g_l(j)) g_l(k):
 * the 1D factor tables of every level, concatenated level by level
 * (sum_l n_l doubles, n_l = p 2^(l+1)).  fmg_create fills them with the load
 * integrals of the manufactured RHS; fmg_set_rhs uploads caller tables from
 * HOST memory (asynchronous on the context stream; pinned memory recommended)
 * and fmg_get_rhs copies them back (synchronous).  fmg_rhs_size returns the
 * table length. */
int64_t fmg_rhs_size(fmg_ctx* c);
int fmg_set_rhs(fmg_ctx* c, const double* host_tables);
int fmg_get_rhs(fmg_ctx* c, double* host_tables);

/* Export the compact solution ú_0..ú_L (device storage layout: per level l,
 * nblk_l * stride_l uint32 words -- block b at word b*stride_l, stride_l =
 * w_u(l, levels-1) -- followed by nblk_l exponent bytes) into `host` (pinned
 * host memory recommended; asynchronous on the context stream).  Returns the
 * number of bytes needed (host == NULL or cap too small copies nothing), or a
 * negative FMG error code. */
int64_t fmg_export_solution(fmg_ctx* c, void* host, int64_t cap);

void fmg_destroy(fmg_ctx* c);          /* idempotent on NULL */
const char* fmg_strerror(int code);

/* Standalone BFP codec (K1).  x, mant, exps are DEVICE pointers
 * (caller-owned); n is a multiple of 32; width in [2,54]; asynchronous on
 * `stream` (cudaStream_t, NULL = default).  bfp_encode reports FMG_ERANGE
 * through the next synchronous call of bfp_status. */
int bfp_encode(const double* x, int64_t n, int width, uint32_t* mant, int8_t* exps, void* stream);
int bfp_decode(const uint32_t* mant, const int8_t* exps, int64_t n, int width, double* x, void* stream);
/* Returns and clears the sticky codec error status (synchronises `stream`). */
int bfp_status(void* stream);

/* Streaming-exponent BFP (§8(f) row N3, readings R19-R21,
 * DESIGN.md §N3).  The running maximum of the entry exponents is the exponent
 * each mantissa is normalised to; a block starts at each increase; only the
 * `width` largest block exponents are kept and entries before the first kept
 * block are stored as 0 (they are below half a unit of single-exponent BFP).
 * All pointers are DEVICE pointers, caller-owned:
 *   x       n doubles (n % 32 == 0; width in [2,54])
 *   mant    n*width/32 words; entry i at stream bits [i w, i w + w), two's
 *           complement (the block codec's packing)
 *   xexp    int32[width]: kept block exponents X_k, increasing
 *   xstart  int64[width]: index of the first entry of block k, increasing
 *   nblocks one int32: number of kept blocks (<= width; 0 for an all-zero x)
 *   work    scratch of bfp_stream_work_bytes(n) bytes, unused between calls
 * Asynchronous on `stream`.  Non-finite input or an exponent above 1024 is
 * reported as FMG_ERANGE by the next bfp_status call.
 * x_i decodes to m_i 2^(X_k - q), q = width - 1, for the block k with
 * xstart[k] <= i < xstart[k+1]; 0 before xstart[0]. */
int64_t bfp_stream_work_bytes(int64_t n);  /* negative FMG error code on bad n */
int bfp_stream_encode(const double* x, int64_t n, int width, uint32_t* mant, int32_t* xexp, int64_t* xstart,
                      int32_t* nblocks, void* work, void* stream);
int bfp_stream_decode(const uint32_t* mant, const int32_t* xexp, const int64_t* xstart, const int32_t* nblocks,
                      int64_t n, int width, double* x, void* stream);

#ifdef __cplusplus
}
#endif
#endif
