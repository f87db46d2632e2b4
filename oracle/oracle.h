/*
 * oracle.h -- CPU ORACLE for the compact-FMG hot path (arXiv 2511.19036).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load liboracle.so.
 * The product path (paper_2511_19036_b200/, libfmg.so) never includes, links
 * or calls anything in this directory, and this directory never includes
 * anything from the product path.
 *
 * The oracle is a plain, slow, sequential FP64 implementation of
 *   Alg 3.3 cFmg  o  Alg 3.2 fmgResidual
 *   o  Alg 3.1 cFas with nu = 1 (ν=1 gives s = 0)
 * on the Lagrange Q_p discretisation of -Δu = f on (0,1)^d,
 * with its own BFP codec (fixed 32-entry blocks,
 * DESIGN.md reading R8).  Every floating-point expression follows the
 * canonical evaluation order written in DESIGN.md §3 with explicit fma();
 * compile with -ffp-contract=off.
 *
 * Parity status per function: see the header comment of each .c file.
 */
#ifndef FMG_ORACLE_H
#define FMG_ORACLE_H
#include <stdint.h>

#define ORC_OK 0
#define ORC_EINVAL 1
#define ORC_ERANGE 2
#define ORC_ENOMEM 3
#define ORC_MAXLEV 16

/* ---- schedule (tab:precisions PAPER.md:820-841) ---- */
typedef struct {
  int b_u, k_u;      /* solution width  w_u(l,L) = b_u + k_u (L-l)  (b1, increment p+1) */
  int b_r, k_r;      /* residual/correction width w_r = b_r + k_r (L-l) (b2, increment m=1) */
  int n_ir;          /* N: IR iterations per FMG level (Alg 3.3) */
  int cheb_degree;   /* k: Chebyshev-Jacobi degree (reading R4) */
  double lambda_hi;  /* upper eigenvalue bound of D^-1 A used by Chebyshev */
  double alpha;      /* lower bound = lambda_hi / alpha */
  int smoother;      /* 0 Chebyshev-Jacobi (R4), 1 multicolor Gauss-Seidel with
                        (p+1)^d colours, 2 lexicographic Gauss-Seidel (PAPER.md:689-690,
                        1624; oracle only) -- SURVEY §8f N1 */
  int nu;            /* V(0,1) cycles of cFas per IR iteration (Alg 3.1, PAPER.md:633-661;
                        SURVEY §8f N2); cycles after the first start from the previous
                        correction: fine-to-coarse s sweep and nonzero-guess terms
                        (reading R23).  0 or 1: one cycle from zero. */
  int cfas_fp32;     /* cFas in FP32 (tab:precisions PAPER.md:820-841: the cFas working
                        precision is at most L + b_r <= 15 bits at the configurations;
                        reading R28): z, b, the Chebyshev iterates and w in float with
                        the FP64 constants rounded to float; the coarse solve, the
                        correction and everything of the residual stay FP64.  Chebyshev,
                        nu = 1 only. */
} orc_schedule;

/* ---- grid geometry of level l ---- */
typedef struct {
  int n;        /* p * 2^(l+1): nodes 0..n-1 stored per dim, node 0 = boundary */
  int NX;       /* stored x extent = roundup(n, 32) */
  int NY, NZ;   /* n, n (3D) or 1 (2D) */
  int64_t size; /* NX*NY*NZ */
  int64_t nblk; /* size / 32 */
} orc_level;

void orc_level_geom(int d, int p, int l, orc_level* g);
/* OpenMP threads the oracle's per-point loops use (OMP_NUM_THREADS; results
 * do not depend on it: every output is one canonical chain of one thread,
 * every norm a sequential sum). */
int orc_threads(void);
void orc_set_threads(int n);

/* ---- BFP codec (orc_bfp.c) ---- */
int orc_block_encode(const double* x, int w, int64_t* m, int* E);
double orc_block_decode_one(int64_t m, int E, int w);
void orc_pack_block(const int64_t* m, int w, uint32_t* words);
void orc_unpack_block(const uint32_t* words, int w, int64_t* m);
int orc_bfp_encode(const double* x, int64_t n, int width, uint32_t* mant, int8_t* exps);
int orc_bfp_decode(const uint32_t* mant, const int8_t* exps, int64_t n, int width, double* x);
/* streaming-exponent BFP (readings R19-R21): xexp/xstart
 * have room for `width` kept blocks; *nblocks <= width. */
int orc_stream_encode(const double* x, int64_t n, int width, uint32_t* mant, int32_t* xexp,
                      int64_t* xstart, int32_t* nblocks);
int orc_stream_decode(const uint32_t* mant, const int32_t* xexp, const int64_t* xstart, int32_t nblocks,
                      int64_t n, int width, double* x);

/* ---- discretisation (orc_fem.c) ---- */
void orc_ref_matrices(int p, int64_t* Knum, int64_t* Kden, int64_t* Mnum, int64_t* Mden);
void orc_coef_A(int p, double* Kc, double* Mc); /* [p][2p+1] assembled 1D rows */
void orc_coef_P(int p, double* W);              /* [2p][p+1] prolongation weights */
void orc_coef_R(int p, double* Rw);             /* [p][4p-1] restriction weights  */
void orc_apply_A(int d, int p, int l, const double* u, double* out);
void orc_apply_A_f32(int d, int p, int l, const float* u, float* out);   /* same tree in float */
void orc_prolong_f32(int d, int p, int lf, const float* coarse, float* fine);
void orc_prolong(int d, int p, int lf, const double* coarse, double* fine);
void orc_restrict(int d, int p, int lf, const double* fine, double* coarse);
void orc_rhs_table(int p, int l, double* g);    /* g[0..n-1], 1D load integrals */
void orc_rhs(int d, int p, int l, double* f);
double orc_rhs_const(int d);
void orc_inv_diag_ref(int d, int p, double* invd); /* [p^d] by node type */
void orc_inv_diag(int d, int p, int l, double* invD); /* full array */
int orc_coarse_n(int d, int p);
void orc_coarse_matrix(int d, int p, double* A0);  /* A_0 dense (n0 x n0) */
int orc_coarse_inverse(int d, int p, double* Ainv);
void orc_cheb_coefs(const orc_schedule* s, double* inv_theta, double* alpha, double* beta);

/* ---- compact FMG (orc_cfmg.c) ---- */
typedef struct orc_ctx orc_ctx;
int orc_create(int d, int p, int levels, const orc_schedule* s, orc_ctx** out);
/* Plane-streamed mode (orc_stream.c; Alg 5.3/5.4 PAPER.md:999-1157 at plane
 * granularity): the same sections and norms as orc_create's simple mode, bit
 * for bit, with O(planes) FP64 temporaries instead of full-size arrays.
 * Chebyshev smoother, nu = 1, FP64 cFas; orc_get_array (l > 0),
 * orc_decode_solution and orc_smooth return ORC_EINVAL on such a context. */
int orc_create_streamed(int d, int p, int levels, const orc_schedule* s, orc_ctx** out);
int64_t orc_stream_bytes(const orc_ctx* c);   /* peak bytes of its plane windows */
void orc_destroy(orc_ctx* c);
int orc_solve(orc_ctx* c);                         /* Alg 3.3 from scratch */
int orc_smooth(orc_ctx* c, int l, const double* b, double* y); /* cFas smoother from y = 0 */
int orc_solve_upto(orc_ctx* c, int Lstop, int iters_last); /* partial solve, for tests */
int orc_residual(orc_ctx* c, int L, double* norms);/* Alg 3.2 at FMG level L */
int orc_cfas_correct(orc_ctx* c, int L);           /* Alg 3.1 + correction */
const double* orc_norms(orc_ctx* c);               /* [Lmax+1][N][Lmax+1] */
int orc_lmax(orc_ctx* c);
int orc_get_section(orc_ctx* c, int which, int l, uint32_t* mant, int8_t* exps, int* width);
int orc_set_section(orc_ctx* c, int which, int l, const double* x, int width);
int orc_decode_solution(orc_ctx* c, int L, double* uhat);
int orc_errors(int d, int p, int l, const double* uhat, double* err3);
int orc_get_array(orc_ctx* c, int which, int l, double* dst);

/* ---- standard FP64 reference solver (orc_std.c) ---- */
int orc_std_solve(int d, int p, int levels, const orc_schedule* s, int cycles, double* uhat);
int orc_std_vcycle_rho(int d, int p, int levels, const orc_schedule* s, int iters, double* rho);

#endif
