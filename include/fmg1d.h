/*
 * fmg1d.h -- C-ABI of the 1D B-spline compact FMG in libfmg.so (§8(f) row N4):
 * the paper's other workloads, solved in batches on the GPU.
 *
 * Problem (R24-R27):
 *   Poisson  -u'' = f,  u = 0 at 0 and 1                (m = 1)
 *   biharmonic u'''' = f, u = u' = 0 at 0 and 1         (m = 2)
 *   on (0, 1), B-splines of degree p (1 <= p <= 7, p >= 2m - 1) on the open
 *   uniform knot vector with 2^(l+1) elements at level l; homogeneous
 *   Dirichlet data removes the m B-splines at each end, so level l has
 *   n_l = 2^(l+1) + p - 2m unknowns (fmg1d_size).
 *
 * Method: Alg 3.3 / 3.2 / 3.1 with ONE V(0,1) cycle per IR
 *   iteration, the coarse solve by the explicit A_0^-1, the smoother one
 *   Gauss-Seidel sweep from zero (lexicographic; or
 *   multicolour, rows i mod (p+1) -- DESIGN.md R27), and the solution,
 *   residual and correction sections in the 32-entry BFP of fmg.h at widths
 *   w_u(l,L) = b1 + (p+1)(L-l), w_r(l,L) = b2 + m(L-l)
 *   (tab:experiments-params).  Matrices, f and every
 *   temporary are FP64 (R26).  Every product is evaluated in the order of
 *   reading R27 (row terms summed from 0.0, ascending storage index), which
 *   makes the result bit-identical to the oracle (oracle/bspline1d.py).
 *
 * Operator layouts (R27), all row-major FP64, host memory, copied at create:
 *   A_l band   n_l x (2p+1): Ab[i][k] = (A_l)_{i, i-p+k}, 0 outside 0..n_l-1.
 *   P_l ELL    n_l x kp_l (fmg1d_ell_width): Pv[i][k] = (P_l)_{i, c0_l(i)+k},
 *              c0_l(i) = the first coarse unknown whose B-spline support
 *              contains that of fine unknown i; entries past the last such
 *              coarse unknown are 0.  R_l = P_l^T is derived by the library.
 *   A_0^-1     n_0 x n_0.
 *
 * Batches: `batch` independent problems share the operators; problem b has its
 *   own load vectors f_l (b-major: f[l][b * n_l + i]) and its own sections.
 *   One CTA solves one problem.
 * Errors: FMG_OK or the fmg.h codes; FMG_ERANGE when an encode meets a
 *   non-finite value or an exponent above 127 (reported by fmg1d_sync).
 */
#ifndef FMG1D_H
#define FMG1D_H
#include <stdint.h>

#include "fmg.h"

#ifdef __cplusplus
extern "C" {
#endif

#define FMG1D_LEX 0  /* lexicographic Gauss-Seidel (the paper's smoother) */
#define FMG1D_MCGS 1 /* multicolour Gauss-Seidel, p + 1 colours */

/* N: IR iterations per FMG level; b1, b2: Table 3's base widths (the
 * increments are p+1 and m); smoother: FMG1D_LEX or FMG1D_MCGS. */
typedef struct {
  int N;
  int b1;
  int b2;
  int smoother;
} fmg1d_schedule;

typedef struct fmg1d_ctx fmg1d_ctx;

/* n_l, or -1 for bad arguments.  Host only. */
int fmg1d_size(int p, int m, int l);

/* kp_l: the ELL width of P_l (l >= 1), or -1.  Host only. */
int fmg1d_ell_width(int p, int m, int l);

/* Native assembly (host, FP64, no GPU).  Writes the band of A_l (n_l*(2p+1)
 * doubles) by Gauss-Legendre quadrature with p+3 points per element
 * (K_ij = int B_i^(m) B_j^(m)). */
int fmg1d_assemble_operator(int p, int m, int l, double* Ab);

/* Native two-scale matrix P_l in the ELL layout (n_l*kp_l doubles, l >= 1) by
 * the discrete B-spline (Oslo) recurrence of midpoint knot insertion. */
int fmg1d_assemble_prolongation(int p, int m, int l, double* Pv);

/* Native load vector of the paper's manufactured problem:
 * m = 1: u = x(1-x)cos(pi x/2), f = -u''; m = 2: u = 1 - cos(2 pi x), f = u''''.
 * f_i = int f B_i, p+6 Gauss points per element; n_l doubles. */
int fmg1d_assemble_load(int p, int m, int l, double* f);

/* Create a context for `levels` FMG levels (1 <= levels <= 20) and `batch`
 * problems (>= 1).  Ab[l], Pv[l] (Pv[0] unused) and A0inv are host arrays in
 * the layouts above; passing Ab = NULL (resp. Pv, A0inv) assembles them
 * natively (A0inv by Gauss-Jordan elimination in long double).  The load
 * vectors start at zero.  Widths must stay in [2, 54]: b1 + (p+1)(levels-1)
 * and b2 + m(levels-1) <= 54.  `stream` is a cudaStream_t (NULL: legacy). */
int fmg1d_create(int p, int m, int levels, const fmg1d_schedule* s, int batch, const double* const* Ab,
                 const double* const* Pv, const double* A0inv, void* stream, fmg1d_ctx** out);
int fmg1d_destroy(fmg1d_ctx* c);

/* Host -> device copy of the load vectors: f[l] holds batch*n_l doubles
 * (b-major), l = 0..levels-1.  Asynchronous on the context's stream; the host
 * arrays must stay valid until the next fmg1d_sync. */
int fmg1d_set_load(fmg1d_ctx* c, const double* const* f);

/* One full solve of every problem of the batch (Alg 3.3 up to the finest
 * level): a single kernel launch, asynchronous. */
int fmg1d_solve_async(fmg1d_ctx* c);
/* Wait for the stream; returns FMG_ERANGE if an encode failed. */
int fmg1d_sync(fmg1d_ctx* c);

/* End to end with host buffers: copies f (as fmg1d_set_load) in, solves, and
 * copies the finest-level solution of every problem (batch*n_L doubles,
 * b-major) to `u`.  Synchronous. */
int fmg1d_solve_host(fmg1d_ctx* c, const double* const* f, double* u);

/* Finest-level solution (standard form, FP64) of problem b: n_L doubles to
 * host `u`.  Synchronous. */
int fmg1d_solution(fmg1d_ctx* c, int b, double* u);

/* Device pointer of the solutions (batch*n_L doubles, b-major); valid until
 * destroy. */
int fmg1d_solution_device(fmg1d_ctx* c, double** u);

/* Section of problem b after the solve: which = 0 solution u_l, 1 residual
 * r_l, 2 correction y_l (of the last IR iteration at the finest level).
 * Copies nblk_l*w words (w words per 32-entry block) to `mant`, nblk_l
 * exponents to `exps` and the width to *w.  Synchronous. */
int fmg1d_section(fmg1d_ctx* c, int which, int l, int b, uint32_t* mant, int8_t* exps, int* w);

#ifdef __cplusplus
}
#endif
#endif
