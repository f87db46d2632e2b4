/*
 * orc_internal.h -- oracle-private declarations shared by orc_cfmg.c (simple
 * mode) and orc_stream.c (plane-streamed mode).  TEST INFRASTRUCTURE ONLY
 * (see oracle.h).
 */
#ifndef FMG_ORACLE_INTERNAL_H
#define FMG_ORACLE_INTERNAL_H
#include "oracle.h"

typedef struct {
  int w;          /* current stored width */
  int64_t* m;     /* mantissas, one per stored entry */
  int8_t* E;      /* one exponent per 32-entry block */
} sec_t;

struct orc_ctx {
  int d, p, levels, Lmax;
  orc_schedule s;
  orc_level g[ORC_MAXLEV];
  sec_t u[ORC_MAXLEV];    /* compact solution sections ú_l */
  sec_t r[ORC_MAXLEV];    /* residual sections r_l */
  sec_t y[ORC_MAXLEV];    /* correction sections ý_l */
  double* f[ORC_MAXLEV];  /* f_l (only the current FMG level is used) */
  double* invD[ORC_MAXLEV];
  double* ut[ORC_MAXLEV]; /* decoded standard representation temporaries u_l */
  double* tt[ORC_MAXLEV]; /* residual temporaries t_l */
  double* wt[ORC_MAXLEV]; /* w_l = z_l + dec ý_l */
  double* Ainv;
  int n0;
  double inv_theta, cal[8], cbe[8];
  double* norms;          /* [Lmax+1][N][Lmax+1] */
  int streamed;           /* plane-streamed mode (orc_stream.c): no full-size FP64
                             temporaries above level 0 */
  int64_t stream_bytes;   /* peak bytes of the streamed mode's plane windows */
};


int orc_wu(const orc_ctx* c, int l, int L);   /* w_u(l,L) = b_u + k_u (L-l) */
int orc_wr(const orc_ctx* c, int l, int L);   /* w_r(l,L) = b_r + k_r (L-l) */
void orc_sec_decode(const sec_t* s, const orc_level* g, double* x);
int orc_sec_encode(sec_t* s, const orc_level* g, const double* x, int w);
void orc_coarse_solve(const orc_ctx* c, const double* x, double* y);

/* One canonical 1D pass (orc_fem.c pass1d) over arrays of logical node counts
 * nin/nout (x extent stored rounded up to 32). kind: 0 = A taps, 1 = P, 2 = R. */
void orc_pass1d(int p, int kind, const double* C, int axis, const double* in, const int nin[3],
                double* out, const int nout[3]);
/* f_l and invD_l restricted to plane `z` of the last axis (3D: z; 2D: the row
 * y), as orc_rhs / orc_inv_diag compute them. */
void orc_rhs_plane(int d, int p, int l, const double* gtab, int z, double* f);
void orc_inv_diag_plane(int d, int p, int l, const double* ref, int z, double* invD);

int orc_stream_residual(orc_ctx* c, int L, double* norms);  /* Alg 5.4 (orc_stream.c) */
int orc_stream_cfas(orc_ctx* c, int L);                     /* Alg 5.3 */
int orc_stream_correct(orc_ctx* c, int L);                  /* PAPER.md:798, blockwise */

#endif
