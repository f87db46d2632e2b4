/*
 * orc_stream.c -- the oracle's plane-streamed mode.  TEST INFRASTRUCTURE ONLY
 * (see oracle.h).
 *
 * The linear-space forms of the two sweeps, at plane granularity (a "node" of
 * the paper's lstCol conditions is one plane of the last axis: z in 3D, the
 * row y in 2D):
 *   Alg 5.4 fmgResidual (alg:fmg-residual-opt-recursive):
 *     c2f(l): while i_l < n_l and lstCol(P_l, i_l) < i_{l-1}:
 *               u_{l,i} = ú_{l,i} + (P_l u_{l-1})_i;  i_l++;
 *               l = L ? f2c(L) : c2f(l+1)
 *     f2c(l): while j_l < n_l and (l = L ? lstCol(A_L, j_L) < i_L
 *                                       : lstCol(R_{l+1}, j_l) < j_{l+1}):
 *               t_{l,j} = l = L ? f_{L,j} - (A_L u_L)_j : (R_{l+1} t_{l+1})_j;
 *               r_{l,j} = fix(t_{l,j});  j_l++;  l > 0 ? f2c(l-1)
 *   Alg 5.3 cFas (alg:cfas-opt-recursive), nu = 1 from
 *   ý = 0, z_0 = 0:
 *     c2f(l): while i_l < n_l and lstCol(P_l, i_l) < j_{l-1}:
 *               z_{l,i} = (P_l w_{l-1})_i;  i_l++;
 *               every plane j of ý_l whose smoother stencil is available;
 *               l < L ? c2f(l+1)
 * Each temporary (u_l, t_l, z_l, the smoother iterates) lives in a window of
 * a few planes ("empty buffer with a capacity of δ(·) DoFs ... drop oldest
 * value"; eq:tail-len PAPER.md:918-934): the
 * windows hold O(p k) planes per level, so the temporaries take linear space in
 * the finest plane, not in the grid.  Every value is computed by the same
 * canonical expression as the simple mode (orc_cfmg.c), so the two modes are
 * bit-identical (tests/test_oracle_stream.py).  Readings:
 *   - z_l = P_l (z_{l-1} + ý_{l-1}) as one application on the sum (reading R23
 *     of the simple mode; the paper writes P ý + P z);
 *   - the Chebyshev-Jacobi smoother of degree k is M_l = a polynomial of
 *     degree k-1 in D^-1 A_l: its k applications of A_l are pipelined stages,
 *     stage s lagging stage s-1 by the reach p of A_l (lstCol(A_l, j) = j + p);
 *   - the intermediate per-plane results of the in-plane passes (x, then y in
 *     3D) are what the windows keep: they are functions of one plane.
 * Scope: Chebyshev smoother, nu = 1, FP64 cFas (orc_create_streamed refuses the
 * others).
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include "orc_internal.h"

enum { K_A = 0, K_P = 1, K_R = 2 };

/* A window of planes: plane q lives in slot q % cap, tagged with q; reading a
 * plane that has been dropped is an oracle bug and aborts. */
typedef struct {
  int cap;
  int64_t ps;
  double* buf;
  int64_t* tag;
} win_t;

static int64_t g_bytes;

static void win_init(win_t* w, int cap, int64_t ps) {
  w->cap = cap;
  w->ps = ps;
  w->buf = malloc(sizeof(double) * cap * ps);
  w->tag = malloc(sizeof(int64_t) * cap);
  if (!w->buf || !w->tag) { fprintf(stderr, "orc_stream: out of memory\n"); abort(); }
  for (int i = 0; i < cap; ++i) w->tag[i] = -1;
  g_bytes += (int64_t)sizeof(double) * cap * ps;
}
static void win_free(win_t* w) {
  free(w->buf); free(w->tag);
  w->buf = NULL; w->tag = NULL;
}
static double* win_put(win_t* w, int64_t q) {
  int s = (int)(q % w->cap);
  w->tag[s] = q;
  return w->buf + s * w->ps;
}
static const double* win_get(const win_t* w, int64_t q) {
  int s = (int)(q % w->cap);
  if (w->tag[s] != q) {
    fprintf(stderr, "orc_stream: plane %lld dropped from its window (cap %d)\n", (long long)q, w->cap);
    abort();
  }
  return w->buf + s * w->ps;
}

/* ---------------------------------------------------------------- geometry */
typedef struct {
  int d, p;
  int n[ORC_MAXLEV];     /* planes (= nodes per axis) of level l */
  int64_t ps[ORC_MAXLEV];/* stored entries per plane */
  int NX[ORC_MAXLEV];
  double Kc[3 * 7], Mc[3 * 7], W[6 * 4], Rw[3 * 11];
} geo_t;

static void geo_init(geo_t* G, const orc_ctx* c, int L) {
  G->d = c->d; G->p = c->p;
  for (int l = 0; l <= L; ++l) {
    G->n[l] = c->g[l].n;
    G->NX[l] = c->g[l].NX;
    G->ps[l] = (int64_t)c->g[l].NX * (c->d == 3 ? c->g[l].NY : 1);
  }
  orc_coef_A(c->p, G->Kc, G->Mc);
  orc_coef_P(c->p, G->W);
  orc_coef_R(c->p, G->Rw);
}

/* logical node counts of one plane of level l (3D: n x n; 2D: the row, n) */
static void pdims(const geo_t* G, int nx, int ny, int out[3]) {
  out[0] = nx; out[1] = G->d == 3 ? ny : 1; out[2] = 1;
}

/* lstCol at plane granularity: the last plane of the coarser (P) / finer (R)
 * level or of the same level (A) that output plane i reads. */
static int lst_P(const geo_t* G, int l, int i) {
  int p = G->p, b = p * (i / (2 * p)) + p;
  return b < G->n[l - 1] - 1 ? b : G->n[l - 1] - 1;
}
static int lst_A(const geo_t* G, int l, int j) {
  int b = j + G->p;
  return b < G->n[l] - 1 ? b : G->n[l] - 1;
}
static int lst_R(const geo_t* G, int l, int j) {  /* coarse plane j of level l */
  int b = 2 * j + 2 * G->p - 1;
  return b < G->n[l + 1] - 1 ? b : G->n[l + 1] - 1;
}

/* ------------------------------------------------------- in-plane passes --
 * The passes of orc_apply_A / orc_prolong / orc_restrict along the axes of a
 * plane, applied to one plane (each output of pass1d along x or y depends on
 * one plane only). */

/* prolongation of a level-(l-1) plane to level l in-plane extents */
static void inplane_P(const geo_t* G, int l, const double* in, double* out, double* tmp) {
  int nf = G->n[l], nc = G->n[l - 1], a[3], b[3], e[3];
  pdims(G, nc, nc, a);
  pdims(G, nf, nc, b);
  pdims(G, nf, nf, e);
  if (G->d == 3) {
    orc_pass1d(G->p, K_P, G->W, 0, in, a, tmp, b);
    orc_pass1d(G->p, K_P, G->W, 1, tmp, b, out, e);
  } else {
    orc_pass1d(G->p, K_P, G->W, 0, in, a, out, e);
  }
}

/* restriction of a level-(l+1) plane to level l in-plane extents */
static void inplane_R(const geo_t* G, int l, const double* in, double* out, double* tmp) {
  int nf = G->n[l + 1], nc = G->n[l], a[3], b[3], e[3];
  pdims(G, nf, nf, a);
  pdims(G, nc, nf, b);
  pdims(G, nc, nc, e);
  if (G->d == 3) {
    orc_pass1d(G->p, K_R, G->Rw, 0, in, a, tmp, b);
    orc_pass1d(G->p, K_R, G->Rw, 1, tmp, b, out, e);
  } else {
    orc_pass1d(G->p, K_R, G->Rw, 0, in, a, out, e);
  }
}

/* the in-plane part of A_l (orc_apply_A): 3D: a = Mx u, b = Kx u, c = My a,
 * s = Ky a + My b -> (X1, X2) = (c, s);  2D: (X1, X2) = (Mx u, Kx u). */
static void inplane_A(const geo_t* G, int l, const double* u, double* X1, double* X2, double* t) {
  int n = G->n[l], g[3];
  int64_t ps = G->ps[l];
  pdims(G, n, n, g);
  if (G->d == 3) {
    double *a = t, *b = t + ps, *dd = t + 2 * ps, *e = t + 3 * ps;
    orc_pass1d(G->p, K_A, G->Mc, 0, u, g, a, g);
    orc_pass1d(G->p, K_A, G->Kc, 0, u, g, b, g);
    orc_pass1d(G->p, K_A, G->Kc, 1, a, g, dd, g);
    orc_pass1d(G->p, K_A, G->Mc, 1, b, g, e, g);
    orc_pass1d(G->p, K_A, G->Mc, 1, a, g, X1, g);
    for (int64_t i = 0; i < ps; ++i) X2[i] = dd[i] + e[i];
  } else {
    orc_pass1d(G->p, K_A, G->Mc, 0, u, g, X1, g);
    orc_pass1d(G->p, K_A, G->Kc, 0, u, g, X2, g);
  }
}

/* x index of entry i of a plane, and whether it is an unknown of the plane */
static int unknown_in_plane(const geo_t* G, int l, int64_t i, int z) {
  int NX = G->NX[l], n = G->n[l], x = (int)(i % NX);
  int y = G->d == 3 ? (int)(i / NX) : z;
  return x >= 1 && x < n && y >= 1 && (G->d == 2 || z >= 1);
}

/* ------------------------------------------------------ last-axis passes -- */
/* (A_l v) at plane z from the windows X1, X2 of inplane_A(v); masked to the
 * unknowns as orc_apply_A does. */
static void stream_A(const geo_t* G, int l, const win_t* X1, const win_t* X2, int z, double* out) {
  int p = G->p, n = G->n[l], R = 2 * p + 1, tau = z % p;
  int64_t ps = G->ps[l];
  const double* c1[7];
  const double* c2[7];
  for (int o = -p; o <= p; ++o) {
    int j = z + o;
    int ok = j >= 1 && j <= n - 1;
    c1[o + p] = ok ? win_get(X1, j) : NULL;
    c2[o + p] = ok ? win_get(X2, j) : NULL;
  }
  if (G->d == 3) {
    double h = ldexp(1.0, -(l + 1));
    for (int64_t i = 0; i < ps; ++i) {
      if (z < 1) { out[i] = 0.0; continue; }
      double acc = 0.0;
      for (int o = -p; o <= p; ++o) acc = fma(G->Kc[tau * R + o + p], c1[o + p] ? c1[o + p][i] : 0.0, acc);
      for (int o = -p; o <= p; ++o) acc = fma(G->Mc[tau * R + o + p], c2[o + p] ? c2[o + p][i] : 0.0, acc);
      out[i] = h * acc;
    }
  } else {
    for (int64_t i = 0; i < ps; ++i) {
      int x = (int)i;
      double dd = 0.0, e = 0.0;
      if (!(z < 1 || z > n - 1 || x >= n)) {
        for (int o = -p; o <= p; ++o) dd = fma(G->Kc[tau * R + o + p], c1[o + p] ? c1[o + p][i] : 0.0, dd);
        for (int o = -p; o <= p; ++o) e = fma(G->Mc[tau * R + o + p], c2[o + p] ? c2[o + p][i] : 0.0, e);
      }
      out[i] = dd + e;
    }
  }
  for (int64_t i = 0; i < ps; ++i)
    if (!unknown_in_plane(G, l, i, z)) out[i] = 0.0;
}

/* (P_l v) at fine plane i from the window of in-plane prolonged coarse planes */
static void stream_P(const geo_t* G, int l, const win_t* PX, int i, double* out) {
  int p = G->p, nf = G->n[l], nc = G->n[l - 1], r = i % (2 * p), b = p * (i / (2 * p));
  int64_t ps = G->ps[l];
  if (i < 1 || i > nf - 1) {
    memset(out, 0, sizeof(double) * ps);
    return;
  }
  const double* v[4];
  for (int t = 0; t <= p; ++t) {
    int j = b + t;
    v[t] = (j >= 1 && j <= nc - 1) ? win_get(PX, j) : NULL;
  }
  for (int64_t e = 0; e < ps; ++e) {
    if ((int)(e % G->NX[l]) >= nf) { out[e] = 0.0; continue; }
    double acc = 0.0;
    for (int t = 0; t <= p; ++t) acc = fma(G->W[r * (p + 1) + t], v[t] ? v[t][e] : 0.0, acc);
    out[e] = acc;
  }
}

/* (R_{l+1} v) at coarse plane j of level l from the window of in-plane
 * restricted fine planes (indexed by the fine plane) */
static void stream_R(const geo_t* G, int l, const win_t* T2, int j, double* out) {
  int p = G->p, nc = G->n[l], nf = G->n[l + 1], tau = j % p, S = 4 * p - 1;
  int64_t ps = G->ps[l];
  if (j < 1 || j > nc - 1) {
    memset(out, 0, sizeof(double) * ps);
    return;
  }
  const double* v[11];
  for (int s = 0; s < S; ++s) {
    int jj = 2 * j - (2 * p - 1) + s;
    v[s] = (jj >= 1 && jj <= nf - 1) ? win_get(T2, jj) : NULL;
  }
  for (int64_t e = 0; e < ps; ++e) {
    if ((int)(e % G->NX[l]) >= nc) { out[e] = 0.0; continue; }
    double acc = 0.0;
    for (int s = 0; s < S; ++s) acc = fma(G->Rw[tau * S + s], v[s] ? v[s][e] : 0.0, acc);
    out[e] = acc;
  }
}

/* section blocks of plane z (a plane is a whole number of 32-entry blocks) */
static void sec_decode_plane(const sec_t* s, int64_t ps, int z, double* x) {
  int64_t o = (int64_t)z * ps;
  for (int64_t i = 0; i < ps; ++i) x[i] = orc_block_decode_one(s->m[o + i], s->E[(o + i) / 32], s->w);
}
static int sec_encode_plane(sec_t* s, int64_t ps, int z, const double* x) {
  int64_t o = (int64_t)z * ps;
  for (int64_t b = 0; b < ps / 32; ++b) {
    int E;
    int rc = orc_block_encode(x + 32 * b, s->w, s->m + o + 32 * b, &E);
    if (rc) return rc;
    s->E[o / 32 + b] = (int8_t)E;
  }
  return ORC_OK;
}

/* =========================================================== Alg 5.4 ==== */
typedef struct {
  orc_ctx* c;
  geo_t G;
  int L;
  int i[ORC_MAXLEV], j[ORC_MAXLEV];
  win_t PX[ORC_MAXLEV];  /* in-plane prolonged u_{l-1} planes (indexed by coarse plane) */
  win_t X1, X2;          /* inplane_A(u_L) */
  win_t T2[ORC_MAXLEV];  /* in-plane restricted t_{l+1} planes (indexed by fine plane) */
  double *u, *t, *f, *au, *tmp, *gtab;
  double nsum[ORC_MAXLEV];
  int rc;
} res_t;

static void res_f2c(res_t* S, int l);

static void res_c2f(res_t* S, int l) {
  const geo_t* G = &S->G;
  while (!S->rc && S->i[l] < G->n[l] && lst_P(G, l, S->i[l]) < S->i[l - 1]) {
    int i = S->i[l];
    stream_P(G, l, &S->PX[l], i, S->au);              /* (P_l u_{l-1})_i */
    sec_decode_plane(&S->c->u[l], G->ps[l], i, S->u);  /* ú_{l,i} */
    for (int64_t e = 0; e < G->ps[l]; ++e) S->u[e] = S->u[e] + S->au[e];
    if (l < S->L) inplane_P(G, l + 1, S->u, win_put(&S->PX[l + 1], i), S->tmp);
    else inplane_A(G, l, S->u, win_put(&S->X1, i), win_put(&S->X2, i), S->tmp);
    S->i[l]++;
    if (l == S->L) res_f2c(S, S->L);
    else res_c2f(S, l + 1);
  }
}

static void res_f2c(res_t* S, int l) {
  const geo_t* G = &S->G;
  const int L = S->L;
  for (;;) {
    if (S->rc || S->j[l] >= G->n[l]) return;
    int can = (l == L) ? lst_A(G, L, S->j[L]) < S->i[L] : lst_R(G, l, S->j[l]) < S->j[l + 1];
    if (!can) return;
    int j = S->j[l];
    if (l == L) {                                       /* t_L = f_L - A_L u_L */
      stream_A(G, L, &S->X1, &S->X2, j, S->au);
      orc_rhs_plane(G->d, G->p, L, S->gtab, j, S->f);
      for (int64_t e = 0; e < G->ps[l]; ++e) S->t[e] = S->f[e] - S->au[e];
    } else {                                            /* t_l = R_{l+1} t_{l+1} */
      stream_R(G, l, &S->T2[l], j, S->t);
    }
    int rc = sec_encode_plane(&S->c->r[l], G->ps[l], j, S->t);   /* r_l = fix(t_l) */
    if (rc) { S->rc = rc; return; }
    for (int64_t e = 0; e < G->ps[l]; ++e) S->nsum[l] += S->t[e] * S->t[e];
    if (l > 0) inplane_R(G, l - 1, S->t, win_put(&S->T2[l - 1], j), S->tmp);
    S->j[l]++;
    if (l > 0) res_f2c(S, l - 1);
  }
}

int orc_stream_residual(orc_ctx* c, int L, double* norms) {
  res_t* S = calloc(1, sizeof(res_t));
  if (!S) return ORC_ENOMEM;
  S->c = c;
  S->L = L;
  geo_init(&S->G, c, L);
  const geo_t* G = &S->G;
  const int p = c->p;
  g_bytes = 0;
  int64_t psL = G->ps[L];
  const int cap = 4 * p + 4;
  for (int l = 1; l <= L; ++l) win_init(&S->PX[l], cap, G->ps[l]);
  for (int l = 0; l < L; ++l) win_init(&S->T2[l], cap, G->ps[l]);
  win_init(&S->X1, cap, psL);
  win_init(&S->X2, cap, psL);
  S->u = malloc(sizeof(double) * psL);
  S->t = malloc(sizeof(double) * psL);
  S->f = malloc(sizeof(double) * psL);
  S->au = malloc(sizeof(double) * psL);
  S->tmp = malloc(sizeof(double) * 4 * psL);
  S->gtab = malloc(sizeof(double) * G->n[L]);
  g_bytes += (int64_t)sizeof(double) * (8 * psL + G->n[L]);
  orc_rhs_table(p, L, S->gtab);
  for (int l = 0; l <= L; ++l) c->r[l].w = orc_wr(c, l, L);
  /* u_0 = ú_0, all planes (i_0 = n_0) */
  for (int z = 0; z < G->n[0]; ++z) {
    sec_decode_plane(&c->u[0], G->ps[0], z, S->u);
    if (L > 0) inplane_P(G, 1, S->u, win_put(&S->PX[1], z), S->tmp);
    else inplane_A(G, 0, S->u, win_put(&S->X1, z), win_put(&S->X2, z), S->tmp);
  }
  S->i[0] = G->n[0];
  if (L > 0) res_c2f(S, 1);
  else res_f2c(S, 0);
  int rc = S->rc;
  for (int l = 0; l <= L && !rc; ++l)
    if (S->i[l] != G->n[l] || S->j[l] != G->n[l]) {
      fprintf(stderr, "orc_stream_residual: level %d incomplete\n", l);
      abort();
    }
  if (!rc && norms)
    for (int l = 0; l <= L; ++l) norms[l] = sqrt(S->nsum[l]);
  c->stream_bytes = g_bytes > c->stream_bytes ? g_bytes : c->stream_bytes;
  for (int l = 0; l <= L; ++l) { win_free(&S->PX[l]); win_free(&S->T2[l]); }
  win_free(&S->X1); win_free(&S->X2);
  free(S->u); free(S->t); free(S->f); free(S->au); free(S->tmp); free(S->gtab);
  free(S);
  return rc;
}

/* =========================================================== Alg 5.3 ==== */
typedef struct {
  win_t PW;              /* in-plane prolonged w_{l-1} planes (indexed by coarse plane) */
  win_t Z, XZ1, XZ2;     /* z_l and inplane_A(z_l) */
  win_t B;               /* b = r_l - A_l z_l */
  win_t DV[9], Y[9];     /* Chebyshev stage s: d and y */
  win_t XY1[9], XY2[9];  /* inplane_A(y_s), s < k */
  int nz, ns[9], nw;
} lev_t;

typedef struct {
  orc_ctx* c;
  geo_t G;
  int L, k;
  lev_t lv[ORC_MAXLEV];
  double *a, *b, *tmp, *idref;
  int rc;
} cf_t;

static void cf_stages(cf_t* S, int l) {
  const geo_t* G = &S->G;
  orc_ctx* c = S->c;
  lev_t* V = &S->lv[l];
  const int n = G->n[l], k = S->k;
  const int64_t ps = G->ps[l];
  double* iD = S->tmp + 4 * ps;
  /* stage 1: b = r_l - A_l z_l;  d = inv_theta (invD b);  y = d */
  while (V->ns[1] < n && lst_A(G, l, V->ns[1]) < V->nz) {
    int m = V->ns[1];
    stream_A(G, l, &V->XZ1, &V->XZ2, m, S->a);
    sec_decode_plane(&c->r[l], ps, m, S->b);
    double* bb = win_put(&V->B, m);
    double* dv = win_put(&V->DV[1], m);
    double* y = win_put(&V->Y[1], m);
    orc_inv_diag_plane(G->d, G->p, l, S->idref, m, iD);
    for (int64_t e = 0; e < ps; ++e) {
      bb[e] = S->b[e] - S->a[e];
      dv[e] = c->inv_theta * (iD[e] * bb[e]);
      y[e] = dv[e];
    }
    if (k >= 2) inplane_A(G, l, y, win_put(&V->XY1[1], m), win_put(&V->XY2[1], m), S->tmp);
    V->ns[1]++;
  }
  /* stages j = 2..k: q = b - A y; d = fma(alpha_j, d, beta_j (invD q)); y = y + d */
  for (int s = 2; s <= k; ++s)
    while (V->ns[s] < V->ns[s - 1] && lst_A(G, l, V->ns[s]) < V->ns[s - 1]) {
      int m = V->ns[s];
      stream_A(G, l, &V->XY1[s - 1], &V->XY2[s - 1], m, S->a);
      const double* bb = win_get(&V->B, m);
      const double* d0 = win_get(&V->DV[s - 1], m);
      const double* y0 = win_get(&V->Y[s - 1], m);
      double* dv = win_put(&V->DV[s], m);
      double* y = win_put(&V->Y[s], m);
      orc_inv_diag_plane(G->d, G->p, l, S->idref, m, iD);
      for (int64_t e = 0; e < ps; ++e) {
        double q = bb[e] - S->a[e];
        dv[e] = fma(c->cal[s - 1], d0[e], c->cbe[s - 1] * (iD[e] * q));
        y[e] = y0[e] + dv[e];
      }
      if (s < k) inplane_A(G, l, y, win_put(&V->XY1[s], m), win_put(&V->XY2[s], m), S->tmp);
      V->ns[s]++;
    }
  /* ý_l = fix(y) at w_r(l, L); w_l = z_l + dec ý_l */
  while (!S->rc && V->nw < V->ns[k]) {
    int m = V->nw;
    int rc = sec_encode_plane(&c->y[l], ps, m, win_get(&V->Y[k], m));
    if (rc) { S->rc = rc; return; }
    sec_decode_plane(&c->y[l], ps, m, S->b);
    const double* z = win_get(&V->Z, m);
    for (int64_t e = 0; e < ps; ++e) S->a[e] = z[e] + S->b[e];
    if (l < S->L) inplane_P(G, l + 1, S->a, win_put(&S->lv[l + 1].PW, m), S->tmp);
    V->nw++;
  }
}

static void cf_c2f(cf_t* S, int l) {
  const geo_t* G = &S->G;
  lev_t* V = &S->lv[l];
  while (!S->rc && V->nz < G->n[l] && lst_P(G, l, V->nz) < S->lv[l - 1].nw) {
    int i = V->nz;
    double* z = win_put(&V->Z, i);
    stream_P(G, l, &V->PW, i, z);                    /* z_l = P_l w_{l-1} */
    inplane_A(G, l, z, win_put(&V->XZ1, i), win_put(&V->XZ2, i), S->tmp);
    V->nz++;
    cf_stages(S, l);
    if (l < S->L) cf_c2f(S, l + 1);
  }
}

int orc_stream_cfas(orc_ctx* c, int L) {
  cf_t* S = calloc(1, sizeof(cf_t));
  if (!S) return ORC_ENOMEM;
  S->c = c;
  S->L = L;
  S->k = c->s.cheb_degree;
  geo_init(&S->G, c, L);
  const geo_t* G = &S->G;
  const int p = c->p, k = S->k;
  g_bytes = 0;
  const int cap = (k + 3) * p + 4;
  const int64_t psL = G->ps[L];
  for (int l = 1; l <= L; ++l) {
    lev_t* V = &S->lv[l];
    const int64_t ps = G->ps[l];
    win_init(&V->PW, cap, ps);
    win_init(&V->Z, cap, ps); win_init(&V->XZ1, cap, ps); win_init(&V->XZ2, cap, ps);
    win_init(&V->B, cap, ps);
    for (int s = 1; s <= k; ++s) {
      win_init(&V->DV[s], cap, ps); win_init(&V->Y[s], cap, ps);
      if (s < k) { win_init(&V->XY1[s], cap, ps); win_init(&V->XY2[s], cap, ps); }
    }
  }
  S->a = malloc(sizeof(double) * psL);
  S->b = malloc(sizeof(double) * psL);
  S->tmp = malloc(sizeof(double) * 5 * psL);
  S->idref = malloc(sizeof(double) * 27);
  g_bytes += (int64_t)sizeof(double) * 7 * psL;
  orc_inv_diag_ref(c->d, p, S->idref);
  for (int l = 0; l <= L; ++l) c->y[l].w = orc_wr(c, l, L);
  /* coarse level PAPER.md:640: ý_0 = fix(A_0^{-1} r_0); w_0 = dec ý_0 (z_0 = 0) */
  {
    const orc_level* g = &c->g[0];
    double* r0 = malloc(sizeof(double) * g->size);
    double* y0 = malloc(sizeof(double) * g->size);
    orc_sec_decode(&c->r[0], g, r0);
    orc_coarse_solve(c, r0, y0);
    int rc = orc_sec_encode(&c->y[0], g, y0, orc_wr(c, 0, L));
    if (!rc) {
      orc_sec_decode(&c->y[0], g, y0);
      for (int z = 0; z < G->n[0] && L > 0; ++z)
        inplane_P(G, 1, y0 + z * G->ps[0], win_put(&S->lv[1].PW, z), S->tmp);
    }
    S->rc = rc;
    S->lv[0].nw = G->n[0];
    free(r0); free(y0);
  }
  if (!S->rc && L > 0) cf_c2f(S, 1);
  int rc = S->rc;
  for (int l = 1; l <= L && !rc; ++l)
    if (S->lv[l].nw != G->n[l]) {
      fprintf(stderr, "orc_stream_cfas: level %d incomplete\n", l);
      abort();
    }
  c->stream_bytes = g_bytes > c->stream_bytes ? g_bytes : c->stream_bytes;
  for (int l = 1; l <= L; ++l) {
    lev_t* V = &S->lv[l];
    win_free(&V->PW); win_free(&V->Z); win_free(&V->XZ1); win_free(&V->XZ2); win_free(&V->B);
    for (int s = 1; s <= k; ++s) {
      win_free(&V->DV[s]); win_free(&V->Y[s]);
      if (s < k) { win_free(&V->XY1[s]); win_free(&V->XY2[s]); }
    }
  }
  free(S->a); free(S->b); free(S->tmp); free(S->idref);
  free(S);
  return rc;
}

/* correction PAPER.md:798 block by block: ú_l <- reg(dec ú_l + dec ý_l) at w_u(l, L) */
int orc_stream_correct(orc_ctx* c, int L) {
  for (int l = 0; l <= L; ++l) {
    const orc_level* g = &c->g[l];
    sec_t* u = &c->u[l];
    const sec_t* y = &c->y[l];
    int wu_old = u->w, wnew = orc_wu(c, l, L);
    double a[32];
    for (int64_t b = 0; b < g->nblk; ++b) {
      for (int j = 0; j < 32; ++j)
        a[j] = orc_block_decode_one(u->m[32 * b + j], u->E[b], wu_old) +
               orc_block_decode_one(y->m[32 * b + j], y->E[b], y->w);
      int E;
      int rc = orc_block_encode(a, wnew, u->m + 32 * b, &E);
      if (rc) return rc;
      u->E[b] = (int8_t)E;
    }
    u->w = wnew;
  }
  return ORC_OK;
}
