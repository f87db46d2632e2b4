/*
 * orc_std.c -- oracle reference solvers and error norms.
 * TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * orc_errors: relative L2, H1-semi and H1 errors of a standard-representation
 *   coefficient vector against u = prod sin(pi x_k) by tensor Gauss-Legendre
 *   quadrature with p+3 points per dimension per element (reading R13;
 *   ||u||_L2^2 = 2^-d, |u|_H1^2 = d pi^2 2^-d).
 * orc_std_solve: standard (non-compact) FP64 full multigrid with V(1,1) cycles of
 *   the correction scheme (supplement sm:alg:fmg / sm:alg:fmg-correction,
 *   PAPER.md:1781-1841) and the same Chebyshev smoother; used to obtain the
 *   discretisation solution u_L of Eq 7.3 (R14).
 * orc_std_vcycle_rho: asymptotic contraction of the V(0,1) cycle, a property
 *   check on the smoother (SURVEY appendix A4 style).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include "oracle.h"

static void gauss_legendre(int n, double* x, double* w) {
  /* nodes/weights on [0,1]; Newton on P_n from the Chebyshev guess */
  for (int i = 0; i < n; ++i) {
    double z = cos(M_PI * (i + 0.75) / (n + 0.5)), pp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = 0.0;
      for (int j = 1; j <= n; ++j) {
        double p2 = p1;
        p1 = p0;
        p0 = ((2.0 * j - 1.0) * z * p1 - (j - 1.0) * p2) / j;
      }
      pp = n * (z * p0 - p1) / (z * z - 1.0);
      double dz = p0 / pp;
      z -= dz;
      if (fabs(dz) < 1e-16) break;
    }
    x[i] = 0.5 * (1.0 - z);
    w[i] = 1.0 / ((1.0 - z * z) * pp * pp);
  }
}

static void lagrange_vals(int p, double xi, double* v, double* dv) {
  for (int a = 0; a <= p; ++a) {
    double val = 1.0, der = 0.0;
    for (int j = 0; j <= p; ++j) {
      if (j == a) continue;
      double fac = (p * xi - j) / (double)(a - j);
      double dfac = p / (double)(a - j);
      der = der * fac + val * dfac;
      val = val * fac;
    }
    v[a] = val;
    dv[a] = der;
  }
}

int orc_errors(int d, int p, int l, const double* uhat, double* err3) {
  orc_level G;
  orc_level_geom(d, p, l, &G);
  int nq = p + 3, nel = 1 << (l + 1);
  double h = ldexp(1.0, -(l + 1));
  double qx[8], qw[8], phi[8][4], dphi[8][4];
  gauss_legendre(nq, qx, qw);
  for (int q = 0; q < nq; ++q) lagrange_vals(p, qx[q], phi[q], dphi[q]);
  double eL2 = 0.0, eH1 = 0.0;
  int nez = d == 3 ? nel : 1, nqz = d == 3 ? nq : 1, pz = d == 3 ? p : 0;
  double loc[64];
  for (int ez = 0; ez < nez; ++ez)
    for (int ey = 0; ey < nel; ++ey)
      for (int ex = 0; ex < nel; ++ex) {
        for (int c = 0; c <= pz; ++c)
          for (int b = 0; b <= p; ++b)
            for (int a = 0; a <= p; ++a) {
              int ix = p * ex + a, iy = p * ey + b, iz = p * ez + c;
              double v = 0.0;
              if (ix < G.n && iy < G.n && (d == 2 || iz < G.n))
                v = uhat[((int64_t)(d == 3 ? iz : 0) * G.NY + iy) * G.NX + ix];
              loc[(c * (p + 1) + b) * (p + 1) + a] = v;
            }
        for (int qz = 0; qz < nqz; ++qz)
          for (int qy = 0; qy < nq; ++qy)
            for (int qxi = 0; qxi < nq; ++qxi) {
              double val = 0.0, gx = 0.0, gy = 0.0, gz = 0.0;
              for (int c = 0; c <= pz; ++c)
                for (int b = 0; b <= p; ++b)
                  for (int a = 0; a <= p; ++a) {
                    double cz = d == 3 ? phi[qz][c] : 1.0, dcz = d == 3 ? dphi[qz][c] : 0.0;
                    double coef = loc[(c * (p + 1) + b) * (p + 1) + a];
                    val += coef * phi[qxi][a] * phi[qy][b] * cz;
                    gx += coef * dphi[qxi][a] * phi[qy][b] * cz;
                    gy += coef * phi[qxi][a] * dphi[qy][b] * cz;
                    gz += coef * phi[qxi][a] * phi[qy][b] * dcz;
                  }
              gx /= h; gy /= h; gz /= h;
              double x = (ex + qx[qxi]) * h, y = (ey + qx[qy]) * h, z = (ez + qx[qz]) * h;
              double sx = sin(M_PI * x), sy = sin(M_PI * y), sz = d == 3 ? sin(M_PI * z) : 1.0;
              double cx = cos(M_PI * x), cy = cos(M_PI * y), cz = d == 3 ? cos(M_PI * z) : 0.0;
              double u = sx * sy * sz;
              double ux = M_PI * cx * sy * sz, uy = M_PI * sx * cy * sz, uz = M_PI * sx * sy * cz;
              double wq = qw[qxi] * qw[qy] * (d == 3 ? qw[qz] : 1.0);
              eL2 += wq * (val - u) * (val - u);
              eH1 += wq * ((gx - ux) * (gx - ux) + (gy - uy) * (gy - uy) +
                           (d == 3 ? (gz - uz) * (gz - uz) : 0.0));
            }
      }
  double vol = (d == 3) ? h * h * h : h * h;
  eL2 *= vol; eH1 *= vol;
  double nL2 = ldexp(1.0, -d), nH1 = d * M_PI * M_PI * ldexp(1.0, -d);
  err3[0] = sqrt(eL2 / nL2);
  err3[1] = sqrt(eH1 / nH1);
  err3[2] = sqrt((eL2 + eH1) / (nL2 + nH1));
  return ORC_OK;
}

/* ------------------------------------------------ standard FP64 multigrid -- */
typedef struct {
  int d, p, levels;
  orc_schedule s;
  orc_level g[ORC_MAXLEV];
  double* invD[ORC_MAXLEV];
  double* Ainv;
  int n0;
  double inv_theta, cal[8], cbe[8];
} std_ctx;

static void std_coarse(const std_ctx* c, const double* b, double* x) {
  const orc_level* g = &c->g[0];
  int m = 2 * c->p - 1;
  double bv[125];
  for (int J = 0; J < c->n0; ++J) {
    int jx = J % m + 1, jy = (J / m) % m + 1, jz = (c->d == 3) ? J / (m * m) + 1 : 0;
    bv[J] = b[((int64_t)jz * g->NY + jy) * g->NX + jx];
  }
  memset(x, 0, sizeof(double) * g->size);
  for (int I = 0; I < c->n0; ++I) {
    double acc = 0.0;
    for (int J = 0; J < c->n0; ++J) acc += c->Ainv[I * c->n0 + J] * bv[J];
    int ix = I % m + 1, iy = (I / m) % m + 1, iz = (c->d == 3) ? I / (m * m) + 1 : 0;
    x[((int64_t)iz * g->NY + iy) * g->NX + ix] = acc;
  }
}

/* x <- x + Cheb_k(b - A x) */
static void std_smooth(const std_ctx* c, int l, const double* b, double* x) {
  const orc_level* g = &c->g[l];
  int64_t N = g->size;
  double* r = malloc(sizeof(double) * N);
  double* y = malloc(sizeof(double) * N);
  double* dv = malloc(sizeof(double) * N);
  double* ay = malloc(sizeof(double) * N);
  orc_apply_A(c->d, c->p, l, x, ay);
  for (int64_t i = 0; i < N; ++i) r[i] = b[i] - ay[i];
  for (int64_t i = 0; i < N; ++i) { dv[i] = c->inv_theta * (c->invD[l][i] * r[i]); y[i] = dv[i]; }
  for (int j = 2; j <= c->s.cheb_degree; ++j) {
    orc_apply_A(c->d, c->p, l, y, ay);
    for (int64_t i = 0; i < N; ++i) {
      double q = r[i] - ay[i];
      dv[i] = c->cal[j - 1] * dv[i] + c->cbe[j - 1] * (c->invD[l][i] * q);
      y[i] += dv[i];
    }
  }
  for (int64_t i = 0; i < N; ++i) x[i] += y[i];
  free(r); free(y); free(dv); free(ay);
}

static void std_vcycle(const std_ctx* c, int l, const double* b, double* x, int nu1, int nu2) {
  if (l == 0) { std_coarse(c, b, x); return; }
  const orc_level* g = &c->g[l];
  const orc_level* gc = &c->g[l - 1];
  for (int k = 0; k < nu1; ++k) std_smooth(c, l, b, x);
  double* r = malloc(sizeof(double) * g->size);
  double* ax = malloc(sizeof(double) * g->size);
  orc_apply_A(c->d, c->p, l, x, ax);
  for (int64_t i = 0; i < g->size; ++i) r[i] = b[i] - ax[i];
  double* rc = malloc(sizeof(double) * gc->size);
  double* xc = calloc(gc->size, sizeof(double));
  orc_restrict(c->d, c->p, l, r, rc);
  std_vcycle(c, l - 1, rc, xc, nu1, nu2);
  orc_prolong(c->d, c->p, l, xc, ax);
  for (int64_t i = 0; i < g->size; ++i) x[i] += ax[i];
  for (int k = 0; k < nu2; ++k) std_smooth(c, l, b, x);
  free(r); free(ax); free(rc); free(xc);
}

static int std_init(std_ctx* c, int d, int p, int levels, const orc_schedule* s) {
  memset(c, 0, sizeof(*c));
  c->d = d; c->p = p; c->levels = levels; c->s = *s;
  for (int l = 0; l < levels; ++l) {
    orc_level_geom(d, p, l, &c->g[l]);
    c->invD[l] = malloc(sizeof(double) * c->g[l].size);
    orc_inv_diag(d, p, l, c->invD[l]);
  }
  c->n0 = orc_coarse_n(d, p);
  c->Ainv = malloc(sizeof(double) * c->n0 * c->n0);
  orc_coarse_inverse(d, p, c->Ainv);
  orc_cheb_coefs(s, &c->inv_theta, c->cal, c->cbe);
  return ORC_OK;
}

static void std_free(std_ctx* c) {
  for (int l = 0; l < c->levels; ++l) free(c->invD[l]);
  free(c->Ainv);
}

/* FMG with `cycles` V(1,1) cycles per level; uhat on the finest level. */
int orc_std_solve(int d, int p, int levels, const orc_schedule* s, int cycles, double* uhat) {
  std_ctx c;
  if (levels < 1 || levels > ORC_MAXLEV) return ORC_EINVAL;
  std_init(&c, d, p, levels, s);
  double* x = NULL;
  for (int l = 0; l < levels; ++l) {
    const orc_level* g = &c.g[l];
    double* f = malloc(sizeof(double) * g->size);
    orc_rhs(d, p, l, f);
    double* xn = calloc(g->size, sizeof(double));
    if (l == 0) std_coarse(&c, f, xn);
    else {
      orc_prolong(d, p, l, x, xn);
      for (int k = 0; k < cycles; ++k) std_vcycle(&c, l, f, xn, 1, 1);
    }
    free(x);
    x = xn;
    free(f);
  }
  memcpy(uhat, x, sizeof(double) * c.g[levels - 1].size);
  free(x);
  std_free(&c);
  return ORC_OK;
}

/* Contraction of the V(0,1) cycle (zero initial guess is the nu = 1 setting):
 * error propagation e <- e - B A e by power iteration from a fixed vector. */
int orc_std_vcycle_rho(int d, int p, int levels, const orc_schedule* s, int iters, double* rho) {
  std_ctx c;
  std_init(&c, d, p, levels, s);
  int l = levels - 1;
  const orc_level* g = &c.g[l];
  double* e = malloc(sizeof(double) * g->size);
  double* b = malloc(sizeof(double) * g->size);
  double* x = malloc(sizeof(double) * g->size);
  unsigned long long st = 12345;
  for (int64_t i = 0; i < g->size; ++i) {
    st = st * 6364136223846793005ULL + 1442695040888963407ULL;
    e[i] = (double)(st >> 11) / 9007199254740992.0 - 0.5;
  }
  double* mask = malloc(sizeof(double) * g->size);
  orc_inv_diag(d, p, l, mask);
  for (int64_t i = 0; i < g->size; ++i) if (mask[i] == 0.0) e[i] = 0.0;
  double prev = 0.0, r = 0.0;
  for (int k = 0; k < iters; ++k) {
    double nrm = 0.0;
    for (int64_t i = 0; i < g->size; ++i) nrm += e[i] * e[i];
    nrm = sqrt(nrm);
    for (int64_t i = 0; i < g->size; ++i) e[i] /= nrm;
    orc_apply_A(d, p, l, e, b);           /* b = A e ; solve A x = b with x0 = 0 */
    memset(x, 0, sizeof(double) * g->size);
    std_vcycle(&c, l, b, x, 0, 1);
    for (int64_t i = 0; i < g->size; ++i) e[i] = e[i] - x[i];
    double n2 = 0.0;
    for (int64_t i = 0; i < g->size; ++i) n2 += e[i] * e[i];
    r = sqrt(n2);
    (void)prev;
    prev = r;
  }
  *rho = r;
  free(e); free(b); free(x); free(mask);
  std_free(&c);
  return ORC_OK;
}
