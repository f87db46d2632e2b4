/*
 * orc_fem.c -- oracle discretisation: Lagrange Q_p on uniform grids of (0,1)^d.
 * TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * Follows PAPER.md:164-181 (nested spaces, Φ_{l-1} = Φ_l P_l)
 * (R_l := P_l^T, Galerkin A_{l-1} = R_l A_l P_l), PAPER.md:882-888 (matrix-free
 * operator, right-hand side assembled on the fly) and the Poisson problem of
 * eq:pde-poisson PAPER.md:1418-1424 with the manufactured solution
 * u = prod_k sin(pi x_k) of BASELINE.json (reading R1/R12).
 * Each operator is applied factor by factor as the Kronecker product it is
 * (A = K⊗M⊗M + M⊗K⊗M + M⊗M⊗K), in the canonical order of DESIGN.md §3.
 *
 * Pins (tests/test_oracle_fem.py): element matrices = exact rational
 * integrals; dense Kronecker assembly vs apply; Galerkin identity; symmetry;
 * exactness of P on Q_p; Φ_{l-1} = Φ_l P_l at sample points; RHS table vs
 * mpmath quadrature; coarse inverse vs numpy.linalg.solve.
 */
#include <math.h>
#include <quadmath.h>
#include <stdlib.h>
#include <string.h>
#include "orc_internal.h"

void orc_level_geom(int d, int p, int l, orc_level* g) {
  g->n = p << (l + 1);
  g->NX = ((g->n + 31) / 32) * 32;
  g->NY = g->n;
  g->NZ = (d == 3) ? g->n : 1;
  g->size = (int64_t)g->NX * g->NY * g->NZ;
  g->nblk = g->size / 32;
}

/* Reference element matrices (element stiffness = K_ref / h, element mass =
 * h M_ref) of the equispaced Lagrange basis of degree p on [0,1]; integer
 * numerators over a common denominator.  Pinned against exact integration in
 * tests/test_oracle_fem.py::test_element_matrices. */
void orc_ref_matrices(int p, int64_t* Knum, int64_t* Kden, int64_t* Mnum, int64_t* Mden) {
  static const int64_t K1[4] = {1, -1, -1, 1}, M1[4] = {2, 1, 1, 2};
  static const int64_t K2[9] = {7, -8, 1, -8, 16, -8, 1, -8, 7};
  static const int64_t M2[9] = {4, 2, -1, 2, 16, 2, -1, 2, 4};
  static const int64_t K3[16] = {148, -189, 54, -13, -189, 432, -297, 54,
                                 54, -297, 432, -189, -13, 54, -189, 148};
  static const int64_t M3[16] = {128, 99, -36, 19, 99, 648, -81, -36,
                                 -36, -81, 648, 99, 19, -36, 99, 128};
  const int64_t *K, *M;
  if (p == 1) { K = K1; M = M1; *Kden = 1; *Mden = 6; }
  else if (p == 2) { K = K2; M = M2; *Kden = 3; *Mden = 30; }
  else { K = K3; M = M3; *Kden = 40; *Mden = 1680; }
  memcpy(Knum, K, sizeof(int64_t) * (p + 1) * (p + 1));
  memcpy(Mnum, M, sizeof(int64_t) * (p + 1) * (p + 1));
}

/* Assembled 1D row of node type tau (= node index mod p), offset o in [-p,p]
 * (numerator over the matrix's denominator).  A vertex node (tau = 0) gets the
 * last local node of its left element and the first of its right element; an
 * interior node tau couples only within its element. */
static int64_t assembled(int p, const int64_t* ref, int tau, int o) {
  if (tau == 0) {
    if (o == 0) return ref[p * (p + 1) + p] + ref[0];
    if (o > 0) return ref[o];                        /* right element, row 0 */
    return ref[p * (p + 1) + (p + o)];               /* left element, row p */
  }
  if (o < -tau || o > p - tau) return 0;
  return ref[tau * (p + 1) + (tau + o)];
}

void orc_coef_A(int p, double* Kc, double* Mc) {
  int64_t Kn[16], Kd, Mn[16], Md;
  orc_ref_matrices(p, Kn, &Kd, Mn, &Md);
  for (int tau = 0; tau < p; ++tau)
    for (int o = -p; o <= p; ++o) {
      Kc[tau * (2 * p + 1) + o + p] = (double)assembled(p, Kn, tau, o) / (double)Kd;
      Mc[tau * (2 * p + 1) + o + p] = (double)assembled(p, Mn, tau, o) / (double)Md;
    }
}

/* Prolongation weights (Φ_{l-1} = Φ_l P_l): fine node i lies in
 * coarse element e = i div 2p at local coordinate xi = (i mod 2p)/(2p); its row
 * holds the coarse Lagrange basis values phi_t(xi), t = 0..p, on coarse nodes
 * p e + t.  phi_t(r/(2p)) = prod_{j!=t} (r - 2j) / (2 (t - j)), exact rational;
 * dyadic for p <= 3, so the double is exact. W[r][t]. */
void orc_coef_P(int p, double* W) {
  for (int r = 0; r < 2 * p; ++r)
    for (int t = 0; t <= p; ++t) {
      int64_t num = 1, den = 1;
      for (int j = 0; j <= p; ++j) {
        if (j == t) continue;
        num *= (r - 2 * j);
        den *= 2 * (t - j);
      }
      W[r * (p + 1) + t] = (double)num / (double)den;
    }
}

/* Restriction R = P^T: coarse node c = p m + tau gathers fine
 * nodes j = 2c - (2p-1) + s, s = 0..4p-2, with weight P[j, c]. */
void orc_coef_R(int p, double* Rw) {
  double W[6 * 4];
  orc_coef_P(p, W);
  for (int tau = 0; tau < p; ++tau)
    for (int s = 0; s <= 4 * p - 2; ++s) {
      int o = 2 * tau - (2 * p - 1) + s;  /* fine node j relative to 2 p m */
      int e = (o >= 0) ? o / (2 * p) : -((-o + 2 * p - 1) / (2 * p));  /* floor */
      int r = o - 2 * p * e;
      int t = tau - p * e;                /* local index of c in element m+e */
      Rw[tau * (4 * p - 1) + s] = (t >= 0 && t <= p) ? W[r * (p + 1) + t] : 0.0;
    }
}

/* ---------------------------------------------------------------- passes -- */
/* An array on a (possibly mixed-level) grid: logical node counts n[axis]
 * (unknowns 1..n-1 along each axis; n = 1 means "no such axis" in 2D), stored
 * x extent sx = roundup(n[0], 32). */
typedef struct { int n[3]; int sx; } dims_t;

static dims_t mkdims(int nx, int ny, int nz) {
  dims_t t;
  t.n[0] = nx; t.n[1] = ny; t.n[2] = nz;
  t.sx = ((nx + 31) / 32) * 32;
  return t;
}
static int64_t dsize(dims_t t) { return (int64_t)t.sx * t.n[1] * t.n[2]; }

enum { TAP_A, TAP_P, TAP_R };

/* One 1D pass along `axis`.  Outputs at non-unknown indices along the axis are
 * 0; inputs outside 1..n_in-1 read as 0.  Accumulation order:
 * acc = 0; acc = fma(c_t, v_t, acc) for taps t in increasing index order. */
static void pass1d(int p, int kind, const double* C, int axis,
                   const double* in, dims_t di, double* out, dims_t dout) {
  int nout = dout.n[axis], nin = di.n[axis];
  int64_t sin[3] = {1, di.sx, (int64_t)di.sx * di.n[1]};
  /* (OpenMP over output rows: every output is one canonical chain computed by
   * one thread, so the result does not depend on the thread count) */
#pragma omp parallel for collapse(2) schedule(static)
  for (int z = 0; z < dout.n[2]; ++z)
    for (int y = 0; y < dout.n[1]; ++y)
      for (int x = 0; x < dout.sx; ++x) {
        int c[3] = {x, y, z};
        int64_t o_idx = ((int64_t)z * dout.n[1] + y) * dout.sx + x;
        int i = c[axis];
        if (i < 1 || i > nout - 1 || x >= dout.n[0]) {
          out[o_idx] = 0.0;
          continue;
        }
        c[axis] = 0;
        int64_t base_idx = (int64_t)c[2] * sin[2] + (int64_t)c[1] * sin[1] + c[0];
        double acc = 0.0;
        if (kind == TAP_A) {
          int tau = i % p;
          for (int o = -p; o <= p; ++o) {
            int j = i + o;
            double v = (j >= 1 && j <= nin - 1) ? in[base_idx + (int64_t)j * sin[axis]] : 0.0;
            acc = fma(C[tau * (2 * p + 1) + o + p], v, acc);
          }
        } else if (kind == TAP_P) {
          int r = i % (2 * p), b = p * (i / (2 * p));
          for (int t = 0; t <= p; ++t) {
            int j = b + t;
            double v = (j >= 1 && j <= nin - 1) ? in[base_idx + (int64_t)j * sin[axis]] : 0.0;
            acc = fma(C[r * (p + 1) + t], v, acc);
          }
        } else {
          int tau = i % p;
          for (int s = 0; s <= 4 * p - 2; ++s) {
            int j = 2 * i - (2 * p - 1) + s;
            double v = (j >= 1 && j <= nin - 1) ? in[base_idx + (int64_t)j * sin[axis]] : 0.0;
            acc = fma(C[tau * (4 * p - 1) + s], v, acc);
          }
        }
        out[o_idx] = acc;
      }
}

/* Zero every entry that is not an unknown of the grid (boundary index 0 along any
 * axis, x padding). */
static void mask_unknowns(int d, dims_t g, double* v) {
  for (int z = 0; z < g.n[2]; ++z)
    for (int y = 0; y < g.n[1]; ++y)
      for (int x = 0; x < g.sx; ++x) {
        int ok = (x >= 1 && x < g.n[0] && y >= 1 && y < g.n[1] && (d == 2 || z >= 1));
        if (!ok) v[((int64_t)z * g.n[1] + y) * g.sx + x] = 0.0;
      }
}

void orc_pass1d(int p, int kind, const double* C, int axis, const double* in, const int nin[3],
                double* out, const int nout[3]) {
  pass1d(p, kind, C, axis, in, mkdims(nin[0], nin[1], nin[2]), out, mkdims(nout[0], nout[1], nout[2]));
}

/* A_l u, A_l = h^(d-2) Â, Â = Kz My Mx + Mz Ky Mx + Mz My Kx:
 *   a = Mx u, b = Kx u, c = My a, d = Ky a, e = My b, s = d + e;
 *   2D: Â u = s;   3D: Â u = chain(Kz over c, then Mz over s);  A u = h Â u. */
void orc_apply_A(int d, int p, int l, const double* u, double* out) {
  int n = p << (l + 1);
  dims_t g = mkdims(n, n, d == 3 ? n : 1);
  int64_t N = dsize(g);
  double Kc[3 * 7], Mc[3 * 7];
  orc_coef_A(p, Kc, Mc);
  double* a = malloc(sizeof(double) * N);
  double* b = malloc(sizeof(double) * N);
  double* dd = malloc(sizeof(double) * N);
  double* e = malloc(sizeof(double) * N);
  pass1d(p, TAP_A, Mc, 0, u, g, a, g);
  pass1d(p, TAP_A, Kc, 0, u, g, b, g);
  pass1d(p, TAP_A, Kc, 1, a, g, dd, g);
  pass1d(p, TAP_A, Mc, 1, b, g, e, g);
  if (d == 2) {
    for (int64_t i = 0; i < N; ++i) out[i] = dd[i] + e[i];
  } else {
    double* c = malloc(sizeof(double) * N);
    pass1d(p, TAP_A, Mc, 1, a, g, c, g);
    for (int64_t i = 0; i < N; ++i) dd[i] = dd[i] + e[i]; /* s */
    double h = ldexp(1.0, -(l + 1));
    int64_t sz = (int64_t)g.sx * g.n[1];
#pragma omp parallel for collapse(2) schedule(static)
    for (int z = 0; z < n; ++z)
      for (int y = 0; y < n; ++y)
        for (int x = 0; x < g.sx; ++x) {
          int64_t idx = ((int64_t)z * n + y) * g.sx + x;
          if (z < 1) { out[idx] = 0.0; continue; }
          int tau = z % p;
          double acc = 0.0;
          for (int o = -p; o <= p; ++o) {
            int j = z + o;
            double v = (j >= 1 && j <= n - 1) ? c[idx + (int64_t)o * sz] : 0.0;
            acc = fma(Kc[tau * (2 * p + 1) + o + p], v, acc);
          }
          for (int o = -p; o <= p; ++o) {
            int j = z + o;
            double v = (j >= 1 && j <= n - 1) ? dd[idx + (int64_t)o * sz] : 0.0;
            acc = fma(Mc[tau * (2 * p + 1) + o + p], v, acc);
          }
          out[idx] = h * acc;
        }
    free(c);
  }
  mask_unknowns(d, g, out);
  free(a); free(b); free(dd); free(e);
}

/* ------------------------------------------------- FP32 cFas (reading R28) --
 * The same 1D passes and trees in float (fmaf from +0.0f, taps in increasing
 * index order); the float constants are the FP64 constants rounded to float
 * (the prolongation weights are dyadic, hence exact). */
static void pass1d_f32(int p, int kind, const float* C, int axis,
                       const float* in, dims_t di, float* out, dims_t dout) {
  int nout = dout.n[axis], nin = di.n[axis];
  int64_t sin[3] = {1, di.sx, (int64_t)di.sx * di.n[1]};
#pragma omp parallel for collapse(2) schedule(static)
  for (int z = 0; z < dout.n[2]; ++z)
    for (int y = 0; y < dout.n[1]; ++y)
      for (int x = 0; x < dout.sx; ++x) {
        int c[3] = {x, y, z};
        int64_t o_idx = ((int64_t)z * dout.n[1] + y) * dout.sx + x;
        int i = c[axis];
        if (i < 1 || i > nout - 1 || x >= dout.n[0]) {
          out[o_idx] = 0.0f;
          continue;
        }
        c[axis] = 0;
        int64_t base_idx = (int64_t)c[2] * sin[2] + (int64_t)c[1] * sin[1] + c[0];
        float acc = 0.0f;
        if (kind == TAP_A) {
          int tau = i % p;
          for (int o = -p; o <= p; ++o) {
            int j = i + o;
            float v = (j >= 1 && j <= nin - 1) ? in[base_idx + (int64_t)j * sin[axis]] : 0.0f;
            acc = fmaf(C[tau * (2 * p + 1) + o + p], v, acc);
          }
        } else {
          int r = i % (2 * p), b = p * (i / (2 * p));
          for (int t = 0; t <= p; ++t) {
            int j = b + t;
            float v = (j >= 1 && j <= nin - 1) ? in[base_idx + (int64_t)j * sin[axis]] : 0.0f;
            acc = fmaf(C[r * (p + 1) + t], v, acc);
          }
        }
        out[o_idx] = acc;
      }
}

static void coefs_f32(int p, float* Kf, float* Mf) {
  double Kc[3 * 7], Mc[3 * 7];
  orc_coef_A(p, Kc, Mc);
  for (int i = 0; i < 3 * 7; ++i) {
    Kf[i] = (float)Kc[i];
    Mf[i] = (float)Mc[i];
  }
}

void orc_apply_A_f32(int d, int p, int l, const float* u, float* out) {
  int n = p << (l + 1);
  dims_t g = mkdims(n, n, d == 3 ? n : 1);
  int64_t N = dsize(g);
  float Kc[3 * 7], Mc[3 * 7];
  coefs_f32(p, Kc, Mc);
  float* a = malloc(sizeof(float) * N);
  float* b = malloc(sizeof(float) * N);
  float* dd = malloc(sizeof(float) * N);
  float* e = malloc(sizeof(float) * N);
  pass1d_f32(p, TAP_A, Mc, 0, u, g, a, g);
  pass1d_f32(p, TAP_A, Kc, 0, u, g, b, g);
  pass1d_f32(p, TAP_A, Kc, 1, a, g, dd, g);
  pass1d_f32(p, TAP_A, Mc, 1, b, g, e, g);
  if (d == 2) {
    for (int64_t i = 0; i < N; ++i) out[i] = dd[i] + e[i];
  } else {
    float* c = malloc(sizeof(float) * N);
    pass1d_f32(p, TAP_A, Mc, 1, a, g, c, g);
    for (int64_t i = 0; i < N; ++i) dd[i] = dd[i] + e[i]; /* s */
    const float h = ldexpf(1.0f, -(l + 1));
    int64_t sz = (int64_t)g.sx * g.n[1];
#pragma omp parallel for collapse(2) schedule(static)
    for (int z = 0; z < n; ++z)
      for (int y = 0; y < n; ++y)
        for (int x = 0; x < g.sx; ++x) {
          int64_t idx = ((int64_t)z * n + y) * g.sx + x;
          if (z < 1) { out[idx] = 0.0f; continue; }
          int tau = z % p;
          float acc = 0.0f;
          for (int o = -p; o <= p; ++o) {
            int j = z + o;
            float v = (j >= 1 && j <= n - 1) ? c[idx + (int64_t)o * sz] : 0.0f;
            acc = fmaf(Kc[tau * (2 * p + 1) + o + p], v, acc);
          }
          for (int o = -p; o <= p; ++o) {
            int j = z + o;
            float v = (j >= 1 && j <= n - 1) ? dd[idx + (int64_t)o * sz] : 0.0f;
            acc = fmaf(Mc[tau * (2 * p + 1) + o + p], v, acc);
          }
          out[idx] = h * acc;
        }
    free(c);
  }
  for (int z = 0; z < g.n[2]; ++z)   /* mask_unknowns */
    for (int y = 0; y < g.n[1]; ++y)
      for (int x = 0; x < g.sx; ++x) {
        int ok = (x >= 1 && x < g.n[0] && y >= 1 && y < g.n[1] && (d == 2 || z >= 1));
        if (!ok) out[((int64_t)z * g.n[1] + y) * g.sx + x] = 0.0f;
      }
  free(a); free(b); free(dd); free(e);
}

void orc_prolong_f32(int d, int p, int lf, const float* coarse, float* fine) {
  int nf = p << (lf + 1), nc = nf / 2;
  double W[6 * 4];
  float Wf[6 * 4];
  orc_coef_P(p, W);
  for (int i = 0; i < 6 * 4; ++i) Wf[i] = (float)W[i];
  if (d == 2) {
    dims_t g0 = mkdims(nc, nc, 1), g1 = mkdims(nf, nc, 1), g2 = mkdims(nf, nf, 1);
    float* t1 = malloc(sizeof(float) * dsize(g1));
    pass1d_f32(p, TAP_P, Wf, 0, coarse, g0, t1, g1);
    pass1d_f32(p, TAP_P, Wf, 1, t1, g1, fine, g2);
    free(t1);
  } else {
    dims_t g0 = mkdims(nc, nc, nc), g1 = mkdims(nf, nc, nc), g2 = mkdims(nf, nf, nc), g3 = mkdims(nf, nf, nf);
    float* t1 = malloc(sizeof(float) * dsize(g1));
    float* t2 = malloc(sizeof(float) * dsize(g2));
    pass1d_f32(p, TAP_P, Wf, 0, coarse, g0, t1, g1);
    pass1d_f32(p, TAP_P, Wf, 1, t1, g1, t2, g2);
    pass1d_f32(p, TAP_P, Wf, 2, t2, g2, fine, g3);
    free(t1); free(t2);
  }
}

/* fine = P_lf coarse: x pass, then y, then z. */
void orc_prolong(int d, int p, int lf, const double* coarse, double* fine) {
  int nf = p << (lf + 1), nc = nf / 2;
  double W[6 * 4];
  orc_coef_P(p, W);
  if (d == 2) {
    dims_t g0 = mkdims(nc, nc, 1), g1 = mkdims(nf, nc, 1), g2 = mkdims(nf, nf, 1);
    double* t1 = malloc(sizeof(double) * dsize(g1));
    pass1d(p, TAP_P, W, 0, coarse, g0, t1, g1);
    pass1d(p, TAP_P, W, 1, t1, g1, fine, g2);
    free(t1);
  } else {
    dims_t g0 = mkdims(nc, nc, nc), g1 = mkdims(nf, nc, nc), g2 = mkdims(nf, nf, nc),
           g3 = mkdims(nf, nf, nf);
    double* t1 = malloc(sizeof(double) * dsize(g1));
    double* t2 = malloc(sizeof(double) * dsize(g2));
    pass1d(p, TAP_P, W, 0, coarse, g0, t1, g1);
    pass1d(p, TAP_P, W, 1, t1, g1, t2, g2);
    pass1d(p, TAP_P, W, 2, t2, g2, fine, g3);
    free(t1); free(t2);
  }
}

/* coarse = R_lf fine = P_lf^T fine: x pass, then y, then z. */
void orc_restrict(int d, int p, int lf, const double* fine, double* coarse) {
  int nf = p << (lf + 1), nc = nf / 2;
  double Rw[3 * 11];
  orc_coef_R(p, Rw);
  if (d == 2) {
    dims_t g0 = mkdims(nf, nf, 1), g1 = mkdims(nc, nf, 1), g2 = mkdims(nc, nc, 1);
    double* t1 = malloc(sizeof(double) * dsize(g1));
    pass1d(p, TAP_R, Rw, 0, fine, g0, t1, g1);
    pass1d(p, TAP_R, Rw, 1, t1, g1, coarse, g2);
    free(t1);
  } else {
    dims_t g0 = mkdims(nf, nf, nf), g1 = mkdims(nc, nf, nf), g2 = mkdims(nc, nc, nf),
           g3 = mkdims(nc, nc, nc);
    double* t1 = malloc(sizeof(double) * dsize(g1));
    double* t2 = malloc(sizeof(double) * dsize(g2));
    pass1d(p, TAP_R, Rw, 0, fine, g0, t1, g1);
    pass1d(p, TAP_R, Rw, 1, t1, g1, t2, g2);
    pass1d(p, TAP_R, Rw, 2, t2, g2, coarse, g3);
    free(t1); free(t2);
  }
}

/* ------------------------------------------------------------------ RHS -- */
/* g_l(i) = ∫_0^1 sin(pi x) phi_i(x) dx (reading R12), in __float128:
 * on element e = [eH, (e+1)H], x = eH + H xi, sin(b + a xi) = sin b cos(a xi) +
 * cos b sin(a xi) with a = pi H, b = pi e H; both expanded in their Taylor
 * series and integrated term by term against phi_t:  ∫ xi^m phi_t = mu_t(m)
 * (exact moments of the monomial coefficients of phi_t).  Rounded once to
 * double.  Independent of the GPU library, which uses Gauss-Legendre
 * quadrature in __float128. */
void orc_rhs_table(int p, int l, double* g) {
  int n = p << (l + 1), nel = 1 << (l + 1);
  __float128 H = ldexpq(1.0Q, -(l + 1));
  __float128 a = M_PIq * H;
  __float128 coef[4][4];  /* monomial coefficients of phi_t */
  for (int t = 0; t <= p; ++t) {
    __float128 c[4] = {1, 0, 0, 0};
    int deg = 0;
    for (int j = 0; j <= p; ++j) {
      if (j == t) continue;
      /* multiply by (p xi - j) / (t - j) */
      __float128 nc[4] = {0, 0, 0, 0};
      for (int k = 0; k <= deg; ++k) {
        nc[k + 1] += c[k] * p;
        nc[k] -= c[k] * j;
      }
      deg++;
      for (int k = 0; k <= deg; ++k) c[k] = nc[k] / (__float128)(t - j);
    }
    for (int k = 0; k < 4; ++k) coef[t][k] = (k <= p) ? c[k] : 0;
  }
  /* S_cos[t] = sum_k (-1)^k a^{2k}/(2k)! mu_t(2k), S_sin[t] similarly (odd) */
  __float128 Sc[4], Ss[4];
  for (int t = 0; t <= p; ++t) {
    __float128 sc = 0, ss = 0, fac = 1;  /* fac = a^m / m! */
    for (int m = 0; m < 80; ++m) {
      if (m > 0) fac = fac * a / m;
      __float128 mu = 0;
      for (int k = 0; k <= p; ++k) mu += coef[t][k] / (m + k + 1);
      __float128 term = fac * mu;
      int sgn = ((m / 2) % 2 == 0) ? 1 : -1;
      if (m % 2 == 0) sc += sgn * term; else ss += sgn * term;
      if (fac < 1e-45Q) break;
    }
    Sc[t] = sc; Ss[t] = ss;
  }
  __float128* acc = calloc(n + 1, sizeof(__float128));
  for (int e = 0; e < nel; ++e) {
    __float128 b = M_PIq * H * e;
    __float128 sb = sinq(b), cb = cosq(b);
    for (int t = 0; t <= p; ++t) acc[p * e + t] += H * (sb * Sc[t] + cb * Ss[t]);
  }
  g[0] = 0.0;
  for (int i = 1; i < n; ++i) g[i] = (double)acc[i];
  free(acc);
}

double orc_rhs_const(int d) { return (double)((__float128)d * M_PIq * M_PIq); }

/* f_l at node (i,j,k) = ((C_d g(i)) g(j)) g(k), C_d = RN(d pi^2);
 * 0 at non-unknowns.  orc_rhs_plane: plane z of the last axis (3D z, 2D y). */
void orc_rhs_plane(int d, int p, int l, const double* g, int z, double* f) {
  orc_level G;
  orc_level_geom(d, p, l, &G);
  double C = orc_rhs_const(d);
  int ny = d == 3 ? G.NY : 1;
  for (int yy = 0; yy < ny; ++yy)
    for (int x = 0; x < G.NX; ++x) {
      int y = d == 3 ? yy : z;
      int64_t idx = (int64_t)yy * G.NX + x;
      int ok = (x >= 1 && x < G.n && y >= 1 && (d == 2 || z >= 1));
      if (!ok) { f[idx] = 0.0; continue; }
      double v = C * g[x];
      v = v * g[y];
      if (d == 3) v = v * g[z];
      f[idx] = v;
    }
}

void orc_rhs(int d, int p, int l, double* f) {
  orc_level G;
  orc_level_geom(d, p, l, &G);
  double* g = malloc(sizeof(double) * G.n);
  orc_rhs_table(p, l, g);
  int64_t ps = (int64_t)G.NX * (d == 3 ? G.NY : 1);
  for (int z = 0; z < G.n; ++z) orc_rhs_plane(d, p, l, g, z, f + z * ps);
  free(g);
}

/* ------------------------------------------------------------- diagonal -- */
/* diag(Â) at node type (tx, ty[, tz]) as an exact rational; invD_ref =
 * RN(den / num).  invd[tz][ty][tx]. */
void orc_inv_diag_ref(int d, int p, double* invd) {
  int64_t Kn[16], Kd, Mn[16], Md;
  orc_ref_matrices(p, Kn, &Kd, Mn, &Md);
  int64_t kd[3], md[3];
  for (int t = 0; t < p; ++t) { kd[t] = assembled(p, Kn, t, 0); md[t] = assembled(p, Mn, t, 0); }
  for (int tz = 0; tz < (d == 3 ? p : 1); ++tz)
    for (int ty = 0; ty < p; ++ty)
      for (int tx = 0; tx < p; ++tx) {
        int64_t num, den;
        if (d == 2) {
          num = kd[ty] * md[tx] + md[ty] * kd[tx];
          den = Kd * Md;
        } else {
          num = kd[tz] * md[ty] * md[tx] + md[tz] * kd[ty] * md[tx] + md[tz] * md[ty] * kd[tx];
          den = Kd * Md * Md;
        }
        invd[(tz * p + ty) * p + tx] = (double)den / (double)num;
      }
}

/* invD of A_l = h^(d-2) Â: invD_ref * 2^((l+1)(d-2)), 0 at non-unknowns.
 * orc_inv_diag_plane: plane z of the last axis (3D z, 2D y); ref from
 * orc_inv_diag_ref. */
void orc_inv_diag_plane(int d, int p, int l, const double* ref, int z, double* invD) {
  orc_level G;
  orc_level_geom(d, p, l, &G);
  double sc = ldexp(1.0, (l + 1) * (d - 2));
  int ny = d == 3 ? G.NY : 1;
  for (int yy = 0; yy < ny; ++yy)
    for (int x = 0; x < G.NX; ++x) {
      int y = d == 3 ? yy : z;
      int64_t idx = (int64_t)yy * G.NX + x;
      int ok = (x >= 1 && x < G.n && y >= 1 && (d == 2 || z >= 1));
      invD[idx] = ok ? ref[((d == 3 ? z % p : 0) * p + y % p) * p + x % p] * sc : 0.0;
    }
}

void orc_inv_diag(int d, int p, int l, double* invD) {
  orc_level G;
  orc_level_geom(d, p, l, &G);
  double ref[27];
  orc_inv_diag_ref(d, p, ref);
  int64_t ps = (int64_t)G.NX * (d == 3 ? G.NY : 1);
  for (int z = 0; z < G.n; ++z) orc_inv_diag_plane(d, p, l, ref, z, invD + z * ps);
}

/* ----------------------------------------------------------- coarse grid -- */
int orc_coarse_n(int d, int p) {
  int m = 2 * p - 1;
  return d == 2 ? m * m : m * m * m;
}

/* Dense Â_0 (level 0, n = 2p nodes per dim, unknowns 1..2p-1, x fastest):
 * entry = RN(num/den) of the exact Kronecker-sum rational. */
static void coarse_hat(int d, int p, double* A0) {
  int64_t Kn[16], Kd, Mn[16], Md;
  orc_ref_matrices(p, Kn, &Kd, Mn, &Md);
  int m = 2 * p - 1, n0 = orc_coarse_n(d, p);
  for (int I = 0; I < n0; ++I)
    for (int J = 0; J < n0; ++J) {
      int ix = I % m + 1, iy = (I / m) % m + 1, iz = (d == 3) ? I / (m * m) + 1 : 0;
      int jx = J % m + 1, jy = (J / m) % m + 1, jz = (d == 3) ? J / (m * m) + 1 : 0;
      int ox = jx - ix, oy = jy - iy, oz = jz - iz;
      int64_t num = 0, den;
      if (ox < -p || ox > p || oy < -p || oy > p || oz < -p || oz > p) {
        A0[I * n0 + J] = 0.0;
        continue;
      }
      int64_t kx = assembled(p, Kn, ix % p, ox), mx = assembled(p, Mn, ix % p, ox);
      int64_t ky = assembled(p, Kn, iy % p, oy), my = assembled(p, Mn, iy % p, oy);
      if (d == 2) {
        num = ky * mx + my * kx;
        den = Kd * Md;
      } else {
        int64_t kz = assembled(p, Kn, iz % p, oz), mz = assembled(p, Mn, iz % p, oz);
        num = kz * my * mx + mz * ky * mx + mz * my * kx;
        den = Kd * Md * Md;
      }
      A0[I * n0 + J] = (double)num / (double)den;
    }
}

void orc_coarse_matrix(int d, int p, double* A0) {
  int n0 = orc_coarse_n(d, p);
  coarse_hat(d, p, A0);
  double h = 0.5;
  if (d == 3)
    for (int i = 0; i < n0 * n0; ++i) A0[i] = A0[i] * h;
}

/* A_0^{-1} (coarse-grid solve, Alg 3.3 line PAPER.md:786): Gauss-Jordan without
 * pivoting on [Â_0 | I] in the canonical order of DESIGN.md §3.7, then scaled by
 * h_0^(2-d). */
int orc_coarse_inverse(int d, int p, double* Ainv) {
  int n = orc_coarse_n(d, p), w = 2 * n;
  double* A = malloc(sizeof(double) * n * n);
  double* M = malloc(sizeof(double) * n * w);
  coarse_hat(d, p, A);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < w; ++j) M[i * w + j] = (j < n) ? A[i * n + j] : (j - n == i ? 1.0 : 0.0);
  for (int k = 0; k < n; ++k) {
    double piv = M[k * w + k];
    if (piv == 0.0) { free(A); free(M); return ORC_EINVAL; }
    for (int j = 0; j < w; ++j) M[k * w + j] = M[k * w + j] / piv;
    for (int i = 0; i < n; ++i) {
      if (i == k) continue;
      double f = M[i * w + k];
      for (int j = 0; j < w; ++j) M[i * w + j] = M[i * w + j] - f * M[k * w + j];
    }
  }
  double sc = (d == 3) ? 2.0 : 1.0;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) Ainv[i * n + j] = M[i * w + n + j] * sc;
  free(A); free(M);
  return ORC_OK;
}

/* Chebyshev-Jacobi constants (reading R4 / §3.5):
 * hi = lambda_hi, lo = hi/alpha, theta = (hi+lo)/2, delta = (hi-lo)/2,
 * sigma = theta/delta, rho_1 = 1/sigma; for j >= 2: rho_j = 1/(2 sigma - rho_{j-1}),
 * alpha_j = rho_j rho_{j-1}, beta_j = (2 rho_j)/delta.  Index j-1 in the arrays. */
void orc_cheb_coefs(const orc_schedule* s, double* inv_theta, double* al, double* be) {
  double hi = s->lambda_hi, lo = hi / s->alpha;
  double theta = (hi + lo) / 2.0, delta = (hi - lo) / 2.0;
  double sigma = theta / delta;
  *inv_theta = 1.0 / theta;
  double rho = 1.0 / sigma;
  al[0] = 0.0; be[0] = 0.0;
  for (int j = 2; j <= s->cheb_degree; ++j) {
    double rn = 1.0 / (2.0 * sigma - rho);
    al[j - 1] = rn * rho;
    be[j - 1] = (2.0 * rn) / delta;
    rho = rn;
  }
}

/* Threads the OpenMP loops of the oracle use (1 without OpenMP). */
#ifdef _OPENMP
#include <omp.h>
int orc_threads(void) { return omp_get_max_threads(); }
void orc_set_threads(int n) { omp_set_num_threads(n > 0 ? n : 1); }
#else
int orc_threads(void) { return 1; }
void orc_set_threads(int n) { (void)n; }
#endif
