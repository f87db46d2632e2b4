// fmg1d_assembly.cpp -- native host assembly of the 1D B-spline operators
// (§8(f) row N4; include/fmg1d.h).  Setup code of the product path, FP64 on
// the host; written independently of the oracle (different algorithms where
// there is a choice: the two-scale matrix comes from the discrete B-spline
// recurrence of knot insertion here, from an L2 projection in the oracle).
//
//   knots        open uniform vector, 2^(l+1) elements (R24)
//   basis        local Cox-de Boor triangle, derivatives by the difference
//                formula D N_{j,q} = q [N_{j,q-1}/(t_{j+q}-t_j) - N_{j+1,q-1}/(t_{j+q+1}-t_{j+1})]
//   quadrature   Gauss-Legendre nodes by Newton on P_n (p+3 points for A, p+6 for f)
//   P_l          Oslo algorithm 1: P_ij = alpha_{j,p}(i), the discrete B-spline of the
//                coarse knots at the fine knots (Cohen, Lyche, Riesenfeld 1980)
//   A_0^-1       Gauss-Jordan with partial pivoting in long double
#include <cmath>
#include <cstring>
#include <vector>

#include "../../include/fmg1d.h"
#include "fmg1d_internal.h"

namespace fmg1d {

static bool args_ok(int p, int m, int l) { return p >= 1 && p <= 7 && (m == 1 || m == 2) && p >= 2 * m - 1 && l >= 0 && l <= 24; }

int nel(int l) { return 1 << (l + 1); }
int n_unknowns(int p, int m, int l) { return nel(l) + p - 2 * m; }

std::vector<double> knot_vector(int p, int l) {
  const int ne = nel(l);
  std::vector<double> t;
  for (int i = 0; i <= p; ++i) t.push_back(0.0);
  for (int i = 1; i < ne; ++i) t.push_back((double)i / ne);  // dyadic: exact
  for (int i = 0; i <= p; ++i) t.push_back(1.0);
  return t;
}

// Support structure of P_l: for fine unknown i, the coarse unknowns j whose
// B-spline support contains the fine one's (the only possible nonzeros).
void structure(int p, int m, int l, std::vector<int>& c0, std::vector<int>& c1) {
  const std::vector<double> tf = knot_vector(p, l), tc = knot_vector(p, l - 1);
  const int nf = n_unknowns(p, m, l), nc = n_unknowns(p, m, l - 1);
  c0.assign(nf, -1);
  c1.assign(nf, -1);
  for (int i = 0; i < nf; ++i) {
    const double a = tf[i + m], b = tf[i + m + p + 1];
    for (int j = 0; j < nc; ++j) {
      if (tc[j + m] <= a && b <= tc[j + m + p + 1]) {
        if (c0[i] < 0) c0[i] = j;
        c1[i] = j;
      }
    }
  }
}

int ell_width(int p, int m, int l) {
  std::vector<int> c0, c1;
  structure(p, m, l, c0, c1);
  int kp = 0;
  for (size_t i = 0; i < c0.size(); ++i) kp = std::max(kp, c1[i] - c0[i] + 1);
  return kp;
}

// Gauss-Legendre nodes / weights on [-1, 1].
static void gauss_legendre(int n, std::vector<double>& x, std::vector<double>& w) {
  x.assign(n, 0.0);
  w.assign(n, 0.0);
  auto legendre = [n](long double z, long double& pn, long double& dp) {
    long double p0 = 1, p1 = z;
    for (int j = 2; j <= n; ++j) {
      const long double p2 = ((2 * j - 1) * z * p1 - (j - 1) * p0) / j;
      p0 = p1;
      p1 = p2;
    }
    pn = p1;                                  // P_n(z)
    dp = n * (z * p1 - p0) / (z * z - 1);     // P_n'(z)
  };
  for (int k = 0; k < n; ++k) {
    long double z = cosl(3.14159265358979323846264338327950288L * (k + 0.75L) / (n + 0.5L)), pn, dp;
    for (int it = 0; it < 8; ++it) {  // Newton converges quadratically from this guess
      legendre(z, pn, dp);
      z -= pn / dp;
    }
    legendre(z, pn, dp);
    x[k] = (double)z;
    w[k] = (double)(2 / ((1 - z * z) * dp * dp));
  }
}

// Values (der = 0) or der-th derivatives of the p+1 B-splines nonzero on the
// span s (t[s] <= x < t[s+1]): out[r] belongs to function s - p + r.
static void basis_local(const std::vector<double>& t, int p, int s, double x, int der, double* out) {
  // N[q][j - (s - q)] = N_{j,q}(x) for j in [s-q, s]
  double N[8][8] = {};
  N[0][0] = 1.0;
  for (int q = 1; q <= p; ++q) {
    for (int r = 0; r <= q; ++r) {
      const int j = s - q + r;
      double v = 0.0;
      // N_{j,q-1} lives at r-1 + ... : index of j in row q-1 is j - (s - q + 1) = r - 1
      if (r >= 1) {
        const double d = t[j + q] - t[j];
        if (d > 0) v += (x - t[j]) / d * N[q - 1][r - 1];
      }
      if (r <= q - 1) {
        const double d = t[j + q + 1] - t[j + 1];
        if (d > 0) v += (t[j + q + 1] - x) / d * N[q - 1][r];
      }
      N[q][r] = v;
    }
  }
  // derivatives: coefficients c over the degree-(p-der) functions
  // D^der N_{i,p} = sum_k c_k N_{i+k, p-der}
  for (int r = 0; r <= p; ++r) {
    const int i = s - p + r;
    double c[8] = {};
    c[0] = 1.0;
    int q = p;
    for (int d = 0; d < der; ++d, --q) {
      double nc[8] = {};
      for (int k = 0; k <= d; ++k) {
        const int j = i + k;
        const double d1 = t[j + q] - t[j];
        const double d2 = t[j + q + 1] - t[j + 1];
        if (d1 > 0) nc[k] += q * c[k] / d1;
        if (d2 > 0) nc[k + 1] -= q * c[k] / d2;
      }
      memcpy(c, nc, sizeof(c));
    }
    double v = 0.0;
    for (int k = 0; k <= der; ++k) {
      const int j = i + k;  // degree q = p - der function j; nonzero only for j in [s-q, s]
      if (j >= s - q && j <= s) v += c[k] * N[q][j - (s - q)];
    }
    out[r] = v;
  }
}

void assemble_operator(int p, int m, int l, double* Ab) {
  const std::vector<double> t = knot_vector(p, l);
  const int ne = nel(l), n = n_unknowns(p, m, l), W = 2 * p + 1;
  std::vector<double> gx, gw;
  gauss_legendre(p + 3, gx, gw);
  memset(Ab, 0, sizeof(double) * n * W);
  const double h = 1.0 / ne;
  for (int e = 0; e < ne; ++e) {
    const int s = e + p;  // span of element e
    double ke[8][8] = {};
    for (size_t q = 0; q < gx.size(); ++q) {
      const double x = e * h + 0.5 * h * (gx[q] + 1.0), wq = 0.5 * h * gw[q];
      double d[8];
      basis_local(t, p, s, x, m, d);
      for (int a = 0; a <= p; ++a)
        for (int b = 0; b <= p; ++b) ke[a][b] += wq * d[a] * d[b];
    }
    for (int a = 0; a <= p; ++a) {
      const int i = s - p + a - m;
      if (i < 0 || i >= n) continue;
      for (int b = 0; b <= p; ++b) {
        const int j = s - p + b - m;
        if (j < 0 || j >= n) continue;
        Ab[(size_t)i * W + (j - i + p)] += ke[a][b];
      }
    }
  }
}

static double manufactured_f(int m, double x) {
  const double pi = 3.14159265358979323846;
  if (m == 1) {  // u = x(1-x) cos(pi x / 2), f = -u''
    const double a = pi / 2, c = cos(a * x), sn = sin(a * x);
    const double g = x - x * x, g1 = 1 - 2 * x, g2 = -2.0;
    return -(g2 * c - 2 * a * g1 * sn - a * a * g * c);
  }
  const double a = 2 * pi;  // u = 1 - cos(2 pi x), f = u''''
  return -a * a * a * a * cos(a * x);
}

void assemble_load(int p, int m, int l, double* f) {
  const std::vector<double> t = knot_vector(p, l);
  const int ne = nel(l), n = n_unknowns(p, m, l);
  std::vector<double> gx, gw;
  gauss_legendre(p + 6, gx, gw);
  memset(f, 0, sizeof(double) * n);
  const double h = 1.0 / ne;
  for (int e = 0; e < ne; ++e) {
    const int s = e + p;
    for (size_t q = 0; q < gx.size(); ++q) {
      const double x = e * h + 0.5 * h * (gx[q] + 1.0), wq = 0.5 * h * gw[q];
      double v[8];
      basis_local(t, p, s, x, 0, v);
      const double fx = manufactured_f(m, x);
      for (int a = 0; a <= p; ++a) {
        const int i = s - p + a - m;
        if (i >= 0 && i < n) f[i] += wq * fx * v[a];
      }
    }
  }
}

void assemble_prolongation(int p, int m, int l, double* Pv) {
  const std::vector<double> tf = knot_vector(p, l), tc = knot_vector(p, l - 1);
  std::vector<int> c0, c1;
  structure(p, m, l, c0, c1);
  const int nf = n_unknowns(p, m, l), kp = ell_width(p, m, l);
  memset(Pv, 0, sizeof(double) * nf * kp);
  for (int i = 0; i < nf; ++i) {
    const int I = i + m;  // all-function index on the fine knots
    for (int k = 0; k <= c1[i] - c0[i]; ++k) {
      const int J = c0[i] + k + m;  // coarse all-function index
      // alpha_{J+r, q}(I) for r = 0..p-q, built up from q = 0
      double a[8];
      for (int r = 0; r <= p; ++r) a[r] = (tc[J + r] <= tf[I] && tf[I] < tc[J + r + 1]) ? 1.0 : 0.0;
      for (int q = 1; q <= p; ++q) {
        for (int r = 0; r <= p - q; ++r) {
          const int j = J + r;
          double v = 0.0;
          const double d1 = tc[j + q] - tc[j], d2 = tc[j + q + 1] - tc[j + 1];
          if (d1 > 0) v += (tf[I + q] - tc[j]) / d1 * a[r];
          if (d2 > 0) v += (tc[j + q + 1] - tf[I + q]) / d2 * a[r + 1];
          a[r] = v;
        }
      }
      Pv[(size_t)i * kp + k] = a[0];
    }
  }
}

bool invert(int n, const double* Ab, int p, double* out) {
  std::vector<long double> A((size_t)n * 2 * n, 0.0L);
  for (int i = 0; i < n; ++i) {
    for (int k = 0; k < 2 * p + 1; ++k) {
      const int j = i - p + k;
      if (j >= 0 && j < n) A[(size_t)i * 2 * n + j] = Ab[(size_t)i * (2 * p + 1) + k];
    }
    A[(size_t)i * 2 * n + n + i] = 1.0L;
  }
  for (int c = 0; c < n; ++c) {
    int piv = c;
    for (int r = c + 1; r < n; ++r)
      if (fabsl(A[(size_t)r * 2 * n + c]) > fabsl(A[(size_t)piv * 2 * n + c])) piv = r;
    if (A[(size_t)piv * 2 * n + c] == 0.0L) return false;
    if (piv != c)
      for (int k = 0; k < 2 * n; ++k) std::swap(A[(size_t)c * 2 * n + k], A[(size_t)piv * 2 * n + k]);
    const long double d = A[(size_t)c * 2 * n + c];
    for (int k = 0; k < 2 * n; ++k) A[(size_t)c * 2 * n + k] /= d;
    for (int r = 0; r < n; ++r) {
      if (r == c) continue;
      const long double f = A[(size_t)r * 2 * n + c];
      if (f == 0.0L) continue;
      for (int k = 0; k < 2 * n; ++k) A[(size_t)r * 2 * n + k] -= f * A[(size_t)c * 2 * n + k];
    }
  }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) out[(size_t)i * n + j] = (double)A[(size_t)i * 2 * n + n + j];
  return true;
}

}  // namespace fmg1d

using namespace fmg1d;

extern "C" {

int fmg1d_size(int p, int m, int l) { return args_ok(p, m, l) ? n_unknowns(p, m, l) : -1; }

int fmg1d_ell_width(int p, int m, int l) { return (args_ok(p, m, l) && l >= 1) ? ell_width(p, m, l) : -1; }

int fmg1d_assemble_operator(int p, int m, int l, double* Ab) {
  if (!args_ok(p, m, l) || !Ab) return FMG_EINVAL;
  assemble_operator(p, m, l, Ab);
  return FMG_OK;
}

int fmg1d_assemble_prolongation(int p, int m, int l, double* Pv) {
  if (!args_ok(p, m, l) || l < 1 || !Pv) return FMG_EINVAL;
  assemble_prolongation(p, m, l, Pv);
  return FMG_OK;
}

int fmg1d_assemble_load(int p, int m, int l, double* f) {
  if (!args_ok(p, m, l) || !f) return FMG_EINVAL;
  assemble_load(p, m, l, f);
  return FMG_OK;
}

}  // extern "C"
