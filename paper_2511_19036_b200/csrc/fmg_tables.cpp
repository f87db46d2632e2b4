// fmg_tables.cpp -- host-side operator / RHS tables of libfmg (product path).
//
// Written independently of oracle/: the element matrices are obtained here by
// exact rational integration of the Lagrange basis (the oracle hard-codes
// them), prolongation weights by exact evaluation of the basis, the RHS load
// integrals by 20-point Gauss-Legendre quadrature in __float128 (the oracle
// uses a Taylor series), all rounded once to double.  Canonical forms:
// DESIGN.md §3.  Compiled with -ffp-contract=off.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <quadmath.h>
#include <vector>

#include "fmg_internal.h"

namespace fmg {
namespace {

struct Q {  // exact rational, den > 0, reduced
  __int128 n, d;
  Q(__int128 a = 0, __int128 b = 1) : n(a), d(b) { norm(); }
  static __int128 gcd(__int128 a, __int128 b) {
    if (a < 0) a = -a;
    while (b) { __int128 t = a % b; a = b; b = t; }
    return a;
  }
  void norm() {
    if (d < 0) { n = -n; d = -d; }
    __int128 g = gcd(n, d);
    if (g > 1) { n /= g; d /= g; }
    if (n == 0) d = 1;
  }
  Q operator+(const Q& o) const { return Q(n * o.d + o.n * d, d * o.d); }
  Q operator-(const Q& o) const { return Q(n * o.d - o.n * d, d * o.d); }
  Q operator*(const Q& o) const { return Q(n * o.n, d * o.d); }
  Q operator/(const Q& o) const { return Q(n * o.d, d * o.n); }
  double to_double() const { return (double)(int64_t)n / (double)(int64_t)d; }  // both < 2^53 here
};

using Poly = std::vector<Q>;  // coefficients in xi

Poly pmul(const Poly& a, const Poly& b) {
  Poly r(a.size() + b.size() - 1, Q(0));
  for (size_t i = 0; i < a.size(); ++i)
    for (size_t j = 0; j < b.size(); ++j) r[i + j] = r[i + j] + a[i] * b[j];
  return r;
}
Poly pder(const Poly& a) {
  Poly r;
  for (size_t k = 1; k < a.size(); ++k) r.push_back(a[k] * Q((__int128)k));
  if (r.empty()) r.push_back(Q(0));
  return r;
}
Q pint01(const Poly& a) {
  Q s(0);
  for (size_t k = 0; k < a.size(); ++k) s = s + a[k] / Q((__int128)(k + 1));
  return s;
}
Q peval(const Poly& a, const Q& x) {
  Q s(0), xp(1);
  for (size_t k = 0; k < a.size(); ++k) { s = s + a[k] * xp; xp = xp * x; }
  return s;
}

// phi_t(xi) = prod_{j != t} (p xi - j) / (t - j), equispaced nodes j/p.
Poly lagrange(int p, int t) {
  Poly c{Q(1)};
  for (int j = 0; j <= p; ++j) {
    if (j == t) continue;
    c = pmul(c, Poly{Q(-j, t - j), Q(p, t - j)});
  }
  return c;
}

// Exact reference element matrices K_ref[a][b] = ∫ phi_a' phi_b', M_ref = ∫ phi_a phi_b.
void element_matrices(int p, Q K[4][4], Q M[4][4]) {
  for (int a = 0; a <= p; ++a)
    for (int b = 0; b <= p; ++b) {
      Poly la = lagrange(p, a), lb = lagrange(p, b);
      K[a][b] = pint01(pmul(pder(la), pder(lb)));
      M[a][b] = pint01(pmul(la, lb));
    }
}

// Assembled 1D rows around node i on a three-element patch (nodes 0..3p):
// row of node p + tau (tau = 0 is a vertex).  out[o+p], o in [-p, p].
void assembled_row(int p, Q E[4][4], int tau, Q* out) {
  int nn = 3 * p + 1;
  std::vector<Q> G((size_t)nn * nn, Q(0));
  for (int e = 0; e < 3; ++e)
    for (int a = 0; a <= p; ++a)
      for (int b = 0; b <= p; ++b) G[(size_t)(p * e + a) * nn + p * e + b] = G[(size_t)(p * e + a) * nn + p * e + b] + E[a][b];
  int i = p + tau;
  for (int o = -p; o <= p; ++o) out[o + p] = G[(size_t)i * nn + i + o];
}

}  // namespace

void build_coefs(int dim, int p, double lambda_hi, double alpha, int cheb_degree, Coefs* c) {
  std::memset(c, 0, sizeof(Coefs));
  Q K[4][4], M[4][4];
  element_matrices(p, K, M);
  Q Krow[3][7], Mrow[3][7];
  for (int tau = 0; tau < p; ++tau) {
    assembled_row(p, K, tau, Krow[tau]);
    assembled_row(p, M, tau, Mrow[tau]);
    for (int o = 0; o <= 2 * p; ++o) {
      c->Kc[tau][o] = Krow[tau][o].to_double();
      c->Mc[tau][o] = Mrow[tau][o].to_double();
    }
  }
  // Prolongation: fine node i in coarse element i div 2p at xi = (i mod 2p)/(2p).
  for (int r = 0; r < 2 * p; ++r)
    for (int t = 0; t <= p; ++t) c->Pw[r][t] = peval(lagrange(p, t), Q(r, 2 * p)).to_double();
  // Restriction R = P^T: coarse node cn = p*m + tau (m = 4 keeps indices positive)
  // gathers fine nodes j = 2cn - (2p-1) + s with weight P[j][cn].
  for (int tau = 0; tau < p; ++tau) {
    int cn = 4 * p + tau;
    for (int s = 0; s <= 4 * p - 2; ++s) {
      int j = 2 * cn - (2 * p - 1) + s;
      int e = j / (2 * p), r = j % (2 * p);
      int t = cn - p * e;
      c->Rw[tau][s] = (t >= 0 && t <= p) ? peval(lagrange(p, t), Q(r, 2 * p)).to_double() : 0.0;
    }
  }
  // 1/diag(Â) by node type: 2D Ky Mx + My Kx; 3D Kz My Mx + Mz Ky Mx + Mz My Kx.
  for (int tz = 0; tz < (dim == 3 ? p : 1); ++tz)
    for (int ty = 0; ty < p; ++ty)
      for (int tx = 0; tx < p; ++tx) {
        Q kx = Krow[tx][p], mx = Mrow[tx][p], ky = Krow[ty][p], my = Mrow[ty][p];
        Q dg;
        if (dim == 2) dg = ky * mx + my * kx;
        else {
          Q kz = Krow[tz][p], mz = Mrow[tz][p];
          dg = kz * my * mx + mz * ky * mx + mz * my * kx;
        }
        Q inv = Q(1) / dg;
        c->invd[(tz * p + ty) * p + tx] = inv.to_double();
      }
  // Chebyshev constants.
  double hi = lambda_hi, lo = hi / alpha;
  double theta = (hi + lo) / 2.0, delta = (hi - lo) / 2.0;
  double sigma = theta / delta;
  c->inv_theta = 1.0 / theta;
  double rho = 1.0 / sigma;
  for (int j = 2; j <= cheb_degree && j <= 8; ++j) {
    double rn = 1.0 / (2.0 * sigma - rho);
    c->cal[j - 1] = rn * rho;
    c->cbe[j - 1] = (2.0 * rn) / delta;
    rho = rn;
  }
  c->rhs_c = (double)((__float128)dim * M_PIq * M_PIq);
}

// g_l(i) = ∫ sin(pi x) phi_i(x) dx by 20-point Gauss-Legendre per element in
// __float128, rounded once to double.
void build_rhs_table(int p, int l, double* g) {
  const int NG = 20;
  __float128 xg[NG], wg[NG];
  for (int i = 0; i < NG; ++i) {
    __float128 z = cosq(M_PIq * (i + 0.75Q) / (NG + 0.5Q)), dp = 0;
    for (int it = 0; it < 100; ++it) {
      __float128 p0 = 1, p1 = 0;
      for (int j = 1; j <= NG; ++j) {
        __float128 p2 = p1;
        p1 = p0;
        p0 = ((2 * j - 1) * z * p1 - (j - 1) * p2) / j;
      }
      dp = NG * (z * p0 - p1) / (z * z - 1);
      __float128 dz = p0 / dp;
      z -= dz;
      if (fabsq(dz) < 1e-34Q) break;
    }
    xg[i] = (1 - z) / 2;
    wg[i] = 1 / ((1 - z * z) * dp * dp);  // = (2/((1-z^2) P'^2)) / 2
  }
  // basis values at the Gauss points (exact rational coefficients, evaluated in quad)
  __float128 phi[4][NG];
  for (int t = 0; t <= p; ++t) {
    Poly L = lagrange(p, t);
    for (int q = 0; q < NG; ++q) {
      __float128 s = 0, xp = 1;
      for (size_t k = 0; k < L.size(); ++k) {
        s += ((__float128)(int64_t)L[k].n / (__float128)(int64_t)L[k].d) * xp;
        xp *= xg[q];
      }
      phi[t][q] = s;
    }
  }
  int n = p << (l + 1), nel = 1 << (l + 1);
  __float128 H = ldexpq(1.0Q, -(l + 1));
  std::vector<__float128> acc(n + 1, 0);
  for (int e = 0; e < nel; ++e) {
    __float128 sv[NG];
    for (int q = 0; q < NG; ++q) sv[q] = sinq(M_PIq * (e * H + H * xg[q]));
    for (int t = 0; t <= p; ++t) {
      __float128 s = 0;
      for (int q = 0; q < NG; ++q) s += wg[q] * sv[q] * phi[t][q];
      acc[p * e + t] += H * s;
    }
  }
  g[0] = 0.0;
  for (int i = 1; i < n; ++i) g[i] = (double)acc[i];
}

int coarse_count(int dim, int p) {
  int m = 2 * p - 1;
  return dim == 2 ? m * m : m * m * m;
}

// A_0^{-1}: Â_0 entries as correctly rounded exact rationals, Gauss-Jordan
// without pivoting on [Â_0 | I] in the canonical order of DESIGN.md §3.7, then
// scaled by h_0^(2-d).
int build_coarse_inverse(int dim, int p, double* Ainv) {
  Q K[4][4], M[4][4];
  element_matrices(p, K, M);
  // full 1D matrices on level 0: nodes 0..2p (two elements)
  int nn = 2 * p + 1;
  std::vector<Q> K1((size_t)nn * nn, Q(0)), M1((size_t)nn * nn, Q(0));
  for (int e = 0; e < 2; ++e)
    for (int a = 0; a <= p; ++a)
      for (int b = 0; b <= p; ++b) {
        K1[(size_t)(p * e + a) * nn + p * e + b] = K1[(size_t)(p * e + a) * nn + p * e + b] + K[a][b];
        M1[(size_t)(p * e + a) * nn + p * e + b] = M1[(size_t)(p * e + a) * nn + p * e + b] + M[a][b];
      }
  int m = 2 * p - 1, n = coarse_count(dim, p), w = 2 * n;
  std::vector<double> Mx((size_t)n * w);
  for (int I = 0; I < n; ++I) {
    int ix = I % m + 1, iy = (I / m) % m + 1, iz = dim == 3 ? I / (m * m) + 1 : 0;
    for (int J = 0; J < n; ++J) {
      int jx = J % m + 1, jy = (J / m) % m + 1, jz = dim == 3 ? J / (m * m) + 1 : 0;
      Q kx = K1[(size_t)ix * nn + jx], mx = M1[(size_t)ix * nn + jx];
      Q ky = K1[(size_t)iy * nn + jy], my = M1[(size_t)iy * nn + jy];
      Q v;
      if (dim == 2) v = ky * mx + my * kx;
      else {
        Q kz = K1[(size_t)iz * nn + jz], mz = M1[(size_t)iz * nn + jz];
        v = kz * my * mx + mz * ky * mx + mz * my * kx;
      }
      Mx[(size_t)I * w + J] = v.to_double();
    }
    for (int J = 0; J < n; ++J) Mx[(size_t)I * w + n + J] = (I == J) ? 1.0 : 0.0;
  }
  for (int k = 0; k < n; ++k) {
    double piv = Mx[(size_t)k * w + k];
    if (piv == 0.0) return 1;
    for (int j = 0; j < w; ++j) Mx[(size_t)k * w + j] = Mx[(size_t)k * w + j] / piv;
    for (int i = 0; i < n; ++i) {
      if (i == k) continue;
      double f = Mx[(size_t)i * w + k];
      for (int j = 0; j < w; ++j) Mx[(size_t)i * w + j] = Mx[(size_t)i * w + j] - f * Mx[(size_t)k * w + j];
    }
  }
  double sc = dim == 3 ? 2.0 : 1.0;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) Ainv[(size_t)i * n + j] = Mx[(size_t)i * w + n + j] * sc;
  return 0;
}

}  // namespace fmg
