// fmg1d_internal.h -- host-side helpers shared by fmg1d_assembly.cpp and
// fmg1d.cu (the 1D B-spline compact FMG, include/fmg1d.h).
#pragma once
#include <cstdint>
#include <vector>

namespace fmg1d {

constexpr int kMaxLevels = 20;

int nel(int l);
int n_unknowns(int p, int m, int l);
std::vector<double> knot_vector(int p, int l);
void structure(int p, int m, int l, std::vector<int>& c0, std::vector<int>& c1);
int ell_width(int p, int m, int l);
void assemble_operator(int p, int m, int l, double* Ab);
void assemble_prolongation(int p, int m, int l, double* Pv);
void assemble_load(int p, int m, int l, double* f);
bool invert(int n, const double* Ab, int p, double* out);

// Device-side description of one level (all pointers device memory).
struct Level1 {
  int n;        // unknowns
  int nblk;     // 32-entry blocks
  int kp;       // ELL width of P_l (l >= 1)
  int kr;       // ELL width of R_l = P_l^T
  int ustride;  // words per block of the u section (max width over L)
  int rstride;  // words per block of the r / y sections
  const double* Ab;  // n x (2p+1)
  const double* Pv;  // n x kp
  const int* c0;     // n
  const double* Rv;  // n_{l-1} x kr
  const int* r0;     // n_{l-1}
  long long uoff, roff;  // word offsets of the level's sections inside a problem's slab
  long long eoff;        // exponent offset (blocks) inside a problem's slab
};

struct Args1 {
  int p, m, levels, N, b1, b2, smoother;
  int batch;
  Level1 lv[kMaxLevels];
  const double* A0inv;   // n0 x n0
  const double* f;       // batch x ftot (b-major; level l at foff[l])
  long long foff[kMaxLevels];
  long long ftot;
  uint32_t* umant;       // batch x mwords
  uint32_t* rmant;
  uint32_t* ymant;
  long long mwords_u, mwords_r;
  int8_t* uexp;          // batch x eblk
  int8_t* rexp;
  int8_t* yexp;
  long long eblk;
  double* tmp;           // batch x 8 x nL
  double* sol;           // batch x nL
  int* status;
  int nL;
};

}  // namespace fmg1d
