// fmg_internal.h -- types shared by the host driver (fmg_api.cpp, fmg_tables.cpp)
// and the CUDA kernels (fmg_kernels.cu).  Product path only; nothing here is
// shared with oracle/.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace fmg {

constexpr int kMaxLev = 16;

// Geometry of one level.
struct Geom {
  int n;            // p 2^(l+1): stored nodes per dim (node 0 = boundary)
  int NX, NY, NZ;   // stored extents (NX = roundup(n, 32); NZ = 1 in 2D)
  long long size;   // NX*NY*NZ
  long long nblk;   // size / 32
  int l;            // level index
};

// Operator tables (passed by value to kernels -> constant bank).
struct Coefs {
  double Kc[3][7];    // assembled 1D stiffness rows (reference, h-free) by node type, offsets -p..p
  double Mc[3][7];    // assembled 1D mass rows
  double Pw[6][4];    // prolongation weights [i mod 2p][t]
  double Rw[3][11];   // restriction weights [c mod p][s], fine j = 2c-(2p-1)+s
  double invd[27];    // 1/diag(Â) by node type (tz*p+ty)*p+tx
  double inv_theta;   // Chebyshev 1/theta
  double cal[8], cbe[8];  // Chebyshev alpha_j, beta_j (index j-1)
  double rhs_c;       // RN(dim pi^2)
};

// A BFP section stored with a fixed block stride (>= current width).
struct Sec {
  uint32_t* mant;
  int8_t* exps;
  int stride;         // words per block slot (max width over the solve)
};

// Host-side table builders (fmg_tables.cpp).
void build_coefs(int dim, int p, double lambda_hi, double alpha, int cheb_degree, Coefs* c);
void build_rhs_table(int p, int l, double* g);       // g[0..n-1]
int coarse_count(int dim, int p);
int build_coarse_inverse(int dim, int p, double* Ainv);  // 0 on success

// Kernel launchers (fmg_kernels.cu).  All asynchronous on `st`.
struct Launch {
  int dim, p;
  cudaStream_t st;
};
void launch_prolong_decode(const Launch& L, double* out, const Geom& gf, const double* coarse,
                           const Geom& gc, const uint32_t* mant, const int8_t* exps, int w,
                           int stride, const Coefs& cf);
void launch_residual(const Launch& L, const double* U, double* T, const Geom& g, const double* gtab,
                     Sec r, int wr, double* partials, const Coefs& cf, int* status);
void launch_restrict(const Launch& L, const double* Tf, const Geom& gf, double* Tc, const Geom& gc,
                     Sec r, int wr, double* partials, const Coefs& cf, int* status);
void launch_coarse(const Launch& L, int mode, const Geom& g0, const double* gtab0, const double* Ainv,
                   int n0, Sec u, int wu_in, int wu_out, Sec r, int wr, double* W0, const Coefs& cf,
                   int* status);
// cFas level kernels.  step = 1: b = dec r - A Z, first Chebyshev step.
// step >= 2: q = B - A Yin.  finalize (last step): encode ý, W = Z + dec ý,
// ú <- enc(dec ú + dec ý).
struct CfasArgs {
  const double* Z; double* B; const double* Yin; double* Yout; double* Dv;
  double* W;  // may be null (finest level)
  Sec r; int wr;
  Sec u; int wu_in, wu_out;
  int step, last;
};
void launch_cfas_step(const Launch& L, const Geom& g, const CfasArgs& a, const Coefs& cf, int* status);
void launch_norms(cudaStream_t st, const double* partials, const long long* offs, const int* counts,
                  int nlev, double* out);
int tile_count(int dim, int p, int kind, const Geom& g);  // CTAs of residual (0) / restrict (1)
void launch_errors(const Launch& L, const double* U, const Geom& g, double* partials, int* nparts);
void set_kernel_attributes();
void launch_bfp_encode(const double* x, long long n, int w, uint32_t* mant, int8_t* exps, int* status,
                       cudaStream_t st);
void launch_bfp_decode(const uint32_t* mant, const int8_t* exps, long long n, int w, double* x,
                       cudaStream_t st);

}  // namespace fmg
