// TMA helper probe (tools only): loads a 34 x 1 FP64 box with the fmg_device.cuh
// helpers, (a) map as a bare __grid_constant__ parameter, (b) inside a struct.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -Ipaper_2511_19036_b200/csrc tools/tma_probe.cu -o tools/tma_probe.bin
#include <cstdio>
#include <cuda.h>
#include <cudaTypedefs.h>
#include "../paper_2511_19036_b200/csrc/fmg_device.cuh"
using namespace fmg;

struct Wrap { int a, b; alignas(64) CUtensorMap tm; int tma; };

__global__ void k_bare(const __grid_constant__ CUtensorMap tm, double* out, int x, int y) {
  __shared__ __align__(128) double buf[64];
  __shared__ unsigned long long bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init_fence(); }
  __syncthreads();
  if (threadIdx.x == 0) tma_load_2d(buf, &tm, x, y, &bar, 34 * 8);
  mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < 34; i += 32) out[i] = buf[i];
}
__global__ void k_struct(const __grid_constant__ Wrap w, double* out, int x, int y) {
  __shared__ __align__(128) double buf[64];
  __shared__ unsigned long long bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); mbar_init_fence(); }
  __syncthreads();
  if (threadIdx.x == 0) tma_load_2d(buf, &w.tm, x, y, &bar, 34 * 8);
  mbar_wait(&bar, 0);
  for (int i = threadIdx.x; i < 34; i += 32) out[i] = buf[i];
}

int main() {
  const int NX = 64, NY = 8;
  double h[NX * NY];
  for (int i = 0; i < NX * NY; ++i) h[i] = i;
  double *d, *o;
  cudaMalloc(&d, sizeof(h)); cudaMalloc(&o, 64 * 8);
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  void* fn = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  CUtensorMap tm;
  cuuint64_t dims[2] = {NX, NY}, str[1] = {NX * 8};
  cuuint32_t box[2] = {34, 1}, es[2] = {1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  double ho[34];
  k_bare<<<1, 32>>>(tm, o, -1, 3);
  printf("bare: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  cudaMemcpy(ho, o, 34 * 8, cudaMemcpyDeviceToHost);
  printf("  %g %g %g ... %g\n", ho[0], ho[1], ho[2], ho[33]);
  Wrap w{}; w.tm = tm;
  k_struct<<<1, 32>>>(w, o, 30, 7);
  printf("struct: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  cudaMemcpy(ho, o, 34 * 8, cudaMemcpyDeviceToHost);
  printf("  %g %g %g ... %g\n", ho[0], ho[1], ho[2], ho[33]);
  return 0;
}
