// Microbenchmark: FP64 / FP32 FMA throughput on the B200 (used for the "alu"
// roofline peak in DESIGN.md). Each thread runs 8 independent FMA chains.
#include <cstdio>
#include <cuda_runtime.h>
template <typename T>
__global__ void fma_loop(T* out, int iters, T a, T b) {
  T x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
template <typename T>
double run(const char* name, int blocks, int threads, int iters) {
  T* out; cudaMalloc(&out, sizeof(T) * blocks * threads);
  fma_loop<T><<<blocks, threads>>>(out, 10, (T)0.999, (T)0.001);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  fma_loop<T><<<blocks, threads>>>(out, iters, (T)0.999, (T)0.001);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
  double tf = flops / (ms * 1e-3) / 1e12;
  printf("%s: %.2f TFLOP/s (%.3f ms)\n", name, tf, ms);
  cudaFree(out);
  return tf;
}
__global__ void copy_k(const double4* __restrict__ a, double4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}
int main() {
  int dev; cudaGetDevice(&dev); cudaDeviceProp pr; cudaGetDeviceProperties(&pr, dev);
  printf("device %s SMs %d clock %d kHz\n", pr.name, pr.multiProcessorCount, pr.clockRate);
  int sms = pr.multiProcessorCount;
  for (int k = 0; k < 3; ++k) run<double>("fp64", sms * 8, 256, 4000);
  for (int k = 0; k < 3; ++k) run<float>("fp32", sms * 8, 256, 8000);
  size_t n = (size_t)1 << 27;  // double4 elements = 4 GiB each
  double4 *a, *b; cudaMalloc(&a, n * 32); cudaMalloc(&b, n * 32);
  cudaMemset(a, 0, n * 32);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int k = 0; k < 5; ++k) {
    cudaEventRecord(e0); copy_k<<<sms * 16, 256>>>(a, b, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("copy: %.1f GB/s\n", 2.0 * n * 32 / (ms * 1e-3) / 1e9);
  }
  return 0;
}
