// Microbenchmark: cost of a 16-CTA cluster barrier phase on B200 (KC design check).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void csync_ra() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void csync_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;\n\tbarrier.cluster.wait.aligned;" ::: "memory");
}
__global__ void k(int mode, int iters, double* buf, unsigned long long* out) {
  unsigned long long t0, t1;
  double acc = 0;
  int tid = blockIdx.x * blockDim.x + threadIdx.x;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int i = 0; i < iters; ++i) {
    if (mode == 0) csync_ra();
    else if (mode == 1) csync_relaxed();
    else if (mode == 2) { buf[tid] = acc + i; csync_ra(); acc += buf[(tid + 512) % (blockDim.x * gridDim.x)]; }
    else if (mode == 3) { buf[tid] = acc + i; __threadfence(); csync_relaxed(); acc += __ldcg(buf + (tid + 512) % (blockDim.x * gridDim.x)); }
    else if (mode == 4) { buf[tid] = acc + i; csync_ra(); 
      double s = 0; for (int j = 0; j < 8; ++j) s += buf[(tid + 512 * j + 7) % (blockDim.x * gridDim.x)]; acc += s; }
  }
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (tid == 0) { out[0] = t1 - t0; buf[0] = acc; }
}
int main() {
  double* buf; unsigned long long* out;
  cudaMalloc(&buf, 1 << 24); cudaMalloc(&out, 64);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {16, 8}) for (int mode = 0; mode < 5; ++mode) {
    cudaLaunchConfig_t cfg{}; cfg.gridDim = dim3(cs); cfg.blockDim = dim3(512);
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    int iters = 1000;
    cudaLaunchKernelEx(&cfg, k, mode, iters, buf, out);
    cudaLaunchKernelEx(&cfg, k, mode, iters, buf, out);
    unsigned long long ns; cudaMemcpy(&ns, out, 8, cudaMemcpyDeviceToHost);
    printf("cluster %d mode %d: %.3f us per phase (%s)\n", cs, mode, ns / 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
  }
}
