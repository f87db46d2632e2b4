// Timeline probe of the streaming-exponent encode (tools only): compiles
// fmg_stream.cu with SX_PROBE and prints per-chunk stamp statistics.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -DSX_PROBE \
//        -Ipaper_2511_19036_b200/csrc tools/sx_probe.cu -o /tmp/sx_probe
#include <cstdio>
#include <vector>
#include <algorithm>
#include "../paper_2511_19036_b200/csrc/fmg_stream.cu"

int main() {
  const long long n = 1LL << 27;
  const int w = 8;
  std::vector<double> h(n);
  for (long long i = 0; i < n; ++i) h[i] = sin(0.001 * i) + 1e-6 * ((i * 7919) % 1000);
  double* x; uint32_t* mant; int32_t *xe, *nbk; int64_t* xs; int* status; void* work;
  cudaMalloc(&x, n * 8); cudaMalloc(&mant, n / 32 * w * 4); cudaMalloc(&xe, 256); cudaMalloc(&xs, 512);
  cudaMalloc(&nbk, 4); cudaMalloc(&status, 4); cudaMemset(status, 0, 4);
  long long wb = fmg::stream_work_bytes(n);
  cudaMalloc(&work, wb);
  cudaMemcpy(x, h.data(), n * 8, cudaMemcpyHostToDevice);
  const long long nc = (n / 32 + fmg::SX_GPC - 1) / fmg::SX_GPC;
  unsigned long long* pb; cudaMalloc(&pb, nc * 32);
  cudaMemset(pb, 0, nc * 32);
  for (int rep = 0; rep < 3; ++rep) {
    unsigned long long* arg = rep == 2 ? pb : nullptr;
    cudaMemcpyToSymbol(fmg::sx_probe_buf, &arg, sizeof(arg));
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    fmg::launch_stream_encode(x, n, w, mant, xe, xs, nbk, work, status, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("rep %d: %.3f ms  err=%s\n", rep, ms, cudaGetErrorString(cudaGetLastError()));
  }
  std::vector<unsigned long long> p(nc * 4);
  cudaMemcpy(p.data(), pb, nc * 32, cudaMemcpyDeviceToHost);
  unsigned long long t0 = ~0ULL, tmax = 0;
  for (long long c = 0; c < nc; ++c) { t0 = std::min(t0, p[c * 4]); tmax = std::max(tmax, p[c * 4 + 2]); }
  std::vector<double> lb, pk, rounds;
  for (long long c = 1; c < nc; ++c) {
    lb.push_back((p[c * 4 + 1] - p[c * 4]) * 1e-3);
    pk.push_back((p[c * 4 + 2] - p[c * 4 + 1]) * 1e-3);
    rounds.push_back((double)p[c * 4 + 3]);
  }
  auto med = [](std::vector<double> v) { std::sort(v.begin(), v.end()); return v[v.size() / 2]; };
  auto p90 = [](std::vector<double> v) { std::sort(v.begin(), v.end()); return v[v.size() * 9 / 10]; };
  printf("chunks %lld, span %.3f ms\n", nc, (tmax - t0) * 1e-6);
  printf("land->lookback done: med %.2f us p90 %.2f us\n", med(lb), p90(lb));
  printf("lookback->end (pack+store): med %.2f us p90 %.2f us\n", med(pk), p90(pk));
  printf("lookback distance walked: med %.0f p90 %.0f\n", med(rounds), p90(rounds));
  for (long long c : {1000LL, 1001LL, 1002LL, 1003LL, 20000LL, 20001LL})
    printf("chunk %lld: land %.2f lb %.2f end %.2f us dist %llu\n", c, (p[c * 4] - t0) * 1e-3,
           (p[c * 4 + 1] - t0) * 1e-3, (p[c * 4 + 2] - t0) * 1e-3, p[c * 4 + 3]);
  return 0;
}
