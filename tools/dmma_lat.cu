// DMMA m8n8k4.f64 latency / issue probe (one warp): dependent chain vs 8 independent chains
#include <cstdio>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
__global__ void k(double* out, long long* cyc, int it) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c0 = 0, c1 = 0;
  long long t0 = clock64();
  for (int i = 0; i < it; i++) dmma(c0, c1, a, b);
  long long t1 = clock64();
  double d0[8] = {0}, d1[8] = {0};
  for (int i = 0; i < it; i++) {
#pragma unroll
    for (int u = 0; u < 8; u++) dmma(d0[u], d1[u], a, b);
  }
  long long t2 = clock64();
  double s = c0 + c1;
  for (int u = 0; u < 8; u++) s += d0[u] + d1[u];
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 256 * 8); cudaMalloc(&c, 16);
  const int it = 1024;
  k<<<1, 32>>>(o, c, it); k<<<1, 32>>>(o, c, it);
  long long h[2]; cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
  printf("DMMA dependent latency %.1f cyc; 8 independent chains: %.1f cyc per DMMA\n", h[0] / (double)it, h[1] / (8.0 * it));
  return 0;
}
