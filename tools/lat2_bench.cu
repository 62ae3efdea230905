// single-warp latency probes: dependent rsqrt(double) chain, dependent 64-bit shuffle chain,
// STS + __syncwarp + LDS round trip, DMUL chain
#include <cstdio>
__global__ void k(double* out, long long* cyc, int iters) {
  __shared__ double sm[64];
  const int lane = threadIdx.x;
  double x = 1.0 + lane, y = 2.0;
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) x = rsqrt(x) + 1.0;
  long long t1 = clock64();
  for (int i = 0; i < iters; i++) y = __shfl_sync(0xffffffffu, y, (lane + 1) & 31) * 1.0000001;
  long long t2 = clock64();
  double z = lane;
  for (int i = 0; i < iters; i++) { sm[lane] = z; __syncwarp(); z = sm[(lane + 1) & 31] * 1.0000001; __syncwarp(); }
  long long t3 = clock64();
  double u = lane;
  for (int i = 0; i < iters; i++) u = u * 1.0000001;
  long long t4 = clock64();
  if (lane == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; }
  out[lane] = x + y + z + u;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 256); cudaMalloc(&c, 64);
  int it = 4096;
  k<<<1, 32>>>(o, c, it); k<<<1, 32>>>(o, c, it);
  long long h[4]; cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
  printf("rsqrt+add %.1f cyc, shfl64+dmul %.1f cyc, sts+syncwarp+lds+dmul %.1f cyc, dmul %.1f cyc\n",
         h[0] / (double)it, h[1] / (double)it, h[2] / (double)it, h[3] / (double)it);
  return 0;
}
