// single-warp latency probes: dependent DFMA chain, dependent LDS.64 chain, LDS+DFMA+STS RMW chain
#include <cstdio>
__global__ void k(double* out, long long* cyc, int iters) {
  __shared__ double sm[1024];
  int lane = threadIdx.x;
  for (int i = lane; i < 1024; i += 32) sm[i] = i * 0.001;
  __syncwarp();
  double x = lane, a = 1.0000001, b = 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < iters; i++) x = fma(x, a, b);
  long long t1 = clock64();
  int idx = lane;
  double y = 0;
  for (int i = 0; i < iters; i++) { y += sm[idx]; idx = (idx + (int)(y * 0) + 33) & 1023; }
  long long t2 = clock64();
  for (int i = 0; i < iters; i++) { int j = (lane + i * 32) & 1023; sm[j] = sm[j] - x * 1e-30; }
  long long t3 = clock64();
  double z0 = 1, z1 = 2, z2 = 3, z3 = 4, z4 = 5, z5 = 6, z6 = 7, z7 = 8;
  for (int i = 0; i < iters; i++) { z0 = fma(z0, a, b); z1 = fma(z1, a, b); z2 = fma(z2, a, b); z3 = fma(z3, a, b); z4 = fma(z4, a, b); z5 = fma(z5, a, b); z6 = fma(z6, a, b); z7 = fma(z7, a, b); }
  long long t4 = clock64();
  if (lane == 0) { cyc[0] = (t1 - t0); cyc[1] = (t2 - t1); cyc[2] = (t3 - t2); cyc[3] = t4 - t3; }
  out[lane] = x + y + sm[lane] + z0 + z1 + z2 + z3 + z4 + z5 + z6 + z7;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 256); cudaMalloc(&c, 64);
  int it = 4096;
  k<<<1, 32>>>(o, c, it); k<<<1, 32>>>(o, c, it);
  long long h[4]; cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
  printf("dep DFMA %.1f cyc, dep LDS.64 %.1f cyc, smem RMW (LDS+DFMA+STS) %.1f cyc, 8 indep DFMA chains %.1f cyc/iter\n",
         h[0] / (double)it, h[1] / (double)it, h[2] / (double)it, h[3] / (double)it);
}
