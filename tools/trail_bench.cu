// variants of the single-warp trailing update T -= L L^T (m x m lower, L m x 8) in shared memory
#include <cstdio>
#include "dense.cuh"
using namespace kkt;
// v2: minimal -- lane = row i (i < m <= 64, 2 rows per lane), columns j loop, L row values in regs,
// column values by shuffle from the owning lane, T column-major (ld m), 32-bit indexing
__device__ void trail_v2(double* T, const double* Lp, int m, int lane) {
  double a0[8], a1[8];
  const int i0 = lane, i1 = lane + 32;
#pragma unroll
  for (int c = 0; c < 8; c++) { a0[c] = (i0 < m) ? Lp[c * m + i0] : 0.0; a1[c] = (i1 < m) ? Lp[c * m + i1] : 0.0; }
  for (int j = 0; j < m; j++) {
    const int src = j & 31;
    double lj[8];
#pragma unroll
    for (int c = 0; c < 8; c++) lj[c] = __shfl_sync(0xffffffffu, (j < 32) ? a0[c] : a1[c], src);
    double s0 = 0, s1 = 0;
#pragma unroll
    for (int c = 0; c < 8; c++) { s0 = fma(a0[c], lj[c], s0); s1 = fma(a1[c], lj[c], s1); }
    if (i0 >= j && i0 < m) T[j * m + i0] -= s0;
    if (i1 >= j && i1 < m) T[j * m + i1] -= s1;
  }
}
__global__ void bench(int m, int reps, long long* out, double* chk) {
  extern __shared__ double sm[];
  const int lane = threadIdx.x;
  double* T = sm; double* Lp = sm + 64 * 64; double* F = Lp + 64 * 8;
  long long t1 = 0, t2 = 0;
  for (int rep = 0; rep < reps; rep++) {
    for (int q = lane; q < m * m; q += 32) T[q] = 1.0;
    for (int q = lane; q < m * 8; q += 32) Lp[q] = 0.001 * q;
    __syncwarp();
    long long a = clock64();
    trail_v2(T, Lp, m, lane);
    __syncwarp();
    long long b = clock64();
    // library routine on an equivalent front: r = m + 8, w = 8 (panel = [.. ; L], U = T packed)
    const int r = m + 8, w = 8;
    for (int q = lane; q < r * w; q += 32) F[q] = 0.001 * q;
    double* U = F + r * w;
    for (int q = lane; q < m * (m + 1) / 2; q += 32) U[q] = 1.0;
    __syncwarp();
    long long c = clock64();
    trailing_update_rows_any<8, 2>(F, U, r, w, 0, 8, 0, 1, lane);
    __syncwarp();
    long long d = clock64();
    t1 += b - a; t2 += d - c;
  }
  if (lane == 0) { out[0] = t1 / reps; out[1] = t2 / reps; chk[0] = T[5] + F[3]; }
}
int main() {
  long long* d; double* c; cudaMalloc(&d, 64); cudaMalloc(&c, 64);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 150 * 1024);
  for (int m : {16, 32, 40, 64}) {
    bench<<<148, 32, 150 * 1024>>>(m, 400, d, c);
    long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("m=%d: minimal shuffle version %lld cyc, library trailing_update_rows %lld cyc\n", m, h[0], h[1]);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
