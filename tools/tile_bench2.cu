// Interference probe for the huge-front critical path: warp 0 times POTRF / TRSM / UPDATE while
// warps 1..7 of the same CTA (a) idle, (b) run tile UPDATEs (DMMA), (c) poll a flag, (d) run
// TRSMs (DFMA); one CTA per SM on all SMs so L2 traffic is realistic.
#include <cstdio>
#include <climits>
#include "huge.cuh"
using namespace kkt;

__global__ void bench(double* Fall, double* dinv, long long* out, int reps, int mode, int* flag) {
  extern __shared__ double sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  HFront H;
  H.F = Fall + (size_t)blockIdx.x * 512 * 512; H.U = nullptr; H.r = 512; H.w = 512; H.nb = 16; H.nt = 16;
  double* ws = sm + warp * HB * HB;
  int fail = INT_MAX;
  __shared__ volatile int stop;
  if (threadIdx.x == 0) stop = 0;
  __syncthreads();
  if (warp == 0) {
    long long t0 = clock64();
    for (int i = 0; i < reps; i++) tile_potrf(H, 0, dinv, ws, lane, &fail);
    long long t1 = clock64();
    for (int i = 0; i < reps; i++) tile_trsm(H, 1, 0, dinv, ws, lane);
    long long t2 = clock64();
    for (int i = 0; i < reps; i++) tile_update(H, 1, 1, 0, lane);
    long long t3 = clock64();
    if (lane == 0 && blockIdx.x == 0) { out[0] = (t1 - t0) / reps; out[1] = (t2 - t1) / reps; out[2] = (t3 - t2) / reps; }
    if (lane == 0) stop = 1;
  } else {
    int it = 0;
    while (!stop) {
      if (mode == 1) tile_update(H, 4 + warp, 3 + warp, 2, lane);
      else if (mode == 2) { if (ld_volatile(flag) > 1000000) break; }
      else if (mode == 3) tile_trsm(H, 4 + warp, 2, dinv, ws, lane);
      else break;
      it++;
    }
  }
}

int main() {
  const int n = 512, G = 148;
  double* hF = new double[(size_t)n * n];
  for (int j = 0; j < n; j++)
    for (int i = 0; i < n; i++) hF[(size_t)j * n + i] = (i == j) ? 1e6 : 1.0 / (1 + i + j);
  double *F, *dinv; long long* out; int* flag;
  cudaMalloc(&F, (size_t)G * n * n * 8); cudaMalloc(&dinv, 8 * 4096); cudaMalloc(&out, 64); cudaMalloc(&flag, 64);
  cudaMemset(dinv, 0, 8 * 4096); cudaMemset(flag, 0, 64);
  for (int g = 0; g < G; g++) cudaMemcpy(F + (size_t)g * n * n, hF, (size_t)n * n * 8, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 32 * 32 * 8);
  const char* names[] = {"idle", "DMMA updates", "flag polling", "DFMA trsm"};
  for (int mode = 0; mode < 4; mode++) {
    bench<<<G, 256, 8 * 32 * 32 * 8>>>(F, dinv, out, 20, mode, flag);
    bench<<<G, 256, 8 * 32 * 32 * 8>>>(F, dinv, out, 20, mode, flag);
    cudaDeviceSynchronize();
    long long h[3];
    cudaMemcpy(h, out, 24, cudaMemcpyDeviceToHost);
    printf("others %-14s: POTRF %6lld  TRSM %6lld  UPDATE(diag) %6lld cycles  (%s)\n", names[mode], h[0], h[1], h[2],
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
