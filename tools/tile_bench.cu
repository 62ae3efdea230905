// One-warp timing of the huge-front tile kernels (huge.cuh): POTRF, TRSM, UPDATE (diag / off-diag)
// on a 1024 x 1024 front resident in L2; clock64 per call, averaged.
// build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2405_14236_b200/csrc tools/tile_bench.cu -o tools/tile_bench
#include <cstdio>
#include <climits>
#include "huge.cuh"
using namespace kkt;

__global__ void bench(double* F, double* dinv, long long* out, int reps, int nwarps_busy) {
  extern __shared__ double sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  HFront H;
  H.F = F; H.U = nullptr; H.r = 1024; H.w = 1024; H.nb = 32; H.nt = 32;
  double* ws = sm + warp * HB * HB;
  int fail = INT_MAX;
  if (warp >= nwarps_busy) return;
  long long t0 = clock64();
  for (int i = 0; i < reps; i++) tile_potrf(H, 0, dinv, ws, lane, &fail);
  long long t1 = clock64();
  for (int i = 0; i < reps; i++) tile_trsm(H, 1 + warp, 0, dinv, ws, lane);
  long long t2 = clock64();
  for (int i = 0; i < reps; i++) tile_update(H, 2 + warp, 1 + warp, 0, lane);
  long long t3 = clock64();
  for (int i = 0; i < reps; i++) tile_update(H, 2 + warp, 2 + warp, 0, lane);
  long long t4 = clock64();
  for (int i = 0; i < reps; i++) tile_publish((int*)(dinv + 2048) + warp, i + 1, lane);
  long long t5 = clock64();
  if (lane == 0 && warp == 0) {
    out[0] = (t1 - t0) / reps; out[1] = (t2 - t1) / reps; out[2] = (t3 - t2) / reps;
    out[3] = (t4 - t3) / reps; out[4] = (t5 - t4) / reps;
  }
}

// cold single call (fresh launch): POTRF then TRSM then UPDATE, globaltimer ns
__global__ void cold(double* F, double* dinv, long long* out) {
  extern __shared__ double sm[];
  const int lane = threadIdx.x & 31;
  HFront H;
  H.F = F; H.U = nullptr; H.r = 1024; H.w = 1024; H.nb = 32; H.nt = 32;
  int fail = INT_MAX;
  long long t0 = gtimer();
  tile_potrf(H, 0, dinv, sm, lane, &fail);
  long long t1 = gtimer();
  tile_trsm(H, 1, 0, dinv, sm, lane);
  long long t2 = gtimer();
  tile_update(H, 1, 1, 0, lane);
  long long t3 = gtimer();
  tile_potrf(H, 1, dinv, sm, lane, &fail);
  long long t4 = gtimer();
  if (lane == 0) { out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; out[3] = t4 - t3; }
}

int main() {
  const int n = 1024;
  double* hF = new double[(size_t)n * n];
  for (int j = 0; j < n; j++)
    for (int i = 0; i < n; i++) hF[(size_t)j * n + i] = (i == j) ? 1e6 : 1.0 / (1 + i + j);
  double *F, *dinv; long long* out;
  cudaMalloc(&F, (size_t)n * n * 8); cudaMalloc(&dinv, 8 * 4096); cudaMalloc(&out, 64);
  cudaMemset(dinv, 0, 8 * 4096);
  cudaMemcpy(F, hF, (size_t)n * n * 8, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 32 * 32 * 8);
  for (int nw : {1, 8}) {
    for (int rep = 0; rep < 2; rep++) bench<<<1, 256, 8 * 32 * 32 * 8>>>(F, dinv, out, 20, nw);
    cudaDeviceSynchronize();
    long long h[5];
    cudaMemcpy(h, out, 40, cudaMemcpyDeviceToHost);
    printf("busy warps %d: cycles per call  POTRF %lld  TRSM %lld  UPDATE offdiag %lld  UPDATE diag %lld  publish %lld  (%s)\n",
           nw, h[0], h[1], h[2], h[3], h[4], cudaGetErrorString(cudaGetLastError()));
  }
  // several CTAs: one per SM, 8 busy warps each (L2 contention)
  bench<<<148, 256, 8 * 32 * 32 * 8>>>(F, dinv, out, 20, 8);
  cudaDeviceSynchronize();
  long long h[5];
  cudaMemcpy(h, out, 40, cudaMemcpyDeviceToHost);
  printf("148 CTAs x 8 warps: POTRF %lld  TRSM %lld  UPDATE offdiag %lld  UPDATE diag %lld  publish %lld\n", h[0], h[1], h[2], h[3], h[4]);
  cudaFuncSetAttribute(cold, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 32 * 32 * 8);
  for (int rep = 0; rep < 3; rep++) {
    cold<<<1, 32, 8 * 32 * 32 * 8>>>(F, dinv, out);
    cudaDeviceSynchronize();
    long long hc[4];
    cudaMemcpy(hc, out, 32, cudaMemcpyDeviceToHost);
    printf("(%s) cold launch %d: POTRF %lld ns  TRSM %lld ns  UPDATE(diag) %lld ns  POTRF again %lld ns\n", cudaGetErrorString(cudaGetLastError()), rep, hc[0], hc[1], hc[2], hc[3]);
  }
  return 0;
}
