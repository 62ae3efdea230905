// Microbenchmark of the warp-level dense front kernels (dense.cuh): cycles per call of
// panel_factor_warp, trailing_update and front_factor_warp on an r x r front held in smem.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2405_14236_b200/csrc tools/dense_bench.cu -o tools/dense_bench
#include <cstdio>
#include <vector>
#include "dense.cuh"
using namespace kkt;

__global__ void bench(int r, int w, int reps, long long* out, double* chk) {
  extern __shared__ double sm[];
  const int lane = threadIdx.x & 31;
  const int R = r - w;
  double* F = sm;
  double* U = sm + r * w;
  double* dinv = U + R * (R + 1) / 2 + 1;
  long long t_panel = 0, t_trail = 0, t_full = 0;
  for (int rep = 0; rep < reps; rep++) {
    // SPD front: diag dominant
    for (int q = lane; q < r * w; q += 32) { int j = q / r, i = q % r; F[q] = (i == j) ? 4.0 * r : ((i > j) ? 0.5 / (1 + i + j) : 0.0); }
    for (int q = lane; q < R * (R + 1) / 2; q += 32) U[q] = 0.0;
    __syncwarp();
    int fk = -1;
    long long t0 = clock64();
    panel_factor_warp_any<8, 2>(F, r, 0, w < 8 ? w : 8, lane, dinv, &fk);
    __syncwarp();
    long long t1 = clock64();
    trailing_update_rows_any<8, 2>(F, U, r, w, 0, w < 8 ? w : 8, 0, 1, lane);
    __syncwarp();
    long long t2 = clock64();
    t_panel += t1 - t0; t_trail += t2 - t1;
    for (int q = lane; q < r * w; q += 32) { int j = q / r, i = q % r; F[q] = (i == j) ? 4.0 * r : ((i > j) ? 0.5 / (1 + i + j) : 0.0); }
    for (int q = lane; q < R * (R + 1) / 2; q += 32) U[q] = 0.0;
    __syncwarp();
    long long t3 = clock64();
    front_factor_warp(F, U, r, w, lane, dinv, &fk);
    __syncwarp();
    long long t4 = clock64();
    t_full += t4 - t3;
  }
  if (lane == 0) { out[0] = t_panel / reps; out[1] = t_trail / reps; out[2] = t_full / reps; chk[0] = F[0] + U[0]; }
}

int main() {
  long long* d; double* c; cudaMalloc(&d, 64); cudaMalloc(&c, 64);
  int cases[][2] = {{12, 4}, {40, 12}, {46, 2}, {64, 16}, {40, 8}};
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (auto& cs : cases) {
    int r = cs[0], w = cs[1];
    bench<<<1, 32, 64 * 1024>>>(r, w, 20, d, c);
    long long h[3]; cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
    printf("r=%d w=%d: panel(8 cols) %lld cyc, trailing(1 block) %lld cyc, full front %lld cyc (%.2f us @1.965GHz)\n",
           r, w, h[0], h[1], h[2], h[2] / 1965.0);
  }
  cudaError_t e = cudaDeviceSynchronize(); printf("%s\n", cudaGetErrorString(e));
}
