// One-CTA timing + agreement of front_factor_cta<8> (current) vs front_factor_cta_ll (left-looking,
// 32-column blocks) on SPD fronts held in shared memory.
// build: nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I paper_2405_14236_b200/csrc tools/ll_bench.cu -o tools/ll_bench
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "dense.cuh"
using namespace kkt;

__device__ void ll_timed(double* F, double* U, int r, int w, double* dinv, int* s_fail, long long* ph) {
  __shared__ double sinv[32];
  __shared__ __align__(16) double L11s[32 * 32];
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  long long t = clock64();
  auto stamp = [&](int k) { __syncthreads(); long long u = clock64(); ph[k] += u - t; t = u; };
  for (int c0 = 0; c0 < w; c0 += 32) {
    const int kb = (w - c0) < 32 ? (w - c0) : 32;
    if (c0 > 0) ll_block_update(F, r, c0, kb, warp, nw, lane);
    stamp(0);
    if (warp == 0) ll_diag_warp(F, r, c0, kb, lane, dinv, sinv, L11s, s_fail);
    stamp(1);
    ll_trsm_rows1(F, r, c0, kb, sinv, L11s, tid, nt);
    stamp(2);
  }
  schur_tiles22(F, U, r, w, warp, nw, lane);
  stamp(3);
}

__global__ void bench(const double* F0, const double* U0, double* Fo, double* Uo, int r, int w, double* dinv,
                      long long* out, int reps, int mode) {
  extern __shared__ double sm[];
  __shared__ int s_fail;
  const int R = r - w;
  const int pw = r * w, usz = R * (R + 1) / 2;
  double* F = sm;
  double* U = sm + pw;
  long long tot = 0, ph[4] = {0, 0, 0, 0};
  for (int it = 0; it < reps; it++) {
    for (int q = threadIdx.x; q < pw; q += blockDim.x) F[q] = F0[q];
    for (int q = threadIdx.x; q < usz; q += blockDim.x) U[q] = U0[q];
    if (threadIdx.x == 0) s_fail = -1;
    __syncthreads();
    long long t0 = clock64();
    if (mode == 0) front_factor_cta<8>(F, U, r, w, dinv, &s_fail);
    else if (mode == 1) front_factor_cta_ll(F, U, r, w, dinv, &s_fail);
    else if (mode == 2) ll_timed(F, U, r, w, dinv, &s_fail, ph);
    else {
      __shared__ double si[32];
      __shared__ __align__(16) double L11s[1024];
      const int kb = w < 32 ? w : 32;
      if (threadIdx.x < 32) ll_diag_warp(F, r, 0, kb, threadIdx.x, dinv, si, L11s, &s_fail);
      __syncthreads();
      long long t1 = clock64();
      ll_trsm_rows1(F, r, 0, kb, si, L11s, threadIdx.x, blockDim.x);
      __syncthreads();
      long long t2 = clock64();
      ph[0] += t1 - t0; ph[1] += t2 - t1;
    }
    __syncthreads();
    tot += clock64() - t0;
  }
  for (int q = threadIdx.x; q < pw; q += blockDim.x) Fo[q] = F[q];
  for (int q = threadIdx.x; q < usz; q += blockDim.x) Uo[q] = U[q];
  if (threadIdx.x == 0) { out[0] = tot / reps; out[1] = s_fail; for (int k = 0; k < 4; k++) out[2 + k] = ph[k] / reps; }
}

int main() {
  int shapes[][2] = {{115, 115}, {150, 35}, {136, 26}, {124, 32}, {120, 42}, {98, 14}, {66, 22},
                     {200, 64}, {226, 40}, {160, 160}, {180, 100}, {33, 33}, {40, 7}};
  srand(7);
  for (auto& sh : shapes) {
    const int r = sh[0], w = sh[1], R = r - w;
    // SPD: A = B B^T / r + diag spanning 1e-2..1e2
    std::vector<double> B(r * r), A(r * r);
    for (auto& v : B) v = (rand() / (double)RAND_MAX) - 0.5;
    for (int i = 0; i < r; i++)
      for (int j = 0; j <= i; j++) {
        double s = 0;
        for (int k = 0; k < r; k++) s += B[i * r + k] * B[j * r + k];
        A[i * r + j] = A[j * r + i] = s / r + (i == j ? pow(10.0, -2 + 4.0 * (i % 7) / 6.0) : 0.0);
      }
    std::vector<double> hF(r * w), hU(R * (R + 1) / 2 + 1);
    for (int j = 0; j < w; j++)
      for (int i = 0; i < r; i++) hF[j * r + i] = i >= j ? A[i * r + j] : 0.0;
    int q = 0;
    for (int j = 0; j < R; j++)
      for (int i = j; i < R; i++) hU[q++] = A[(w + i) * r + (w + j)];
    double *F, *U, *Fo, *Uo, *dinv;
    long long* out;
    const size_t ub = (R * (R + 1) / 2 + 1) * 8;
    cudaMalloc(&F, r * w * 8); cudaMalloc(&U, ub); cudaMalloc(&Fo, r * w * 8); cudaMalloc(&Uo, ub);
    cudaMalloc(&dinv, 8 * r); cudaMalloc(&out, 64);
    cudaMemcpy(F, hF.data(), r * w * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(U, hU.data(), ub, cudaMemcpyHostToDevice);
    const int smem = (r * w + R * (R + 1) / 2) * 8;
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    std::vector<double> rF[2], rU[2];
    long long cyc[2];
    long long phs[4];
    long long iso[2];
    for (int mode = 0; mode < 4; mode++) {
      bench<<<1, 256, smem>>>(F, U, Fo, Uo, r, w, dinv, out, 5, mode);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
      long long h[6];
      cudaMemcpy(h, out, 48, cudaMemcpyDeviceToHost);
      if (mode == 2) { for (int k = 0; k < 4; k++) phs[k] = h[2 + k]; continue; }
      if (mode == 3) { iso[0] = h[2]; iso[1] = h[3]; continue; }
      cyc[mode] = h[0];
      rF[mode].resize(r * w); rU[mode].resize(R * (R + 1) / 2 + 1);
      cudaMemcpy(rF[mode].data(), Fo, r * w * 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(rU[mode].data(), Uo, ub, cudaMemcpyDeviceToHost);
    }
    double ef = 0, mf = 0, eu = 0, mu = 0;
    for (int j = 0; j < w; j++)
      for (int i = j; i < r; i++) {
        ef = fmax(ef, fabs(rF[0][j * r + i] - rF[1][j * r + i]));
        mf = fmax(mf, fabs(rF[0][j * r + i]));
      }
    for (int k = 0; k < R * (R + 1) / 2; k++) { eu = fmax(eu, fabs(rU[0][k] - rU[1][k])); mu = fmax(mu, fabs(rU[0][k])); }
    printf("r=%4d w=%4d  cta<8> %7lld cyc (%6.2f us)  ll %7lld cyc (%6.2f us)  x%.2f   dF %.1e dU %.1e\n", r, w,
           cyc[0], cyc[0] / 1965.0, cyc[1], cyc[1] / 1965.0, (double)cyc[0] / cyc[1], ef / (mf + 1e-300),
           eu / (mu + 1e-300));
    printf("      ll phases: update %lld diag %lld trsm %lld schur %lld | isolated first block: diag %lld trsm %lld\n", phs[0], phs[1], phs[2], phs[3], iso[0], iso[1]);
    cudaFree(F); cudaFree(U); cudaFree(Fo); cudaFree(Uo); cudaFree(dinv); cudaFree(out);
  }
  return 0;
}
