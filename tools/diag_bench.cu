// one-warp 32x32 Cholesky step-chain probe: variants of ll_diag_warp's loop body
#include <cstdio>
#include "dense.cuh"
using namespace kkt;
template <int V>
__global__ void k(double* out, long long* cyc) {
  __shared__ __align__(16) double L11s[1024];
  const int lane = threadIdx.x;
  double a[32];
#pragma unroll
  for (int c = 0; c < 32; c++) a[c] = (c == lane) ? 64.0 : (c < lane ? 1.0 / (1 + c + lane) : 0.0);
  long long t0 = clock64();
  double d = shfl_idx_d(a[0], 0);
  double inv = rsqrt_fast(d);
#pragma unroll
  for (int c = 0; c < 32; c++) {
    const double l = (lane > c) ? a[c] * inv : (lane == c ? d * inv : 0.0);
    a[c] = l;
    if (V != 2) L11s[c * 32 + lane] = l;
    if (c + 1 < 32) {
      d = shfl_idx_d(fma(-l, l, a[c + 1]), c + 1);
      inv = (V == 3) ? d * 0.5 : rsqrt_fast(d);
    }
    if (V != 2) warp_bar();
    if (V == 0 || V == 3) {
      const double* col = L11s + c * 32;
#pragma unroll
      for (int cc = c + 1; cc < 32; cc++) a[cc] = fma(-l, col[cc], a[cc]);
    } else if (V == 1) {
      if (c + 1 < 32) a[c + 1] = fma(-l, L11s[c * 32 + c + 1], a[c + 1]);
    }
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < 32; c++) s += a[c];
  out[lane] = s;
  if (lane == 0) cyc[V] = t1 - t0;
}
__global__ void kr(double* out, long long* cyc, int kb) {
  __shared__ __align__(16) double L11s[1024];
  __shared__ double F[32 * 40];
  __shared__ double sinv[32];
  __shared__ int fk;
  const int lane = threadIdx.x, r = 40;
  for (int q = lane; q < 32 * 40; q += 32) { int i = q % r, j = q / r; F[q] = (i == j) ? 64.0 : 1.0 / (1 + i + j); }
  fk = -1;
  __syncwarp();
  long long t0 = clock64();
  ll_diag_warp(F, r, 0, kb, lane, out + 64, sinv, L11s, &fk);
  long long t1 = clock64();
  __syncwarp();
  out[lane] = F[lane * r + lane] + sinv[lane];
  if (lane == 0) cyc[4] = t1 - t0;
}
template <int V>
__global__ void kt(double* out, long long* cyc) {
  __shared__ __align__(16) double L11s[1024];
  __shared__ double F[32 * 128];
  __shared__ double sinv[32];
  const int r = 128;
  for (int q = threadIdx.x; q < 32 * 128; q += blockDim.x) { int i = q % r, j = q / r; F[q] = (i == j) ? 64.0 : 1.0 / (1 + i + j); }
  for (int q = threadIdx.x; q < 1024; q += blockDim.x) L11s[q] = ((q & 31) >= (q >> 5)) ? 0.1 : 0.0;
  if (threadIdx.x < 32) sinv[threadIdx.x] = 0.125;
  __syncthreads();
  long long t0 = clock64();
  if (V == 1) ll_trsm_rows1(F, r, 0, 32, sinv, L11s, threadIdx.x, blockDim.x);
  else ll_trsm_rows2(F, r, 0, 32, sinv, L11s, threadIdx.x, blockDim.x);
  __syncthreads();
  long long t1 = clock64();
  out[threadIdx.x] = F[threadIdx.x + 40];
  if (threadIdx.x == 0) cyc[5 + V] = t1 - t0;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 4096); cudaMalloc(&c, 128);
  for (int rep = 0; rep < 2; rep++) { k<0><<<1, 32>>>(o, c); k<1><<<1, 32>>>(o, c); k<2><<<1, 32>>>(o, c); k<3><<<1, 32>>>(o, c); }
  kr<<<1, 32>>>(o, c, 32); kr<<<1, 32>>>(o, c, 32);
  long long h[5]; cudaMemcpy(h, c, 40, cudaMemcpyDeviceToHost);
  kt<1><<<1, 256>>>(o, c); kt<2><<<1, 256>>>(o, c); kt<1><<<1, 256>>>(o, c); kt<2><<<1, 256>>>(o, c);
  long long h2[8]; cudaMemcpy(h2, c, 64, cudaMemcpyDeviceToHost);
  printf("trsm 96 rows x 32: 1-row/thread %lld, 2-rows/thread %lld\n", h2[6], h2[7]);
  printf("real ll_diag_warp (kb=32): %lld\n", h[4]);
  printf("full %lld | chain+1 bcast %lld | chain only (no smem) %lld | full without rsqrt %lld  (cycles / 32 steps)\n", h[0], h[1], h[2], h[3]);
  return 0;
}
