// Variants of the 32-column warp Cholesky of tiles.cuh (tile_diag32) to find what bounds its
// ~265 cycles per column.  Build: nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a
//   -o tools/diag_bench2 tools/diag_bench2.cu
#include <cstdio>
#include <vector>
#include "../paper_2405_14236_b200/csrc/tiles.cuh"
using namespace kkt;

template <int V>
__device__ __forceinline__ void diag_v(double* T, int kb, int lane, double* dinv, double* sinv, double* L11s, int* fail_k) {
  const int row = lane;
  double a[32];
#pragma unroll
  for (int c = 0; c < 32; c++) a[c] = (lane < kb && c < kb && c <= lane) ? T[tsw(row, c)] : (c == lane ? 1.0 : 0.0);
  double myinv = 0.0;
  unsigned bad = 0;
  double d = shfl_idx_d(a[0], 0);
  double inv = (V == 3) ? 1.0 / sqrt(d) : rsqrt_fast(d);
#pragma unroll
  for (int c = 0; c < 32; c++) {
    bool b_ = false;
    if (V != 2) { b_ = pivot_bad(d); bad |= (b_ ? 1u : 0u) << c; }
    const double iv = b_ ? nan_d() : inv;
    if (lane == c) myinv = iv;
    const double l = (lane > c) ? a[c] * iv : (lane == c ? d * iv : 0.0);
    a[c] = l;
    L11s[c * 32 + lane] = l;
    if (c + 1 < 32) {
      d = shfl_idx_d(fma(-l, l, a[c + 1]), c + 1);
      inv = (V == 3) ? 1.0 / sqrt(d) : (V == 4 ? d : rsqrt_fast(d));   // V4: no rsqrt at all (timing only)
    }
    warp_bar();
    const double2* col2 = reinterpret_cast<const double2*>(L11s + c * 32);
    if ((c + 1) & 1) a[c + 1] = fma(-l, L11s[c * 32 + c + 1], a[c + 1]);
#pragma unroll
    for (int q = (c + 2) / 2; q < 16; q++) {
      const double2 l2 = col2[q];
      a[2 * q] = fma(-l, l2.x, a[2 * q]);
      a[2 * q + 1] = fma(-l, l2.y, a[2 * q + 1]);
    }
    if (V != 1) asm volatile("" ::: "memory");
  }
#pragma unroll
  for (int c = 0; c < 32; c++)
    if (c < kb) T[tsw(row, c)] = (lane < kb && c <= lane) ? a[c] : 0.0;
  if (lane < kb) { sinv[lane] = myinv; dinv[lane] = myinv; }
  if (lane == 0 && bad && *fail_k < 0) *fail_k = __ffs(bad) - 1;
  warp_bar();
}

template <int V>
__global__ void __launch_bounds__(256, 1) bench(int reps, double* g, double* dinv, long long* out) {
  extern __shared__ __align__(16) double sm[];
  __shared__ int sf;
  double* gt = g + (long long)blockIdx.x * TBD;
  if (threadIdx.x == 0) sf = -1;
  long long t0 = clock64();
  for (int r = 0; r < reps; r++) {
    tile_load_async(sm, gt); cp_async_wait_all(); __syncthreads();
    long long a = clock64();
    if (threadIdx.x < 32) diag_v<V>(sm, 32, threadIdx.x, dinv + blockIdx.x * 64, sm + TBD, sm + TBD + 64, &sf);
    __syncthreads();
    if (r == 0) t0 -= clock64() - a;  // placeholder to keep a dependency
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / reps;
}

int main() {
  const int nb = 1;
  std::vector<double> h((size_t)nb * TBD);
  for (int c = 0; c < 64; c++) for (int r = 0; r < 64; r++) h[c * 64 + r] = (r == c) ? 70.0 : 0.5 / (1 + r + c);
  double *g, *dinv; long long* out;
  cudaMalloc(&g, h.size() * 8); cudaMalloc(&dinv, 64 * 8); cudaMalloc(&out, 8);
  cudaMemcpy(g, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  const char* names[] = {"V0 current", "V1 no asm clobber", "V2 no pivot checks", "V3 1/sqrt", "V4 no rsqrt (timing)"};
  void (*ks[])(int, double*, double*, long long*) = {bench<0>, bench<1>, bench<2>, bench<3>, bench<4>};
  for (int v = 0; v < 5; v++) {
    cudaFuncSetAttribute(ks[v], cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    long long o = 0;
    // reps 1 and 21: difference / 20 = per call incl. the tile load
    ks[v]<<<1, 256, 64 * 1024>>>(1, g, dinv, out); cudaDeviceSynchronize();
    ks[v]<<<1, 256, 64 * 1024>>>(21, g, dinv, out); cudaDeviceSynchronize();
    cudaMemcpy(&o, out, 8, cudaMemcpyDeviceToHost);
    printf("%-22s %8lld cycles per (load + diag32)\n", names[v], o);
  }
  return 0;
}
