// One-CTA timing of front_factor_cta (dense.cuh) on fronts held in shared memory, as used by
// factor_big_kernel for medium supernodes.  build like tile_bench.
#include <cstdio>
#include "dense.cuh"
using namespace kkt;

// instrumented copy of front_factor_cta: accumulates panel / trailing cycles
template <int NB>
__device__ void ffc_timed(double* F, double* U, int r, int w, double* dinv, int* s_fail, long long* tp, long long* tt) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  for (int k0 = 0; k0 < w; k0 += NB) {
    const int kb = (w - k0) < NB ? (w - k0) : NB;
    long long a = clock64();
    if (r - k0 <= 128) {
      if (warp == 0) panel_factor_warp_any<NB, 4>(F, r, k0, kb, lane, dinv, s_fail);
    } else {
      panel_factor_group<NB>(F, r, k0, kb, tid, blockDim.x, dinv, s_fail, [] { __syncthreads(); });
    }
    __syncthreads();
    long long b = clock64();
    trailing_update_rows_any<NB, 4>(F, U, r, w, k0, kb, warp, nw, lane);
    __syncthreads();
    long long c = clock64();
    *tp += b - a; *tt += c - b;
  }
}

// dissected single round of trailing_tiles<8> for one warp: what=1 loads+MMA only, 2 RMW only, 3 both
template <int TPI>
__device__ long long tt_round(double* F, double* U, int r, int w, int k0, int kb, int lane, int what, double* sink) {
  const int j0 = k0 + kb, m = r - j0;
  const int ntl = (m + 7) >> 3;
  const int lr = lane >> 2, lc = lane & 3;
  long long t0 = clock64();
  int TI[TPI], TJ[TPI];
  int ti = 0, tj = 0;
#pragma unroll
  for (int u = 0; u < TPI; u++) { TI[u] = ti; TJ[u] = tj; if (++ti >= ntl) { tj++; ti = tj; } }
  double c0[TPI], c1[TPI];
#pragma unroll
  for (int u = 0; u < TPI; u++) { c0[u] = 0.0; c1[u] = 0.0; }
  if (what & 1) {
    for (int kk = 0; kk < kb; kk += 4) {
      const double* Fc = F + (k0 + kk + lc) * r;
      double a[TPI], b[TPI];
#pragma unroll
      for (int u = 0; u < TPI; u++) { a[u] = Fc[j0 + TI[u] * 8 + lr]; b[u] = Fc[j0 + TJ[u] * 8 + lr]; }
#pragma unroll
      for (int u = 0; u < TPI; u++) dmma8x8x4(c0[u], c1[u], a[u], b[u]);
    }
  }
  long long t1 = clock64();
  if (what & 2) {
    double* p0[TPI]; double* p1[TPI]; double o0[TPI], o1[TPI];
#pragma unroll
    for (int u = 0; u < TPI; u++) {
      const int i = j0 + TI[u] * 8 + lr, jb = j0 + TJ[u] * 8 + lc * 2;
      p0[u] = (i < r && jb <= i) ? front_at(F, U, r, w, i, jb) : nullptr;
      p1[u] = (i < r && jb + 1 <= i) ? front_at(F, U, r, w, i, jb + 1) : nullptr;
      o0[u] = p0[u] ? *p0[u] : 0.0;
      o1[u] = p1[u] ? *p1[u] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < TPI; u++) { if (p0[u]) *p0[u] = o0[u] - c0[u]; if (p1[u]) *p1[u] = o1[u] - c1[u]; }
  }
  long long t2 = clock64();
  double s = 0;
  for (int u = 0; u < TPI; u++) s += c0[u] + c1[u];
  sink[lane] = s;
  return (t1 - t0) * 100000 + (t2 - t1);
}

// variant: warp2 panel + DMMA tile trailing update, no look-ahead
template <int NB>
__device__ void ffc_dmma(double* F, double* U, int r, int w, double* dinv, int* s_fail, long long* tp, long long* tt) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  for (int k0 = 0; k0 < w; k0 += NB) {
    const int kb = (w - k0) < NB ? (w - k0) : NB;
    long long a = clock64();
    if (warp == 0) { if (r - k0 <= 128) panel_factor_warp2<NB, 4>(F, r, k0, kb, lane, dinv, s_fail); else panel_factor_warp2<NB, 8>(F, r, k0, kb, lane, dinv, s_fail); }
    __syncthreads();
    long long b = clock64();
    trailing_update(F, U, r, w, k0, kb, warp, nw, lane);
    __syncthreads();
    long long c = clock64();
    *tp += b - a; *tt += c - b;
  }
}

template <int NB>
__global__ void bench(const double* F0, const double* U0, int r, int w, double* dinv, long long* out, int reps, int mode) {
  extern __shared__ double sm[];
  __shared__ int s_fail;
  const int R = r - w;
  const int pw = r * w, usz = R * (R + 1) / 2;
  double* F = sm;
  double* U = sm + pw;
  long long tot = 0, tp = 0, tt = 0;
  for (int it = 0; it < reps; it++) {
    for (int q = threadIdx.x; q < pw; q += blockDim.x) F[q] = F0[q];
    for (int q = threadIdx.x; q < usz; q += blockDim.x) U[q] = U0[q];
    if (threadIdx.x == 0) s_fail = -1;
    __syncthreads();
    long long t0 = clock64();
    if (mode == 0) ffc_timed<NB>(F, U, r, w, dinv, &s_fail, &tp, &tt);
    else if (mode == 1) front_factor_cta_la<NB>(F, U, r, w, dinv, &s_fail);
    else if (mode == 2) front_factor_cta_la2<NB>(F, U, r, w, dinv, &s_fail);
    else if (mode == 3) { if (threadIdx.x < 32) panel_factor_warp_any<NB, 8>(F, r, 0, NB, threadIdx.x, dinv, &s_fail); }
    else if (mode == 5) ffc_dmma<NB>(F, U, r, w, dinv, &s_fail, &tp, &tt);
    else if (mode == 6) front_factor_cta_tiles(F, U, r, w, dinv, &s_fail);
    else if (mode == 7) trailing_tiles<8>(F, U, r, w, 0, 8, 0, 1 << 30, threadIdx.x >> 5, 8, threadIdx.x & 31);
    else if (mode == 8) { if (threadIdx.x < 32) trailing_tiles<8>(F, U, r, w, 0, 8, 0, 1 << 30, 0, 1000, threadIdx.x & 31); }
    else if (mode == 9) trailing_update_rows_any<8, 4>(F, U, r, w, 0, 8, threadIdx.x >> 5, 8, threadIdx.x & 31);
    else if (mode >= 10) { if (threadIdx.x < 32) { long long v = tt_round<8>(F, U, r, w, 0, 8, threadIdx.x, mode - 9, dinv + 64); if (threadIdx.x == 0) tp += v; } }
    else if (mode == 4) { if (threadIdx.x < 32) { if (r <= 128) panel_factor_warp2<NB, 4>(F, r, 0, NB, threadIdx.x, dinv, &s_fail); else panel_factor_warp2<NB, 8>(F, r, 0, NB, threadIdx.x, dinv, &s_fail); } }
    __syncthreads();
    tot += clock64() - t0;
  }
  if (threadIdx.x == 0) { out[0] = tot / reps; out[1] = s_fail; out[2] = tp / reps; out[3] = tt / reps; }
}

int main() {
  int shapes[][2] = {{115, 115}, {150, 35}, {136, 26}, {120, 42}, {66, 22}, {200, 64}};
  for (auto& sh : shapes) {
    const int r = sh[0], w = sh[1], R = r - w;
    // SPD front: A = I*r + small symmetric
    double* hF = new double[r * w];
    double* hU = new double[R * (R + 1) / 2 + 1];
    for (int j = 0; j < w; j++)
      for (int i = 0; i < r; i++) hF[j * r + i] = (i == j) ? r : 1.0 / (1 + i + j);
    int q = 0;
    for (int j = 0; j < R; j++)
      for (int i = j; i < R; i++) hU[q++] = (i == j) ? r : 1.0 / (1 + i + j);
    double *F, *U, *dinv; long long* out;
    cudaMalloc(&F, r * w * 8); cudaMalloc(&U, (R * (R + 1) / 2 + 1) * 8); cudaMalloc(&dinv, 8 * r); cudaMalloc(&out, 32);
    cudaMemcpy(F, hF, r * w * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(U, hU, (R * (R + 1) / 2 + 1) * 8, cudaMemcpyHostToDevice);
    const int smem = (r * w + R * (R + 1) / 2) * 8;
    cudaFuncSetAttribute(bench<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int mode = 0; mode < 13; mode++) {
    bench<8><<<1, 256, smem>>>(F, U, r, w, dinv, out, 5, mode);
    cudaDeviceSynchronize();
    long long h[4];
    cudaMemcpy(h, out, 32, cudaMemcpyDeviceToHost);
    // checksum of the factor against mode 0
    static double ref[65536];
    double* cur = new double[r * w];
    cudaMemcpy(cur, dinv, 8 * w, cudaMemcpyDeviceToHost);
    double err = 0;
    if (mode == 0) for (int i = 0; i < w; i++) ref[i] = cur[i];
    else if (mode < 3 || (mode >= 5 && mode < 7)) for (int i = 0; i < w; i++) err = fmax(err, fabs(cur[i] - ref[i]) / fabs(ref[i]));
    printf("mode %d dinv relerr vs mode0 %.2e\n", mode, err);
    printf("r=%4d w=%4d  NB=8: %7lld cycles (%.1f us @1.9GHz) panel %lld trailing %lld fail=%lld  %s\n", r, w, h[0], h[0] / 1900.0,
           h[2], h[3], h[1], cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
