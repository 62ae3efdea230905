// one-warp timing of front_factor_warp (small supernodes) on SPD fronts in shared memory
#include <cstdio>
#include <vector>
#include <cmath>
#include "dense.cuh"
using namespace kkt;
__global__ void k(const double* F0, int r, int w, double* dinv, long long* out, int reps, int mode, double* res) {
  __shared__ double sm[KKT_SCAP];
  const int R = r - w, pw = r * w, usz = R * (R + 1) / 2, lane = threadIdx.x;
  long long tot = 0;
  for (int it = 0; it < reps; it++) {
    for (int q = lane; q < pw + usz; q += 32) sm[q] = F0[q];
    __syncwarp();
    int fk = -1;
    long long t0 = clock64();
    if (mode == 0) front_factor_warp(sm, sm + pw, r, w, lane, dinv, &fk); else front_factor_warp2(sm, sm + pw, r, w, lane, dinv, &fk);
    __syncwarp();
    tot += clock64() - t0;
  }
  if (lane == 0) out[0] = tot / reps;
  for (int q = lane; q < pw + usz; q += 32) res[q] = sm[q];
}
int main() {
  int shapes[][2] = {{46, 2}, {40, 12}, {38, 8}, {40, 16}, {28, 4}, {24, 4}, {19, 5}, {15, 2}, {12, 4}, {8, 2}, {60, 20}, {32, 32}};
  for (auto& sh : shapes) {
    int r = sh[0], w = sh[1], R = r - w;
    std::vector<double> h(r * w + R * (R + 1) / 2);
    for (int j = 0; j < w; j++) for (int i = 0; i < r; i++) h[j * r + i] = (i == j) ? 2.0 * r : (i > j ? 1.0 / (1 + i + j) : 0.0);
    int q = r * w;
    for (int j = 0; j < R; j++) for (int i = j; i < R; i++) h[q++] = (i == j) ? 2.0 * r : 1.0 / (1 + i + j);
    double *F, *dv; long long* o;
    cudaMalloc(&F, h.size() * 8); cudaMalloc(&dv, 8 * r); cudaMalloc(&o, 8);
    cudaMemcpy(F, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    double* res; cudaMalloc(&res, h.size() * 8);
    std::vector<double> o0(h.size()), o1(h.size());
    long long c[2];
    for (int m = 0; m < 2; m++) {
      k<<<1, 32>>>(F, r, w, dv, o, 5, m, res);
      cudaMemcpy(&c[m], o, 8, cudaMemcpyDeviceToHost);
      cudaMemcpy(m ? o1.data() : o0.data(), res, h.size() * 8, cudaMemcpyDeviceToHost);
    }
    double e = 0, mx = 0;
    for (int j = 0; j < w; j++) for (int i = j; i < r; i++) { e = fmax(e, fabs(o0[j * r + i] - o1[j * r + i])); mx = fmax(mx, fabs(o0[j * r + i])); }
    for (size_t t = r * w; t < h.size(); t++) { e = fmax(e, fabs(o0[t] - o1[t])); mx = fmax(mx, fabs(o0[t])); }
    printf("r=%3d w=%3d old %6lld cyc (%.2f us)  new %6lld cyc (%.2f us)  x%.1f  maxdiff %.1e  %s\n", r, w, c[0], c[0] / 1965.0,
           c[1], c[1] / 1965.0, (double)c[0] / c[1], e / mx, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
