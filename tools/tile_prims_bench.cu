// Micro-benchmark of the tile-task primitives of tiles.cuh (one CTA per SM, each repeats the
// primitive; reports cycles per call).  Build: nvcc -std=c++17 -O3 -gencode
// arch=compute_100a,code=sm_100a -o tools/tile_prims_bench tools/tile_prims_bench.cu
#include <cstdio>
#include <vector>
#include <cmath>
#include "../paper_2405_14236_b200/csrc/tiles.cuh"
using namespace kkt;

__global__ void __launch_bounds__(256, 1) bench(int which, int reps, double* g, double* dinv, long long* out) {
  extern __shared__ __align__(16) double sm[];
  __shared__ int sf;
  double* gt = g + (long long)blockIdx.x * 4 * TBD;
  if (threadIdx.x == 0) sf = -1;
  tile_load_async(sm, gt); tile_load_async(sm + TBD, gt + TBD); tile_load_async(sm + 2 * TBD, gt + 2 * TBD);
  cp_async_wait_all();
  __syncthreads();
  long long t0 = clock64();
  for (int r = 0; r < reps; r++) {
    if (which == 0) {          // potrf64 (re-load the SPD tile each rep)
      tile_load_async(sm, gt); cp_async_wait_all(); __syncthreads();
      tile_potrf64(sm, 64, dinv + blockIdx.x * 64, sm + 3 * TBD, sm + 3 * TBD + 64, &sf);
    } else if (which == 1) {   // trsm64 against the factored tile in sm+TBD
      tile_load_async(sm, gt + 2 * TBD); cp_async_wait_all(); __syncthreads();
      tile_trsm64(sm, sm + TBD, sm + 3 * TBD);
    } else if (which == 2) {   // gemm into global C
      tile_gemm_nt_global(gt + 3 * TBD, sm, sm + TBD);
      __syncthreads();
    } else if (which == 3) {   // load 2 tiles
      tile_load_async(sm, gt); tile_load_async(sm + TBD, gt + TBD); cp_async_wait_all(); __syncthreads();
    } else if (which == 4) {   // diag32 only
      if (threadIdx.x < 32) tile_diag32<0>(sm, 32, threadIdx.x, dinv + blockIdx.x * 64, sm + 3 * TBD, sm + 3 * TBD + 64, &sf);
      __syncthreads();
    } else if (which == 5) {   // rowsolve32 64 rows
      tile_rowsolve32<0>(sm + 2 * TBD, 0, 64, sm + TBD, sm + 3 * TBD);
      __syncthreads();
    } else if (which == 6) {   // gemm into smem C
      tile_gemm_nt_smem(sm + 2 * TBD, sm, sm + TBD);
    } else if (which == 7) {   // store a tile + panel copy + fence (publish cost)
      tile_store(gt + 3 * TBD, sm);
      TFront F{}; F.r = 700; F.w = 651; F.nbp = 11; F.nt = 11;
      tile_to_panel(F, sm, g + (long long)gridDim.x * 4 * TBD + (long long)blockIdx.x * 64 * 700, 1, 0);
      __syncthreads();
      if (threadIdx.x == 0) __threadfence();
      __syncthreads();
    } else if (which == 10 || which == 11) {   // syrk+potrf: 10 = separate (gemm_smem + potrf64), 11 = fused, no follower
      tile_load_async(sm + 2 * TBD, gt); cp_async_wait_all(); __syncthreads();
      if (which == 10) { tile_gemm_nt_smem(sm + 2 * TBD, sm + TBD, sm + TBD); tile_potrf64(sm + 2 * TBD, 64, dinv + blockIdx.x * 64, sm + 3 * TBD, sm + 3 * TBD + 64, &sf); }
      else tile_syrk_potrf64<false>(sm + 2 * TBD, sm + TBD, 64, dinv + blockIdx.x * 64, sm + 3 * TBD, sm + 3 * TBD + 64, &sf);
    } else if (which == 12) {  // fused with the follower
      tile_load_async(sm + 2 * TBD, gt); cp_async_wait_all(); __syncthreads();
      tile_syrk_potrf64<true>(sm + 2 * TBD, sm + TBD, 64, dinv + blockIdx.x * 64, sm + 3 * TBD, sm + 3 * TBD + 64, &sf);
    } else if (which == 9) {   // current CRIT body: trsm + store + fence + fused syrk/potrf + store + fence
      tile_load_async(sm, gt + TBD); tile_load_async(sm + TBD, gt + 2 * TBD); tile_load_async(sm + 2 * TBD, gt); cp_async_wait_all(); __syncthreads();
      long long c0 = clock64();
      tile_trsm64(sm + TBD, sm, sm + 3 * TBD);
      __syncthreads(); long long c1 = clock64();
      tile_store(gt + 3 * TBD, sm + TBD);
      __syncthreads(); if (threadIdx.x == 0) __threadfence(); __syncthreads();
      long long c2 = clock64();
      tile_syrk_potrf64(sm + 2 * TBD, sm + TBD, 64, dinv + blockIdx.x * 64, sm + 3 * TBD, sm + 3 * TBD + 64, &sf);
      long long c3 = clock64();
      tile_store(gt + 3 * TBD, sm + 2 * TBD);
      __syncthreads(); if (threadIdx.x == 0) __threadfence(); __syncthreads();
      long long c4 = clock64();
      if (threadIdx.x == 0 && blockIdx.x == 0 && r == reps - 1) printf("crit parts: trsm %lld store+fence %lld syrk+potrf %lld store+fence %lld\n", c1 - c0, c2 - c1, c3 - c2, c4 - c3);
    } else if (which == 8) {   // the whole CRIT body without waits
      tile_load_async(sm, gt + TBD); tile_load_async(sm + TBD, gt + 2 * TBD); tile_load_async(sm + 2 * TBD, gt); cp_async_wait_all(); __syncthreads();
      tile_trsm64(sm + TBD, sm, sm + 3 * TBD);
      tile_store(gt + 3 * TBD, sm + TBD);
      TFront F{}; F.r = 700; F.w = 651; F.nbp = 11; F.nt = 11;
      tile_to_panel(F, sm + TBD, g + (long long)gridDim.x * 4 * TBD + (long long)blockIdx.x * 64 * 700, 1, 0);
      __syncthreads(); if (threadIdx.x == 0) __threadfence(); __syncthreads();
      tile_gemm_nt_smem(sm + 2 * TBD, sm + TBD, sm + TBD);
      tile_potrf64(sm + 2 * TBD, 64, dinv + blockIdx.x * 64, sm + 3 * TBD, sm + 3 * TBD + 64, &sf);
      tile_store(gt + 3 * TBD, sm + 2 * TBD);
      tile_to_panel(F, sm + 2 * TBD, g + (long long)gridDim.x * 4 * TBD + (long long)blockIdx.x * 64 * 700, 1, 1);
      __syncthreads(); if (threadIdx.x == 0) __threadfence(); __syncthreads();
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / reps;
}

int main() {
  const int nb = 296;
  std::vector<double> h((size_t)nb * 4 * TBD);
  // tile 0: SPD (diagonally dominant), tile 1: its factor is produced by which=0 (we fake: identity-ish lower),
  for (int b = 0; b < nb; b++) {
    double* t = h.data() + (size_t)b * 4 * TBD;
    for (int c = 0; c < 64; c++) for (int r = 0; r < 64; r++) {
      t[c * 64 + r] = (r == c) ? 70.0 : 0.5 / (1 + r + c);                  // SPD
      t[TBD + c * 64 + r] = (r == c) ? 2.0 : (r > c ? 0.01 : 0.0);          // lower "L"
      t[2 * TBD + c * 64 + r] = 0.3 * std::sin(r + 2.0 * c);
      t[3 * TBD + c * 64 + r] = 0.0;
    }
  }
  double *g, *dinv; long long* out;
  cudaMalloc(&g, h.size() * 8 + (size_t)nb * 64 * 700 * 8 * 2); cudaMalloc(&dinv, nb * 64 * 8); cudaMalloc(&out, nb * 8);
  cudaMemcpy(g, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, TILE_SMEM_BYTES);
  const char* names[] = {"potrf64", "trsm64", "gemm_global", "load2tiles", "diag32", "rowsolve32x64", "gemm_smem",
                         "store+panel+fence", "crit_body", "crit_now", "syrk_potrf_sep", "syrk_potrf_fused", "syrk_potrf_follow"};
  for (int w = 0; w < 13; w++) {
    for (int grid : {1, 148, 296}) {
      bench<<<grid, 256, TILE_SMEM_BYTES>>>(w, 20, g, dinv, out);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<long long> o(nb);
      cudaMemcpy(o.data(), out, (grid < nb ? grid : nb) * 8, cudaMemcpyDeviceToHost);
      printf("%-14s grid %3d: %8lld cycles/call (%.2f us @1.965GHz)  %s\n", names[w], grid, o[0], o[0] / 1965.0,
             e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  }
  return 0;
}
