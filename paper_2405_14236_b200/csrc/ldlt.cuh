// ldlt.cuh -- pivot-free LDL^T with inertia (factor_kind = 1; P:370-375,
// P:424-429 eq. ipm:inertia; the paper's GPU factorisation is cuDSS LDL^T).
//
// The factor is kept in "signed Cholesky" form K = L~ S L~^T with S = diag(s_j), s_j = +-1 and
// l~_jj = sqrt(|d_j|) > 0; the LDL^T factors are L = L~ diag(l~)^-1 (unit lower) and
// D = S diag(l~)^2 (d_j = s_j l~_jj^2) -- the same pivots, so inertia(K) = (#s_j = +1, #s_j = -1,
// #zero pivots) by Sylvester's law.  Keeping L~ lets the triangular solves and the
// L11^-1 products run unchanged: K^-1 b = L~^-T S L~^-1 b (S is applied between the sweeps).
//
// Column j (left-looking blocks as front_factor_cta_ll, dense.cuh):
//   d_j = a_jj - sum_k l~_jk^2 s_k ;  s_j = sign(d_j) ;  |d_j| <= 1e-14 |K_jj| counts as a zero
//   pivot (R6) and is replaced by s_j max(1e-14 |K_jj|, 1e-300) so that the sweep stays finite ;
//   l~_jj = sqrt(|d_j|) ;  l~_ij = (a_ij - sum_k l~_ik s_k l~_jk) s_j / l~_jj
// Every Schur / block update is A -= L~ S L~^T (the A operand of the DMMA scaled by s_k).
// A non-finite pivot is a breakdown (fail column, as for LL^T).  Inertia counts are integer
// atomics (deterministic).
#pragma once
#include "dense.cuh"

namespace kkt {

// Pivot rule shared by the CTA and tile kernels: returns |d| after the zero-pivot substitution,
// sets s (+-1), zero, bad.
__device__ __forceinline__ double ldlt_pivot(double d, double kjj, double& s, bool& zero, bool& bad) {
  s = (d < 0.0) ? -1.0 : 1.0;
  bad = !isfinite(d);
  const double thr = 1e-14 * fabs(kjj);
  double ad = fabs(d);
  zero = !(ad > thr);
  if (zero && !bad) ad = fmax(thr, 1e-300);
  return ad;
}

// Signed Cholesky of the kb x kb diagonal block at (c0, c0) of a column-major front F (ld r) by one
// warp (lane = row; identity padding beyond kb).  Writes L~ (zeros above the diagonal), inverse
// pivots 1 / l~_jj into dinv and sinv, signs into ssg (shared) and sg_out (global), the first
// non-finite pivot column into *fail_k, and adds the block's (positive, negative, zero) pivot
// counts to cnt3.  Kv/Kp/col0: the condensed matrix (internal lower CSC, diagonal first in each
// column) and the supernode's first column -- K_jj gives the zero-pivot threshold.
__device__ __forceinline__ void ll_diag_warp_signed(double* F, int r, int c0, int kb, int lane, double* dinv,
                                                    double* sinv, double* ssg, double* L11s, int* fail_k,
                                                    double* sg_out, const double* Kv, const int* Kp, int col0,
                                                    int* cnt3) {
  const int row = c0 + lane;
  double a[32];
#pragma unroll
  for (int c = 0; c < 32; c++)
    a[c] = (lane < kb && c < kb && c <= lane) ? F[(c0 + c) * r + row] : (c == lane ? 1.0 : 0.0);
  const double kjj_lane = (lane < kb) ? __ldg(Kv + __ldg(Kp + col0 + c0 + lane)) : 1.0;  // K_jj (diagonal first)
  double myinv = 0.0, mys = 1.0;
  unsigned bad = 0;
  int npos = 0, nneg = 0, nzero = 0;
#pragma unroll
  for (int c = 0; c < 32; c++) {
    const double d = shfl_idx_d(a[c], c);
    const double kjj = shfl_idx_d(kjj_lane, c);
    double s;
    bool zero, b_;
    const double ad = ldlt_pivot(d, kjj, s, zero, b_);
    if (c < kb) {
      bad |= (b_ ? 1u : 0u) << c;
      if (zero) nzero++; else if (s > 0) npos++; else nneg++;
    }
    const double inv = 1.0 / sqrt(ad);
    if (lane == c) { myinv = inv; mys = s; }
    const double l = (lane > c) ? a[c] * inv * s : (lane == c ? ad * inv : 0.0);
    a[c] = l;
    L11s[c * 32 + lane] = l;
    warp_bar();
    const double ls = l * s;
#pragma unroll
    for (int cc = c + 1; cc < 32; cc++) a[cc] = fma(-ls, L11s[c * 32 + cc], a[cc]);
    asm volatile("" ::: "memory");
  }
#pragma unroll
  for (int c = 0; c < 32; c++)
    if (lane < kb && c < kb) F[(long long)(c0 + c) * r + row] = (c <= lane) ? a[c] : 0.0;
  sinv[lane] = myinv;
  ssg[lane] = (lane < kb) ? mys : 1.0;
  if (lane < kb) { dinv[c0 + lane] = myinv; sg_out[c0 + lane] = mys; }
  bad &= (kb < 32) ? ((1u << kb) - 1u) : 0xffffffffu;
  if (lane == 0) {
    if (bad && *fail_k < 0) *fail_k = c0 + __ffs(bad) - 1;
    if (npos) atomicAdd(cnt3, npos);
    if (nneg) atomicAdd(cnt3 + 1, nneg);
    if (nzero) atomicAdd(cnt3 + 2, nzero);
  }
}

// L~21 = A21 L~11^-T S11: the usual row solve (unsigned, inverse pivots sinv), signs at the store.
__device__ __forceinline__ void ll_trsm_rows1_signed(double* F, int r, int c0, int kb, const double* sinv,
                                                     const double* ssg, const double* L11s, int tid, int nt) {
  for (int i = c0 + kb + tid; i < r; i += nt) {
    double x[32];
#pragma unroll
    for (int c = 0; c < 32; c++) x[c] = (c < kb) ? F[(c0 + c) * r + i] : 0.0;
#pragma unroll
    for (int c = 0; c < 32; c++) {
      x[c] *= sinv[c];
#pragma unroll
      for (int cc = c + 1; cc < 32; cc++) x[cc] = fma(-x[c], L11s[c * 32 + cc], x[cc]);
      asm volatile("" ::: "memory");
    }
#pragma unroll
    for (int c = 0; c < 32; c++)
      if (c < kb) F[(c0 + c) * r + i] = x[c] * ssg[c];
  }
}

// A(c0:r, blk) -= L~(c0:r, 0:c0) S L~(blk, 0:c0)^T  (ll_block_update with the A operand * s_k)
__device__ __forceinline__ void ll_block_update_signed(double* F, int r, int c0, int kb, int warp, int nw, int lane,
                                                       const double* sg) {
  const int lr = lane >> 2, lc = lane & 3;
  const int nst = (r - c0 + 7) >> 3;
  const int ntc = (kb + 7) >> 3;
  for (int st = warp; st < nst; st += nw) {
    const int row = c0 + st * 8 + lr;
    const bool rok = row < r;
    double acc0[4], acc1[4];
#pragma unroll
    for (int t = 0; t < 4; t++) { acc0[t] = 0.0; acc1[t] = 0.0; }
    for (int k = 0; k < c0; k += 4) {
      const double* Fk = F + (k + lc) * r;
      const double a = rok ? Fk[row] * sg[k + lc] : 0.0;
      double b[4];
#pragma unroll
      for (int t = 0; t < 4; t++) {
        const int col = c0 + 8 * t + lr;
        b[t] = (t < ntc && col < c0 + kb) ? Fk[col] : 0.0;
      }
#pragma unroll
      for (int t = 0; t < 4; t++)
        if (t < ntc && t <= st) dmma8x8x4(acc0[t], acc1[t], a, b[t]);
    }
#pragma unroll
    for (int t = 0; t < 4; t++) {
      const int col = c0 + 8 * t + lc * 2;
      if (t < ntc && t <= st && rok) {
        if (col < c0 + kb && col <= row) F[col * r + row] -= acc0[t];
        if (col + 1 < c0 + kb && col + 1 <= row) F[(col + 1) * r + row] -= acc1[t];
      }
    }
  }
}

// U -= L~21 S L~21^T (schur_tiles22 with the A operand * s_k)
__device__ __forceinline__ void schur_tiles22_signed(double* F, double* U, int r, int w, int warp, int nw, int lane,
                                                     const double* sg) {
  const int R = r - w;
  if (R <= 0) return;
  const int lr = lane >> 2, lc = lane & 3;
  const int nm = (R + 15) >> 4;
  const int nmt = nm * (nm + 1) / 2;
  for (int t = warp; t < nmt; t += nw) {
    int J = 0, rem = t;
    while (rem >= nm - J) { rem -= nm - J; J++; }
    const int I = J + rem;
    const int ra0 = w + 16 * I + lr, ra1 = ra0 + 8, rb0 = w + 16 * J + lr, rb1 = rb0 + 8;
    const bool oa0 = ra0 < r, oa1 = ra1 < r, ob0 = rb0 < r, ob1 = rb1 < r;
    double c00 = 0, c01 = 0, c10 = 0, c11 = 0, c20 = 0, c21 = 0, c30 = 0, c31 = 0;
    for (int k = 0; k < w; k += 4) {
      const int kc = k + lc;
      const bool kin = kc < w;
      const double* Fk = F + kc * r;
      const double sk = kin ? sg[kc] : 0.0;
      const double a0 = (kin && oa0) ? Fk[ra0] * sk : 0.0, a1 = (kin && oa1) ? Fk[ra1] * sk : 0.0;
      const double b0 = (kin && ob0) ? Fk[rb0] : 0.0, b1 = (kin && ob1) ? Fk[rb1] : 0.0;
      dmma8x8x4(c00, c01, a0, b0);
      dmma8x8x4(c10, c11, a0, b1);
      dmma8x8x4(c20, c21, a1, b0);
      dmma8x8x4(c30, c31, a1, b1);
    }
    const double cv[4][2] = {{c00, c01}, {c10, c11}, {c20, c21}, {c30, c31}};
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const int i = w + 16 * I + 8 * (q >> 1) + lr;
      const int j = w + 16 * J + 8 * (q & 1) + 2 * lc;
#pragma unroll
      for (int e = 0; e < 2; e++)
        if (i < r && j + e <= i) U[upk(i - w, j + e - w, R)] -= cv[q][e];
    }
  }
}

// Left-looking signed partial factorisation of a front in shared memory (front_factor_cta_ll's
// schedule).  sg: global signs of the supernode's columns; kdiag: K_jj of its columns.
__device__ __noinline__ void front_factor_cta_ldlt(double* F, double* U, int r, int w, double* dinv, int* s_fail,
                                                   double* sg, const double* Kv, const int* Kp, int col0, int* cnt3) {
  __shared__ double sinv[32], ssg[32];
  __shared__ __align__(16) double L11s[32 * 32];
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  for (int c0 = 0; c0 < w; c0 += 32) {
    const int kb = (w - c0) < 32 ? (w - c0) : 32;
    if (c0 > 0) {
      ll_block_update_signed(F, r, c0, kb, warp, nw, lane, sg);
      __syncthreads();
    }
    if (warp == 0) ll_diag_warp_signed(F, r, c0, kb, lane, dinv, sinv, ssg, L11s, s_fail, sg, Kv, Kp, col0, cnt3);
    __syncthreads();
    ll_trsm_rows1_signed(F, r, c0, kb, sinv, ssg, L11s, tid, nt);
    __syncthreads();
  }
  schur_tiles22_signed(F, U, r, w, warp, nw, lane, sg);
}

// y <- S y between the forward and the backward sweep (internal numbering, all instances)
__global__ void ldlt_sign_kernel(long long total, double* y, const double* __restrict__ sg) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x)
    y[i] *= sg[i];
}

}  // namespace kkt
