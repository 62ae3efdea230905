// trsv.cuh -- supernodal triangular solves L y = P b, L^T z = y, x = P^T z (P:1376-1377,
// SURVEY §8(a) a3), multifrontal form:
//   forward (bottom-up):  v = [b(cols(s)); 0] + sum_children extend(u_c);
//                         y_s = L11^-1 v[0:w);  u_s = v[w:r) - L21 y_s  (passed to the parent)
//   backward (top-down):  x_s = L11^-T (y_s - L21^T x(R_s[w:r)))
// Same small (warp per supernode) / big (CTA per supernode) split as the factorisation.
// Forward: continuation scheduling (last child continues with the parent, no waiting).
// Backward: a finished supernode continues with its first child and pushes the others on a
// work queue (slot flags are reset by their consumer); workers exit once every task is done.
#pragma once
#include "factor.cuh"

namespace kkt {

// encoded task = s * batch + b
struct TaskQueue {
  int* q;      // [ns * batch] task slots
  int* flag;   // [ns * batch] 1 = slot published
};

// ---------------------------------------------------------------- CTA-blocked sweeps (big)
// Forward sweep of one supernode by a CTA, v[0:r) in shared memory, L read from L2/HBM:
// per 32-column block, warp 0 solves the diagonal block in registers (lane = row; the block's
// rows are fetched while the previous block's rows are updated), then every thread updates
// rows below with the block (thread per row, 32 independent loads in flight).
__device__ __forceinline__ void cta_fwd_blocked(const double* __restrict__ L, int r, int w,
                                                const double* __restrict__ dv, double* v, int tid, int nt) {
  const int lane = tid & 31, warp = tid >> 5;
  const unsigned full = 0xffffffffu;
  double ld[32];
  if (warp == 0) {
#pragma unroll
    for (int c = 0; c < 32; c++) ld[c] = (lane < w && c < lane) ? __ldg(L + (long long)c * r + lane) : 0.0;
  }
  for (int c0 = 0; c0 < w; c0 += 32) {
    const int kb = min(32, w - c0);
    if (warp == 0) {
      const int row = c0 + lane;
      double x = (lane < kb) ? v[row] : 0.0;
      const double di = (lane < kb) ? __ldg(dv + row) : 0.0;
#pragma unroll
      for (int k = 0; k < 32; k++) {
        if (k < kb) {
          const double yk = __shfl_sync(full, x * di, k);
          if (lane == k) x = yk;
          else if (lane > k) x = fma(-ld[k], yk, x);
        }
      }
      if (lane < kb) v[row] = x;
      // next diagonal block (L is read-only here)
      const int n0 = c0 + 32, nkb = min(32, w - n0);
#pragma unroll
      for (int c = 0; c < 32; c++)
        ld[c] = (lane < nkb && c < lane) ? __ldg(L + (long long)(n0 + c) * r + n0 + lane) : 0.0;
    }
    __syncthreads();
    for (int i = c0 + kb + tid; i < r; i += nt) {
      double l[32];
#pragma unroll
      for (int c = 0; c < 32; c++) l[c] = (c < kb) ? __ldg(L + (long long)(c0 + c) * r + i) : 0.0;
      double a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int c = 0; c < 32; c += 2) {
        a0 = fma(l[c], (c < kb) ? v[c0 + c] : 0.0, a0);
        a1 = fma(l[c + 1], (c + 1 < kb) ? v[c0 + c + 1] : 0.0, a1);
      }
      v[i] -= a0 + a1;
    }
    __syncthreads();
  }
}

// Backward sweep of one supernode by a CTA, xa[0:r) in shared memory (own part = y on entry,
// ancestor part = x): per 32-column block, last first, every thread accumulates its rows'
// products L_ic x_i for the block's 32 columns, a 31-shuffle transpose-reduce gives each lane
// its column's warp sum, and warp 0 adds the warp partials in fixed order and solves the
// transposed diagonal block in registers.  part: [8][32] shared scratch.
__device__ __forceinline__ void cta_bwd_blocked(const double* __restrict__ L, int r, int w,
                                                const double* __restrict__ dv, double* xa, double* part,
                                                int tid, int nt) {
  const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  const unsigned full = 0xffffffffu;
  for (int c0 = ((w - 1) / 32) * 32; c0 >= 0; c0 -= 32) {
    const int kb = min(32, w - c0);
    double ld[32];
    double y0 = 0.0, di = 0.0;
    if (warp == 0) {  // column c0+lane of the diagonal block, rows below the diagonal
      if (lane < kb) { y0 = xa[c0 + lane]; di = __ldg(dv + c0 + lane); }
#pragma unroll
      for (int k = 0; k < 32; k++)
        ld[k] = (lane < kb && k > lane && k < kb) ? __ldg(L + (long long)(c0 + lane) * r + c0 + k) : 0.0;
    }
    double p[32];
#pragma unroll
    for (int c = 0; c < 32; c++) p[c] = 0.0;
    for (int i = c0 + kb + tid; i < r; i += nt) {
      const double xi = xa[i];
#pragma unroll
      for (int c = 0; c < 32; c++) p[c] = fma((c < kb) ? __ldg(L + (long long)(c0 + c) * r + i) : 0.0, xi, p[c]);
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      const bool up = (lane & o) != 0;
#pragma unroll
      for (int c = 0; c < o; c++) {
        const double send = up ? p[c] : p[c + o];
        const double keep = up ? p[c + o] : p[c];
        p[c] = keep + __shfl_xor_sync(full, send, o);
      }
    }
    part[warp * 32 + lane] = p[0];
    __syncthreads();
    if (warp == 0) {
      double a = y0;
      for (int q = 0; q < nw; q++) a -= part[q * 32 + lane];
#pragma unroll
      for (int k = 31; k >= 0; k--) {
        if (k < kb) {
          const double xk = __shfl_sync(full, a * di, k);
          if (lane == k) a = xk;
          else if (lane < k) a = fma(-ld[k], xk, a);
        }
      }
      if (lane < kb) xa[c0 + lane] = a;
    }
    __syncthreads();
  }
}

// =====================================================================================
// Inverse-diagonal-block supernodal sweeps for the big (CTA) supernodes.  After the numeric
// factorization, linv_kernel forms Li = L11^-1 of every big non-huge supernode (all in
// parallel, off the tree's critical path); the solves then replace the w-step dependent
// substitution on L11 by two data-parallel products per supernode:
//   forward:   y1 = Li v[0:w),            u = v[w:r) - L21 y1
//   backward:  z = y1 - L21^T x(anc),     x1 = Li^T z
// (the same operator L11^-1 applied as a matrix; the refinement loop measures and corrects
// the result against the unassembled operator exactly as before).
// =====================================================================================
// Shared-memory budget of linv_kernel in doubles (host and device decide residency with it).
#define KKT_LINV_CAP 28160
// packed block-lower-triangular staging of L11: block (I, K), K <= I, of 32 x 33 doubles
__host__ __device__ __forceinline__ int linv_packed(int nb) { return nb * (nb + 1) / 2 * 1056; }
__host__ __device__ __forceinline__ bool linv_resident(int nb) {
  return linv_packed(nb) + 1024 + nb * 1024 + nb * 32 * 32 <= KKT_LINV_CAP;
}
// wavefront variant: every X block (I, J <= I) and every partial sum T_IJ (J < I) in shared memory
__host__ __device__ __forceinline__ int linv_wave_need(int nb) {
  return linv_packed(nb) + 1024 + nb * (nb + 1) / 2 * 1024 + nb * (nb - 1) / 2 * 1024;
}
__host__ __device__ __forceinline__ bool linv_wave(int nb) { return nb >= 2 && linv_wave_need(nb) <= KKT_LINV_CAP; }

__global__ void __launch_bounds__(KKT_BNT) linv_kernel(DevPlan P, const double* __restrict__ Lx_all,
                                                       const double* __restrict__ Dv_all, double* Li_all) {
  // L11 staged in shared memory as its lower 32 x 32 blocks (packed, row pitch 33), padded to
  // nb*32 with the identity: L11(i, k) = Ls[(I(I+1)/2 + K) * 1056 + (i%32) * 33 + k%32].
  // Phase 1: warp I inverts diagonal block I (lane j: column j in registers, substitution with
  //          broadcast rows of L11).
  // Phase 2: warp J forms the blocks below it in block column J, top to bottom:
  //          X_IJ = -X_II * sum_{K=J}^{I-1} L_IK X_KJ   (X_KJ and X_II read back from Li).
  extern __shared__ double Ls[];
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  const long long tasks = (long long)P.ns_b * P.batch;
  // Tasks in reverse topological order: the roots -- the widest blocks, the longest tasks --
  // start in the first wave instead of queueing behind the leaves (longest-first scheduling).
  for (long long t0 = blockIdx.x; t0 < tasks; t0 += gridDim.x) {
    const long long t = tasks - 1 - t0;
    const int b = (int)(t % P.batch);
    const int s = __ldg(P.order_b + t / P.batch);
    const long long lip = __ldg(P.sn_Lip + s);
    if (lip < 0) continue;  // huge: solved by the whole-GPU path
    const SnInfo I = P.sn[s];
    const int w = I.w, r = I.r, nb = (w + 31) >> 5, LD = nb * 32;
    const double* L = Lx_all + (long long)b * P.nnzL_stored + I.Lp;
    const double* dv = Dv_all + (long long)b * P.n + I.f0;
    double* Li = Li_all + (long long)b * P.linv_doubles + lip;  // column-major w x w
#ifdef KKT_LINV_PROF  // tuning build (-DKKT_LINV_PROF): per-task cycles of staging / phase 1 / phase 2
    const long long pc0 = clock64();
#endif
    double* Ts = Ls + linv_packed(nb);         // [32][32]
    const bool resident = linv_resident(nb);   // X's diagonal blocks + current block column in smem
    double* Xd = Ts + 1024;                    // [nb][32][32] diagonal inverses (row-major blocks)
    double* Xc = Xd + nb * 1024;               // [LD][32] current block column
    const bool wave = linv_wave(nb);
    double* Xw = Ts + 1024;                    // wave: packed X blocks (I, J <= I), row-major 32 x 32
    double* Tw = Xw + nb * (nb + 1) / 2 * 1024;  // wave: T blocks (I, J < I) at (I(I-1)/2 + J)
    __syncthreads();
    for (int q0 = tid; q0 < LD * LD; q0 += nt * 16) {  // coalesced along the columns of L11, 16 loads in flight
      double v8[16];
#pragma unroll
      for (int u = 0; u < 16; u++) {
        const int q = q0 + u * nt, k = q / LD, i = q % LD;
        v8[u] = (q < LD * LD && i < w && k < w && k <= i) ? __ldg(L + (long long)k * r + i) : 0.0;  // k <= i: lower blocks only
      }
#pragma unroll
      for (int u = 0; u < 16; u++) {
        const int q = q0 + u * nt, k = q / LD, i = q % LD;
        if (q < LD * LD && (k >> 5) <= (i >> 5))
          Ls[((i >> 5) * ((i >> 5) + 1) / 2 + (k >> 5)) * 1056 + (i & 31) * 33 + (k & 31)] =
              (i < w && k < w) ? v8[u] : (i == k ? 1.0 : 0.0);
      }
    }
    __syncthreads();
#ifdef KKT_LINV_PROF
    const long long pc1 = clock64();
#endif
    // phase 1: diagonal blocks
    for (int Ib = warp; Ib < nb; Ib += nw) {
      const int o = Ib * 32;
      const int j = lane;
      // Right-looking (column) substitution: x[i] accumulates sum_{k<i} L(i,k) x[k] in ascending
      // k -- the same fma sequence as the row-oriented dot product, hence bitwise the same
      // result -- but the dependent chain is 32 finalizations, not the 496 fmas of the dots.
      double x[32];
#pragma unroll
      for (int i = 0; i < 32; i++) x[i] = 0.0;
#pragma unroll
      for (int k = 0; k < 32; k++) {
        const double dk = (o + k < w) ? __ldg(dv + o + k) : 1.0;
        x[k] = (k < j) ? 0.0 : (k == j ? dk : -dk * x[k]);
        const double* Lcol = Ls + (Ib * (Ib + 1) / 2 + Ib) * 1056 + (k + 1) * 33 + k;
#pragma unroll
        for (int i = k + 1; i < 32; i++) x[i] = fma(Lcol[(i - k - 1) * 33], x[k], x[i]);
      }
#pragma unroll
      for (int i = 0; i < 32; i++)
        if (o + i < w && o + j < w) Li[(long long)(o + j) * w + o + i] = x[i];
      if (resident || wave) {
        double* xd = wave ? Xw + (Ib * (Ib + 1) / 2 + Ib) * 1024 : Xd + Ib * 1024;
#pragma unroll
        for (int i = 0; i < 32; i++) xd[i * 32 + j] = x[i];
      }
    }
    __syncthreads();
#ifdef KKT_LINV_PROF
    const long long pc2 = clock64();
#endif
    if (wave) {
      // phase 2, wavefront form (right-looking over block rows K): step K adds L_IK X_KJ to every
      // T_IJ (I > K, J <= K) at once, then finalizes block row K+1: X_{K+1,J} = -X_{K+1,K+1} T.
      // Each T_IJ accumulates the same fma sequence (K, k ascending, from 0) as the column form.
      for (int Kb = 0; Kb + 1 < nb; Kb++) {
        const int nJ = Kb + 1, items = (nb - 1 - Kb) * nJ * 32;
        for (int it = warp * 4; it < items; it += nw * 4) {
          const int blk = it >> 5, i0 = it & 31, Ib = Kb + 1 + blk / nJ, Jb = blk % nJ;
          double* T = Tw + (Ib * (Ib - 1) / 2 + Jb) * 1024 + i0 * 32 + lane;
          const double* Lb = Ls + (Ib * (Ib + 1) / 2 + Kb) * 1056 + i0 * 33;
          const double* X = Xw + (Kb * (Kb + 1) / 2 + Jb) * 1024 + lane;
          double tq[4];
#pragma unroll
          for (int u = 0; u < 4; u++) tq[u] = (Jb == Kb) ? 0.0 : T[u * 32];
#pragma unroll 8
          for (int k = 0; k < 32; k++) {
            const double xk = X[k * 32];
#pragma unroll
            for (int u = 0; u < 4; u++) tq[u] = fma(Lb[u * 33 + k], xk, tq[u]);
          }
#pragma unroll
          for (int u = 0; u < 4; u++) T[u * 32] = tq[u];
        }
        __syncthreads();
        const int Ib = Kb + 1, oi = Ib * 32;
        for (int it = warp * 4; it < nJ * 32; it += nw * 4) {
          const int Jb = it >> 5, i0 = it & 31, oj = Jb * 32;
          const double* T = Tw + (Ib * (Ib - 1) / 2 + Jb) * 1024;
          const double* Xii = Xw + (Ib * (Ib + 1) / 2 + Ib) * 1024;
          double* Xo = Xw + (Ib * (Ib + 1) / 2 + Jb) * 1024;
#pragma unroll
          for (int u = 0; u < 4; u++) {
            const int i = i0 + u;
            double a0 = 0.0, a1 = 0.0;
#pragma unroll
            for (int k = 0; k < 32; k += 2) {
              a0 = fma(Xii[i * 32 + k], T[k * 32 + lane], a0);
              a1 = fma(Xii[i * 32 + k + 1], T[(k + 1) * 32 + lane], a1);
            }
            const double xo = -(a0 + a1);  // X_II is zero above its diagonal
            Xo[i * 32 + lane] = xo;
            if (oj + lane < w && oi + i < w) Li[(long long)(oj + lane) * w + oi + i] = xo;
          }
        }
        __syncthreads();
      }
#ifdef KKT_LINV_PROF
      if (tid == 0) printf("linv wave s=%d w=%d nb=%d stage=%lld p1=%lld p2=%lld\n", s, w, nb, pc1 - pc0, pc2 - pc1, clock64() - pc2);
#endif
      continue;
    }
    if (resident) {
      // phase 2, shared-memory resident (nb <= 5): block column J at a time (X_IJ needs only
      // X_KJ, J <= K < I, and X_II), the current block column kept in Xc [LD][32]
      for (int Jb = 0; Jb + 1 < nb; Jb++) {
        const int oj = Jb * 32, j = lane;
        const bool jin = oj + j < w;
        for (int q = tid; q < 1024; q += nt) Xc[(oj + (q >> 5)) * 32 + (q & 31)] = Xd[Jb * 1024 + q];
        __syncthreads();
        for (int Ib = Jb + 1; Ib < nb; Ib++) {
          const int oi = Ib * 32;
          double tq[4] = {0.0, 0.0, 0.0, 0.0};
          for (int Kb = Jb; Kb < Ib; Kb++) {
            const int ok = Kb * 32;
            const double* Lb = Ls + (Ib * (Ib + 1) / 2 + Kb) * 1056 + warp * 33;
#pragma unroll 8
            for (int k = 0; k < 32; k++) {
              const double xk = Xc[(ok + k) * 32 + j];
#pragma unroll
              for (int u = 0; u < 4; u++) tq[u] = fma(Lb[u * 8 * 33 + k], xk, tq[u]);
            }
          }
#pragma unroll
          for (int u = 0; u < 4; u++) Ts[(warp + 8 * u) * 32 + j] = tq[u];
          __syncthreads();
#pragma unroll
          for (int u = 0; u < 4; u++) {
            const int i = warp + 8 * u;
            const double* xr = Xd + Ib * 1024 + i * 32;
            double a0 = 0.0, a1 = 0.0;
#pragma unroll
            for (int k = 0; k < 32; k += 2) {
              a0 = fma(xr[k], Ts[k * 32 + j], a0);
              a1 = fma(xr[k + 1], Ts[(k + 1) * 32 + j], a1);
            }
            const double xo = -(a0 + a1);  // X_II is zero above its diagonal
            Xc[(oi + i) * 32 + j] = xo;
            if (jin && oi + i < w) Li[(long long)(oj + j) * w + oi + i] = xo;
          }
          __syncthreads();
        }
      }
#ifdef KKT_LINV_PROF
      if (tid == 0) printf("linv s=%d w=%d nb=%d stage=%lld p1=%lld p2=%lld\n", s, w, nb, pc1 - pc0, pc2 - pc1, clock64() - pc2);
#endif
      continue;
    }
    // phase 2: below-diagonal blocks in dependency order (block distance d = I - J), one block
    // at a time by the whole CTA: warp q forms rows q, q+8, q+16, q+24 of T = sum_K L_IK X_KJ
    // (lane = column), then of X_IJ = -X_II T (T staged in shared memory).
    for (int d = 1; d < nb; d++) {
      for (int Jb = 0; Jb + d < nb; Jb++) {
        const int Ib = Jb + d, oi = Ib * 32, oj = Jb * 32, j = lane;
        const bool jin = oj + j < w;
        double tq[4] = {0.0, 0.0, 0.0, 0.0};
        for (int Kb = Jb; Kb < Ib; Kb++) {
          const int ok = Kb * 32;
          double xk[32];
#pragma unroll
          for (int k = 0; k < 32; k++) xk[k] = (jin && ok + k < w) ? Li[(long long)(oj + j) * w + ok + k] : 0.0;
#pragma unroll
          for (int u = 0; u < 4; u++) {
            const double* Lrow = Ls + (Ib * (Ib + 1) / 2 + Kb) * 1056 + (warp + 8 * u) * 33;
            double a = tq[u];
#pragma unroll
            for (int k = 0; k < 32; k++) a = fma(Lrow[k], xk[k], a);
            tq[u] = a;
          }
        }
#pragma unroll
        for (int u = 0; u < 4; u++) Ts[(warp + 8 * u) * 32 + j] = tq[u];
        __syncthreads();
#pragma unroll
        for (int u = 0; u < 4; u++) {
          const int i = warp + 8 * u;
          double xii[32];  // row i of X_II: independent loads, all in flight together
#pragma unroll
          for (int k = 0; k < 32; k++)
            xii[k] = (k <= i && oi + i < w && oi + k < w) ? Li[(long long)(oi + k) * w + oi + i] : 0.0;
          double a = 0.0;
#pragma unroll
          for (int k = 0; k < 32; k++) a = fma(xii[k], Ts[k * 32 + j], a);
          if (jin && oi + i < w) Li[(long long)(oj + j) * w + oi + i] = -a;
        }
        __syncthreads();
      }
    }
  }
}

// Row dot products of the big-supernode sweeps: acc = sum_k A[k * lda + i] x[k] for k < kend,
// four accumulators (a_j takes k = j mod 4 while a full group of four fits, the tail goes to
// a0), combined as (a0 + a1) + (a2 + a3).  The loads of 16 consecutive k are issued before
// their FMAs (16 in flight per thread: the products are latency-bound, one row per thread).
__device__ __forceinline__ double row_dot4(const double* __restrict__ A, long long lda, int i, const double* x,
                                           int kend) {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  const int k4 = kend & ~3;  // groups of four: k + 3 < kend
  int k = 0;
  for (; k + 16 <= k4; k += 16) {
    double l[16];
#pragma unroll
    for (int u = 0; u < 16; u++) l[u] = __ldg(A + (long long)(k + u) * lda + i);
#pragma unroll
    for (int u = 0; u < 16; u += 4) {
      a0 = fma(l[u], x[k + u], a0);
      a1 = fma(l[u + 1], x[k + u + 1], a1);
      a2 = fma(l[u + 2], x[k + u + 2], a2);
      a3 = fma(l[u + 3], x[k + u + 3], a3);
    }
  }
  {  // remaining groups of four (< 16 values), loads first
    double l[12];
    const int ng = (k4 - k) >> 2;
#pragma unroll
    for (int u = 0; u < 12; u++) l[u] = (u < 4 * ng) ? __ldg(A + (long long)(k + u) * lda + i) : 0.0;
#pragma unroll
    for (int u = 0; u < 12; u += 4) {
      if (u < 4 * ng) {
        a0 = fma(l[u], x[k + u], a0);
        a1 = fma(l[u + 1], x[k + u + 1], a1);
        a2 = fma(l[u + 2], x[k + u + 2], a2);
        a3 = fma(l[u + 3], x[k + u + 3], a3);
      }
    }
    k += 4 * ng;
  }
  for (; k < kend; k++) a0 = fma(__ldg(A + (long long)k * lda + i), x[k], a0);
  return (a0 + a1) + (a2 + a3);
}

// forward sweep of a big supernode with Li: v[0:r) in shared memory; tmp: >= w doubles
__device__ __forceinline__ void cta_fwd_inv(const double* __restrict__ L, const double* __restrict__ Li, int r,
                                            int w, double* v, double* tmp, int tid, int nt) {
  for (int i = tid; i < w; i += nt) tmp[i] = row_dot4(Li, w, i, v, i + 1);  // y1 = Li v[0:w) (lower)
  __syncthreads();
  for (int i = tid; i < w; i += nt) v[i] = tmp[i];
  for (int i = w + tid; i < r; i += nt) v[i] -= row_dot4(L, r, i, tmp, w);  // u = v[w:r) - L21 y1
  __syncthreads();
}

// backward sweep of a big supernode with Li: xa[0:w) = y1 on entry, xa[w:r) = ancestors' x;
// on return xa[0:w) = x1.  Warp per column (lanes along the contiguous column), fixed-order
// shuffle reductions; a warp takes four columns at a time so that their loads are in flight
// together (each column's sum keeps its own order).  tmp: >= w doubles.
__device__ __forceinline__ void cta_bwd_inv(const double* __restrict__ L, const double* __restrict__ Li, int r,
                                            int w, double* xa, double* tmp, int tid, int nt) {
  const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  constexpr int CB = 4, RB = 4;  // columns per warp at once, row chunks of 32 with loads in flight
  for (int k0 = warp; k0 < w; k0 += nw * CB) {  // z_k = y_k - L21(:,k)^T x(anc)
    double a[CB];
#pragma unroll
    for (int c = 0; c < CB; c++) a[c] = 0.0;
    for (int i0 = w + lane; i0 < r; i0 += 32 * RB) {
      double l[CB][RB], xv[RB];
#pragma unroll
      for (int q = 0; q < RB; q++) xv[q] = (i0 + 32 * q < r) ? xa[i0 + 32 * q] : 0.0;
#pragma unroll
      for (int c = 0; c < CB; c++)
#pragma unroll
        for (int q = 0; q < RB; q++) {
          const int k = k0 + c * nw, i = i0 + 32 * q;
          l[c][q] = (k < w && i < r) ? __ldg(L + (long long)k * r + i) : 0.0;
        }
#pragma unroll
      for (int c = 0; c < CB; c++)
#pragma unroll
        for (int q = 0; q < RB; q++)
          if (i0 + 32 * q < r) a[c] = fma(l[c][q], xv[q], a[c]);
    }
#pragma unroll
    for (int c = 0; c < CB; c++) {
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) a[c] += __shfl_xor_sync(0xffffffffu, a[c], o);
      const int k = k0 + c * nw;
      if (lane == 0 && k < w) tmp[k] = xa[k] - a[c];
    }
  }
  __syncthreads();
  for (int k0 = warp; k0 < w; k0 += nw * CB) {  // x_k = sum_{i>=k} Li(i,k) z_i
    double a[CB];
#pragma unroll
    for (int c = 0; c < CB; c++) a[c] = 0.0;
    // column k's lane covers rows k + lane + 32 j (the per-column order of the sequential form)
    for (int j0 = 0; k0 + j0 < w; j0 += 32 * RB) {
      double l[CB][RB];
#pragma unroll
      for (int c = 0; c < CB; c++)
#pragma unroll
        for (int q = 0; q < RB; q++) {
          const int k = k0 + c * nw, i = k + lane + j0 + 32 * q;
          l[c][q] = (k < w && i < w) ? __ldg(Li + (long long)k * w + i) : 0.0;
        }
#pragma unroll
      for (int c = 0; c < CB; c++)
#pragma unroll
        for (int q = 0; q < RB; q++) {
          const int k = k0 + c * nw, i = k + lane + j0 + 32 * q;
          if (k < w && i < w) a[c] = fma(l[c][q], tmp[i], a[c]);
        }
    }
#pragma unroll
    for (int c = 0; c < CB; c++) {
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) a[c] += __shfl_xor_sync(0xffffffffu, a[c], o);
      const int k = k0 + c * nw;
      if (lane == 0 && k < w) xa[k] = a[c];
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------- forward, small (warp)
__device__ __forceinline__ void fwd_sweep_any(const double* Lp, int r, int w, const double* dv,
                                              double* v, int lane) {
  if (r <= 32) fwd_sweep_warp<1>(Lp, r, w, dv, v, lane);
  else if (r <= 64) fwd_sweep_warp<2>(Lp, r, w, dv, v, lane);
  else if (r <= 128) fwd_sweep_warp<4>(Lp, r, w, dv, v, lane);
  else fwd_sweep_warp<8>(Lp, r, w, dv, v, lane);  // callers guarantee r <= 256
}
__device__ __forceinline__ void bwd_sweep_any(const double* Lp, int r, int w, const double* dv,
                                              double* xa, int lane) {
  if (w <= 32) bwd_sweep_warp<1>(Lp, r, w, dv, xa, lane);
  else if (w <= 64) bwd_sweep_warp<2>(Lp, r, w, dv, xa, lane);
  else bwd_sweep_warp<4>(Lp, r, w, dv, xa, lane);  // callers guarantee w <= 128
}

// Forward-solve input of a small supernode (one warp, r <= 64): panel -> Pn (shared), and
// v = [b(perm(cols)); 0] + extend-add of the children's update vectors (in child order).
// All loads are issued before the first dependent use: child metadata arrives with the panel
// and permutation, then the right-hand side and up to 8 chunks of 32 update entries per lane
// are in flight together; only the (rare) remainder falls back to a chunk-by-chunk loop.
__device__ __forceinline__ void stage_in(const DevPlan& P, const SnInfo& I, const double* __restrict__ L,
                                         const double* __restrict__ bb, const double* uv, double* Pn,
                                         double* v, int lane) {
  const int r = I.r, w = I.w, rw = r * w, nch = I.c1 - I.c0;
  if (nch > 32) {  // many children: plain chunk-by-chunk path
    copy_g2s<false>(Pn, L, rw, lane, 32);
    for (int q = lane; q < r; q += 32) v[q] = (q < w) ? bb[__ldg(P.perm + I.f0 + q)] : 0.0;
    __syncwarp();
    for (int c = I.c0; c < I.c1; c++) {
      const SnInfo C = P.chinfo[c];
      const int Rq = C.r - C.w;
      for (int q = lane; q < Rq; q += 32) v[__ldg(P.sn_rel + C.rp0 + C.w + q)] += ldcg(uv + C.uvp + q);
      __syncwarp();
    }
    return;
  }
  // metadata
  const int p0 = (lane < w) ? __ldg(P.perm + I.f0 + lane) : 0;
  const int p1 = (lane + 32 < w) ? __ldg(P.perm + I.f0 + lane + 32) : 0;
  int cR = 0, cRel = 0, cU = 0;
  if (lane < nch) {
    const int4 h = __ldg(reinterpret_cast<const int4*>(P.chinfo + I.c0 + lane));  // f0, w, r, rp0
    cR = h.z - h.y;
    cRel = h.w + h.y;
    cU = __ldg(reinterpret_cast<const int*>(P.chinfo + I.c0 + lane) + 10);        // uvp
  }
  // panel
  double lv[8];
#pragma unroll
  for (int u = 0; u < 8; u++) lv[u] = (lane + 32 * u < rw) ? __ldg(L + lane + 32 * u) : 0.0;
  // right-hand side (own columns)
  const double b0 = (lane < w) ? bb[p0] : 0.0;
  const double b1 = (lane + 32 < w) ? bb[p1] : 0.0;
  // children's update entries: slot k <-> (child ci, chunk base), uniform across the warp
  int bpos[8], bch[8];
  double bval[8];
  int ci = 0, base = 0;
  int Rc = nch > 0 ? __shfl_sync(0xffffffffu, cR, 0) : 0;
#pragma unroll
  for (int k = 0; k < 8; k++) {
    while (ci < nch && base >= Rc) {
      ci++;
      base = 0;
      Rc = (ci < nch) ? __shfl_sync(0xffffffffu, cR, ci) : 0;
    }
    bch[k] = ci;
    bpos[k] = -1;
    bval[k] = 0.0;
    if (ci < nch) {
      const int relp = __shfl_sync(0xffffffffu, cRel, ci), up = __shfl_sync(0xffffffffu, cU, ci);
      const int q = base + lane;
      if (q < Rc) { bpos[k] = __ldg(P.sn_rel + relp + q); bval[k] = ldcg(uv + up + q); }
      base += 32;
    }
  }
  // stores: panel, v init, then the children in order
#pragma unroll
  for (int u = 0; u < 8; u++) if (lane + 32 * u < rw) Pn[lane + 32 * u] = lv[u];
  if (rw > 256) copy_g2s<false>(Pn + 256, L + 256, rw - 256, lane, 32);
  if (lane < r) v[lane] = (lane < w) ? b0 : 0.0;
  if (lane + 32 < r) v[lane + 32] = (lane + 32 < w) ? b1 : 0.0;
  __syncwarp();
#pragma unroll
  for (int k = 0; k < 8; k++) {
    if (k > 0 && bch[k] != bch[k - 1]) __syncwarp();
    if (bpos[k] >= 0) v[bpos[k]] += bval[k];
  }
  __syncwarp();
  // remainder (more than 8 chunks of children entries)
  while (ci < nch) {
    while (ci < nch && base >= Rc) {
      ci++;
      base = 0;
      Rc = (ci < nch) ? __shfl_sync(0xffffffffu, cR, ci) : 0;
      __syncwarp();
    }
    if (ci >= nch) break;
    const int relp = __shfl_sync(0xffffffffu, cRel, ci), up = __shfl_sync(0xffffffffu, cU, ci);
    const int q = base + lane;
    if (q < Rc) v[__ldg(P.sn_rel + relp + q)] += ldcg(uv + up + q);
    base += 32;
  }
  __syncwarp();
}

__global__ void __launch_bounds__(KKT_WPB * 32) fwd_small_kernel(DevPlan P, const double* __restrict__ Lx_all,
                                                                 const double* __restrict__ Dv_all,
                                                                 const double* __restrict__ rhs, long long rs,
                                                                 double* Y_all, double* uv_all, int* cnt_all,
                                                                 int* ctl, const int* __restrict__ done) {
  extern __shared__ double sm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* Pn = sm + (long long)wid * (P.max_rw_small + P.max_r_small);
  double* v = Pn + P.max_rw_small;
  const int ninit = P.n_up_s * P.batch;
  pdl_launch_dependents();
  if (done && done[P.batch] == 0) return;  // every instance has finished refining
  for (;;) {
    const int t = warp_ticket(ctl);
    if (t >= ninit) break;
    const int b = t % P.batch;
    if (done && done[b]) continue;
    int s = __ldg(P.up_s + t / P.batch);
    int* cnt = cnt_all + (long long)b * P.ns;
    const double* Lb = Lx_all + (long long)b * P.nnzL_stored;
    const double* Dv = Dv_all + (long long)b * P.n;
    double* uv = uv_all + (long long)b * P.uvec_doubles;
    const double* bb = rhs + (long long)b * rs;
    double* Y = Y_all + (long long)b * P.n;
    SnInfo I = P.sn[s];
    for (;;) {
      if (lane == 0) trace_stamp(P, 1, s, b, 0);
      const int r = I.r, w = I.w;
      const double* L = Lb + I.Lp;
      // every independent load of the supernode is issued before the first use (one memory
      // round trip for metadata, one for values): parent info, own permutation entries,
      // children's info (lane c holds child c), the panel (registers), then the right-hand
      // side and the children's update vectors
      SnInfo Ip;
      if (I.par >= 0) Ip = P.sn[I.par];
      stage_in(P, I, L, bb, uv, Pn, v, lane);
      fwd_sweep_any(Pn, r, w, Dv + I.f0, v, lane);
      __syncwarp();
      for (int q = lane; q < w; q += 32) Y[I.f0 + q] = v[q];
      if (lane == 0) trace_stamp(P, 1, s, b, 1);
      if (I.par < 0) break;
      const int R = r - w;
      double* us = uv + I.uvp;
      for (int q = lane; q < R; q += 32) us[q] = v[w + q];
      if (!warp_signal_parent(I, Ip, cnt, lane, true)) break;
      s = I.par;
      I = Ip;
    }
  }
  warp_exit(ctl, gridDim.x * KKT_WPB);
}

// ---------------------------------------------------------------- forward, big (CTA)
__global__ void __launch_bounds__(KKT_BNT) fwd_big_kernel(DevPlan P, const double* __restrict__ Lx_all,
                                                          const double* __restrict__ Dv_all,
                                                          const double* __restrict__ rhs, long long rs,
                                                          double* Y_all, double* uv_all, int* cnt_all,
                                                          int* ctl, const int* __restrict__ done,
                                                          int pcap, const double* __restrict__ Li_all) {
  extern __shared__ double sm[];
  __shared__ int s_task, s_last;
  __shared__ int s_cR[32], s_cRel[32], s_cU[32];
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int ninit = P.n_up_bf * P.batch;
  double* v = sm;                         // [max_front]
  if (done && done[P.batch] == 0) return;  // every instance has finished refining
  for (;;) {
    const int t = next_task(ctl, &s_task);
    if (t >= ninit) break;
    const int b = t % P.batch;
    if (done && done[b]) continue;
    int s = __ldg(P.up_bf + t / P.batch);
    int* cnt = cnt_all + (long long)b * P.ns;
    const double* Lb = Lx_all + (long long)b * P.nnzL_stored;
    double* uv = uv_all + (long long)b * P.uvec_doubles;
    const double* bb = rhs + (long long)b * rs;
    double* Y = Y_all + (long long)b * P.n;
    if (tid == 0) {  // all children are small: wait for the small phase to have counted them
      const SnInfo I0 = P.sn[s];
      wait_children_reset(cnt + s, I0.c1 - I0.c0);
    }
    __syncthreads();
    SnInfo I = P.sn[s];
    for (;;) {
      if (tid == 0) trace_stamp(P, 1, s, b, 0);
      const int r = I.r, w = I.w, R = r - w, nch = I.c1 - I.c0;
      const double* L = Lb + I.Lp;
      // all independent loads first: parent info and big-children count (for the hand-off),
      // permutation, children's metadata (thread c: child c), then rhs and children's entries
      SnInfo Ip;
      int pnbig = 0;
      if (I.par >= 0) { Ip = P.sn[I.par]; pnbig = __ldg(P.sn_nbig + I.par); }
      const bool fast = nch <= 32;
      if (fast && tid < nch) {
        const int4 h4 = __ldg(reinterpret_cast<const int4*>(P.chinfo + I.c0 + tid));  // f0, w, r, rp0
        s_cR[tid] = h4.z - h4.y;
        s_cRel[tid] = h4.w + h4.y;
        s_cU[tid] = __ldg(reinterpret_cast<const int*>(P.chinfo + I.c0 + tid) + 10);  // uvp
      }
      for (int q = tid; q < r; q += nt) v[q] = (q < w) ? bb[__ldg(P.perm + I.f0 + q)] : 0.0;
      __syncthreads();
      if (fast) {
        // children's update entries: slot k <-> (child ci, chunk base), uniform across the CTA
        int bpos[6], bch[6];
        double bval[6];
        int ci = 0, base = 0, Rc = nch > 0 ? s_cR[0] : 0;
#pragma unroll
        for (int k = 0; k < 6; k++) {
          while (ci < nch && base >= Rc) { ci++; base = 0; Rc = (ci < nch) ? s_cR[ci] : 0; }
          bch[k] = ci; bpos[k] = -1; bval[k] = 0.0;
          if (ci < nch) {
            const int q = base + tid;
            if (q < Rc) { bpos[k] = __ldg(P.sn_rel + s_cRel[ci] + q); bval[k] = ldcg(uv + s_cU[ci] + q); }
            base += nt;
          }
        }
#pragma unroll
        for (int k = 0; k < 6; k++) {
          if (k > 0 && bch[k] != bch[k - 1]) __syncthreads();
          if (bpos[k] >= 0) v[bpos[k]] += bval[k];
        }
        __syncthreads();
        while (ci < nch) {  // remainder beyond 6 chunks
          while (ci < nch && base >= Rc) { ci++; base = 0; Rc = (ci < nch) ? s_cR[ci] : 0; __syncthreads(); }
          if (ci >= nch) break;
          const int q = base + tid;
          if (q < Rc) v[__ldg(P.sn_rel + s_cRel[ci] + q)] += ldcg(uv + s_cU[ci] + q);
          base += nt;
        }
        __syncthreads();
      } else {
        for (int c = I.c0; c < I.c1; c++) {
          const SnInfo C = P.chinfo[c];
          const int Rq = C.r - C.w;
          for (int q = tid; q < Rq; q += nt) v[__ldg(P.sn_rel + C.rp0 + C.w + q)] += ldcg(uv + C.uvp + q);
          __syncthreads();
        }
      }
      const long long lip = Li_all ? __ldg(P.sn_Lip + s) : -1;
      if (lip >= 0) cta_fwd_inv(L, Li_all + (long long)b * P.linv_doubles + lip, r, w, v, sm + P.max_front, tid, nt);
      else cta_fwd_blocked(L, r, w, Dv_all + (long long)b * P.n + I.f0, v, tid, nt);
      for (int q = tid; q < w; q += nt) Y[I.f0 + q] = v[q];
      if (tid == 0) trace_stamp(P, 1, s, b, 1);
      if (I.par < 0) break;
      double* us = uv + I.uvp;
      for (int q = tid; q < R; q += nt) us[q] = v[w + q];
      __threadfence();
      __syncthreads();
      if (Ip.huge && !P.solve_huge_cta) break;  // the whole-GPU phase (hsolve.cuh) takes it from here
      if (tid == 0) s_last = big_child_arrive_n(cnt + I.par, pnbig, Ip.c1 - Ip.c0);
      __syncthreads();
      if (!s_last) break;
      s = I.par;
      I = Ip;
    }
  }
  persistent_exit(ctl);
}

// ---------------------------------------------------------------- top-down queue helpers
// Pop the next task for a worker: the static ready list first, then the dynamic queue.
// Returns -1 when every task of the phase is done.  Called by one lane / thread.
__device__ __forceinline__ int pop_task(int* ctl, const int* init, int ninit_nodes, int batch,
                                        TaskQueue Q, int total) {
  const int h = atomicAdd(ctl, 1);
  const int ninit = ninit_nodes * batch;
  if (h < ninit) return __ldg(init + h / batch) * batch + h % batch;
  const int slot = h - ninit;
  if (slot >= total) return -1;
  for (int polls = 1;; polls++) {
    if (ld_volatile(Q.flag + slot)) break;
    // every task of the phase done?  (checked every 16th poll: one hot word for all pollers)
    if ((polls & 15) == 0 && ld_volatile(ctl + 8)) return -1;
    __nanosleep(32);
  }
  __threadfence();
  const int task = ld_volatile(Q.q + slot);
  Q.flag[slot] = 0;
  return task;
}

// Continue with the first eligible child, push the others.  Called by one lane / thread after
// the supernode's results are globally visible.  One slot reservation for all pushed children;
// a supernode with an eligible child cannot be the phase's last completion (the child completes
// after it), so it counts itself with a fire-and-forget reduction and only childless supernodes
// wait for the counter (all-done detection) -- the continuation pays at most one round trip.
__device__ __forceinline__ int spawn_children(const DevPlan& P, const SnInfo& I, int b, int* ctl,
                                              TaskQueue Q, bool big_phase, int total) {
  int next = -1, nextra = 0;
  for (int ci = I.c0; ci < I.c1; ci++) {
    if (big_phase && !P.chinfo[ci].big) continue;  // small children start phase 2 from dn_s
    if (next < 0) next = __ldg(P.sn_ch + ci) * P.batch + b;
    else nextra++;
  }
  if (nextra > 0) {
    int slot = atomicAdd(ctl + 2, nextra);
    bool first = true;
    for (int ci = I.c0; ci < I.c1; ci++) {
      if (big_phase && !P.chinfo[ci].big) continue;
      if (first) { first = false; continue; }
      Q.q[slot] = __ldg(P.sn_ch + ci) * P.batch + b;
      st_release(Q.flag + slot, 1);
      slot++;
    }
  }
  if (next >= 0) {
    atomicAdd(ctl + 3, 1);  // result unused -> RED
  } else {
    __threadfence();
    if (atomicAdd(ctl + 3, 1) == total - 1) st_release(ctl + 8, 1);  // completed -> all done
  }
  return next;
}

// Backward hand-off from a big (CTA) supernode to its small children, which the small kernel
// may already be polling (programmatic launch): the flag holds the number of small children
// still to consume it; each consumer decrements it, so every flag is back to 0 after a solve.
__device__ __forceinline__ void release_small_children(const DevPlan& P, const SnInfo& I, int s, int b, int* bflag) {
  int nsm = 0;
  for (int ci = I.c0; ci < I.c1; ci++) nsm += P.chinfo[ci].big ? 0 : 1;
  if (nsm) st_release(bflag + (long long)b * P.ns + s, nsm);
}

// ---------------------------------------------------------------- backward, big (CTA)
__global__ void __launch_bounds__(KKT_BNT) bwd_big_kernel(DevPlan P, const double* __restrict__ Lx_all,
                                                          const double* __restrict__ Dv_all,
                                                          const double* __restrict__ Y_all, double* Xp_all,
                                                          double* xout, long long xs, TaskQueue Q,
                                                          int* ctl, const int* __restrict__ done, int pcap,
                                                          int* bflag, const double* __restrict__ Li_all) {
  extern __shared__ double sm[];
  __shared__ int s_task;
  __shared__ int s_cid[32], s_cbig[32];
  pdl_launch_dependents();
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  const int total = P.ns_bn * P.batch;
  double* xa = sm;                   // [max_front]  x over R_s (own columns then ancestors)
  double* part = sm + P.max_front;   // [8 * 32] warp partials
  if (done && done[P.batch] == 0) return;  // every instance has finished refining
  int task = -1, cn_task = -1;
  SnInfo Cn;  // first child's metadata, prefetched (usually the continuation)
  for (;;) {
    if (task < 0) {
      if (tid == 0) s_task = pop_task(ctl, P.dn_b, P.n_dn_b, P.batch, Q, total);
      __syncthreads();
      task = s_task;
      __syncthreads();
      if (task < 0) break;
    }
    const int s = task / P.batch, b = task % P.batch;
    if (done && done[b]) {  // finished instance: account for its whole subtree without work
      if (tid == 0) { release_small_children(P, P.sn[s], s, b, bflag); s_task = spawn_children(P, P.sn[s], b, ctl, Q, true, total); }
      __syncthreads();
      task = s_task;
      cn_task = -1;
      __syncthreads();
      continue;
    }
    if (tid == 0) trace_stamp(P, 2, s, b, 0);
    const SnInfo I = (task == cn_task) ? Cn : P.sn[s];
    const int r = I.r, w = I.w, nch = I.c1 - I.c0;
    const double* L = Lx_all + (long long)b * P.nnzL_stored + I.Lp;
    double* Xp = Xp_all + (long long)b * P.n;
    const double* Y = Y_all + (long long)b * P.n;
    // independent loads first: children ids / classes, big-children count, first child's info
    const bool fast = nch <= 32;
    if (fast && tid < nch) { s_cid[tid] = __ldg(P.sn_ch + I.c0 + tid); s_cbig[tid] = P.chinfo[I.c0 + tid].big; }
    const int nbig = __ldg(P.sn_nbig + s);
    cn_task = -1;
    if (nch > 0) { Cn = P.chinfo[I.c0]; cn_task = __ldg(P.sn_ch + I.c0) * P.batch + b; }
    for (int q = tid; q < r; q += nt) xa[q] = (q < w) ? ldcg(Y + I.f0 + q) : ldcg(Xp + __ldg(P.sn_rows + I.rp0 + q));
    __syncthreads();
    const long long lip = Li_all ? __ldg(P.sn_Lip + s) : -1;
    if (lip >= 0) cta_bwd_inv(L, Li_all + (long long)b * P.linv_doubles + lip, r, w, xa, part, tid, nt);
    else cta_bwd_blocked(L, r, w, Dv_all + (long long)b * P.n + I.f0, xa, part, tid, nt);
    double* xo = xout + (long long)b * xs;
    for (int q = tid; q < w; q += nt) {
      Xp[I.f0 + q] = xa[q];
      xo[__ldg(P.perm + I.f0 + q)] = xa[q];
    }
    if (tid == 0) trace_stamp(P, 2, s, b, 1);
    __threadfence();
    __syncthreads();
    if (tid == 0) {
      if (nch - nbig > 0) st_release(bflag + (long long)b * P.ns + s, nch - nbig);  // small children's hand-off
      if (fast) {  // continue with the first big child, publish the others (one slot reservation)
        int next = -1;
        if (nbig > 1) {
          int slot = atomicAdd(ctl + 2, nbig - 1);
          for (int c = 0; c < nch; c++) {
            if (!s_cbig[c]) continue;
            const int tk = s_cid[c] * P.batch + b;
            if (next < 0) { next = tk; continue; }
            Q.q[slot] = tk;
            st_release(Q.flag + slot, 1);
            slot++;
          }
        } else if (nbig == 1) {
          for (int c = 0; c < nch; c++) if (s_cbig[c]) { next = s_cid[c] * P.batch + b; break; }
        }
        if (next >= 0) {
          atomicAdd(ctl + 3, 1);
        } else {
          __threadfence();
          if (atomicAdd(ctl + 3, 1) == total - 1) st_release(ctl + 8, 1);
        }
        s_task = next;
      } else {
        s_task = spawn_children(P, I, b, ctl, Q, true, total);
      }
    }
    __syncthreads();
    task = s_task;
    __syncthreads();
  }
  persistent_exit(ctl);
}

// ---------------------------------------------------------------- backward, small (warp)
__global__ void __launch_bounds__(KKT_WPB * 32) bwd_small_kernel(DevPlan P, const double* __restrict__ Lx_all,
                                                                 const double* __restrict__ Dv_all,
                                                                 const double* __restrict__ Y_all, double* Xp_all,
                                                                 double* xout, long long xs, TaskQueue Q,
                                                                 int* ctl, const int* __restrict__ done,
                                                                 int* bflag, int pdl) {
  extern __shared__ double sm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* Pn = sm + (long long)wid * (P.max_rw_small + P.max_r_small);
  double* xa = Pn + P.max_rw_small;
  const int total = P.ns_s * P.batch;
  (void)pdl;
  if (done && done[P.batch] == 0) return;  // every instance has finished refining
  int task = -1;
  SnInfo Cn;           // first child's metadata, prefetched (the continuation's next supernode)
  int cn_task = -1;
  for (;;) {
    if (task < 0) {
      int t = 0;
      if (lane == 0) t = pop_task(ctl, P.dn_s, P.n_dn_s, P.batch, Q, total);
      task = __shfl_sync(0xffffffffu, t, 0);
      if (task < 0) break;
    }
    const int s = task / P.batch, b = task % P.batch;
    const SnInfo I = (task == cn_task) ? Cn : P.sn[s];
    if (I.par >= 0 && task != cn_task) {  // a small root under a big (CTA) parent: take its hand-off
      int t = 0;
      if (lane == 0) {
        const SnInfo Ipar = P.sn[I.par];
        if (Ipar.big && (!Ipar.huge || P.solve_huge_cta)) {
          int* f = bflag + (long long)b * P.ns + I.par;
          while (ld_volatile(f) <= 0) { __nanosleep(64); }
          fence_acq_rel();
          atomicSub(f, 1);
        }
      }
      t = __shfl_sync(0xffffffffu, t, 0);
    }
    if (done && done[b]) {
      int t = 0;
      if (lane == 0) t = spawn_children(P, I, b, ctl, Q, false, total);
      task = __shfl_sync(0xffffffffu, t, 0);
      cn_task = -1;
      continue;
    }
    if (lane == 0) trace_stamp(P, 2, s, b, 0);
    const int r = I.r, w = I.w, rw = r * w;
    const double* L = Lx_all + (long long)b * P.nnzL_stored + I.Lp;
    double* Xp = Xp_all + (long long)b * P.n;
    const double* Y = Y_all + (long long)b * P.n;
    // every independent load first: child metadata, row indices / permutation, panel, y;
    // then the ancestors' x (dependent on the row indices)
    cn_task = -1;
    if (I.c0 < I.c1) { Cn = P.chinfo[I.c0]; cn_task = __ldg(P.sn_ch + I.c0) * P.batch + b; }
    const int q0 = lane, q1 = lane + 32;
    const int i0 = (q0 >= w && q0 < r) ? __ldg(P.sn_rows + I.rp0 + q0) : 0;
    const int i1 = (q1 >= w && q1 < r) ? __ldg(P.sn_rows + I.rp0 + q1) : 0;
    const int p0 = (q0 < w) ? __ldg(P.perm + I.f0 + q0) : 0;
    const int p1 = (q1 < w) ? __ldg(P.perm + I.f0 + q1) : 0;
    double lv[8];
#pragma unroll
    for (int u = 0; u < 8; u++) lv[u] = (lane + 32 * u < rw) ? __ldg(L + lane + 32 * u) : 0.0;
    double x0 = (q0 < w) ? ldcg(Y + I.f0 + q0) : 0.0, x1 = (q1 < w) ? ldcg(Y + I.f0 + q1) : 0.0;
    if (q0 >= w && q0 < r) x0 = ldcg(Xp + i0);
    if (q1 >= w && q1 < r) x1 = ldcg(Xp + i1);
#pragma unroll
    for (int u = 0; u < 8; u++) if (lane + 32 * u < rw) Pn[lane + 32 * u] = lv[u];
    if (rw > 256) copy_g2s<false>(Pn + 256, L + 256, rw - 256, lane, 32);
    if (q0 < r) xa[q0] = x0;
    if (q1 < r) xa[q1] = x1;
    for (int q = lane + 64; q < r; q += 32) xa[q] = (q < w) ? ldcg(Y + I.f0 + q) : ldcg(Xp + __ldg(P.sn_rows + I.rp0 + q));
    __syncwarp();
    if (w <= 128) {
      bwd_sweep_any(Pn, r, w, Dv_all + (long long)b * P.n + I.f0, xa, lane);
      __syncwarp();
    } else {
      for (int k = w - 1; k >= 0; k--) {
        double acc = 0.0;
        for (int i = k + 1 + lane; i < r; i += 32) acc = fma(Pn[k * r + i], xa[i], acc);
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        const double xk = (xa[k] - acc) / Pn[k * r + k];
        __syncwarp();
        if (lane == 0) xa[k] = xk;
        __syncwarp();
      }
    }
    double* xo = xout + (long long)b * xs;
    if (q0 < w) { Xp[I.f0 + q0] = xa[q0]; xo[p0] = xa[q0]; }
    if (q1 < w) { Xp[I.f0 + q1] = xa[q1]; xo[p1] = xa[q1]; }
    for (int q = lane + 64; q < w; q += 32) {
      Xp[I.f0 + q] = xa[q];
      xo[__ldg(P.perm + I.f0 + q)] = xa[q];
    }
    if (lane == 0) trace_stamp(P, 2, s, b, 1);
    __syncwarp();  // lanes' x writes are ordered before lane 0's release (spawn_children)
    int t = 0;
    if (lane == 0) t = spawn_children(P, I, b, ctl, Q, false, total);
    task = __shfl_sync(0xffffffffu, t, 0);
  }
  warp_exit(ctl, gridDim.x * KKT_WPB);
}

}  // namespace kkt
