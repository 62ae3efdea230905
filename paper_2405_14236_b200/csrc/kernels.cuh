// kernels.cuh -- sm_100a kernels of the condensed-KKT hot path (arXiv 2405.14236).
//
//   dweights_kernel   D_r in fp64 and double-double
//   condense_kernel   K = W + D_x + dw I + J^T D J, gather per K entry
//   factor_kernel     persistent multifrontal supernodal Cholesky           (§8(a) a2)
//   fwd_kernel/bwd_kernel  persistent supernodal triangular solves         (a3)
//   resid_rows/cols   double-double residual of the unassembled operator   (R8, a4)
//   CG kernels        HyKKT Schur-complement CG on G K_gamma^-1 G^T         (a5)
//
// Determinism: no floating-point atomics anywhere; every sum has a fixed order, so results
// are bitwise reproducible run to run and independent of the GPU count.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "devplan.h"

namespace kkt {

#define KKT_NT 128          // threads per CTA of the persistent kernels
#define KKT_NPART 64        // reduction partials per instance

// ------------------------------------------------------------------ memory-model helpers
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// producer data written earlier in the same launch by another CTA: bypass L1
__device__ __forceinline__ double ldcg(const double* p) { return __ldcg(p); }

__device__ __forceinline__ void atomic_max_pos(unsigned long long* a, double v) {
  // non-negative doubles order like their bit patterns; NaN maps above +inf
  unsigned long long b = isnan(v) ? 0x7ff8000000000000ULL : __double_as_longlong(v);
  atomicMax(a, b);
}

// ------------------------------------------------------------------ double-double
struct dd { double hi, lo; };
__device__ __forceinline__ dd two_sum(double a, double b) {
  double s = a + b, bb = s - a;
  return {s, (a - (s - bb)) + (b - bb)};
}
__device__ __forceinline__ dd quick_two_sum(double a, double b) {
  double s = a + b;
  return {s, b - (s - a)};
}
__device__ __forceinline__ dd two_prod(double a, double b) {
  double p = a * b;
  return {p, fma(a, b, -p)};
}
__device__ __forceinline__ dd dd_add(dd a, dd b) {
  dd s = two_sum(a.hi, b.hi), t = two_sum(a.lo, b.lo);
  s.lo += t.hi;
  s = quick_two_sum(s.hi, s.lo);
  s.lo += t.lo;
  return quick_two_sum(s.hi, s.lo);
}
__device__ __forceinline__ dd dd_mul(dd a, dd b) {
  dd p = two_prod(a.hi, b.hi);
  p.lo += a.hi * b.lo + a.lo * b.hi;
  return quick_two_sum(p.hi, p.lo);
}
__device__ __forceinline__ dd dd_mul_d(dd a, double b) {
  dd p = two_prod(a.hi, b);
  p.lo = fma(a.lo, b, p.lo);
  return quick_two_sum(p.hi, p.lo);
}
__device__ __forceinline__ dd dd_div(dd a, dd b) {
  double q1 = a.hi / b.hi;
  dd r = dd_add(a, dd_mul_d(b, -q1));
  double q2 = r.hi / b.hi;
  r = dd_add(r, dd_mul_d(b, -q2));
  double q3 = r.hi / b.hi;
  dd q = quick_two_sum(q1, q2);
  return dd_add(q, dd{q3, 0.0});
}

// =====================================================================================
// D_r: gamma for r < m_eq; else t = Sigma_s + dw, D = t / (1 + dc t).
// Written in fp64 (Dh, used by the condensation) and as a double-double (Dh + Dl, used by
// the refinement residual, R8).  An explicit override D[m] replaces every row weight.
// =====================================================================================
__global__ void dweights_kernel(DevPlan P, const double* __restrict__ Ss, const double* __restrict__ Dov,
                                double dw, double dc, double gamma, double* Dh, double* Dl) {
  long long total = (long long)P.batch * P.m;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    int b = (int)(idx / P.m), r = (int)(idx % P.m);
    dd D;
    if (Dov) {
      D = {Dov[idx], 0.0};
    } else if (r < P.m_eq) {
      D = {gamma, 0.0};
    } else {
      dd t = two_sum(Ss[(long long)b * (P.m - P.m_eq) + (r - P.m_eq)], dw);
      if (dc != 0.0) {
        dd den = dd_add(dd{1.0, 0.0}, dd_mul_d(t, dc));
        D = dd_div(t, den);
      } else {
        D = t;
      }
    }
    Dh[idx] = D.hi;
    Dl[idx] = D.lo;
  }
}

// =====================================================================================
// Condensation: one thread per K entry (internal lower-CSC order), gather form:
//   K_k = W[kw] + [diag](Sigma_x + dw) + sum_q D[row(pa_q)] J[pa_q] J[pb_q]
// Fixed summation order (W, diagonal, then J rows ascending) -- deterministic, no atomics.
// =====================================================================================
__global__ void __launch_bounds__(256) condense_kernel(DevPlan P, const double* __restrict__ Wv,
                                                       const double* __restrict__ Jv,
                                                       const double* __restrict__ Sx,
                                                       const double* __restrict__ Dh, double dw,
                                                       double* __restrict__ Kv) {
  long long total = (long long)P.batch * P.nnzK;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    int b = (int)(idx / P.nnzK), k = (int)(idx % P.nnzK);
    const double* W = Wv + (long long)b * P.nnzW;
    const double* J = Jv + (long long)b * P.nnzJ;
    const double* D = Dh + (long long)b * P.m;
    int w = __ldg(P.kw + k), dg = __ldg(P.kdiag + k);
    double v = (w >= 0) ? __ldg(W + w) : 0.0;
    if (dg >= 0) v += __ldg(Sx + (long long)b * P.n + dg) + dw;
    int q0 = __ldg(P.pptr + k), q1 = __ldg(P.pptr + k + 1);
    for (int q = q0; q < q1; q++) {
      int a = __ldg(P.pa + q), c = __ldg(P.pb + q);
      v = fma(__ldg(D + __ldg(P.jrow + a)) * __ldg(J + a), __ldg(J + c), v);
    }
    Kv[idx] = v;
  }
}

// =====================================================================================
// Persistent-kernel task protocol.  Tasks are (supernode in level order, instance) pairs,
// dequeued in increasing order with a global ticket; a task's dependencies always carry
// smaller ticket numbers and are therefore held by running CTAs -> no deadlock for any grid
// size.  Dependency counters are reset by their consumer; the ticket is reset by the last
// CTA to exit (ctl[0] = ticket, ctl[1] = exit count).
// =====================================================================================
__device__ __forceinline__ int next_task(int* ctl, int* s_task) {
  __syncthreads();
  if (threadIdx.x == 0) *s_task = atomicAdd(ctl, 1);
  __syncthreads();
  return *s_task;
}
__device__ __forceinline__ void persistent_exit(int* ctl) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    int e = atomicAdd(ctl + 1, 1);
    if (e == (int)gridDim.x - 1) {
      ctl[0] = 0;
      ctl[1] = 0;
      __threadfence();
    }
  }
}

__device__ __forceinline__ long long upk(int i, int j, int R) {  // packed lower col-major
  return (long long)j * R - (long long)j * (j - 1) / 2 + (i - j);
}

// ---------------------------------------------------------------------------------
// Dense partial factorisation of a front held as [panel F (r x w, ld r) | update U (packed,
// R = r - w)].  F and U are either shared memory or the global L / update buffers.
//   F <- [L11; L21] with L11 L11^T = F11, L21 = F21 L11^-T   (unblocked right-looking)
//   U <- U - L21 L21^T                                       (SYRK into the update matrix)
// Returns (through *fail) the first non-positive pivot column or -1.
// ---------------------------------------------------------------------------------
__device__ void front_factor(double* F, double* U, int r, int w, int* s_fail) {
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int k = 0; k < w; k++) {
    double* Fk = F + (long long)k * r;
    if (tid == 0) {
      double d = Fk[k];
      if (!(d > 0.0) || !isfinite(d)) {
        if (*s_fail < 0) *s_fail = k;
        d = __longlong_as_double(0x7ff8000000000000LL);  // NaN propagates, never hangs
      }
      Fk[k] = sqrt(d);
    }
    __syncthreads();
    double inv = 1.0 / Fk[k];
    for (int i = k + 1 + tid; i < r; i += nt) Fk[i] *= inv;
    __syncthreads();
    // rank-1 update of the remaining panel columns j in (k, w)
    int cols = w - k - 1;
    if (cols > 0) {
      for (int j = k + 1; j < w; j++) {
        double ljk = Fk[j];
        double* Fj = F + (long long)j * r;
        for (int i = j + tid; i < r; i += nt) Fj[i] = fma(-Fk[i], ljk, Fj[i]);
      }
      __syncthreads();
    }
  }
  // SYRK: U(i,j) -= sum_k L21(i,k) L21(j,k),  i >= j, packed column-major; warps over j
  const int R = r - w;
  if (R > 0 && U) {
    const int lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
    for (int j = warp; j < R; j += nw) {
      const long long cs = upk(j, j, R);
      const double* Fj = F + w + j;
      for (int i = j + lane; i < R; i += 32) {
        double acc = U[cs + (i - j)];
        const double* Fi = F + w + i;
        for (int k = 0; k < w; k++) acc = fma(-Fi[(long long)k * r], Fj[(long long)k * r], acc);
        U[cs + (i - j)] = acc;
      }
    }
  }
  __syncthreads();
}

// =====================================================================================
// Multifrontal supernodal Cholesky, persistent.  Task (s, b):
//   wait until all children of s finished;  assemble the front: K columns of s scattered
//   via kpos, then each child's update matrix extend-added through its relative-index map
//   (children in fixed order -> deterministic);  dense partial factorisation;  write the
//   panel to L and the update matrix to the update buffer;  signal the parent.
// Fronts that fit `smem_cap` doubles are factorised in shared memory, larger ones in place
// in global memory (L2-resident).
// =====================================================================================
__global__ void __launch_bounds__(KKT_NT) factor_kernel(DevPlan P, const double* __restrict__ Kv_all,
                                                        double* Lx_all, double* U_all, int* cnt_all,
                                                        int* ctl, int* fail_all, long long smem_cap) {
  extern __shared__ double sm[];
  __shared__ int s_task, s_fail;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int total = P.ns * P.batch;
  for (;;) {
    int t = next_task(ctl, &s_task);
    if (t >= total) break;
    const int oi = t / P.batch, b = t % P.batch;
    const int s = __ldg(P.order + oi);
    const int f0 = __ldg(P.sn_first + s), w = __ldg(P.sn_first + s + 1) - f0;
    const int rp0 = __ldg(P.sn_rp + s), r = __ldg(P.sn_rp + s + 1) - rp0, R = r - w;
    const int par = __ldg(P.sn_parent + s);
    const int c0 = __ldg(P.sn_cp + s), c1 = __ldg(P.sn_cp + s + 1);
    int* cnt = cnt_all + (long long)b * P.ns;
    double* Lx = Lx_all + (long long)b * P.nnzL_stored;
    double* Ub = U_all + (long long)b * P.update_doubles;
    const double* Kv = Kv_all + (long long)b * P.nnzK;
    if (tid == 0) {
      s_fail = -1;
      if (c1 > c0) {
        while (ld_acquire(cnt + s) < c1 - c0) __nanosleep(20);
        cnt[s] = 0;  // consumer resets
      }
    }
    __syncthreads();
    const long long pw = (long long)r * w;
    const long long usz = (par >= 0) ? (long long)R * (R + 1) / 2 : 0;
    const bool in_smem = (pw + usz) <= smem_cap;
    double* F = in_smem ? sm : Lx + __ldg(P.sn_Lp + s);
    double* U = in_smem ? sm + pw : (usz ? Ub + __ldg(P.sn_Up + s) : nullptr);
    // ---- assemble ----
    for (long long q = tid; q < pw; q += nt) F[q] = 0.0;
    for (long long q = tid; q < usz; q += nt) U[q] = 0.0;
    __syncthreads();
    {
      int k0 = __ldg(P.Kp + f0), k1 = __ldg(P.Kp + f0 + w);
      for (int k = k0 + tid; k < k1; k += nt) F[__ldg(P.kpos + k)] = __ldg(Kv + k);
    }
    __syncthreads();
    for (int ci = c0; ci < c1; ci++) {
      const int c = __ldg(P.sn_ch + ci);
      const int cf = __ldg(P.sn_first + c), cw = __ldg(P.sn_first + c + 1) - cf;
      const int crp = __ldg(P.sn_rp + c), Rc = __ldg(P.sn_rp + c + 1) - crp - cw;
      const int* rel = P.sn_rel + crp + cw;
      const double* Uc = Ub + __ldg(P.sn_Up + c);
      // warps over child columns jc, lanes over rows ic >= jc
      const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
      for (int jc = warp; jc < Rc; jc += nw) {
        const int pj = __ldg(rel + jc);
        const long long cs = upk(jc, jc, Rc);
        for (int ic = jc + lane; ic < Rc; ic += 32) {
          const int pi = __ldg(rel + ic);
          const double v = ldcg(Uc + cs + (ic - jc));
          if (pj < w) F[(long long)pj * r + pi] += v;
          else U[upk(pi - w, pj - w, R)] += v;
        }
      }
      __syncthreads();
    }
    // ---- factor ----
    front_factor(F, U, r, w, &s_fail);
    // ---- write back ----
    if (in_smem) {
      double* Lg = Lx + __ldg(P.sn_Lp + s);
      for (long long q = tid; q < pw; q += nt) Lg[q] = F[q];
      if (usz) {
        double* Ug = Ub + __ldg(P.sn_Up + s);
        for (long long q = tid; q < usz; q += nt) Ug[q] = U[q];
      }
    }
    if (tid == 0 && s_fail >= 0) atomicMin(fail_all, f0 + s_fail);
    __threadfence();
    __syncthreads();
    if (tid == 0 && par >= 0) red_release_add(cnt + par, 1);
  }
  persistent_exit(ctl);
}

// =====================================================================================
// Forward solve L y = P b, multifrontal form (bottom-up, persistent).  Task (s, b):
//   v[0:w) = b[perm[f0 + t]], v[w:r) = 0;  v += children's update vectors (relative map);
//   L11 y = v[0:w) (warp 0, from shared memory);  u_s = v[w:r) - L21 y;  signal parent.
// `done` (per instance, may be NULL) skips finished instances (refinement early exit).
// =====================================================================================
__global__ void __launch_bounds__(KKT_NT) fwd_kernel(DevPlan P, const double* __restrict__ Lx_all,
                                                     const double* __restrict__ rhs, long long rhs_stride,
                                                     double* Y_all, double* uv_all, int* cnt_all,
                                                     int* ctl, const int* __restrict__ done) {
  extern __shared__ double sm[];
  __shared__ int s_task;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int total = P.ns * P.batch;
  double* v = sm;                         // [max_front]
  double* L11 = sm + P.max_front;         // [64 * 64] staging for w <= 64
  for (;;) {
    int t = next_task(ctl, &s_task);
    if (t >= total) break;
    const int oi = t / P.batch, b = t % P.batch;
    if (done && done[b]) continue;
    const int s = __ldg(P.order + oi);
    const int f0 = __ldg(P.sn_first + s), w = __ldg(P.sn_first + s + 1) - f0;
    const int rp0 = __ldg(P.sn_rp + s), r = __ldg(P.sn_rp + s + 1) - rp0, R = r - w;
    const int par = __ldg(P.sn_parent + s);
    const int c0 = __ldg(P.sn_cp + s), c1 = __ldg(P.sn_cp + s + 1);
    int* cnt = cnt_all + (long long)b * P.ns;
    const double* L = Lx_all + (long long)b * P.nnzL_stored + __ldg(P.sn_Lp + s);
    double* uv = uv_all + (long long)b * P.uvec_doubles;
    const double* bb = rhs + (long long)b * rhs_stride;
    if (tid == 0 && c1 > c0) {
      while (ld_acquire(cnt + s) < c1 - c0) __nanosleep(20);
      cnt[s] = 0;
    }
    for (int q = tid; q < r; q += nt) v[q] = (q < w) ? bb[__ldg(P.perm + f0 + q)] : 0.0;
    const bool stage = (w <= 64);
    if (stage)
      for (int q = tid; q < w * w; q += nt) {
        int k = q / w, i = q % w;
        L11[q] = (i >= k) ? __ldg(L + (long long)k * r + i) : 0.0;
      }
    __syncthreads();
    for (int ci = c0; ci < c1; ci++) {
      const int c = __ldg(P.sn_ch + ci);
      const int cw = __ldg(P.sn_first + c + 1) - __ldg(P.sn_first + c);
      const int crp = __ldg(P.sn_rp + c), Rc = __ldg(P.sn_rp + c + 1) - crp - cw;
      const int* rel = P.sn_rel + crp + cw;
      const double* u = uv + __ldg(P.sn_uvp + c);
      for (int q = tid; q < Rc; q += nt) v[__ldg(rel + q)] += ldcg(u + q);
      __syncthreads();
    }
    // L11 y = v[0:w)
    if (stage) {
      if (warp == 0) {
        for (int k = 0; k < w; k++) {
          double yk = v[k] / L11[k * w + k];
          __syncwarp();
          if (lane == 0) v[k] = yk;
          for (int i = k + 1 + lane; i < w; i += 32) v[i] = fma(-L11[k * w + i], yk, v[i]);
          __syncwarp();
        }
      }
    } else {
      for (int k = 0; k < w; k++) {
        double yk = v[k] / __ldg(L + (long long)k * r + k);
        __syncthreads();
        if (tid == 0) v[k] = yk;
        for (int i = k + 1 + tid; i < w; i += nt) v[i] = fma(-__ldg(L + (long long)k * r + i), yk, v[i]);
        __syncthreads();
      }
    }
    __syncthreads();
    // u_s = v[w:r) - L21 y
    double* Y = Y_all + (long long)b * P.n;
    for (int q = tid; q < w; q += nt) Y[f0 + q] = v[q];
    if (par >= 0) {
      double* us = uv + __ldg(P.sn_uvp + s);
      for (int i = tid; i < R; i += nt) {
        double acc = v[w + i];
        const double* Li = L + w + i;
        int k = 0;
        for (; k + 4 <= w; k += 4) {
          double l0 = __ldg(Li + (long long)k * r), l1 = __ldg(Li + (long long)(k + 1) * r);
          double l2 = __ldg(Li + (long long)(k + 2) * r), l3 = __ldg(Li + (long long)(k + 3) * r);
          acc = fma(-l0, v[k], acc); acc = fma(-l1, v[k + 1], acc);
          acc = fma(-l2, v[k + 2], acc); acc = fma(-l3, v[k + 3], acc);
        }
        for (; k < w; k++) acc = fma(-__ldg(Li + (long long)k * r), v[k], acc);
        us[i] = acc;
      }
    }
    __threadfence();
    __syncthreads();
    if (tid == 0 && par >= 0) red_release_add(cnt + par, 1);
  }
  persistent_exit(ctl);
}

// =====================================================================================
// Backward solve L^T z = y, x = P^T z (top-down, persistent; tasks in reverse level order).
//   wait for the parent;  xa = x[R_s[w:r)] (ancestors, already final);
//   z = y_s - L21^T xa (warp per column, fixed reduction tree);  L11^T x_s = z (warp 0);
//   write x_s (internal and original order);  release every child.
// =====================================================================================
__global__ void __launch_bounds__(KKT_NT) bwd_kernel(DevPlan P, const double* __restrict__ Lx_all,
                                                     const double* __restrict__ Y_all, double* Xp_all,
                                                     double* xout, long long xout_stride, int* flag_all,
                                                     int* ctl, const int* __restrict__ done) {
  extern __shared__ double sm[];
  __shared__ int s_task;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  const int total = P.ns * P.batch;
  double* xa = sm;                   // [max_front]
  double* z = sm + P.max_front;      // [w] (<= max_front)
  double* L11 = z + P.max_front;     // [64*64]
  for (;;) {
    int t = next_task(ctl, &s_task);
    if (t >= total) break;
    const int oi = P.ns - 1 - t / P.batch, b = t % P.batch;
    if (done && done[b]) continue;
    const int s = __ldg(P.order + oi);
    const int f0 = __ldg(P.sn_first + s), w = __ldg(P.sn_first + s + 1) - f0;
    const int rp0 = __ldg(P.sn_rp + s), r = __ldg(P.sn_rp + s + 1) - rp0, R = r - w;
    const int par = __ldg(P.sn_parent + s);
    const int c0 = __ldg(P.sn_cp + s), c1 = __ldg(P.sn_cp + s + 1);
    int* flag = flag_all + (long long)b * P.ns;
    const double* L = Lx_all + (long long)b * P.nnzL_stored + __ldg(P.sn_Lp + s);
    double* Xp = Xp_all + (long long)b * P.n;
    const double* Y = Y_all + (long long)b * P.n;
    if (tid == 0 && par >= 0) {
      while (ld_acquire(flag + s) == 0) __nanosleep(20);
      flag[s] = 0;
    }
    __syncthreads();
    for (int q = tid; q < R; q += nt) xa[q] = ldcg(Xp + __ldg(P.sn_rows + rp0 + w + q));
    const bool stage = (w <= 64);
    if (stage)
      for (int q = tid; q < w * w; q += nt) {
        int k = q / w, i = q % w;
        L11[q] = (i >= k) ? __ldg(L + (long long)k * r + i) : 0.0;
      }
    __syncthreads();
    for (int k = warp; k < w; k += nw) {
      const double* Lk = L + (long long)k * r + w;
      double acc = 0.0;
      for (int i = lane; i < R; i += 32) acc = fma(__ldg(Lk + i), xa[i], acc);
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) z[k] = ldcg(Y + f0 + k) - acc;
    }
    __syncthreads();
    if (stage) {
      if (warp == 0) {
        for (int k = w - 1; k >= 0; k--) {
          double xk = z[k] / L11[k * w + k];
          __syncwarp();
          if (lane == 0) z[k] = xk;
          for (int i = lane; i < k; i += 32) z[i] = fma(-L11[i * w + k], xk, z[i]);
          __syncwarp();
        }
      }
    } else {
      for (int k = w - 1; k >= 0; k--) {
        double xk = z[k] / __ldg(L + (long long)k * r + k);
        __syncthreads();
        if (tid == 0) z[k] = xk;
        for (int i = tid; i < k; i += nt) z[i] = fma(-__ldg(L + (long long)i * r + k), xk, z[i]);
        __syncthreads();
      }
    }
    __syncthreads();
    double* xo = xout + (long long)b * xout_stride;
    for (int q = tid; q < w; q += nt) {
      Xp[f0 + q] = z[q];
      xo[__ldg(P.perm + f0 + q)] = z[q];
    }
    __threadfence();
    __syncthreads();
    if (tid == 0)
      for (int ci = c0; ci < c1; ci++) st_release(flag + __ldg(P.sn_ch + ci), 1);
  }
  persistent_exit(ctl);
}

// =====================================================================================
// Double-double residual of the unassembled operator (R8), two passes.
//   rows:  t_r = D_r (J_r x)  (dd)          [mode 1 (saddle): rows r < m_eq carry t_r = dy_r
//                                             and res2_r = rbar2_r - J_r x]
//          a_r = |D_r| (|J_r| |x|)           (fp64, for the componentwise denominator)
//   cols:  y_i = (W x)_i + (Sx_i + dw) x_i + sum_r J_ri t_r   (dd);  res_i = b_i - y_i
//          omega = max_i |res_i| / (|W||x| + |Sx+dw||x| + |J|^T a + |b|)_i
// =====================================================================================
__global__ void resid_rows_kernel(DevPlan P, const double* __restrict__ Jv, const double* __restrict__ Dh,
                                  const double* __restrict__ Dl, const double* __restrict__ x,
                                  long long xs, int mode, const double* __restrict__ dy,
                                  const double* __restrict__ rb2, double* res2, double2* T,
                                  double* A, const int* __restrict__ done) {
  long long total = (long long)P.batch * P.m;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    int b = (int)(idx / P.m), r = (int)(idx % P.m);
    if (done && done[b]) continue;
    const double* J = Jv + (long long)b * P.nnzJ;
    const double* xb = x + (long long)b * xs;
    int p0 = P.Jrp[r], p1 = P.Jrp[r + 1];
    dd acc = {0.0, 0.0};
    double aa = 0.0;
    for (int p = p0; p < p1; p++) {
      double jv = J[p], xv = xb[P.Jci[p]];
      acc = dd_add(acc, two_prod(jv, xv));
      aa = fma(fabs(jv), fabs(xv), aa);
    }
    if (mode == 1 && r < P.m_eq) {
      T[idx] = make_double2(dy[(long long)b * P.m_eq + r], 0.0);
      A[idx] = fabs(dy[(long long)b * P.m_eq + r]);
      dd rr = dd_add(dd{rb2[(long long)b * P.m_eq + r], 0.0}, dd{-acc.hi, -acc.lo});
      res2[(long long)b * P.m_eq + r] = rr.hi + rr.lo;
    } else {
      dd D = {Dh[idx], Dl[idx]};
      dd t = dd_mul(acc, D);
      T[idx] = make_double2(t.hi, t.lo);
      A[idx] = fabs(D.hi) * aa;
    }
  }
}

__global__ void resid_cols_kernel(DevPlan P, const double* __restrict__ Wv, const double* __restrict__ Jv,
                                  const double* __restrict__ Sx, double dw, const double* __restrict__ x,
                                  long long xs, const double* __restrict__ rhs, long long rs,
                                  const double2* __restrict__ T, const double* __restrict__ A,
                                  double* res, unsigned long long* omega, const int* __restrict__ done) {
  long long total = (long long)P.batch * P.n;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    int b = (int)(idx / P.n), i = (int)(idx % P.n);
    if (done && done[b]) continue;
    const double* W = Wv + (long long)b * P.nnzW;
    const double* J = Jv + (long long)b * P.nnzJ;
    const double* xb = x + (long long)b * xs;
    const double2* Tb = T + (long long)b * P.m;
    const double* Ab = A + (long long)b * P.m;
    double xi = xb[i];
    dd s = two_sum(Sx[idx], dw);
    dd y = dd_mul_d(s, xi);
    double den = fabs(s.hi) * fabs(xi);
    for (int p = P.Wf_p[i]; p < P.Wf_p[i + 1]; p++) {
      double wv = W[P.Wf_k[p]], xv = xb[P.Wf_c[p]];
      y = dd_add(y, two_prod(wv, xv));
      den = fma(fabs(wv), fabs(xv), den);
    }
    for (int p = P.Jt_p[i]; p < P.Jt_p[i + 1]; p++) {
      int r = P.Jt_r[p];
      double jv = J[P.Jt_k[p]];
      double2 t = Tb[r];
      y = dd_add(y, dd_mul_d(dd{t.x, t.y}, jv));
      den = fma(fabs(jv), Ab[r], den);
    }
    double bi = rhs[(long long)b * rs + i];
    dd rr = dd_add(dd{bi, 0.0}, dd{-y.hi, -y.lo});
    double rv = rr.hi + rr.lo;
    res[idx] = rv;
    den += fabs(bi);
    if (omega) {
      double om = (den > 0.0) ? fabs(rv) / den : (rv != 0.0 ? INFINITY : 0.0);
      atomic_max_pos(omega + b, om);
    }
  }
}

}  // namespace kkt
