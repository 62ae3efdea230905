// cg_kernels.cuh -- refinement control and HyKKT CG kernels.
// All reductions are deterministic: fixed per-block trees, partials summed in block order by
// the last-arriving block (no floating-point atomics).
#pragma once
#include "common.cuh"

namespace kkt {

__device__ __forceinline__ double bits2d(unsigned long long b) { return __longlong_as_double((long long)b); }

// ---------------------------------------------------------------- refinement control
__global__ void refine_init_kernel(int batch, DevCtrl C) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b == 0) { C.done[batch] = batch; *C.sweep = 0; }  // done[batch]: instances still refining
  if (b >= batch) return;
  C.done[b] = 0; C.refine_iters[b] = 0; C.grow[b] = 0;
  C.omega[b] = 0ULL; C.omega_prev[b] = INFINITY; C.omega_last[b] = 0.0;
  C.dxn[b] = 0ULL; C.xn[b] = 0ULL; C.dxprev[b] = INFINITY;
}

// Stopping rules (R9): omega <= tol (only if tol > 0); the correction just applied was
// negligible, ||dx_k|| <= 1e-14 ||x||; geometric convergence over the last two corrections
// (rho = ||dx_k|| / ||dx_k-1|| < 1/2) predicts rho ||dx_k|| / (1 - rho) <= 1e-14 ||x||; omega grew
// in two consecutive sweeps; max_refine corrections applied (the last check only measures).
__global__ void refine_decide_kernel(int batch, DevCtrl C, double tol, int max_refine) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  const int sweep = *C.sweep;
  const bool last = sweep >= max_refine;
  if (C.done[b]) return;
  double om = bits2d(C.omega[b]);
  C.omega[b] = 0ULL;
  C.omega_last[b] = om;
  bool stop = last || isnan(om) || (tol > 0.0 && om <= tol);
  if (sweep > 0) {
    double dxn = bits2d(C.dxn[b]), xn = bits2d(C.xn[b]);
    C.dxn[b] = 0ULL; C.xn[b] = 0ULL;
    // the last correction was negligible, or (geometric convergence, rate rho = ||dx_k|| /
    // ||dx_k-1|| < 1/2) the next one would be: rho ||dx_k|| / (1 - rho) <= 1e-14 ||x||   (R9)
    // the rate test needs two corrections: after the first one dxprev is still +inf (rho = 0
    // would stop every instance after one correction whatever its convergence state)
    const bool have_prev = isfinite(C.dxprev[b]);
    const double rho = have_prev ? dxn / C.dxprev[b] : 1.0;
    C.dxprev[b] = dxn;
    if (dxn <= 1e-14 * xn) stop = true;
    if (have_prev && rho < 0.5 && rho * dxn / (1.0 - rho) <= 1e-14 * xn) stop = true;
    if (om > C.omega_prev[b]) { if (++C.grow[b] >= 2) stop = true; }
    else C.grow[b] = 0;
  }
  C.omega_prev[b] = om;
  if (stop) {
    C.done[b] = 1;
    atomicSub(C.done + batch, 1);
  } else {
    C.refine_iters[b] += 1;
  }
}

// End of a sweep: advance the sweep counter and, inside the solve graph, set the condition of
// the refinement WHILE node (another sweep iff some instance is still refining).
__global__ void refine_cond_kernel(int batch, DevCtrl C, cudaGraphConditionalHandle handle, int use_handle) {
  *C.sweep += 1;
  if (use_handle) cudaGraphSetConditional(handle, C.done[batch] > 0 ? 1u : 0u);
}

// x += dx for the instances still refining; ||dx||_inf, ||x||_inf by block reductions.
// grid (gx, batch): the instance is block-uniform.
__global__ void refine_update_kernel(int batch, int n, double* x, const double* __restrict__ dx, DevCtrl C) {
  const int b = blockIdx.y;
  if (C.done[batch] == 0 || C.done[b]) return;  // block-uniform exits
  double mdx = 0.0, mx = 0.0;
  const long long o = (long long)b * n;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double d = dx[o + i], xv = x[o + i] + d;
    x[o + i] = xv;
    mdx = (isnan(d) || isnan(mdx)) ? NAN : fmax(mdx, fabs(d));  // NaN propagates
    mx = (isnan(xv) || isnan(mx)) ? NAN : fmax(mx, fabs(xv));
  }
  block_max_atomic(C.dxn + b, mdx);
  block_max_atomic(C.xn + b, mx);
}

// ---------------------------------------------------------------- G^T and G products
// out_i = base_i + alpha * sum_{r < m_eq} J_ri y_r   (the G^T prefix of every J^T column)
__global__ void gt_kernel(DevPlan P, const double* __restrict__ Jv, const double* __restrict__ y,
                          double alpha, const double* __restrict__ base, double* out,
                          const int* __restrict__ skip) {
  long long total = (long long)P.batch * P.n;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    int b = (int)(idx / P.n), i = (int)(idx % P.n);
    if (skip && skip[b]) continue;
    const double* J = Jv + (long long)b * P.nnzJ;
    const double* yb = y + (long long)b * P.m_eq;
    double acc = 0.0;
    int p = P.Jt_p[i];
    const int pe = P.Gt_end[i];
    for (; p + 4 <= pe; p += 4) {  // four terms' loads in flight, the same fma order
      const int k0 = P.Jt_k[p], k1 = P.Jt_k[p + 1], k2 = P.Jt_k[p + 2], k3 = P.Jt_k[p + 3];
      const int r0 = P.Jt_r[p], r1 = P.Jt_r[p + 1], r2 = P.Jt_r[p + 2], r3 = P.Jt_r[p + 3];
      const double j0 = J[k0], j1 = J[k1], j2 = J[k2], j3 = J[k3];
      const double y0 = yb[r0], y1 = yb[r1], y2 = yb[r2], y3 = yb[r3];
      acc = fma(j0, y0, acc); acc = fma(j1, y1, acc); acc = fma(j2, y2, acc); acc = fma(j3, y3, acc);
    }
    for (; p < pe; p++) acc = fma(J[P.Jt_k[p]], yb[P.Jt_r[p]], acc);
    out[idx] = base ? fma(alpha, acc, base[idx]) : alpha * acc;
  }
}

// Block tree reduction (fixed order) of one double per thread; result valid in thread 0.
__device__ __forceinline__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int k = 0; k < nw; k++) s += red[k];
  return s;
}

// Ordered sums over the KKT_NPART blocks of instance b of NV values per block: returns true in
// thread 0 of the last-arriving block, with sum[v] = partials summed in block order (no
// floating-point atomics: deterministic).
template <int NV>
__device__ __forceinline__ bool finish_dots(DevCtrl C, int b, const double* part, double* sum) {
  __shared__ bool last;
  if (threadIdx.x == 0) {
    for (int v = 0; v < NV; v++) C.partial[((long long)b * 2 + v) * KKT_NPART + blockIdx.x] = part[v];
    __threadfence();
    unsigned int a = atomicAdd(C.part_cnt + b, 1u);
    last = (a == KKT_NPART - 1);
    if (last) {
      __threadfence();
      for (int v = 0; v < NV; v++) {
        double s = 0.0;
        for (int k = 0; k < KKT_NPART; k++) s += __ldcg(C.partial + ((long long)b * 2 + v) * KKT_NPART + k);
        sum[v] = s;
      }
      C.part_cnt[b] = 0u;
    }
  }
  __syncthreads();
  return last && threadIdx.x == 0;
}

// Krylov state of one HyKKT pass, per instance: cg_done[b] = 0 running, 1 converged, 2 maxit
// reached, 3 skipped (outer refinement already finished); cg_done[batch] = instances running
// (the solve kernels and the graph WHILE node test it).
__device__ __forceinline__ void cg_mark_done(DevCtrl C, int batch, int b, int code) {
  C.cg_done[b] = code;
  atomicSub(C.cg_done + batch, 1);
}

// Start of a pass: instances whose outer refinement finished are skipped for the whole pass.
__global__ void cg_init_kernel(int batch, DevCtrl C, int use_odone) {
  __shared__ int cnt;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  for (int b = threadIdx.x; b < batch; b += blockDim.x) {
    const int skip = use_odone && C.odone[b];
    C.cg_done[b] = skip ? 3 : 0;
    C.cg_iters[b] = 0;
    if (!skip) atomicAdd(&cnt, 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) C.cg_done[batch] = cnt;
}

// mode 0 (start):       r = G z - rbar2 ; p = r ; dy = 0 ; rr = rr0 = r.r
// mode 1 (CG step):     q = G z ; alpha = rr / p.q
// mode 2 (CR start):    s = q = G z (= S r0) ; rs = r.s ; qq = s.s ; alpha = rs / qq
// mode 3 (CR step):     s = G z (= S r) ; beta = r.s / rs ; rs = r.s
// grid (KKT_NPART, batch), KKT_CGT threads
__global__ void __launch_bounds__(KKT_CGT) g_kernel(DevPlan P, const double* __restrict__ Jv, const double* __restrict__ z,
                         const double* __restrict__ sub, double* out, double* p, double* dy,
                         DevCtrl C, int mode, int first, double* q) {
  __shared__ double red[32];
  const int b = blockIdx.y;
  if (C.cg_done[b]) return;   // converged, or skipped for this pass (block-uniform)
  const int me = P.m_eq;
  const double* J = Jv + (long long)b * P.nnzJ;
  const double* zb = z + (long long)b * P.n;
  double part[2] = {0.0, 0.0};
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < me; r += KKT_NPART * blockDim.x) {
    double acc = 0.0;
    int t = P.Jrp[r];
    const int te = P.Jrp[r + 1];
    for (; t + 4 <= te; t += 4) {  // four terms' loads in flight, the same fma order
      const int c0 = P.Jci[t], c1 = P.Jci[t + 1], c2 = P.Jci[t + 2], c3 = P.Jci[t + 3];
      const double j0 = J[t], j1 = J[t + 1], j2 = J[t + 2], j3 = J[t + 3];
      const double z0 = zb[c0], z1 = zb[c1], z2 = zb[c2], z3 = zb[c3];
      acc = fma(j0, z0, acc); acc = fma(j1, z1, acc); acc = fma(j2, z2, acc); acc = fma(j3, z3, acc);
    }
    for (; t < te; t++) acc = fma(J[t], zb[P.Jci[t]], acc);
    const long long o = (long long)b * me + r;
    if (mode == 0) {
      acc -= sub[o];
      out[o] = acc;
      p[o] = acc;
      dy[o] = 0.0;
      part[0] = fma(acc, acc, part[0]);
    } else if (mode == 1) {
      out[o] = acc;
      part[0] = fma(p[o], acc, part[0]);
    } else if (mode == 2) {        // out = s, q = s ; p (= r) holds r0
      out[o] = acc;
      q[o] = acc;
      part[0] = fma(p[o], acc, part[0]);
      part[1] = fma(acc, acc, part[1]);
    } else {                       // mode 3: out = s ; sub = r
      out[o] = acc;
      part[0] = fma(sub[o], acc, part[0]);
    }
  }
  double sv[2];
  sv[0] = block_sum(part[0], red);
  if (mode == 2) sv[1] = block_sum(part[1], red);
  double tot[2];
  const bool last = (mode == 2) ? finish_dots<2>(C, b, sv, tot) : finish_dots<1>(C, b, sv, tot);
  if (last) {
    if (mode == 0) {
      C.rr[b] = tot[0]; C.rr0[b] = tot[0];
      if (first) C.rr0_first[b] = tot[0];
      if (tot[0] == 0.0) cg_mark_done(C, P.batch, b, 1);
    } else if (mode == 1) {
      C.pq[b] = tot[0];
      C.alpha[b] = C.rr[b] / tot[0];
    } else if (mode == 2) {
      C.rs[b] = tot[0]; C.qq[b] = tot[1];
      C.alpha[b] = tot[0] / tot[1];
    } else {
      C.beta[b] = tot[0] / C.rs[b];
      C.rs[b] = tot[0];
    }
  }
}

// dy += alpha p ; r -= alpha q ; rr_new = r.r ; convergence ||r|| <= rtol ||r0|| (R10);
// maxit iterations -> stop (reported as KKT_ERR_NOT_CONVERGED by cg_finish_kernel).
// Correction passes of the outer refinement (first == 0) stop at the absolute level
// rtol ||r0 of the first pass|| -- the correction only has to be accurate relative to the
// solution it corrects, not relative to its own (small) right-hand side.
__global__ void __launch_bounds__(KKT_CGT) cg_update_kernel(int batch, int me, double* dy, double* r, const double* __restrict__ p,
                                 const double* __restrict__ q, DevCtrl C, double rtol, int* status, int first,
                                 int maxit) {
  __shared__ double red[32];
  const int b = blockIdx.y;
  if (C.cg_done[b]) return;
  const double a = C.alpha[b];
  double part = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < me; i += KKT_NPART * blockDim.x) {
    long long o = (long long)b * me + i;
    dy[o] = fma(a, p[o], dy[o]);
    double rv = fma(-a, q[o], r[o]);
    r[o] = rv;
    part = fma(rv, rv, part);
  }
  double s = block_sum(part, red), tot;
  if (finish_dots<1>(C, b, &s, &tot)) {
    const int it = (C.cg_iters[b] += 1);
    if (!isfinite(tot) || !isfinite(a)) {
      cg_mark_done(C, batch, b, 1);
      atomicCAS(status, 0, 5 /* KKT_ERR_NONFINITE */);
    } else if (sqrt(tot) <= rtol * sqrt(first ? C.rr0[b] : fmax(C.rr0[b], C.rr0_first[b]))) {
      cg_mark_done(C, batch, b, 1);
    } else if (it >= maxit) {
      cg_mark_done(C, batch, b, 2);
    }
    C.beta[b] = tot / C.rr[b];   // CG's beta (CR overwrites it in g mode 3)
    C.rr[b] = tot;
  }
}

// CG: p = r + beta p
__global__ void cg_p_kernel(int batch, int me, double* p, const double* __restrict__ r, DevCtrl C) {
  const int b = blockIdx.y;
  if (C.cg_done[b]) return;
  const double be = C.beta[b];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < me; i += gridDim.x * blockDim.x) {
    const long long o = (long long)b * me + i;
    p[o] = fma(be, p[o], r[o]);
  }
}

// CR: p = r + beta p ; q = s + beta q ; qq = q.q ; alpha = rs / qq.  grid (KKT_NPART, batch)
__global__ void __launch_bounds__(KKT_CGT) cr_pq_kernel(int batch, int me, double* p, double* q, const double* __restrict__ r,
                             const double* __restrict__ sv, DevCtrl C) {
  __shared__ double red[32];
  const int b = blockIdx.y;
  if (C.cg_done[b]) return;
  const double be = C.beta[b];
  double part = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < me; i += KKT_NPART * blockDim.x) {
    const long long o = (long long)b * me + i;
    p[o] = fma(be, p[o], r[o]);
    const double qv = fma(be, q[o], sv[o]);
    q[o] = qv;
    part = fma(qv, qv, part);
  }
  double s = block_sum(part, red), tot;
  if (finish_dots<1>(C, b, &s, &tot)) {
    C.qq[b] = tot;
    C.alpha[b] = C.rs[b] / tot;
  }
}

// WHILE-node condition of the Krylov loop: another iteration iff some instance is running.
// count_run: called at the end of the body (counts body executions), not before the node.
__global__ void cg_cond_kernel(int batch, DevCtrl C, cudaGraphConditionalHandle handle, int count_run) {
  if (count_run) *C.cg_runs += 1;
  cudaGraphSetConditional(handle, C.cg_done[batch] > 0 ? 1u : 0u);
}

__global__ void cg_finish_kernel(int batch, DevCtrl C, int first, int* status) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  if (C.cg_done[b] == 3) return;   // skipped pass
  if (first) C.cg_iters_first[b] = C.cg_iters[b];
  if (C.cg_done[b] == 2) atomicCAS(status, 0, 4 /* KKT_ERR_NOT_CONVERGED */);
}

// ---------------------------------------------------------------- HyKKT outer refinement
__global__ void outer_init_kernel(int batch, DevCtrl C) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b == 0) { C.odone[batch] = batch; *C.cg_runs = 0; }
  if (b >= batch) return;
  C.odone[b] = 0; C.opass[b] = 0; C.oprev[b] = INFINITY;
  for (int k = 0; k < 4; k++) C.onrm[4 * b + k] = 0ULL;
}

// v += dv for instances still refining, with ||dv||_inf -> onrm[4b + k], ||v||_inf -> onrm[4b + k + 1].
// grid (gx, batch)
__global__ void outer_update_kernel(int batch, long long len, double* v, const double* __restrict__ dv,
                                    DevCtrl C, int k) {
  const int b = blockIdx.y;
  if (C.odone[b]) return;
  double mdv = 0.0, mv = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < len; i += (long long)gridDim.x * blockDim.x) {
    const long long o = (long long)b * len + i;
    const double d = dv[o], nv = v[o] + d;
    v[o] = nv;
    mdv = (isnan(d) || isnan(mdv)) ? NAN : fmax(mdv, fabs(d));
    mv = (isnan(nv) || isnan(mv)) ? NAN : fmax(mv, fabs(nv));
  }
  block_max_atomic(C.onrm + 4 * b + k, mdv);
  block_max_atomic(C.onrm + 4 * b + k + 1, mv);
}

// Stop rule of the saddle-system refinement (R9 analogue on (dx, dy)): the relative correction
// c_k = max(||ddx||/||dx||, ||ddy||/||dy||) just applied is <= 1e-14, or two corrections converge
// geometrically (rho = c_k / c_k-1 < 1/2) with rho c_k / (1 - rho) <= 1e-14.
__global__ void outer_decide_kernel(int batch, DevCtrl C) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch || C.odone[b]) return;
  const double ddx = bits2d(C.onrm[4 * b]), xn = bits2d(C.onrm[4 * b + 1]);
  const double ddy = bits2d(C.onrm[4 * b + 2]), yn = bits2d(C.onrm[4 * b + 3]);
  for (int k = 0; k < 4; k++) C.onrm[4 * b + k] = 0ULL;
  const double c = fmax(xn > 0 ? ddx / xn : ddx, yn > 0 ? ddy / yn : ddy);
  C.opass[b] += 1;
  bool stop = !(c > 1e-14);   // also stops on NaN (reported by the Krylov status)
  if (isfinite(C.oprev[b])) {
    const double rho = c / C.oprev[b];
    if (rho < 0.5 && rho * c / (1.0 - rho) <= 1e-14) stop = true;
  }
  C.oprev[b] = c;
  if (stop) { C.odone[b] = 1; atomicSub(C.odone + batch, 1); }
}

// ---------------------------------------------------------------- NEXT-1 recovery
// dz = -C r2 + D_H (H dx + r4), ds = -(D_s + dw)^-1 (r2 + dz), one thread per row
__global__ void recover_kernel(DevPlan P, const double* __restrict__ Jv, const double* __restrict__ Ss,
                               double dw, double dc, const double* __restrict__ r2,
                               const double* __restrict__ r4, const double* __restrict__ dx, double* dz,
                               double* ds) {
  const int mi = P.m - P.m_eq;
  long long total = (long long)P.batch * mi;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(idx / mi), q = (int)(idx % mi), row = P.m_eq + q;
    const double* J = Jv + (long long)b * P.nnzJ;
    const double* x = dx + (long long)b * P.n;
    double hx = 0.0;
    for (int p = P.Jrp[row]; p < P.Jrp[row + 1]; p++) hx = fma(J[p], x[P.Jci[p]], hx);
    const double t = Ss[idx] + dw;               // D_s + dw
    const double Cr = 1.0 / fma(dc, t, 1.0);     // C
    const double DH = t * Cr;                    // D_H
    const double z = fma(DH, hx + r4[idx], -Cr * r2[idx]);
    dz[idx] = z;
    ds[idx] = -(r2[idx] + z) / t;
  }
}

// du = -(U dx - mu)/X - u ;  dv = -(V ds - mu)/S - v
__global__ void recover_bounds_kernel(long long nx, long long ns, const double* __restrict__ x,
                                      const double* __restrict__ u, const double* __restrict__ s,
                                      const double* __restrict__ v, double mu,
                                      const double* __restrict__ dx, const double* __restrict__ ds,
                                      double* du, double* dv) {
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < nx + ns;
       idx += (long long)gridDim.x * blockDim.x) {
    if (idx < nx) du[idx] = -fma(u[idx], dx[idx], -mu) / x[idx] - u[idx];
    else {
      const long long k = idx - nx;
      dv[k] = -fma(v[k], ds[k], -mu) / s[k] - v[k];
    }
  }
}

}  // namespace kkt
