// k3.cuh -- Richardson refinement on the unreduced KKT system K3 (P:292-317 eq. K3; P:431-439
// "Richardson iterations on the original system (K3) to refine the solution returned by the
// direct sparse linear solver").
//
// Unknowns d = (dx[n], ds[mi], dy[me], dz[mi], du[n], dv[mi]); rows G = J[0, me), H = J[me, m);
// X, S, U, V the diagonal matrices of x, s, u, v.  K3 d = f:
//   (1) W dx + G^T dy + H^T dz - du = f1     (2) dz - dv = f2        (3) G dx = f3
//   (4) H dx + ds = f4                       (5) U dx + X du = f5    (6) V ds + S dv = f6
// One sweep: residual rho = f - K3 d (double-double), then the correction solves K3 with the
// condensed factor (K = W + D_x + dw I + H^T D_H H [+ gamma G^T G], D_x = X^-1 U, D_s = S^-1 V):
//   b1 = rho1 + X^-1 rho5, b2 = rho2 + S^-1 rho6 (eliminate du, dv: P:360-362)
//   c1 = b1 + H^T (D_H rho4 - C b2)            (eliminate ds, dz: P:415-423)
//   [K G^T; G -dc] [ex; ey] = [c1; rho3]       (kkt_solve / HyKKT)
//   ez = D_H (H ex - rho4) + C b2,  es = (b2 - ez) / (D_s + dw),  ev = S^-1 (rho6 - V es),
//   eu = X^-1 (rho5 - U ex);  d += e.
// With dw = dc = 0 the first sweep is the exact (direct) K3 solution; regularisation makes the
// condensed factor a preconditioner and the refinement converges to the unregularised K3 solution.
#pragma once
#include "common.cuh"

namespace kkt {

struct K3Ctx {
  const double *x, *s, *u, *v;                 // [B][n], [B][mi], [B][n], [B][mi]
  const double *f1, *f2, *f3, *f4, *f5, *f6;   // right-hand side blocks
  double *dx, *ds, *dy, *dz, *du, *dv;         // current solution (updated in place)
  double *r5, *b2, *r4, *r6, *c1, *r3;         // sweep scratch: rho5 [n], b2/rho4/rho6 [mi], c1 [n], rho3 [me]
  double2* tw;                                 // [B][m] J^T weights: t_r (residual) in .x, w_r (rhs) in .y
  double *ex, *ey;                             // correction from the condensed solve
  int* done;                                   // [B + 1] finished instances ([B] = still refining)
  unsigned long long* nrm;                     // [B][2] ||e||_inf, ||d||_inf bits
  double* prev;                                // [B] previous relative correction
  int* sweeps;                                 // [B] sweeps applied
  double dw, dc;
  const double* Ss;                            // Sigma_s of the last kkt_condense (= D_s)
};

__global__ void k3_init_kernel(int batch, K3Ctx K) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b == 0) K.done[batch] = batch;
  if (b >= batch) return;
  K.done[b] = 0; K.prev[b] = INFINITY; K.sweeps[b] = 0;
  K.nrm[2 * b] = 0ULL; K.nrm[2 * b + 1] = 0ULL;
}

// rows: rho2, rho3, rho4, rho6 and the J^T weights t_r (residual: dy or dz) and w_r (rhs)
__global__ void k3_rows_kernel(DevPlan P, const double* __restrict__ Jv, K3Ctx K) {
  if (K.done[P.batch] == 0) return;
  const int me = P.m_eq, mi = P.m - P.m_eq;
  const long long total = (long long)P.batch * P.m;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(idx / P.m), r = (int)(idx % P.m);
    if (K.done[b]) continue;
    const double* J = Jv + (long long)b * P.nnzJ;
    const double* dx = K.dx + (long long)b * P.n;
    dd acc = {0.0, 0.0};
    for (int p = P.Jrp[r]; p < P.Jrp[r + 1]; p++) acc = dd_add(acc, two_prod(J[p], dx[P.Jci[p]]));
    if (r < me) {
      const long long o = (long long)b * me + r;
      const dd rr = dd_add(dd{K.f3[o], 0.0}, dd{-acc.hi, -acc.lo});
      K.r3[o] = rr.hi + rr.lo;
      K.tw[idx] = make_double2(K.dy[o], 0.0);
    } else {
      const long long o = (long long)b * mi + (r - me);
      const double dzv = K.dz[o], dvv = K.dv[o], dsv = K.ds[o];
      // rho2 = f2 - dz + dv ; rho4 = f4 - H dx - ds ; rho6 = f6 - V ds - S dv
      const dd r2 = dd_add(two_sum(K.f2[o], -dzv), dd{dvv, 0.0});
      dd r4 = dd_add(dd{K.f4[o], 0.0}, dd{-acc.hi, -acc.lo});
      r4 = dd_add(r4, dd{-dsv, 0.0});
      dd r6 = dd_add(dd{K.f6[o], 0.0}, two_prod(-K.v[o], dsv));
      r6 = dd_add(r6, two_prod(-K.s[o], dvv));
      const double rho2 = r2.hi + r2.lo, rho4 = r4.hi + r4.lo, rho6 = r6.hi + r6.lo;
      const double b2 = rho2 + rho6 / K.s[o];
      const double t = K.Ss[o] + K.dw;          // D_s + dw
      const double Cr = 1.0 / fma(K.dc, t, 1.0);
      const double DH = t * Cr;
      K.b2[o] = b2; K.r4[o] = rho4; K.r6[o] = rho6;
      K.tw[idx] = make_double2(dzv, fma(DH, rho4, -Cr * b2));
    }
  }
}

// columns: rho1, rho5, c1 = rho1 + rho5 / x + H^T w   (one pass over W and J^T per column)
__global__ void k3_cols_kernel(DevPlan P, const double* __restrict__ Wv, const double* __restrict__ Jv, K3Ctx K) {
  if (K.done[P.batch] == 0) return;
  const long long total = (long long)P.batch * P.n;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(idx / P.n), i = (int)(idx % P.n);
    if (K.done[b]) continue;
    const double* W = Wv + (long long)b * P.nnzW;
    const double* J = Jv + (long long)b * P.nnzJ;
    const double* dx = K.dx + (long long)b * P.n;
    const double2* tw = K.tw + (long long)b * P.m;
    dd y = {0.0, 0.0};
    for (int p = P.Wf_p[i]; p < P.Wf_p[i + 1]; p++) y = dd_add(y, two_prod(W[P.Wf_k[p]], dx[P.Wf_c[p]]));
    double wsum = 0.0;
    for (int p = P.Jt_p[i]; p < P.Jt_p[i + 1]; p++) {
      const int r = P.Jt_r[p];
      const double jv = J[P.Jt_k[p]];
      const double2 t = tw[r];
      y = dd_add(y, two_prod(jv, t.x));
      if (r >= P.m_eq) wsum = fma(jv, t.y, wsum);
    }
    const double duv = K.du[idx];
    dd r1 = dd_add(dd{K.f1[idx], 0.0}, dd{-y.hi, -y.lo});
    r1 = dd_add(r1, dd{duv, 0.0});
    dd r5 = dd_add(dd{K.f5[idx], 0.0}, two_prod(-K.u[idx], dx[i]));
    r5 = dd_add(r5, two_prod(-K.x[idx], duv));
    const double rho1 = r1.hi + r1.lo, rho5 = r5.hi + r5.lo;
    K.r5[idx] = rho5;
    K.c1[idx] = rho1 + rho5 / K.x[idx] + wsum;
  }
}

// recovery of the correction and update of d (rows: ez, es, ev, dy += ey), norms per instance;
// grid (gx, batch)
__global__ void k3_update_rows_kernel(DevPlan P, const double* __restrict__ Jv, K3Ctx K) {
  const int b = blockIdx.y;
  if (K.done[b]) return;
  const int me = P.m_eq, mi = P.m - P.m_eq;
  const double* J = Jv + (long long)b * P.nnzJ;
  const double* ex = K.ex + (long long)b * P.n;
  double me_ = 0.0, md_ = 0.0;
  bool bad = false;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < P.m; r += gridDim.x * blockDim.x) {
    if (r < me) {
      const long long o = (long long)b * me + r;
      const double e = K.ey[o], d = K.dy[o] + e;
      K.dy[o] = d;
      me_ = fmax(me_, fabs(e)); md_ = fmax(md_, fabs(d));
      bad |= isnan(e);
    } else {
      const long long o = (long long)b * mi + (r - me);
      double hx = 0.0;
      for (int p = P.Jrp[r]; p < P.Jrp[r + 1]; p++) hx = fma(J[p], ex[P.Jci[p]], hx);
      const double t = K.Ss[o] + K.dw;
      const double Cr = 1.0 / fma(K.dc, t, 1.0);
      const double DH = t * Cr;
      const double ez = fma(DH, hx - K.r4[o], Cr * K.b2[o]);
      const double es = (K.b2[o] - ez) / t;
      const double ev = (K.r6[o] - K.v[o] * es) / K.s[o];
      const double nz = K.dz[o] + ez, ns = K.ds[o] + es, nv = K.dv[o] + ev;
      K.dz[o] = nz; K.ds[o] = ns; K.dv[o] = nv;
      me_ = fmax(me_, fmax(fabs(ez), fmax(fabs(es), fabs(ev))));
      md_ = fmax(md_, fmax(fabs(nz), fmax(fabs(ns), fabs(nv))));
      bad |= isnan(ez) || isnan(es) || isnan(ev);
    }
  }
  block_max_atomic(K.nrm + 2 * b, bad ? NAN : me_);
  block_max_atomic(K.nrm + 2 * b + 1, md_);
}

// columns: eu = X^-1 (rho5 - U ex); dx += ex; du += eu
__global__ void k3_update_cols_kernel(DevPlan P, K3Ctx K) {
  const int b = blockIdx.y;
  if (K.done[b]) return;
  double me_ = 0.0, md_ = 0.0;
  bool bad = false;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.n; i += gridDim.x * blockDim.x) {
    const long long o = (long long)b * P.n + i;
    const double ex = K.ex[o];
    const double eu = (K.r5[o] - K.u[o] * ex) / K.x[o];
    const double nx = K.dx[o] + ex, nu = K.du[o] + eu;
    K.dx[o] = nx; K.du[o] = nu;
    me_ = fmax(me_, fmax(fabs(ex), fabs(eu)));
    md_ = fmax(md_, fmax(fabs(nx), fabs(nu)));
    bad |= isnan(ex) || isnan(eu);
  }
  block_max_atomic(K.nrm + 2 * b, bad ? NAN : me_);
  block_max_atomic(K.nrm + 2 * b + 1, md_);
}

// stop rule (R9 analogue on the whole K3 direction): the relative correction just applied
// c = ||e|| / ||d|| <= tol, or two corrections converge geometrically (rho = c / c_prev < 1/2) with
// rho c / (1 - rho) <= tol, or max_sweeps sweeps (the direct solve + max_refine corrections), or a
// non-finite correction (status KKT_ERR_NONFINITE)
__global__ void k3_decide_kernel(int batch, K3Ctx K, double tol, int max_sweeps, int* status) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch || K.done[b]) return;
  const double e = __longlong_as_double((long long)K.nrm[2 * b]);
  const double d = __longlong_as_double((long long)K.nrm[2 * b + 1]);
  K.nrm[2 * b] = 0ULL; K.nrm[2 * b + 1] = 0ULL;
  const int sw = (K.sweeps[b] += 1);
  const double c = d > 0 ? e / d : e;
  bool stop = sw >= max_sweeps;
  if (!isfinite(c)) { stop = true; atomicCAS(status, 0, 5 /* KKT_ERR_NONFINITE */); }
  if (sw >= 2) {  // sweep 1 is the direct solve; refinement corrections from sweep 2 on
    if (c <= tol) stop = true;
    if (isfinite(K.prev[b])) {
      const double rho = c / K.prev[b];
      if (rho < 0.5 && rho * c / (1.0 - rho) <= tol) stop = true;
    }
    K.prev[b] = c;
  }
  if (stop) { K.done[b] = 1; atomicSub(K.done + batch, 1); }
}

__global__ void k3_finish_kernel(int batch, K3Ctx K, int* refine_iters) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b < batch) refine_iters[b] = K.sweeps[b] - 1;
}

}  // namespace kkt
