// resid.cuh -- double-double residual of the unassembled operator (R8).
#pragma once
#include "common.cuh"

namespace kkt {

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
  if (done && done[P.batch] == 0) return;  // every instance has finished refining
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
    int p = p0;
    for (; p + 4 <= p1; p += 4) {  // four terms' loads in flight; the same summation order
      const int c0 = P.Jci[p], c1 = P.Jci[p + 1], c2 = P.Jci[p + 2], c3 = P.Jci[p + 3];
      const double jv[4] = {J[p], J[p + 1], J[p + 2], J[p + 3]};
      const double xv[4] = {xb[c0], xb[c1], xb[c2], xb[c3]};
#pragma unroll
      for (int u = 0; u < 4; u++) {
        acc = dd_add(acc, two_prod(jv[u], xv[u]));
        aa = fma(fabs(jv[u]), fabs(xv[u]), aa);
      }
    }
    for (; p < p1; p++) {
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

// grid (gx, batch): the instance is block-uniform, so omega is reduced per block (one atomic).
__global__ void resid_cols_kernel(DevPlan P, const double* __restrict__ Wv, const double* __restrict__ Jv,
                                  const double* __restrict__ Sx, double dw, const double* __restrict__ x,
                                  long long xs, const double* __restrict__ rhs, long long rs,
                                  const double2* __restrict__ T, const double* __restrict__ A,
                                  double* res, unsigned long long* omega, const int* __restrict__ done) {
  const int b = blockIdx.y;
  if (done && (done[P.batch] == 0 || done[b])) return;  // block-uniform exits
  const double* W = Wv + (long long)b * P.nnzW;
  const double* J = Jv + (long long)b * P.nnzJ;
  const double* xb = x + (long long)b * xs;
  const double2* Tb = T + (long long)b * P.m;
  const double* Ab = A + (long long)b * P.m;
  double ommax = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.n; i += gridDim.x * blockDim.x) {
    const long long idx = (long long)b * P.n + i;
    double xi = xb[i];
    dd s = two_sum(Sx[idx], dw);
    dd y = dd_mul_d(s, xi);
    double den = fabs(s.hi) * fabs(xi);
    // loads of four terms in flight per step; the summation order is the sequential one
    int p = P.Wf_p[i];
    const int pw = P.Wf_p[i + 1];
    for (; p + 4 <= pw; p += 4) {
      const int k0 = P.Wf_k[p], k1 = P.Wf_k[p + 1], k2 = P.Wf_k[p + 2], k3 = P.Wf_k[p + 3];
      const int c0 = P.Wf_c[p], c1 = P.Wf_c[p + 1], c2 = P.Wf_c[p + 2], c3 = P.Wf_c[p + 3];
      const double wv[4] = {W[k0], W[k1], W[k2], W[k3]};
      const double xv[4] = {xb[c0], xb[c1], xb[c2], xb[c3]};
#pragma unroll
      for (int u = 0; u < 4; u++) {
        y = dd_add(y, two_prod(wv[u], xv[u]));
        den = fma(fabs(wv[u]), fabs(xv[u]), den);
      }
    }
    for (; p < pw; p++) {
      double wv = W[P.Wf_k[p]], xv = xb[P.Wf_c[p]];
      y = dd_add(y, two_prod(wv, xv));
      den = fma(fabs(wv), fabs(xv), den);
    }
    p = P.Jt_p[i];
    const int pj = P.Jt_p[i + 1];
    for (; p + 4 <= pj; p += 4) {
      const int r0 = P.Jt_r[p], r1 = P.Jt_r[p + 1], r2 = P.Jt_r[p + 2], r3 = P.Jt_r[p + 3];
      const int k0 = P.Jt_k[p], k1 = P.Jt_k[p + 1], k2 = P.Jt_k[p + 2], k3 = P.Jt_k[p + 3];
      const double jv[4] = {J[k0], J[k1], J[k2], J[k3]};
      const double2 t[4] = {Tb[r0], Tb[r1], Tb[r2], Tb[r3]};
      const double av[4] = {Ab[r0], Ab[r1], Ab[r2], Ab[r3]};
#pragma unroll
      for (int u = 0; u < 4; u++) {
        y = dd_add(y, dd_mul_d(dd{t[u].x, t[u].y}, jv[u]));
        den = fma(fabs(jv[u]), av[u], den);
      }
    }
    for (; p < pj; p++) {
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
    const double om = (den > 0.0) ? fabs(rv) / den : (rv != 0.0 ? INFINITY : 0.0);
    ommax = (isnan(om) || isnan(ommax)) ? NAN : fmax(ommax, om);
  }
  if (omega) block_max_atomic(omega + b, ommax);
}

// Variant for long columns (dense W, e.g. COPS elec): one WARP per column.  Lanes accumulate a
// strided subset of the column's W and J^T terms in double-double, then a fixed xor-butterfly
// (dd_add) combines them: the summation order is fixed, so results stay deterministic.
// grid (gx, batch); blockDim = 256 (8 columns per block).
__global__ void resid_cols_warp_kernel(DevPlan P, const double* __restrict__ Wv, const double* __restrict__ Jv,
                                       const double* __restrict__ Sx, double dw, const double* __restrict__ x,
                                       long long xs, const double* __restrict__ rhs, long long rs,
                                       const double2* __restrict__ T, const double* __restrict__ A,
                                       double* res, unsigned long long* omega, const int* __restrict__ done) {
  const int b = blockIdx.y;
  if (done && (done[P.batch] == 0 || done[b])) return;  // block-uniform exits
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5, nwb = blockDim.x >> 5;
  const double* W = Wv + (long long)b * P.nnzW;
  const double* J = Jv + (long long)b * P.nnzJ;
  const double* xb = x + (long long)b * xs;
  const double2* Tb = T + (long long)b * P.m;
  const double* Ab = A + (long long)b * P.m;
  double ommax = 0.0;
  for (int i = blockIdx.x * nwb + wib; i < P.n; i += gridDim.x * nwb) {
    const long long idx = (long long)b * P.n + i;
    dd y = {0.0, 0.0};
    double den = 0.0;
    for (int p = P.Wf_p[i] + lane; p < P.Wf_p[i + 1]; p += 32) {
      const double wv = W[P.Wf_k[p]], xv = xb[P.Wf_c[p]];
      y = dd_add(y, two_prod(wv, xv));
      den = fma(fabs(wv), fabs(xv), den);
    }
    for (int p = P.Jt_p[i] + lane; p < P.Jt_p[i + 1]; p += 32) {
      const int r = P.Jt_r[p];
      const double jv = J[P.Jt_k[p]];
      const double2 t = Tb[r];
      y = dd_add(y, dd_mul_d(dd{t.x, t.y}, jv));
      den = fma(fabs(jv), Ab[r], den);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const dd oth = {__shfl_xor_sync(0xffffffffu, y.hi, o), __shfl_xor_sync(0xffffffffu, y.lo, o)};
      // both partners compute the same sum: order the operands by lane so the result is identical
      y = (lane & o) ? dd_add(oth, y) : dd_add(y, oth);
      den += __shfl_xor_sync(0xffffffffu, den, o);
    }
    const double xi = xb[i];
    const dd s2 = two_sum(Sx[idx], dw);
    y = dd_add(dd_mul_d(s2, xi), y);
    den = fma(fabs(s2.hi), fabs(xi), den);
    const double bi = rhs[(long long)b * rs + i];
    const dd rr = dd_add(dd{bi, 0.0}, dd{-y.hi, -y.lo});
    const double rv = rr.hi + rr.lo;
    if (lane == 0) res[idx] = rv;
    den += fabs(bi);
    const double om = (den > 0.0) ? fabs(rv) / den : (rv != 0.0 ? INFINITY : 0.0);
    ommax = (isnan(om) || isnan(ommax)) ? NAN : fmax(ommax, om);
  }
  if (omega) block_max_atomic(omega + b, ommax);
}

}  // namespace kkt
