// condense.cuh -- row weights D_r and the fixed-pattern condensation.
#pragma once
#include "common.cuh"

namespace kkt {

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
    int q = __ldg(P.pptr + k);
    const int q1 = __ldg(P.pptr + k + 1);
    for (; q + 4 <= q1; q += 4) {  // four products' loads in flight, the same fma order
      int a[4], c[4], r[4];
      double ja[4], jc[4], d[4];
#pragma unroll
      for (int u = 0; u < 4; u++) { a[u] = __ldg(P.pa + q + u); c[u] = __ldg(P.pb + q + u); }
#pragma unroll
      for (int u = 0; u < 4; u++) { r[u] = __ldg(P.jrow + a[u]); ja[u] = __ldg(J + a[u]); jc[u] = __ldg(J + c[u]); }
#pragma unroll
      for (int u = 0; u < 4; u++) d[u] = __ldg(D + r[u]);
#pragma unroll
      for (int u = 0; u < 4; u++) v = fma(d[u] * ja[u], jc[u], v);
    }
    for (; q < q1; q++) {
      int a = __ldg(P.pa + q), c = __ldg(P.pb + q);
      v = fma(__ldg(D + __ldg(P.jrow + a)) * __ldg(J + a), __ldg(J + c), v);
    }
    Kv[idx] = v;
  }
}

}  // namespace kkt
