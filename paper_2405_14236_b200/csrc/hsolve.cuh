// hsolve.cuh -- triangular solves through the huge fronts (huge.cuh's class: fronts beyond one
// CTA's shared memory) by the whole GPU, one cooperative kernel:
//
//   forward, levels bottom-up (HugeSched, same CTA groups as the factorisation):
//     gather    v = [b(cols(s)); 0] + extend-add of the children's u vectors (CTA 0 of the group)
//     sweep     row blocks of 32 rows over the group's CTAs, in order: diagonal block t
//               computes v_t - sum_{j<t} L_tj y_j (8 warps split the column blocks j), then
//               y_t = L_tt^-1 (...) in warp 0's registers and publishes y_t by a flag; row
//               blocks of L21 accumulate all column blocks into u = v2 - L21 y
//   backward, levels top-down:
//     column blocks of 32 over the group's CTAs, last block first: block j computes
//     y_j - sum_{i>j} L_ij^T x_i (8 warps split the row blocks; the L21 rows need no wait), then
//     x_j = L_jj^-T (...) and publishes x_j by a flag
//
// A consumer warp loads its 32 x 32 block of L before it waits for the flag of the y / x block
// it multiplies, so the critical path per 32 columns is one flag hand-off, one block product
// and one 32-step register solve.  Flags carry (batch index + 1) and are zeroed at launch;
// reductions are in fixed order (warp partials summed 0..7): results are deterministic.
#pragma once
#include "huge.cuh"

namespace kkt {

#define SB 32  // row / column block of the huge-front solves (one warp lane per row)

__device__ __forceinline__ void wait_flag(const int* f, int target) { spin_acquire(f, target); }

__global__ void __launch_bounds__(256, 1) solve_huge_kernel(DevPlan P, const double* __restrict__ Lx_all,
                                                            const double* __restrict__ Dv_all,
                                                            const double* __restrict__ rhs, long long rs,
                                                            double* Y_all, double* uv_all, double* Xp_all,
                                                            double* xout, long long xs,
                                                            const int* __restrict__ done, HugeSched H) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ double part[8][SB];
  __shared__ double Dg[SB][SB + 1];  // diagonal block of the current task: Dg[k][lane] (warp 0)
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const unsigned full = 0xffffffffu;
  if (done && done[P.batch] == 0) return;  // every instance has finished refining (grid-uniform)
  const int nent = H.lvl_ptr[H.nlev];
  for (int q = blockIdx.x * nt + tid; q < nent; q += gridDim.x * nt) H.ctr[q] = 0;
  for (int q = blockIdx.x * nt + tid; q < 2 * H.nflag; q += gridDim.x * nt) H.flags[q] = 0;
  grid.sync();

  for (int phase = 0; phase < 2; phase++) {
    const bool fwd = (phase == 0);
    for (int Li = 0; Li < H.nlev; Li++) {
      const int L = fwd ? Li : H.nlev - 1 - Li;
      const int e0 = H.lvl_ptr[L], e1 = H.lvl_ptr[L + 1];
      const bool rr = (H.ent[e0].z == 0);
      for (int e = rr ? e0 + (int)blockIdx.x : e0; e < e1; e += rr ? (int)gridDim.x : 1) {
        const int4 E = H.ent[e];
        CtaGroup G;
        if (rr) { G.rank = 0; G.size = 1; }
        else {
          if ((int)blockIdx.x < E.y || (int)blockIdx.x >= E.y + E.z) continue;
          G.rank = blockIdx.x - E.y; G.size = E.z;
        }
        G.ctr = H.ctr + e; G.gen = 0;
        const int s = E.x;
        const SnInfo I = P.sn[s];
        const int r = I.r, w = I.w, R = r - w;
        const int nb = (w + SB - 1) / SB, nR = (R + SB - 1) / SB;
        int* fl = H.flags + (fwd ? 0 : H.nflag) + E.w;
        for (int b = 0; b < P.batch; b++) {
          if (done && done[b]) continue;
          const int tgt = b + 1;
          const double* Lp = Lx_all + (long long)b * P.nnzL_stored + I.Lp;
          const double* dv = Dv_all + (long long)b * P.n + I.f0;
          double* y = Y_all + (long long)b * P.n + I.f0;
          if (G.rank == 0 && tid == 0) trace_stamp(P, fwd ? 1 : 2, s, b, 0);
          if (fwd) {
            double* uvb = uv_all + (long long)b * P.uvec_doubles;
            double* us = uvb + I.uvp;
            // ---- gather (CTA 0; children in fixed order) ----
            if (G.rank == 0) {
              const double* bb = rhs + (long long)b * rs;
              for (int q = tid; q < w; q += nt) y[q] = bb[__ldg(P.perm + I.f0 + q)];
              for (int q = tid; q < R; q += nt) us[q] = 0.0;
              for (int ci = I.c0; ci < I.c1; ci++) {
                const SnInfo C = P.chinfo[ci];
                const int Rc = C.r - C.w;
                const int* rel = P.sn_rel + C.rp0 + C.w;
                const double* u = uvb + C.uvp;
                __syncthreads();
                for (int q = tid; q < Rc; q += nt) {
                  const int pos = __ldg(rel + q);
                  double* d = (pos < w) ? y + pos : us + (pos - w);
                  *d += ldcg(u + q);
                }
              }
            }
            G.sync();
            // ---- row blocks ----
            for (int t = G.rank; t < nb + nR; t += G.size) {
              const bool dg = t < nb;
              const int row0 = dg ? t * SB : w + (t - nb) * SB;
              const int nrow = min(SB, (dg ? w : r) - row0);
              const int row = row0 + lane;
              const bool rv = lane < nrow;
              const int jmax = dg ? t : nb;
              double v0 = 0.0, di = 0.0;
              if (warp == 0) {  // own right-hand side and diagonal block, ahead of the waits
                if (rv) v0 = ldcg(dg ? y + row : us + (row - w));
                if (dg) {
#pragma unroll
                  for (int c = 0; c < SB; c++)
                    Dg[c][lane] = (rv && c < lane) ? __ldg(Lp + (long long)(row0 + c) * r + row) : 0.0;
                  if (rv) di = __ldg(dv + row);
                }
              }
              double acc = 0.0;
              for (int j = warp; j < jmax; j += 8) {
                const int c0 = j * SB, ncol = min(SB, w - c0);
                double l[SB];
#pragma unroll
                for (int c = 0; c < SB; c++)
                  l[c] = (rv && c < ncol) ? __ldg(Lp + (long long)(c0 + c) * r + row) : 0.0;
                wait_flag(fl + j, tgt);
                const double yv = (lane < ncol) ? ldcg(y + c0 + lane) : 0.0;
#pragma unroll
                for (int c = 0; c < SB; c++) acc = fma(l[c], __shfl_sync(full, yv, c), acc);
              }
              part[warp][lane] = acc;
              __syncthreads();
              if (warp == 0) {
                double v = v0;
#pragma unroll
                for (int q = 0; q < 8; q++) v -= part[q][lane];
                if (dg) {
                  double ld[SB];
#pragma unroll
                  for (int c = 0; c < SB; c++) ld[c] = Dg[c][lane];
#pragma unroll
                  for (int k = 0; k < SB; k++) {
                    if (k < nrow) {
                      const double yk = __shfl_sync(full, v * di, k);
                      if (lane == k) v = yk;
                      else if (lane > k) v = fma(-ld[k], yk, v);
                    }
                  }
                  if (rv) y[row] = v;
                  __threadfence();
                  __syncwarp();
                  if (lane == 0) st_release(fl + t, tgt);
                } else if (rv) {
                  us[row - w] = v;
                }
              }
              __syncthreads();
            }
          } else {
            double* Xp = Xp_all + (long long)b * P.n;
            double* x = Xp + I.f0;
            const int* rows = P.sn_rows + I.rp0;
            double* xo = xout + (long long)b * xs;
            for (int t = G.rank; t < nb; t += G.size) {
              const int j = nb - 1 - t;
              const int c0 = j * SB, ncol = min(SB, w - c0);
              const int col = c0 + lane;
              const bool cv = lane < ncol;
              double y0 = 0.0, di = 0.0;
              if (warp == 0) {
                if (cv) { y0 = ldcg(y + col); di = __ldg(dv + col); }
#pragma unroll
                for (int k = 0; k < SB; k++)  // row k of the diagonal block, column col
                  Dg[k][lane] = (cv && k > lane && k < ncol) ? __ldg(Lp + (long long)col * r + c0 + k) : 0.0;
              }
              double p[SB];
#pragma unroll
              for (int c = 0; c < SB; c++) p[c] = 0.0;
              const int nq = nR + (nb - 1 - j);  // L21 row blocks first, then i = nb-1 .. j+1
              for (int q = warp; q < nq; q += 8) {
                int row0, nrow, fi = -1;
                if (q < nR) { row0 = w + q * SB; nrow = min(SB, r - row0); }
                else { fi = nb - 1 - (q - nR); row0 = fi * SB; nrow = min(SB, w - row0); }
                const int row = row0 + lane;
                const bool rv = lane < nrow;
                double l[SB];
#pragma unroll
                for (int c = 0; c < SB; c++)
                  l[c] = (rv && c < ncol) ? __ldg(Lp + (long long)(c0 + c) * r + row) : 0.0;
                double xv = 0.0;
                if (fi >= 0) {
                  wait_flag(fl + fi, tgt);
                  if (rv) xv = ldcg(x + row);
                } else if (rv) {
                  xv = ldcg(Xp + __ldg(rows + row));
                }
#pragma unroll
                for (int c = 0; c < SB; c++) p[c] = fma(l[c], xv, p[c]);
              }
              // transpose-reduce: lane c ends with sum over the warp's rows of p[c] (31 shuffles)
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
              part[warp][lane] = p[0];
              __syncthreads();
              if (warp == 0) {
                double a = y0;
#pragma unroll
                for (int q = 0; q < 8; q++) a -= part[q][lane];
                double ld[SB];
#pragma unroll
                for (int k = 0; k < SB; k++) ld[k] = Dg[k][lane];
#pragma unroll
                for (int k = SB - 1; k >= 0; k--) {
                  if (k < ncol) {
                    const double xk = __shfl_sync(full, a * di, k);
                    if (lane == k) a = xk;
                    else if (lane < k) a = fma(-ld[k], xk, a);
                  }
                }
                if (cv) {
                  x[col] = a;
                  xo[__ldg(P.perm + I.f0 + col)] = a;
                }
                __threadfence();
                __syncwarp();
                if (lane == 0) st_release(fl + j, tgt);
              }
              __syncthreads();
            }
          }
          if (lane == 0) trace_max(P, fwd ? 1 : 2, s, b, 1);
        }
      }
      grid.sync();  // level done: the next level reads these u vectors / x values
    }
  }
}

}  // namespace kkt
