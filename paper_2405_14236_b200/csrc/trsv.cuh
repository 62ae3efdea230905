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

__global__ void __launch_bounds__(KKT_WPB * 32) fwd_small_kernel(DevPlan P, const double* __restrict__ Lx_all,
                                                                 const double* __restrict__ Dv_all,
                                                                 const double* __restrict__ rhs, long long rs,
                                                                 double* Y_all, double* uv_all, int* cnt_all,
                                                                 int* ctl, const int* __restrict__ done) {
  extern __shared__ double sm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* Pn = sm + (long long)wid * (KKT_SCAP + P.max_r_small);
  double* v = Pn + KKT_SCAP;
  const int ninit = P.n_up_s * P.batch;
  if (P.batch == 1 && done && done[0]) return;  // refinement finished: nothing to do
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
    for (;;) {
      if (lane == 0) trace_stamp(P, 1, s, b, 0);
      const SnInfo I = P.sn[s];
      const int r = I.r, w = I.w, R = r - w;
      const double* L = Lb + I.Lp;
      copy_g2s<false>(Pn, L, r * w, lane, 32);
      for (int q = lane; q < r; q += 32) v[q] = (q < w) ? bb[__ldg(P.perm + I.f0 + q)] : 0.0;
      __syncwarp();
      for (int ci = I.c0; ci < I.c1; ci++) {
        const SnInfo C = P.chinfo[ci];
        const int Rc = C.r - C.w;
        const int* rel = P.sn_rel + C.rp0 + C.w;
        const double* u = uv + C.uvp;
        for (int base = lane; base < Rc; base += 32 * 4) {
          int ps[4]; double val[4];
#pragma unroll
          for (int k = 0; k < 4; k++)
            if (base + 32 * k < Rc) { ps[k] = __ldg(rel + base + 32 * k); val[k] = ldcg(u + base + 32 * k); }
#pragma unroll
          for (int k = 0; k < 4; k++)
            if (base + 32 * k < Rc) v[ps[k]] += val[k];
        }
        __syncwarp();
      }
      // sweep: y_k = v_k / L_kk ; v_i -= L_ik y_k for i > k (covers L11 and L21), registers
      fwd_sweep_any(Pn, r, w, Dv + I.f0, v, lane);
      __syncwarp();
      for (int q = lane; q < w; q += 32) Y[I.f0 + q] = v[q];
      if (lane == 0) trace_stamp(P, 1, s, b, 1);
      if (I.par < 0) break;
      double* us = uv + I.uvp;
      for (int q = lane; q < R; q += 32) us[q] = v[w + q];
      const SnInfo Ip = P.sn[I.par];
      if (!warp_signal_parent(I, Ip, cnt, lane, true)) break;
      s = I.par;
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
                                                          int pcap) {
  extern __shared__ double sm[];
  __shared__ int s_task, s_last;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int ninit = P.n_up_bf * P.batch;
  double* v = sm;                         // [max_front]
  double* L11 = sm + P.max_front;         // [64 * 64] (unstaged path)
  double* Pn = L11 + 64 * 64;             // [pcap] staged panel
  if (P.batch == 1 && done && done[0]) return;
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
    if (tid == 0) cnt[s] = 0;
    for (;;) {
      if (tid == 0) trace_stamp(P, 1, s, b, 0);
      const SnInfo I = P.sn[s];
      const int r = I.r, w = I.w, R = r - w;
      const double* L = Lb + I.Lp;
      const bool staged = (r <= 256) && ((long long)r * w <= pcap);
      if (staged) copy_g2s<false>(Pn, L, r * w, tid, nt);
      for (int q = tid; q < r; q += nt) v[q] = (q < w) ? bb[__ldg(P.perm + I.f0 + q)] : 0.0;
      const int wb = staged ? 0 : (w < 64 ? w : 64);
      for (int q = tid; q < wb * wb; q += nt) {
        const int k = q / wb, i = q % wb;
        L11[q] = (i >= k) ? __ldg(L + (long long)k * r + i) : 0.0;
      }
      __syncthreads();
      for (int ci = I.c0; ci < I.c1; ci++) {
        const SnInfo C = P.chinfo[ci];
        const int Rc = C.r - C.w;
        const int* rel = P.sn_rel + C.rp0 + C.w;
        const double* u = uv + C.uvp;
        for (int q = tid; q < Rc; q += nt) v[__ldg(rel + q)] += ldcg(u + q);
        __syncthreads();
      }
      if (staged) {
        if (warp == 0) fwd_sweep_any(Pn, r, w, Dv_all + (long long)b * P.n + I.f0, v, lane);
        __syncthreads();
      } else {
        for (int k0 = 0; k0 < w; k0 += 64) {
          const int kb = (w - k0) < 64 ? (w - k0) : 64;
          if (k0 > 0) {
            for (int q = tid; q < kb * kb; q += nt) {
              const int k = q / kb, i = q % kb;
              L11[q] = (i >= k) ? __ldg(L + (long long)(k0 + k) * r + k0 + i) : 0.0;
            }
            __syncthreads();
          }
          if (warp == 0) {
            for (int k = 0; k < kb; k++) {
              const double yk = v[k0 + k] / L11[k * kb + k];
              __syncwarp();
              if (lane == 0) v[k0 + k] = yk;
              for (int i = k + 1 + lane; i < kb; i += 32) v[k0 + i] = fma(-L11[k * kb + i], yk, v[k0 + i]);
              __syncwarp();
            }
          }
          __syncthreads();
          for (int i = k0 + kb + tid; i < r; i += nt) {
            double acc = v[i];
            const double* Li = L + i;
            int k = 0;
            for (; k + 4 <= kb; k += 4) {
              const double l0 = __ldg(Li + (long long)(k0 + k) * r), l1 = __ldg(Li + (long long)(k0 + k + 1) * r);
              const double l2 = __ldg(Li + (long long)(k0 + k + 2) * r), l3 = __ldg(Li + (long long)(k0 + k + 3) * r);
              acc = fma(-l0, v[k0 + k], acc); acc = fma(-l1, v[k0 + k + 1], acc);
              acc = fma(-l2, v[k0 + k + 2], acc); acc = fma(-l3, v[k0 + k + 3], acc);
            }
            for (; k < kb; k++) acc = fma(-__ldg(Li + (long long)(k0 + k) * r), v[k0 + k], acc);
            v[i] = acc;
          }
          __syncthreads();
        }
      }
      for (int q = tid; q < w; q += nt) Y[I.f0 + q] = v[q];
      if (tid == 0) trace_stamp(P, 1, s, b, 1);
      if (I.par < 0) break;
      double* us = uv + I.uvp;
      for (int q = tid; q < R; q += nt) us[q] = v[w + q];
      __threadfence();
      __syncthreads();
      if (P.sn[I.par].huge) break;  // the whole-GPU phase (hsolve.cuh) takes it from here
      if (tid == 0) {
        const SnInfo Ip = P.sn[I.par];
        const int old = atom_add_acq_rel(cnt + I.par, 1);
        s_last = (old == Ip.c1 - Ip.c0 - 1);
        if (s_last) cnt[I.par] = 0;
      }
      __syncthreads();
      if (!s_last) break;
      s = I.par;
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
// the supernode's results are globally visible.
__device__ __forceinline__ int spawn_children(const DevPlan& P, const SnInfo& I, int b, int* ctl,
                                              TaskQueue Q, bool big_phase, int total) {
  int next = -1;
  for (int ci = I.c0; ci < I.c1; ci++) {
    const int c = __ldg(P.sn_ch + ci);
    if (big_phase && !P.sn[c].big) continue;  // small children start phase 2 from dn_s
    const int task = c * P.batch + b;
    if (next < 0) {
      next = task;
    } else {
      const int slot = atomicAdd(ctl + 2, 1);
      Q.q[slot] = task;
      st_release(Q.flag + slot, 1);
    }
  }
  __threadfence();
  if (atomicAdd(ctl + 3, 1) == total - 1) st_release(ctl + 8, 1);  // completed -> all done
  return next;
}

// ---------------------------------------------------------------- backward, big (CTA)
__global__ void __launch_bounds__(KKT_BNT) bwd_big_kernel(DevPlan P, const double* __restrict__ Lx_all,
                                                          const double* __restrict__ Dv_all,
                                                          const double* __restrict__ Y_all, double* Xp_all,
                                                          double* xout, long long xs, TaskQueue Q,
                                                          int* ctl, const int* __restrict__ done, int pcap) {
  extern __shared__ double sm[];
  __shared__ int s_task;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5, nw = nt >> 5;
  const int total = P.ns_bn * P.batch;
  double* xa = sm;                   // [max_front]  x over R_s (own columns then ancestors)
  double* L11 = sm + P.max_front;    // [64*64] (unstaged path)
  double* Pn = L11 + 64 * 64;        // [pcap] staged panel
  if (P.batch == 1 && done && done[0]) return;
  int task = -1;
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
      if (tid == 0) s_task = spawn_children(P, P.sn[s], b, ctl, Q, true, total);
      __syncthreads();
      task = s_task;
      __syncthreads();
      continue;
    }
    if (tid == 0) trace_stamp(P, 2, s, b, 0);
    const SnInfo I = P.sn[s];
    const int r = I.r, w = I.w;
    const double* L = Lx_all + (long long)b * P.nnzL_stored + I.Lp;
    double* Xp = Xp_all + (long long)b * P.n;
    const double* Y = Y_all + (long long)b * P.n;
    const bool staged = (w <= 128) && ((long long)r * w <= pcap);
    if (staged) copy_g2s<false>(Pn, L, r * w, tid, nt);
    for (int q = tid; q < r; q += nt) xa[q] = (q < w) ? ldcg(Y + I.f0 + q) : ldcg(Xp + __ldg(P.sn_rows + I.rp0 + q));
    __syncthreads();
    if (staged) {
      if (warp == 0) bwd_sweep_any(Pn, r, w, Dv_all + (long long)b * P.n + I.f0, xa, lane);
      __syncthreads();
    }
    const int nblk = staged ? 0 : (w + 63) / 64;
    for (int bk = nblk - 1; bk >= 0; bk--) {
      const int k0 = bk * 64, kb = (w - k0) < 64 ? (w - k0) : 64;
      for (int k = warp; k < kb; k += nw) {
        const double* Lk = L + (long long)(k0 + k) * r;
        double acc = 0.0;
        for (int i = k0 + kb + lane; i < r; i += 32) acc = fma(__ldg(Lk + i), xa[i], acc);
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) xa[k0 + k] -= acc;
      }
      for (int q = tid; q < kb * kb; q += nt) {
        const int k = q / kb, i = q % kb;
        L11[q] = (i >= k) ? __ldg(L + (long long)(k0 + k) * r + k0 + i) : 0.0;
      }
      __syncthreads();
      if (warp == 0) {
        for (int k = kb - 1; k >= 0; k--) {
          const double xk = xa[k0 + k] / L11[k * kb + k];
          __syncwarp();
          if (lane == 0) xa[k0 + k] = xk;
          for (int i = lane; i < k; i += 32) xa[k0 + i] = fma(-L11[i * kb + k], xk, xa[k0 + i]);
          __syncwarp();
        }
      }
      __syncthreads();
    }
    double* xo = xout + (long long)b * xs;
    for (int q = tid; q < w; q += nt) {
      Xp[I.f0 + q] = xa[q];
      xo[__ldg(P.perm + I.f0 + q)] = xa[q];
    }
    if (tid == 0) trace_stamp(P, 2, s, b, 1);
    __threadfence();
    __syncthreads();
    if (tid == 0) s_task = spawn_children(P, I, b, ctl, Q, true, total);
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
                                                                 int* ctl, const int* __restrict__ done) {
  extern __shared__ double sm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* Pn = sm + (long long)wid * (KKT_SCAP + P.max_r_small);
  double* xa = Pn + KKT_SCAP;
  const int total = P.ns_s * P.batch;
  if (P.batch == 1 && done && done[0]) return;
  int task = -1;
  for (;;) {
    if (task < 0) {
      int t = 0;
      if (lane == 0) t = pop_task(ctl, P.dn_s, P.n_dn_s, P.batch, Q, total);
      task = __shfl_sync(0xffffffffu, t, 0);
      if (task < 0) break;
    }
    const int s = task / P.batch, b = task % P.batch;
    const SnInfo I = P.sn[s];
    if (done && done[b]) {
      int t = 0;
      if (lane == 0) t = spawn_children(P, I, b, ctl, Q, false, total);
      task = __shfl_sync(0xffffffffu, t, 0);
      continue;
    }
    if (lane == 0) trace_stamp(P, 2, s, b, 0);
    const int r = I.r, w = I.w;
    const double* L = Lx_all + (long long)b * P.nnzL_stored + I.Lp;
    double* Xp = Xp_all + (long long)b * P.n;
    const double* Y = Y_all + (long long)b * P.n;
    copy_g2s<false>(Pn, L, r * w, lane, 32);
    for (int q = lane; q < r; q += 32) xa[q] = (q < w) ? ldcg(Y + I.f0 + q) : ldcg(Xp + __ldg(P.sn_rows + I.rp0 + q));
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
    for (int q = lane; q < w; q += 32) {
      Xp[I.f0 + q] = xa[q];
      xo[__ldg(P.perm + I.f0 + q)] = xa[q];
    }
    if (lane == 0) trace_stamp(P, 2, s, b, 1);
    __threadfence();
    __syncwarp();
    int t = 0;
    if (lane == 0) t = spawn_children(P, I, b, ctl, Q, false, total);
    task = __shfl_sync(0xffffffffu, t, 0);
  }
  warp_exit(ctl, gridDim.x * KKT_WPB);
}

}  // namespace kkt
