// factor.cuh -- persistent multifrontal supernodal Cholesky, P K P^T = L L^T without pivoting
// ("factorize it using sparse Cholesky").
//
// Front of supernode s (columns f0..f0+w, rows R_s with r = |R_s|, R = r - w):
//   [F | U]:  F = panel r x w column-major (becomes L's columns),  U = packed lower R x R
//   assembly:  F <- K(R_s, cols(s)) ; U <- 0 ; then for each child c (fixed order):
//              extend-add U_c through the relative-index map rel_c       (deterministic)
//   partial factorisation:  F11 = L11 L11^T, L21 = F21 L11^-T, U <- U - L21 L21^T
//   U is kept for the parent; F is written to L.
//
// Phase 1 (factor_small_kernel): one WARP per supernode for the subtrees whose fronts fit
//   KKT_SCAP doubles; the front lives in a per-warp shared-memory slice.
// Phase 2 (factor_big_kernel): one CTA per remaining (top) supernode; front in shared memory
//   when it fits, otherwise in global memory (L2) with a 64x64 register-tiled SYRK.
#pragma once
#include "dense.cuh"
#include "ldlt.cuh"

namespace kkt {

__device__ __forceinline__ int warp_ticket(int* ctl) {
  int t = 0;
  if ((threadIdx.x & 31) == 0) t = atomicAdd(ctl, 1);
  return __shfl_sync(0xffffffffu, t, 0);
}
__device__ __forceinline__ void warp_exit(int* ctl, int nwarps_total) {
  if ((threadIdx.x & 31) == 0) {
    __threadfence();
    int e = atomicAdd(ctl + 1, 1);
    if (e == nwarps_total - 1) reset_ctl(ctl);
  }
}


// ------------------------------------------------------------------ front assembly
// F, U may live in shared or global memory; `nt`/`tid` describe the cooperating group
// (a warp: nt = 32, tid = lane; a CTA: nt = blockDim, tid = threadIdx).  The caller
// synchronises the group between the zero/scatter/extend-add stages via `sync`.
template <int MLP = KKT_MLP, class Sync>
__device__ __forceinline__ void assemble_front(const DevPlan& P, const SnInfo& I, double* F,
                                               double* U, long long usz,
                                               const double* __restrict__ Kv, const double* Ub,
                                               int tid, int nt, Sync sync) {
  const int w = I.w, r = I.r, R = r - w;
  const long long pw = (long long)r * w;
  for (long long q = tid; q < pw; q += nt) F[q] = 0.0;
  for (long long q = tid; q < usz; q += nt) U[q] = 0.0;
  sync();
  // K entries of the supernode's columns: batched loads, then scatter
  for (int base = I.k0 + tid; base < I.k1; base += nt * MLP) {
    int pos[MLP];
    double val[MLP];
#pragma unroll
    for (int u = 0; u < MLP; u++) {
      const int k = base + u * nt;
      if (k < I.k1) { pos[u] = __ldg(P.kpos + k); val[u] = __ldg(Kv + k); }
    }
#pragma unroll
    for (int u = 0; u < MLP; u++)
      if (base + u * nt < I.k1) F[pos[u]] = val[u];
  }
  sync();
  SnInfo Cn;
  if (I.c0 < I.c1) Cn = P.chinfo[I.c0];
  for (int ci = I.c0; ci < I.c1; ci++) {
    const SnInfo C = Cn;
    if (ci + 1 < I.c1) Cn = P.chinfo[ci + 1];  // prefetch the next child's metadata
    const int Rc = C.r - C.w;
    const int* rel = P.sn_rel + C.rp0 + C.w;
    const double* Uc = Ub + C.Up;
    const long long tot = (long long)Rc * (Rc + 1) / 2;
    // each member walks the packed child matrix with stride nt (monotone q -> incremental
    // column decode); MLP entries are loaded before any is accumulated.  Positions within
    // one child are distinct, so there are no conflicts; children are applied in order.
    int jc = 0;
    long long cs = 0;  // start of column jc
    for (long long base = tid; base < tot; base += (long long)nt * MLP) {
      int pi[MLP], pj[MLP];
      double v[MLP];
#pragma unroll
      for (int u = 0; u < MLP; u++) {
        const long long q = base + (long long)u * nt;
        if (q < tot) {
          while (q >= cs + (Rc - jc)) { cs += Rc - jc; jc++; }
          const int ic = jc + (int)(q - cs);
          pj[u] = __ldg(rel + jc);
          pi[u] = __ldg(rel + ic);
          v[u] = ldcg(Uc + q);
        }
      }
#pragma unroll
      for (int u = 0; u < MLP; u++) {
        if (base + (long long)u * nt < tot) {
          if (pj[u] < w) F[(long long)pj[u] * r + pi[u]] += v[u];
          else U[upk(pi[u] - w, pj[u] - w, R)] += v[u];
        }
      }
    }
    sync();
  }
}

// =====================================================================================
// Spin-free scheduling (bottom-up).  Workers take tasks only from a static ready list
// (leaves); when a worker finishes supernode s it increments its parent's counter with an
// acq_rel atomic, and the LAST child to finish continues with the parent itself.  No worker
// ever waits on a dependency.  Phase 1 (small, warps) stops at a big parent (it only counts);
// phase 2 (big, CTAs) starts from the big supernodes without big children, whose counters
// phase 1 already completed (reset on entry).
// =====================================================================================
__device__ __forceinline__ bool warp_signal_parent(const SnInfo& I, const SnInfo& Ip, int* cnt,
                                                   int lane, bool phase_small) {
  __syncwarp();  // lanes' writes are ordered before lane 0's release (acq_rel / release atomic)
  int last = 0;
  if (lane == 0) {
    if (phase_small && Ip.big) {
      red_release_add(cnt + I.par, 1);
    } else {
      const int old = atom_add_acq_rel(cnt + I.par, 1);
      last = (old == Ip.c1 - Ip.c0 - 1);
      if (last) cnt[I.par] = 0;
    }
  }
  return __shfl_sync(0xffffffffu, last, 0) != 0;
}

// MINB = resident CTAs per SM the register allocation must allow: 1 for latency-bound trees
// (no spills on the critical path), 3 for throughput-bound ones (many small supernodes / batches)
template <int MINB>
__global__ void __launch_bounds__(KKT_WPB * 32, MINB) factor_small_kernel(DevPlan P, const double* __restrict__ Kv_all,
                                                                    double* Lx_all, double* U_all, double* Dv_all,
                                                                    int* cnt_all, int* ctl, int* fail_all) {
  extern __shared__ double sm[];
  __shared__ SnInfo s_ip[KKT_WPB];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* region = sm + (long long)wid * KKT_SCAP;
  const int ninit = P.n_up_s * P.batch;
  auto wsync = [] { __syncwarp(); };
  pdl_launch_dependents();
  for (;;) {
    const int t = warp_ticket(ctl);
    if (t >= ninit) break;
    const int b = t % P.batch;
    int s = __ldg(P.up_s + t / P.batch);
    int* cnt = cnt_all + (long long)b * P.ns;
    double* Lx = Lx_all + (long long)b * P.nnzL_stored;
    double* Ub = U_all + (long long)b * P.update_doubles;
    const double* Kv = Kv_all + (long long)b * P.nnzK;
    bool from_smem = false;  // continuing with the parent: its metadata is already in s_ip
    for (;;) {
      if (lane == 0) trace_stamp(P, 0, s, b, 0);
      const SnInfo I = from_smem ? s_ip[wid] : P.sn[s];
      const int R = I.r - I.w;
      const long long usz = I.par >= 0 ? (long long)R * (R + 1) / 2 : 0;
      double* F = region;
      double* U = region + I.r * I.w;
      assemble_front(P, I, F, U, usz, Kv, Ub, lane, 32, wsync);
      if (lane == 0) trace_stamp(P, 0, s, b, 2);
      int fk = -1;
      front_factor_warp2(F, U, I.r, I.w, lane, Dv_all + (long long)b * P.n + I.f0, &fk);
      if (lane == 0) trace_stamp(P, 0, s, b, 3);
      // parent metadata in flight while the panel and update matrix are written out: lane k < 16
      // holds int k of the parent's 64-byte SnInfo
      const int ipw = (I.par >= 0 && lane < 16) ? __ldg(reinterpret_cast<const int*>(P.sn + I.par) + lane) : 0;
      double* Lg = Lx + I.Lp;
      for (int q = lane; q < I.r * I.w; q += 32) Lg[q] = F[q];
      if (usz) {
        double* Ug = Ub + I.Up;
        for (int q = lane; q < usz; q += 32) Ug[q] = U[q];
      }
      if (lane == 0 && fk >= 0) atomicMin(fail_all, I.f0 + fk);
      if (lane == 0) trace_stamp(P, 0, s, b, 1);
      if (I.par < 0) break;
      if (lane < 16) reinterpret_cast<int*>(s_ip + wid)[lane] = ipw;
      __syncwarp();
      if (!warp_signal_parent(I, s_ip[wid], cnt, lane, true)) break;
      s = I.par;
      from_smem = true;
    }
  }
  warp_exit(ctl, gridDim.x * KKT_WPB);
}

// =====================================================================================
// Phase 2: one CTA per big supernode (continuation scheduling, see above).
// =====================================================================================
template <bool SG>
__global__ void __launch_bounds__(KKT_BNT) factor_big_kernel(DevPlan P, const double* __restrict__ Kv_all,
                                                             double* Lx_all, double* U_all, double* Dv_all,
                                                             int* cnt_all, int* ctl, int* fail_all,
                                                             long long smem_cap) {
  extern __shared__ double sm[];
  __shared__ int s_task, s_fail, s_last, s_pnbig;
  __shared__ SnInfo s_I, s_Ip;  // current supernode, and its parent (prefetched at node start)
  const int tid = threadIdx.x;
  const int ninit = P.n_up_bf * P.batch;
  auto bsync = [] { __syncthreads(); };
  for (;;) {
    const int t = next_task(ctl, &s_task);
    if (t >= ninit) break;
    const int b = t % P.batch;
    int s = __ldg(P.up_bf + t / P.batch);
    int* cnt = cnt_all + (long long)b * P.ns;
    double* Lx = Lx_all + (long long)b * P.nnzL_stored;
    double* Ub = U_all + (long long)b * P.update_doubles;
    const double* Kv = Kv_all + (long long)b * P.nnzK;
    if (tid == 0) {  // all children are small: wait for phase 1 to have counted them
      const SnInfo I0 = P.sn[s];
      s_I = I0;
      wait_children_reset(cnt + s, I0.c1 - I0.c0);
    }
    __syncthreads();
    for (;;) {
      if (tid == 0) trace_stamp(P, 0, s, b, 0);
      const SnInfo I = s_I;
      const int r = I.r, w = I.w, R = r - w;
      if (tid == 0) s_fail = -1;
      if (tid == 32 && I.par >= 0) { s_Ip = P.sn[I.par]; s_pnbig = __ldg(P.sn_nbig + I.par); }  // off the critical warp
      __syncthreads();
      const long long pw = (long long)r * w;
      const long long usz = (I.par >= 0) ? (long long)R * (R + 1) / 2 : 0;
      const bool in_smem = (pw + usz) <= smem_cap;
      double* F = in_smem ? sm : Lx + I.Lp;
      double* U = in_smem ? sm + pw : (usz ? Ub + I.Up : nullptr);
      assemble_front(P, I, F, U, usz, Kv, Ub, tid, blockDim.x, bsync);
      if (tid == 0) trace_stamp(P, 0, s, b, 2);
      double* dv = Dv_all + (long long)b * P.n + I.f0;
      // left-looking 32-column blocks for medium/large fronts in shared memory (one U update,
      // three barriers per block); narrow short fronts keep the 8-column right-looking kernel
      if (SG) front_factor_cta_ldlt(F, U, r, w, dv, &s_fail, P.Sg + (long long)b * P.n + I.f0, Kv, P.Kp, I.f0,
                                    P.inert + 3 * b);
      else if (in_smem && (w >= 20 || r >= 128)) front_factor_cta_ll(F, U, r, w, dv, &s_fail);
      else front_factor_cta<8>(F, U, r, w, dv, &s_fail);
      __syncthreads();
      if (tid == 0) trace_stamp(P, 0, s, b, 3);
      if (tid == 0) trace_stamp(P, 0, s, b, 4);
      if (in_smem) {
        double* Lg = Lx + I.Lp;
        for (long long q = tid; q < pw; q += blockDim.x) Lg[q] = F[q];
        if (usz) {
          double* Ug = Ub + I.Up;
          for (long long q = tid; q < usz; q += blockDim.x) Ug[q] = U[q];
        }
      }
      if (tid == 0 && s_fail >= 0) atomicMin(fail_all, I.f0 + s_fail);
      if (tid == 0) trace_stamp(P, 0, s, b, 1);
      if (I.par < 0) break;
      __syncthreads();  // every thread's panel / U writes precede thread 0's release (cumulative)
      if (tid == 0) {
        const SnInfo Ip = s_Ip;
        if (Ip.huge) {            // the whole-GPU phase takes it from here
          red_release_add(cnt + I.par, 1);
          s_last = 0;
        } else {
          s_last = big_child_arrive_n(cnt + I.par, s_pnbig, Ip.c1 - Ip.c0);
          if (s_last) s_I = Ip;
        }
      }
      __syncthreads();
      if (!s_last) break;
      s = I.par;
    }
  }
  persistent_exit(ctl);
}

}  // namespace kkt
