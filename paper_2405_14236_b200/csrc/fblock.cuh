// fblock.cuh -- multifrontal factorisation of the small supernodes by subtree blocks (P:512,
// P:1344-1346; the partition is built by sblock_plan.cpp: build_fblocks).
//
// One CTA per block (a whole subtree of small supernodes, contiguous in the postorder): the K
// values of the block's columns and their panel positions, the SnInfo records, the relative-
// index map, the children lists and the level lists are staged by TMA bulk copies (one
// mbarrier transaction); then the levels run leaves first, one warp per supernode, entirely in
// shared memory: assemble the front F (scatter of K, extend-add of the children's update
// matrices -- in child order, from shared memory), partial Cholesky by the warp
// (front_factor_warp2: L panel in place, U = Schur complement), panel -> Lx.  The root's U goes
// to the global update storage and the parent is signalled as in factor_small_kernel (a big
// parent counts its small children; a small parent outside every block is continued on warp 0
// by the per-node code).  Same operations in the same order as factor_small_kernel: bitwise
// the same factor.
#pragma once
#include "factor.cuh"
#include "sblock.cuh"

namespace kkt {

constexpr int FB_NT = 128;   // threads per CTA (4 warps)
constexpr int FB_NW = FB_NT / 32;
#ifndef FB_MINB
#define FB_MINB 3
#endif

struct FBPlan {
  const FBlk* blk;
  int nblk;
  const int* meta;
  const int* up_init;   // childless small supernodes outside every block
  int n_up_init;
  int smem_doubles;
};

// One call site of the register-hungry warp front factorisation for both paths of the kernel
__device__ __forceinline__ void fb_front_factor(double* F, double* U, int r, int w, int lane, double* dinv, int* fail_k) {
  front_factor_warp2(F, U, r, w, lane, dinv, fail_k);
}

// Per-node factorisation of a small supernode outside every block by one warp, continued
// upward while this warp's child was the last to arrive (the loop body of factor_small_kernel).
__device__ __forceinline__ void factor_chain_warp(const DevPlan& P, int s, SnInfo I, int b, const double* Kv,
                                                  double* Lx, double* Ub, double* Dv, int* cnt, int* fail_all,
                                                  double* region, int lane) {
  auto wsync = [] { __syncwarp(); };
  for (;;) {
    if (lane == 0) trace_stamp(P, 0, s, b, 0);
    const int R = I.r - I.w;
    const long long usz = I.par >= 0 ? (long long)R * (R + 1) / 2 : 0;
    double* F = region;
    double* U = region + I.r * I.w;
    SnInfo Ip;
    if (I.par >= 0) Ip = P.sn[I.par];
    assemble_front<2>(P, I, F, U, usz, Kv, Ub, lane, 32, wsync);  // MLP 2: the block kernel's register budget
    int fk = -1;
    fb_front_factor(F, U, I.r, I.w, lane, Dv + I.f0, &fk);
    double* Lg = Lx + I.Lp;
    for (int q = lane; q < I.r * I.w; q += 32) Lg[q] = F[q];
    if (usz) {
      double* Ug = Ub + I.Up;
      for (int q = lane; q < usz; q += 32) Ug[q] = U[q];
    }
    if (lane == 0 && fk >= 0) atomicMin(fail_all, I.f0 + fk);
    if (lane == 0) trace_stamp(P, 0, s, b, 1);
    if (I.par < 0) break;
    if (!warp_signal_parent(I, Ip, cnt, lane, true)) break;
    s = I.par;
    I = Ip;
  }
}

template <int MINB>
__global__ void __launch_bounds__(FB_NT, MINB) factor_block_kernel(DevPlan P, FBPlan B, const double* __restrict__ Kv_all,
                                                                  double* Lx_all, double* U_all, double* Dv_all,
                                                                  int* cnt_all, int* ctl, int* fail_all) {
  extern __shared__ __align__(16) double sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ int s_task, s_qc[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) mbar_init(&bar, 1);
  __syncthreads();
  pdl_launch_dependents();
  uint32_t phase = 0;
  const int nblk_t = B.nblk * P.batch, ntask = (B.nblk + B.n_up_init) * P.batch;
  for (;;) {
    const int t = next_task(ctl, &s_task);  // (barrier: the previous task's shared reads are done)
    if (t >= ntask) break;
    const int b = t % P.batch;
    double* Lx = Lx_all + (long long)b * P.nnzL_stored;
    double* Ub = U_all + (long long)b * P.update_doubles;
    double* Dv = Dv_all + (long long)b * P.n;
    const double* Kv = Kv_all + (long long)b * P.nnzK;
    int* cnt = cnt_all + (long long)b * P.ns;
    if (t >= nblk_t) {  // a childless small supernode outside the blocks (warp 0)
      if (warp == 0) {
        const int s = __ldg(B.up_init + (t - nblk_t) / P.batch);
#ifndef FB_NOCHAIN
        factor_chain_warp(P, s, P.sn[s], b, Kv, Lx, Ub, Dv, cnt, fail_all, sm, lane);
#endif
      }
      continue;
    }
    const FBlk K = B.blk[t / P.batch];
    const int nn = K.s_hi - K.s_lo + 1;
    const FBLayout O = fb_layout(nn, K.nlev, K.nL, K.nU, K.nK, K.nr, K.nch);
    const SBRange rK = sb_range(Kv + K.K0, K.nK), rP = sb_range(P.kpos + K.K0, K.nK),
                  rS = sb_range(P.sn + K.s_lo, nn), rR = sb_range(P.sn_rel + K.RP0, K.nr),
                  rC = sb_range(P.sn_ch + K.CP0, K.nch), rM = sb_range(B.meta + K.m0, K.nlev + 1 + nn);
    if (tid == 0) {
      fence_proxy_async_smem();
      mbar_arrive_expect_tx(&bar, rK.bytes + rP.bytes + rS.bytes + rR.bytes + rC.bytes + rM.bytes);
      bulk_g2s(sm + O.sn, rS.g0, rS.bytes, &bar);
      bulk_g2s(sm + O.meta, rM.g0, rM.bytes, &bar);
      if (rK.bytes) bulk_g2s(sm + O.K, rK.g0, rK.bytes, &bar);
      if (rP.bytes) bulk_g2s(sm + O.kpos, rP.g0, rP.bytes, &bar);
      bulk_g2s(sm + O.rel, rR.g0, rR.bytes, &bar);
      if (rC.bytes) bulk_g2s(sm + O.ch, rC.g0, rC.bytes, &bar);
    }
    mbar_wait(&bar, phase);
    phase ^= 1;
    __syncthreads();
    double* Fb = sm + O.F - K.L0;                                 // Fb + I.Lp = front / panel
    double* Ubs = sm + O.U - K.U0;                                // Ubs + I.Up = update matrix
    const double* Ks = sm + O.K + rK.shift - K.K0;                // Ks[k], k in [I.k0, I.k1)
    const int* kp = reinterpret_cast<const int*>(sm + O.kpos) + rP.shift - K.K0;
    const SnInfo* Ss = reinterpret_cast<const SnInfo*>(sm + O.sn) - K.s_lo;
    const int* relb = reinterpret_cast<const int*>(sm + O.rel) + rR.shift - K.RP0;
    const int* chs = reinterpret_cast<const int*>(sm + O.ch) + rC.shift - K.CP0;
    const int* lvl = reinterpret_cast<const int*>(sm + O.meta) + rM.shift;
    const int* nodes = lvl + K.nlev + 1;
    // ready queue: leaves first, a parent pushed by its last child; warps take slots by ticket
    int* rq = reinterpret_cast<int*>(sm + O.q);
    int* pend = rq + nn;
    const int nleaf = lvl[1];
    for (int q = tid; q < nn; q += FB_NT) {
      rq[q] = q < nleaf ? nodes[q] : -1;
      const SnInfo& Iq = Ss[K.s_lo + q];
      pend[q] = Iq.c1 - Iq.c0;
    }
    if (tid == 0) { s_qc[0] = 0; s_qc[1] = nleaf; }
    __syncthreads();
    volatile int* vrq = rq;
    for (;;) {
      int tq = 0, ls = -1;
      if (lane == 0) tq = atomicAdd(s_qc, 1);
      tq = __shfl_sync(0xffffffffu, tq, 0);
      if (tq >= nn) break;
      if (lane == 0) {
        while ((ls = vrq[tq]) < 0) { __nanosleep(40); }
        __threadfence_block();
      }
      ls = __shfl_sync(0xffffffffu, ls, 0);
      {
        const int s = K.s_lo + ls;
        const SnInfo& I = Ss[s];
        if (lane == 0) trace_stamp(P, 0, s, b, 0);
        const int r = I.r, w = I.w, R = r - w;
        const int usz = I.par >= 0 ? R * (R + 1) / 2 : 0;
        double* F = Fb + I.Lp;
        double* U = Ubs + I.Up;
        for (int q = lane; q < r * w; q += 32) F[q] = 0.0;
        for (int q = lane; q < usz; q += 32) U[q] = 0.0;
        __syncwarp();
        for (int k = I.k0 + lane; k < I.k1; k += 32) F[kp[k]] = Ks[k];
        __syncwarp();
        for (int ci = I.c0; ci < I.c1; ci++) {
          const SnInfo& C = Ss[chs[ci]];
          const int Rc = C.r - C.w;
          const int* rel = relb + C.rp0 + C.w;
          const double* Uc = Ubs + C.Up;
          const int tot = Rc * (Rc + 1) / 2;
          int jc = 0, cs = 0;  // column decode of the packed child matrix (monotone per lane)
          for (int q = lane; q < tot; q += 32) {
            while (q >= cs + (Rc - jc)) { cs += Rc - jc; jc++; }
            const int ic = jc + (q - cs);
            const int pj = rel[jc], pi = rel[ic];
            const double v = Uc[q];
            if (pj < w) F[pj * r + pi] += v;
            else U[upk(pi - w, pj - w, R)] += v;
          }
          __syncwarp();
        }
        int fk = -1;
        fb_front_factor(F, U, r, w, lane, Dv + I.f0, &fk);
        double* Lg = Lx + I.Lp;
        for (int q = lane; q < r * w; q += 32) Lg[q] = F[q];
        if (lane == 0) {
          if (fk >= 0) atomicMin(fail_all, I.f0 + fk);
          trace_stamp(P, 0, s, b, 1);
          if (s != K.s_hi) {
            const int pl = I.par - K.s_lo;
            __threadfence_block();
            if (atomicSub(pend + pl, 1) == 1) vrq[atomicAdd(s_qc + 1, 1)] = pl;
          }
        }
      }
    }
    __syncthreads();
    // the root's update matrix to the global storage, then the hand-off to its parent
    const SnInfo I = Ss[K.s_hi];
    if (I.par >= 0) {
      const int R = I.r - I.w, usz = R * (R + 1) / 2;
      const double* U = Ubs + I.Up;
      for (int q = tid; q < usz; q += FB_NT) Ub[I.Up + q] = U[q];
      __syncthreads();  // every thread's U entries precede warp 0's release (warp_signal_parent)
      if (warp == 0) {
        const SnInfo Ip = P.sn[I.par];
        if (warp_signal_parent(I, Ip, cnt, lane, true)) {
          __syncwarp();
#ifndef FB_NOCHAIN
          factor_chain_warp(P, I.par, Ip, b, Kv, Lx, Ub, Dv, cnt, fail_all, sm, lane);
#endif
        }
      }
    }
  }
  persistent_exit(ctl);
}

}  // namespace kkt
