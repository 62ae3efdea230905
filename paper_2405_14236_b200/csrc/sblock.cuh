// sblock.cuh -- triangular solves of the small supernodes by subtree blocks (P:1376-1377,
// SURVEY §8(a) a3; the plan is built by sblock_plan.cpp, see sblock.h).
//
// Forward (bottom-up), one CTA per block:
//   stage   TMA bulk copies of the block's contiguous ranges -- L panels, SnInfo records,
//           relative-index map, children lists, inverse pivots, level lists -- into shared
//           memory (one mbarrier transaction); meanwhile the threads gather b(perm(cols)).
//   levels  leaves first: one warp per supernode, v = [b(cols); 0] + extend-add of the
//           children's u (in child order, from shared memory), y = L11^-1 v[0:w),
//           u = v[w:r) - L21 y (fwd_sweep_warp on the staged panel), y -> Y; CTA barrier.
//   hand-off the root's u goes to the parent exactly as in the per-node kernel
//           (warp_signal_parent); a small parent outside every block is continued on warp 0
//           with the per-node code (fwd_chain_warp).
// Backward (top-down), one CTA per task: a task is a block (staged the same way plus y, the
// permutation and the ancestors' x of the root's update rows; levels root first, x written
// to Xp and to the caller's x) or a single small supernode (warp 0, per-node code).
// The arithmetic per supernode -- order of the extend-add, the sweeps -- is that of the
// per-node kernels (fwd_small_kernel / bwd_small_kernel): results are bitwise identical.
#pragma once
#include "sblock.h"
#include "trsv.cuh"

namespace kkt {

// small supernodes have r <= 64 (r w + R(R+1)/2 <= KKT_SCAP): two register slots at most
__device__ __forceinline__ void fwd_sweep_sm(const double* Lp, int r, int w, const double* dv, double* v, int lane) {
  if (r <= 32) fwd_sweep_warp<1>(Lp, r, w, dv, v, lane);
  else fwd_sweep_warp<2>(Lp, r, w, dv, v, lane);
}
__device__ __forceinline__ void bwd_sweep_sm(const double* Lp, int r, int w, const double* dv, double* xa, int lane) {
  if (w <= 32) bwd_sweep_warp<1>(Lp, r, w, dv, xa, lane);
  else bwd_sweep_warp<2>(Lp, r, w, dv, xa, lane);
}

// resident CTAs per SM the register allocation must allow: 24 warps per SM at <= 85 registers
template <int NT> constexpr int sb_minb() { return 768 / NT; }

struct SBPlan {
  const SBlk* blk;
  int nblk;
  const int* blk_of;    // [ns]: block index of a block root, -2 inside a block, -1 otherwise
  const int* meta;      // level offsets + node lists
  const int* lrow;      // parallel to sn_rows
  int smem_doubles;
  // whole-tree schedules of the solve (small + big supernodes; the huge fronts of the tile
  // solve excluded unless the plan view solves them as CTA supernodes)
  const int* fwd_order; // forward initial tasks (block index >= 0, childless big supernode -s-1),
  int n_fwd;            //   longest estimated path to the top first
  const int2* bwd_order;// backward tasks {supernode, supernode to wait for or -1} in estimated
  int n_bwd;            //   start order (topological: parents first)
  int* zbuf;            // the tile solve's dependency counters, zeroed by the forward kernel
  int zn;               //   (the next kernel in the stream; no separate memset node) or null
};

// one contiguous range staged by TMA: shift = elements between the 16-byte-aligned start and
// the first element; bytes rounded up to 16
struct SBRange {
  const void* g0;
  uint32_t bytes;
  int shift;
};
template <class T>
__device__ __forceinline__ SBRange sb_range(const T* src, long long n) {
  const uintptr_t g = (uintptr_t)src, a = g & ~(uintptr_t)15;
  SBRange r;
  r.g0 = (const void*)a;
  r.shift = (int)((g - a) / sizeof(T));
  r.bytes = (uint32_t)(((g - a) + (uintptr_t)n * sizeof(T) + 15) & ~(uintptr_t)15);
  return r;
}


// ---------------------------------------------------------------- forward, one block
// Stage the block's ranges (TMA), gather b, run the levels leaves first; on return the root's
// v (= [y; u]) is in shared memory at the returned pointer.
template <int NT>
__device__ __forceinline__ const double* fwd_block(const DevPlan& P, const SBPlan& B, const SBlk& K, int b,
                                                   const double* Lb, const double* Dv, const double* bb,
                                                   double* Y, double* sm, uint64_t* bar, uint32_t& phase,
                                                   int* qc, int tid, int lane, int warp) {
  const int nn = K.s_hi - K.s_lo + 1;
  const SBLayout O = sb_layout(nn, K.nlev, K.nL, K.ncol, K.nr, K.nch, K.Rroot, NT / 32);
  const SBRange rL = sb_range(Lb + K.L0, K.nL), rD = sb_range(Dv + K.F0, K.ncol),
                rS = sb_range(P.sn + K.s_lo, nn), rR = sb_range(P.sn_rel + K.RP0, K.nr),
                rC = sb_range(P.sn_ch + K.CP0, K.nch), rM = sb_range(B.meta + K.m0, K.nlev + 1 + nn);
  if (tid == 0) {
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(bar, rL.bytes + rD.bytes + rS.bytes + rR.bytes + rC.bytes + rM.bytes);
    bulk_g2s(sm + O.L, rL.g0, rL.bytes, bar);
    bulk_g2s(sm + O.sn, rS.g0, rS.bytes, bar);
    bulk_g2s(sm + O.meta, rM.g0, rM.bytes, bar);
    if (rR.bytes) bulk_g2s(sm + O.rel, rR.g0, rR.bytes, bar);
    if (rC.bytes) bulk_g2s(sm + O.ch, rC.g0, rC.bytes, bar);
    bulk_g2s(sm + O.D, rD.g0, rD.bytes, bar);
  }
  // right-hand side of the block's columns (generic loads, overlapping the bulk copies)
  double* bcol = sm + O.bcol;
  for (int c = tid; c < K.ncol; c += NT) bcol[c] = bb[__ldg(P.perm + K.F0 + c)];
  mbar_wait(bar, phase);
  phase ^= 1;
  __syncthreads();
  const double* Ls = sm + O.L + rL.shift - K.L0;          // Ls + I.Lp = staged panel
  const double* Ds = sm + O.D + rD.shift - K.F0;          // Ds + I.f0
  const SnInfo* Ss = reinterpret_cast<const SnInfo*>(sm + O.sn) - K.s_lo;
  const int* rel = reinterpret_cast<const int*>(sm + O.rel) + rR.shift - K.RP0;
  const int* chs = reinterpret_cast<const int*>(sm + O.ch) + rC.shift - K.CP0;
  const int* lvl = reinterpret_cast<const int*>(sm + O.meta) + rM.shift;
  const int* nodes = lvl + K.nlev + 1;
  double* vb = sm + O.v - K.RP0;                          // vb + I.rp0 = the supernode's v
  // ready queue of the block's supernodes: leaves (level 0) first, a parent is pushed by its
  // last child (pending counts); warps take queue slots by ticket -- no level barriers
  int* rq = reinterpret_cast<int*>(sm + O.q);
  int* pend = rq + nn;
  const int nleaf = lvl[1];
  for (int t = tid; t < nn; t += NT) {
    rq[t] = t < nleaf ? nodes[t] : -1;
    const SnInfo& It = Ss[K.s_lo + t];
    pend[t] = It.c1 - It.c0;
  }
  if (tid == 0) { qc[0] = 0; qc[1] = nleaf; }
  __syncthreads();
  volatile int* vrq = rq;
  for (;;) {
    int t = 0, ls = -1;
    if (lane == 0) t = atomicAdd(qc, 1);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= nn) break;
    if (lane == 0) {
      while ((ls = vrq[t]) < 0) { __nanosleep(40); }
      __threadfence_block();
    }
    ls = __shfl_sync(0xffffffffu, ls, 0);
    const int s = K.s_lo + ls;
    const SnInfo& I = Ss[s];
    if (lane == 0) trace_stamp(P, 1, s, b, 0);
    const int r = I.r, w = I.w, f0 = I.f0, c0 = I.c0, c1 = I.c1;
    double* v = vb + I.rp0;
    for (int q = lane; q < r; q += 32) v[q] = (q < w) ? bcol[f0 - K.F0 + q] : 0.0;
    __syncwarp();
    for (int c = c0; c < c1; c++) {
      const SnInfo& C = Ss[chs[c]];
      const int Rc = C.r - C.w;
      const double* vc = vb + C.rp0 + C.w;
      const int* rc = rel + C.rp0 + C.w;
      for (int q = lane; q < Rc; q += 32) v[rc[q]] += vc[q];
      __syncwarp();
    }
    fwd_sweep_sm(Ls + I.Lp, r, w, Ds + f0, v, lane);
    __syncwarp();
    for (int q = lane; q < w; q += 32) Y[f0 + q] = v[q];
    if (lane == 0) {
      trace_stamp(P, 1, s, b, 1);
      if (s != K.s_hi) {
        const int pl = I.par - K.s_lo;
        __threadfence_block();
        if (atomicSub(pend + pl, 1) == 1) vrq[atomicAdd(qc + 1, 1)] = pl;
      }
    }
  }
  __syncthreads();
  return vb + Ss[K.s_hi].rp0;
}

// Forward of one small supernode outside every block by one warp (the per-node code of
// fwd_small_kernel with fewer registers; same sums in the same order).  Pn / v: scratch.
__device__ __forceinline__ void fwd_single_warp(const DevPlan& P, const SnInfo& I, int s, int b, const double* Lb,
                                                const double* Dv, const double* bb, double* Y, double* uv,
                                                double* Pn, double* v, int lane) {
  if (lane == 0) trace_stamp(P, 1, s, b, 0);
  const int r = I.r, w = I.w;
  copy_g2s<false>(Pn, Lb + I.Lp, r * w, lane, 32);
  for (int q = lane; q < r; q += 32) v[q] = (q < w) ? bb[__ldg(P.perm + I.f0 + q)] : 0.0;
  __syncwarp();
  for (int c = I.c0; c < I.c1; c++) {
    const int4 h4 = __ldg(reinterpret_cast<const int4*>(P.chinfo + c));  // f0, w, r, rp0
    const int uvp = __ldg(reinterpret_cast<const int*>(P.chinfo + c) + 10);
    const int Rq = h4.z - h4.y;
    for (int q = lane; q < Rq; q += 32) v[__ldg(P.sn_rel + h4.w + h4.y + q)] += ldcg(uv + uvp + q);
    __syncwarp();
  }
  fwd_sweep_sm(Pn, r, w, Dv + I.f0, v, lane);
  __syncwarp();
  for (int q = lane; q < w; q += 32) Y[I.f0 + q] = v[q];
  if (I.par >= 0)
    for (int q = lane; q < r - w; q += 32) uv[I.uvp + q] = v[w + q];
  if (lane == 0) trace_stamp(P, 1, s, b, 1);
}

// Blocked sweeps of a supernode without L11^-1 inside the tree kernels (the CTA view of the
// large fronts), with the arithmetic of cta_fwd_blocked / cta_bwd_blocked but few registers: the
// 32 x 32 diagonal block is staged in shared memory (Ds, pitch 33) instead of registers, the rows
// below take their 32 column values 8 at a time, and the backward partial sums run 8 columns at
// a time (per column the same per-thread order and the same butterfly).  Ds: >= 32 * 33 doubles,
// part: >= 8 * 32 doubles.
template <int NT>
__device__ __forceinline__ void cta_fwd_lite(const double* __restrict__ L, int r, int w, const double* __restrict__ dv,
                                             double* v, double* Ds, int tid) {
  const int lane = tid & 31, warp = tid >> 5;
  for (int c0 = 0; c0 < w; c0 += 32) {
    const int kb = min(32, w - c0);
    for (int q = tid; q < 32 * 32; q += NT) {  // diagonal block, column-major, pitch 33
      const int k = q >> 5, i = q & 31;
      Ds[k * 33 + i] = (i < kb && k < kb && k < i) ? __ldg(L + (long long)(c0 + k) * r + c0 + i) : 0.0;
    }
    __syncthreads();
    if (warp == 0) {
      const int row = c0 + lane;
      double x = (lane < kb) ? v[row] : 0.0;
      const double di = (lane < kb) ? __ldg(dv + row) : 0.0;
      for (int k = 0; k < kb; k++) {
        const double yk = __shfl_sync(0xffffffffu, x * di, k);
        if (lane == k) x = yk;
        else if (lane > k) x = fma(-Ds[k * 33 + lane], yk, x);
      }
      if (lane < kb) v[row] = x;
    }
    __syncthreads();
    for (int i = c0 + kb + tid; i < r; i += NT) {
      double a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int cb = 0; cb < 32; cb += 8) {
        double l[8];
#pragma unroll
        for (int u = 0; u < 8; u++) l[u] = (cb + u < kb) ? __ldg(L + (long long)(c0 + cb + u) * r + i) : 0.0;
#pragma unroll
        for (int u = 0; u < 8; u += 2) {
          a0 = fma(l[u], (cb + u < kb) ? v[c0 + cb + u] : 0.0, a0);
          a1 = fma(l[u + 1], (cb + u + 1 < kb) ? v[c0 + cb + u + 1] : 0.0, a1);
        }
      }
      v[i] -= a0 + a1;
    }
    __syncthreads();
  }
}

template <int NT>
__device__ __forceinline__ void cta_bwd_lite(const double* __restrict__ L, int r, int w, const double* __restrict__ dv,
                                             double* xa, double* Ds, double* part, int tid) {
  const int lane = tid & 31, warp = tid >> 5;
  constexpr int nw = NT / 32;
  for (int c0 = ((w - 1) / 32) * 32; c0 >= 0; c0 -= 32) {
    const int kb = min(32, w - c0);
    for (int q = tid; q < 32 * 32; q += NT) {  // diagonal block, column-major, pitch 33
      const int k = q >> 5, i = q & 31;
      Ds[k * 33 + i] = (i < kb && k < kb && k < i) ? __ldg(L + (long long)(c0 + k) * r + c0 + i) : 0.0;
    }
    double tot = 0.0;  // lane c (warp 0): sum of the warp partials of column c0 + c
    for (int g = 0; g < 32; g += 8) {
      double p[8];
#pragma unroll
      for (int c = 0; c < 8; c++) p[c] = 0.0;
      for (int i = c0 + kb + tid; i < r; i += NT) {
        const double xi = xa[i];
#pragma unroll
        for (int c = 0; c < 8; c++) p[c] = fma((g + c < kb) ? __ldg(L + (long long)(c0 + g + c) * r + i) : 0.0, xi, p[c]);
      }
#pragma unroll
      for (int c = 0; c < 8; c++) {
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) p[c] += __shfl_xor_sync(0xffffffffu, p[c], o);
      }
      if (lane < 8) {
        double pv = p[0];
#pragma unroll
        for (int c = 1; c < 8; c++) pv = (lane == c) ? p[c] : pv;
        part[warp * 32 + g + lane] = pv;
      }
    }
    __syncthreads();
    if (warp == 0) {
      double a = (lane < kb) ? xa[c0 + lane] : 0.0;
      const double di = (lane < kb) ? __ldg(dv + c0 + lane) : 0.0;
      for (int q = 0; q < nw; q++) a -= part[q * 32 + lane];
      (void)tot;
      for (int k = 31; k >= 0; k--) {
        if (k < kb) {
          const double xk = __shfl_sync(0xffffffffu, a * di, k);
          if (lane == k) a = xk;
          else if (lane < k) a = fma(-Ds[lane * 33 + k], xk, a);
        }
      }
      if (lane < kb) xa[c0 + lane] = a;
    }
    __syncthreads();
  }
}

// Forward of one big supernode by the CTA (the per-node code of fwd_big_kernel): gather
// v = [b(cols); 0] + children's u (fixed order), L11^-1 / blocked sweep, y -> Y, u -> uv.
// v: [max_front] shared, tmp: [>= w] shared.
template <bool BLK, int NT>
__device__ __forceinline__ void fwd_big_cta(const DevPlan& P, const SnInfo& I, int s, int b, const double* Lb,
                                            const double* Dv, const double* bb, double* Y, double* uv,
                                            const double* Li_all, double* v, double* tmp, int* s_cR, int* s_cRel,
                                            int* s_cU, int tid) {
  const int nt = NT;
  if (tid == 0) trace_stamp(P, 1, s, b, 0);
  const int r = I.r, w = I.w, R = r - w, nch = I.c1 - I.c0;
  const double* L = Lb + I.Lp;
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
  if (lip >= 0) cta_fwd_inv(L, Li_all + (long long)b * P.linv_doubles + lip, r, w, v, tmp, tid, nt);
  else if (BLK) cta_fwd_blocked(L, r, w, Dv + I.f0, v, tid, nt);
  else cta_fwd_lite<NT>(L, r, w, Dv + I.f0, v, tmp, tid);
  for (int q = tid; q < w; q += nt) Y[I.f0 + q] = v[q];
  if (I.par >= 0)
    for (int q = tid; q < R; q += nt) uv[I.uvp + q] = v[w + q];
  if (tid == 0) trace_stamp(P, 1, s, b, 1);
}

// Arrival of a finished child at its parent (acq_rel: the child's u is visible to whoever
// continues); returns true for the last child, which resets the counter and continues.
__device__ __forceinline__ bool tree_arrive(int* cnt, int par, int nch) {
  const int old = atom_add_acq_rel(cnt + par, 1);
  if (old != nch - 1) return false;
  cnt[par] = 0;
  return true;
}

// Whole-tree forward sweep below the tile solve's huge fronts, one persistent CTA grid:
// initial tasks are the subtree blocks and the childless big supernodes; every finished
// supernode arrives at its parent and the last child continues with it -- a small parent
// outside the blocks on warp 0, a big parent with the whole CTA.  No task ever waits.
// BLK: some big supernode of the tree has no L11^-1 (the blocked substitution is compiled in;
// it needs registers that cost occupancy, so the common case compiles without it)
template <bool BLK, int NT>
__global__ void __launch_bounds__(NT, BLK ? 1 : sb_minb<NT>()) tree_fwd_kernel(DevPlan P, SBPlan B, const double* __restrict__ Lx_all,
                                                                 const double* __restrict__ Dv_all,
                                                                 const double* __restrict__ rhs, long long rs,
                                                                 double* Y_all, double* uv_all, int* cnt_all, int* ctl,
                                                                 const int* __restrict__ done,
                                                                 const double* __restrict__ Li_all) {
  extern __shared__ __align__(16) double sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ int s_task, s_next, s_qc[2];
  __shared__ int s_cR[32], s_cRel[32], s_cU[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) mbar_init(&bar, 1);
  __syncthreads();
  pdl_launch_dependents();
  for (int q = blockIdx.x * NT + tid; q < B.zn; q += gridDim.x * NT) B.zbuf[q] = 0;
  if (done && done[P.batch] == 0) return;  // every instance has finished refining
  uint32_t phase = 0;
  const int ntask = B.n_fwd * P.batch;
  for (;;) {
    const int t = next_task(ctl, &s_task);  // (barrier: the previous task's shared reads are done)
    if (t >= ntask) break;
    const int b = t % P.batch;
    if (done && done[b]) continue;
    const double* Lb = Lx_all + (long long)b * P.nnzL_stored;
    const double* Dv = Dv_all + (long long)b * P.n;
    const double* bb = rhs + (long long)b * rs;
    double* Y = Y_all + (long long)b * P.n;
    double* uv = uv_all + (long long)b * P.uvec_doubles;
    int* cnt = cnt_all + (long long)b * P.ns;
    int s;        // supernode just finished (its u is in uv)
    SnInfo I;
    const int code = __ldg(B.fwd_order + t / P.batch);
    if (code >= 0) {
      const SBlk K = B.blk[code];
      const double* vr = fwd_block<NT>(P, B, K, b, Lb, Dv, bb, Y, sm, &bar, phase, s_qc, tid, lane, warp);
      s = K.s_hi;
      I = P.sn[s];
      if (I.par >= 0)
        for (int q = tid; q < I.r - I.w; q += NT) uv[I.uvp + q] = vr[I.w + q];
    } else {
      s = -code - 1;
      I = P.sn[s];
      fwd_big_cta<BLK, NT>(P, I, s, b, Lb, Dv, bb, Y, uv, Li_all, sm, sm + P.max_front, s_cR, s_cRel, s_cU, tid);
    }
    // continuation up the tree
    for (;;) {
      __syncthreads();  // every thread's u entries are written before the arrival (acq_rel atomic: cumulative)
      if (tid == 0) {
        int nx = -1;
        if (I.par >= 0) {
          const SnInfo Ip = P.sn[I.par];
          if ((!Ip.huge || P.solve_huge_cta) && tree_arrive(cnt, I.par, Ip.c1 - Ip.c0)) nx = I.par;
        }
        s_next = nx;
      }
      __syncthreads();
      const int nx = s_next;
      if (nx < 0) break;
      s = nx;
      I = P.sn[s];
      if (I.big) {
        fwd_big_cta<BLK, NT>(P, I, s, b, Lb, Dv, bb, Y, uv, Li_all, sm, sm + P.max_front, s_cR, s_cRel, s_cU, tid);
      } else if (warp == 0) {
        fwd_single_warp(P, I, s, b, Lb, Dv, bb, Y, uv, sm, sm + P.max_rw_small, lane);
      }
    }
  }
  persistent_exit(ctl);
}

// Backward sweep of one small supernode outside every block by one warp (per-node code of
// bwd_small_kernel).  Pn, xa: per-warp scratch.
__device__ __forceinline__ void bwd_node_warp(const DevPlan& P, const SnInfo& I, int s, int b,
                                              const double* __restrict__ Lx_all, const double* __restrict__ Dv_all,
                                              const double* __restrict__ Y_all, double* Xp_all, double* xout,
                                              long long xs, double* Pn, double* xa, int lane) {
  if (lane == 0) trace_stamp(P, 2, s, b, 0);
  const int r = I.r, w = I.w, rw = r * w;
  const double* L = Lx_all + (long long)b * P.nnzL_stored + I.Lp;
  double* Xp = Xp_all + (long long)b * P.n;
  const double* Y = Y_all + (long long)b * P.n;
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
  __syncwarp();
  bwd_sweep_sm(Pn, r, w, Dv_all + (long long)b * P.n + I.f0, xa, lane);
  __syncwarp();
  double* xo = xout + (long long)b * xs;
  if (q0 < w) { Xp[I.f0 + q0] = xa[q0]; xo[p0] = xa[q0]; }
  if (q1 < w) { Xp[I.f0 + q1] = xa[q1]; xo[p1] = xa[q1]; }
  if (lane == 0) trace_stamp(P, 2, s, b, 1);
}

// Backward of one big supernode by the CTA (per-node code of bwd_big_kernel).
template <bool BLK, int NT>
__device__ __forceinline__ void bwd_big_cta(const DevPlan& P, const SnInfo& I, int s, int b,
                                            const double* __restrict__ Lx_all, const double* __restrict__ Dv_all,
                                            const double* __restrict__ Y_all, double* Xp_all, double* xout,
                                            long long xs, const double* __restrict__ Li_all, double* xa, double* part,
                                            int tid) {
  const int nt = NT;
  if (tid == 0) trace_stamp(P, 2, s, b, 0);
  const int r = I.r, w = I.w;
  const double* L = Lx_all + (long long)b * P.nnzL_stored + I.Lp;
  double* Xp = Xp_all + (long long)b * P.n;
  const double* Y = Y_all + (long long)b * P.n;
  for (int q = tid; q < r; q += nt) xa[q] = (q < w) ? ldcg(Y + I.f0 + q) : ldcg(Xp + __ldg(P.sn_rows + I.rp0 + q));
  __syncthreads();
  const long long lip = Li_all ? __ldg(P.sn_Lip + s) : -1;
  if (lip >= 0) cta_bwd_inv(L, Li_all + (long long)b * P.linv_doubles + lip, r, w, xa, part, tid, nt);
  else if (BLK) cta_bwd_blocked(L, r, w, Dv_all + (long long)b * P.n + I.f0, xa, part, tid, nt);
  else cta_bwd_lite<NT>(L, r, w, Dv_all + (long long)b * P.n + I.f0, xa, part + 8 * 32, part, tid);
  double* xo = xout + (long long)b * xs;
  for (int q = tid; q < w; q += nt) {
    Xp[I.f0 + q] = xa[q];
    xo[__ldg(P.perm + I.f0 + q)] = xa[q];
  }
  if (tid == 0) trace_stamp(P, 2, s, b, 1);
}

// Backward of one block: stage, y and the ancestors' x, then the block's ready queue.
template <int NT>
__device__ __forceinline__ void bwd_block(const DevPlan& P, const SBPlan& B, const SBlk& K, const SnInfo& I, int b,
                                          const double* Lb, const double* Dv, const double* Yb, double* Xp,
                                          double* xo, double* sm, uint64_t* bar, uint32_t& phase,
                                          int* qc, int tid, int lane, int warp) {
  const int nn = K.s_hi - K.s_lo + 1;
  const SBLayout O = sb_layout(nn, K.nlev, K.nL, K.ncol, K.nr, K.nch, K.Rroot, NT / 32);
  const SBRange rL = sb_range(Lb + K.L0, K.nL), rD = sb_range(Dv + K.F0, K.ncol),
                rS = sb_range(P.sn + K.s_lo, nn), rR = sb_range(B.lrow + K.RP0, K.nr),
                rP = sb_range(P.perm + K.F0, K.ncol), rM = sb_range(B.meta + K.m0, K.nlev + 1 + nn),
                rC = sb_range(P.sn_ch + K.CP0, K.nch);
  if (tid == 0) {
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(bar, rL.bytes + rD.bytes + rS.bytes + rR.bytes + rP.bytes + rM.bytes + rC.bytes);
    if (rC.bytes) bulk_g2s(sm + O.ch, rC.g0, rC.bytes, bar);
    bulk_g2s(sm + O.L, rL.g0, rL.bytes, bar);
    bulk_g2s(sm + O.sn, rS.g0, rS.bytes, bar);
    bulk_g2s(sm + O.meta, rM.g0, rM.bytes, bar);
    bulk_g2s(sm + O.rel, rR.g0, rR.bytes, bar);
    bulk_g2s(sm + O.perm, rP.g0, rP.bytes, bar);
    bulk_g2s(sm + O.D, rD.g0, rD.bytes, bar);
  }
  // y of the block's columns and the ancestors' x of the root's update rows (generic loads)
  double* xl = sm + O.v;
  for (int c = tid; c < K.ncol; c += NT) xl[c] = ldcg(Yb + K.F0 + c);
  for (int q = tid; q < K.Rroot; q += NT) xl[K.ncol + q] = ldcg(Xp + __ldg(P.sn_rows + I.rp0 + I.w + q));
  mbar_wait(bar, phase);
  phase ^= 1;
  __syncthreads();
  const double* Ls = sm + O.L + rL.shift - K.L0;
  const double* Ds = sm + O.D + rD.shift - K.F0;
  const SnInfo* Ss = reinterpret_cast<const SnInfo*>(sm + O.sn) - K.s_lo;
  const int* lrow = reinterpret_cast<const int*>(sm + O.rel) + rR.shift - K.RP0;
  const int* perm = reinterpret_cast<const int*>(sm + O.perm) + rP.shift - K.F0;
  const int* lvl = reinterpret_cast<const int*>(sm + O.meta) + rM.shift;
  const int* nodes = lvl + K.nlev + 1;
  const int* chs = reinterpret_cast<const int*>(sm + O.ch) + rC.shift - K.CP0;
  double* xa = sm + O.xa + warp * 64;
  // ready queue: the root, then every supernode pushes its children (tallest first)
  int* rq = reinterpret_cast<int*>(sm + O.q);
  for (int t = tid; t < nn; t += NT) rq[t] = t == 0 ? nn - 1 : -1;
  if (tid == 0) { qc[0] = 0; qc[1] = 1; }
  __syncthreads();
  volatile int* vrq = rq;
  for (;;) {
    int t = 0, ls = -1;
    if (lane == 0) t = atomicAdd(qc, 1);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= nn) break;
    if (lane == 0) {
      while ((ls = vrq[t]) < 0) { __nanosleep(40); }
      __threadfence_block();
    }
    ls = __shfl_sync(0xffffffffu, ls, 0);
    const int sj = K.s_lo + ls;
    const SnInfo& In = Ss[sj];
    if (lane == 0) trace_stamp(P, 2, sj, b, 0);
    const int r = In.r, w = In.w, f0 = In.f0;
    const int* lr = lrow + In.rp0;
    for (int q = lane; q < r; q += 32) xa[q] = xl[lr[q]];
    __syncwarp();
    bwd_sweep_sm(Ls + In.Lp, r, w, Ds + f0, xa, lane);
    __syncwarp();
    for (int q = lane; q < w; q += 32) {
      const double x = xa[q];
      xl[f0 - K.F0 + q] = x;
      Xp[f0 + q] = x;
      xo[perm[f0 + q]] = x;
    }
    __syncwarp();
    if (lane == 0) {
      trace_stamp(P, 2, sj, b, 1);
      const int nc = In.c1 - In.c0;
      if (nc > 0) {
        const int slot = atomicAdd(qc + 1, nc);
        __threadfence_block();
        for (int i = 0; i < nc; i++) vrq[slot + i] = chs[In.c0 + i] - K.s_lo;
      }
    }
  }
  __syncthreads();
}

// Whole-tree backward sweep below the tile solve's huge fronts: a static list of tasks -- big
// supernodes (CTA), small supernodes outside the blocks (warp 0) and blocks (CTA) -- in
// estimated start order (parents before children), taken by ticket; a task waits for its
// parent's done flag (flag == this launch's epoch; no resets).  Every task waits only for a
// task with a smaller ticket, held by a resident CTA: deadlock-free.
template <bool BLK, int NT>
__global__ void __launch_bounds__(NT, BLK ? 1 : sb_minb<NT>()) tree_bwd_kernel(DevPlan P, SBPlan B, const double* __restrict__ Lx_all,
                                                                 const double* __restrict__ Dv_all,
                                                                 const double* __restrict__ Y_all, double* Xp_all,
                                                                 double* xout, long long xs, int* flags_all, int* ctl,
                                                                 const int* __restrict__ done,
                                                                 const double* __restrict__ Li_all) {
  extern __shared__ __align__(16) double sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ int s_task, s_qc[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) mbar_init(&bar, 1);
  __syncthreads();
  if (done && done[P.batch] == 0) return;  // every instance has finished refining
  const int epoch = ld_volatile(ctl + 9) + 1;
  const int ntask = B.n_bwd * P.batch;
  uint32_t phase = 0;
  for (;;) {
    const int t = next_task(ctl, &s_task);  // (barrier: the previous task's shared reads are done)
    if (t >= ntask) break;
    const int b = t % P.batch;
    if (done && done[b]) continue;
    const int2 tk = __ldg(B.bwd_order + t / P.batch);
    const int s = tk.x;
    int* flags = flags_all + (long long)b * P.ns;
    if (tid == 0 && tk.y >= 0) {
      while (ld_volatile(flags + tk.y) != epoch) { __nanosleep(32); }
      fence_acq_rel();
    }
    const SnInfo I = P.sn[s];
    const int bi = I.big ? -1 : __ldg(B.blk_of + s);
    __syncthreads();  // every thread reads the ancestors' x only after thread 0's acquire
    if (I.big) {
      bwd_big_cta<BLK, NT>(P, I, s, b, Lx_all, Dv_all, Y_all, Xp_all, xout, xs, Li_all, sm, sm + P.max_front, tid);
      __syncthreads();
      if (tid == 0) st_release(flags + s, epoch);   // release: cumulative over the barrier
    } else if (bi < 0) {  // single small supernode: warp 0
      if (warp == 0) {
        bwd_node_warp(P, I, s, b, Lx_all, Dv_all, Y_all, Xp_all, xout, xs, sm, sm + P.max_rw_small, lane);
        __syncwarp();  // lanes' x writes are ordered before lane 0's release
        if (lane == 0) st_release(flags + s, epoch);
      }
    } else {
      const SBlk K = B.blk[bi];
      bwd_block<NT>(P, B, K, I, b, Lx_all + (long long)b * P.nnzL_stored, Dv_all + (long long)b * P.n,
                Y_all + (long long)b * P.n, Xp_all + (long long)b * P.n, xout + (long long)b * xs, sm, &bar,
                phase, s_qc, tid, lane, warp);
    }
  }
  __syncthreads();
  if (tid == 0) {  // persistent_exit, plus the epoch of the next launch
    __threadfence();
    const int e = atomicAdd(ctl + 1, 1);
    if (e == (int)gridDim.x - 1) { ctl[9] = epoch; reset_ctl(ctl); }
  }
}

}  // namespace kkt
