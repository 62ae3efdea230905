// common.cuh -- shared device helpers of the sm_100a kernels of the condensed-KKT hot path (arXiv 2405.14236).
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
#define KKT_CGT 1024        // threads per block of the per-instance Krylov reductions (G z, updates)

// ------------------------------------------------------------------ memory-model helpers
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void st_release(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// relaxed gpu-scope flag writes: preceded by one fence_acq_rel() they publish together (one
// release fence for several flags)
__device__ __forceinline__ void st_relaxed(int* p, int v) {
  asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_relaxed_add(int* p, int v) {
  asm volatile("red.relaxed.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int atom_add_acq_rel(int* p, int v) {
  int old;
  asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ int ld_volatile(const int* p) {
  int v;
  asm volatile("ld.volatile.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Wait until *f >= target: relaxed polling (no per-poll L1 invalidation, which would stall the
// SM's other warps), then one acquire fence (relaxed read + fence = acquire pattern).
__device__ __forceinline__ void spin_acquire(const int* f, int target) {
  while (ld_volatile(f) < target) { }
  fence_acq_rel();
}
// Programmatic dependent launch: let the next kernel in the stream start now (its CTAs wait
// on device flags, not on this grid's completion).
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
// Wait until every child of an initial big task has been counted by the small phase (which may
// still be running when the big kernel is a programmatic dependent), then reset the counter.
__device__ __forceinline__ void wait_children_reset(int* c, int nch) {
  while (ld_volatile(c) < nch) { __nanosleep(64); }
  fence_acq_rel();
  *c = 0;
}
// Bottom-up hand-off into a big (CTA) parent whose small children may still be running in the
// overlapped small kernel: big children add 1 << 16 and the LAST big child continues with the
// parent after the small children (each adds 1) have all arrived; it then resets the counter.
// Returns true if the caller continues with the parent.  Called by one thread.
__device__ __forceinline__ bool big_child_arrive_n(int* c, int nbig, int nch) {
  const int nsmall = nch - nbig;
  const int old = atom_add_acq_rel(c, 1 << 16);
  if ((old >> 16) != nbig - 1) return false;
  while ((ld_volatile(c) & 0xffff) < nsmall) { __nanosleep(64); }
  fence_acq_rel();
  *c = 0;
  return true;
}
__device__ __forceinline__ bool big_child_arrive(const DevPlan& P, int* c, int par, int par_c0, int par_c1) {
  const int nbig = __ldg(P.sn_nbig + par);
  const int nsmall = (par_c1 - par_c0) - nbig;
  const int old = atom_add_acq_rel(c, 1 << 16);
  if ((old >> 16) != nbig - 1) return false;
  while ((ld_volatile(c) & 0xffff) < nsmall) { __nanosleep(64); }
  fence_acq_rel();
  *c = 0;
  return true;
}
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// trace stamps (instance 0 only): kind 0 = factor, 1 = forward, 2 = backward;
// which 0 = start, 1 = end, 2..7 = intermediate checkpoints (KKT_TRACE_SLOTS per task)
#define KKT_TRACE_SLOTS 8
__device__ __forceinline__ void trace_stamp(const DevPlan& P, int kind, int s, int b, int which) {
  if (P.trace && b == 0) P.trace[((long long)kind * P.ns + s) * KKT_TRACE_SLOTS + which] = gtimer();
}
// latest-of stamp (several warps finish a phase; the last one counts)
__device__ __forceinline__ void trace_max(const DevPlan& P, int kind, int s, int b, int which) {
  if (P.trace && b == 0)
    atomicMax((unsigned long long*)&P.trace[((long long)kind * P.ns + s) * KKT_TRACE_SLOTS + which],
              (unsigned long long)gtimer());
}
// Coalesced global -> shared copy with KKT_MLP loads in flight per thread (the loads are issued
// back to back before any store, so a copy of n elements costs ~ceil(n / (nt*KKT_MLP)) memory
// round trips instead of ceil(n / nt)).  CG = bypass L1 (data produced in the same launch).
#define KKT_MLP 8
template <bool CG, class T>
__device__ __forceinline__ void copy_g2s(T* dst, const T* src, int n, int tid, int nt) {
  for (int base = tid; base < n; base += nt * KKT_MLP) {
    T t[KKT_MLP];
#pragma unroll
    for (int u = 0; u < KKT_MLP; u++) {
      const int q = base + u * nt;
      if (q < n) t[u] = CG ? __ldcg(src + q) : __ldg(src + q);
    }
#pragma unroll
    for (int u = 0; u < KKT_MLP; u++) {
      const int q = base + u * nt;
      if (q < n) dst[q] = t[u];
    }
  }
}
// producer data written earlier in the same launch by another CTA: bypass L1
__device__ __forceinline__ double ldcg(const double* p) { return __ldcg(p); }

// ------------------------------------------------------------------ TMA bulk copies (1-D)
// cp.async.bulk global -> shared with an mbarrier transaction count: one thread issues the
// copies of a whole staging set, every thread waits on the barrier's phase.  Addresses and
// sizes must be 16-byte multiples (the callers round ranges outwards; every global array has
// >= 16 bytes of slack after its end, kkt_api.cu: vbytes / Carver).
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n.reg .pred P1;\nLAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\nbra LAB_WAIT;\nDONE:\n}" ::"r"(smem_u32(bar)), "r"(phase) : "memory");
}
// generic-proxy accesses of shared memory before this point are ordered before later
// async-proxy (TMA) writes to it (buffer reuse across tasks)
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void atomic_max_pos(unsigned long long* a, double v) {
  // non-negative doubles order like their bit patterns; NaN maps above +inf
  unsigned long long b = isnan(v) ? 0x7ff8000000000000ULL : __double_as_longlong(v);
  atomicMax(a, b);
}

// Block-wide max of non-negative doubles (NaN propagates as the largest value), then ONE
// atomic per block: every thread of the block must call it (block-uniform destination).  A
// per-element atomic on one address serialises ~n atomics in the L2 (measured on C4: the
// refinement update took 0.5 ms for n = 674k).
__device__ __forceinline__ void block_max_atomic(unsigned long long* a, double v) {
  __shared__ unsigned long long red_max[32];
  unsigned long long b = isnan(v) ? 0x7ff8000000000000ULL : (unsigned long long)__double_as_longlong(v);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long t = __shfl_xor_sync(0xffffffffu, b, o);
    b = t > b ? t : b;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  __syncthreads();
  if (lane == 0) red_max[warp] = b;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long m = 0ULL;
    for (int k = 0; k < nw; k++) m = red_max[k] > m ? red_max[k] : m;
    if (m) atomicMax(a, m);
  }
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
// Control block of one persistent launch (KKT_CTL ints, the all-done flag on its own 32-byte
// sector so that pollers do not contend with the completion atomics):
//   ctl[0] = ticket/head, ctl[1] = exit count, ctl[2] = queue tail, ctl[3] = completed tasks,
//   ctl[8] = all tasks done.  The last worker to exit resets it for the next launch.
#define KKT_CTL 16
__device__ __forceinline__ void reset_ctl(int* ctl) {
  ctl[0] = 0; ctl[1] = 0; ctl[2] = 0; ctl[3] = 0; ctl[4] = 0; ctl[5] = 0; ctl[6] = 0; ctl[8] = 0;
  __threadfence();
}
__device__ __forceinline__ void persistent_exit(int* ctl) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    int e = atomicAdd(ctl + 1, 1);
    if (e == (int)gridDim.x - 1) reset_ctl(ctl);
  }
}

__device__ __forceinline__ long long upk(int i, int j, int R) {  // packed lower col-major
  return (long long)j * R - (long long)j * (j - 1) / 2 + (i - j);
}

}  // namespace kkt
