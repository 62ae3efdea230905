// tsolve.cuh -- triangular solves through the large fronts (the huge class of tiles.cuh) as a task
// DAG over the 64 x 64 L tiles of the tile pool, on a persistent CTA grid (SURVEY
// §8(a) a3).  Replaces the level-synchronous whole-GPU wavefront (hsolve.cuh) for these fronts.
//
// Front f (rows in blocks of 64 restarting at w, as the factorisation): forward y1 = L11^-1 v1,
// u = v2 - L21 y1; backward x1 = L11^-T (y1 - L21^T x2).  Row block t of the front keeps its
// working vector in the solve's own buffers: panel blocks in Y (internal numbering, y then z),
// update blocks in the front's u vector (uv + uvp, read by the parent's gather).
//
// Forward tasks:  FG(f, t)   gather v_t = [P b]_t + sum over children (fixed order) of their u
//                            entries landing in block t
//                 FU(f,i,k)  partial P[i][k] = L_ik y_k (i >= k + 2) into its own slot: the
//                            producers of one block run in any order, in parallel
//                 FC(f, k)   chain step: r_k = v_k - sum_j P[k][j] (j ascending), y_k = L_kk^-1 r_k
//                            with the inverse diagonal tile, publish; then P[k+1][k] itself
//                 (the update blocks t >= nbp are finalised by the parent's gathers:
//                 u_t = v_t - sum_k P[t][k], k ascending)
// Backward tasks: BU(f,k,i)  partial Q[k][.] = L_ik^T x_i: update rows in chunks of TS_UCHUNK tiles
//                            (after the parent's backward), panel rows i >= k + 2 one each
//                 BC(f, k)   chain step (k = nbp-1..0): z_k = y_k - sum over update chunks (last
//                            first) - sum_i Q[k][i] (i descending) - L_{k+1,k}^T x_{k+1},
//                            x_k = L_kk^-T z_k, write x
// Counters per instance are zeroed before the launch; every task waits only on tasks earlier in
// the list-schedule order (tile_plan.cpp), all workers resident: deadlock-free.  Every sum has a
// fixed order (no floating-point atomics): deterministic, bitwise identical run to run.
#pragma once
#ifndef TS_SLEEP
#define TS_SLEEP 32   // spin back-off (ns) of the dependency waits
#endif
#include "tiles.cuh"

namespace kkt {

constexpr int TS_GATHER = 0, TS_FU = 1, TS_FC = 2, TS_BU = 3, TS_BC = 4, TS_UF = 5, TS_FCH = 6, TS_BCH = 7;
// chain tasks (FCH / BCH): the whole panel of one front on one CTA, tiles streamed by TMA bulk
// copies through a ring of TS_RING shared-memory slots (one mbarrier each, linear layout), one
// warp per tile product, working vectors in shared memory
constexpr int TS_RING = 6;
constexpr int TS_NBP_MAX = 24;   // panel row blocks per front the chain tasks support
constexpr int TS_SMEM_BYTES = (TS_RING * TBD + 2 * TS_NBP_MAX * 64 + 2 * 64) * 8;
#ifndef TS_UCHUNK_N
#define TS_UCHUNK_N 1   // (shared with tile_plan.cpp; 1 measured faster than 2 on C3/C4)
#endif
constexpr int TS_UCHUNK = TS_UCHUNK_N;   // update-row tiles per backward task (parallel chunks, one slot each)

struct TSolvePlan {
  const int4* tasks;   // x = type | (instance << 4), y = front, z = i, w = k
  int ntask;
  int ncnt;            // counters per instance
  int* cnt;            // [batch][ncnt] + ticket at [batch * ncnt]
  // per front f (counter layout from cbase2[f]): gf[nt] (block gathered), pc[nt] (forward
  // partials present), yf[nbp] (y_k final), ufin (u blocks final), qc[nbp] (backward partials
  // present), xf[nbp] (x_k final), xdone (x blocks final)
  const int* cbase2;   // [nf]
  long long* trace;    // optional [ntask][4]
  double* part;        // [batch][part_doubles] partial products (one 64-slot per producer)
  long long part_doubles;
  int wave;            // chain tasks: tiles per wave (<= min(TS_RING, 4): two warps per tile)
  const long long* pbase;  // [nf]: forward slots P[t][k] (nt x nbp x 64), then backward Q[k][s]
                           // (nbp x nt x 64; s = source panel block i, or nbp + c = update-row chunk c)
};

__device__ __forceinline__ int* ts_gf(const TSolvePlan& S, int* cnt, const TFront& F, int f, int t) { return cnt + S.cbase2[f] + t; }
__device__ __forceinline__ int* ts_pc(const TSolvePlan& S, int* cnt, const TFront& F, int f, int t) { return cnt + S.cbase2[f] + F.nt + t; }
__device__ __forceinline__ int* ts_yf(const TSolvePlan& S, int* cnt, const TFront& F, int f, int k) { return cnt + S.cbase2[f] + 2 * F.nt + k; }
__device__ __forceinline__ int* ts_ufin(const TSolvePlan& S, int* cnt, const TFront& F, int f) { return cnt + S.cbase2[f] + 2 * F.nt + F.nbp; }
__device__ __forceinline__ int* ts_qc(const TSolvePlan& S, int* cnt, const TFront& F, int f, int k) { return cnt + S.cbase2[f] + 2 * F.nt + F.nbp + 1 + k; }
__device__ __forceinline__ int* ts_xf(const TSolvePlan& S, int* cnt, const TFront& F, int f, int k) { return cnt + S.cbase2[f] + 2 * F.nt + 2 * F.nbp + 1 + k; }
__device__ __forceinline__ int* ts_xdone(const TSolvePlan& S, int* cnt, const TFront& F, int f) { return cnt + S.cbase2[f] + 2 * F.nt + 3 * F.nbp + 1; }

// working vector of row block t of front f: Y (panel) or the front's u vector
__device__ __forceinline__ double* ts_vec(const TFront& F, const SnInfo& I, double* Y, double* uvb, int t) {
  return t < F.nbp ? Y + I.f0 + t * TBS : uvb + I.uvp + (t - F.nbp) * TBS;
}

struct TSCtx {
  const DevPlan* P;
  const TilePlan* T;
  const TSolvePlan* S;
  const double* pool;
  const double* inv;   // the instance's inverse diagonal tiles (L_kk^-1)^T
  const double* Dv;
  const double* rhs;
  double* Y;
  double* uvb;
  double* Xp;
  double* xout;
  int* cnt;
  double* part;        // the instance's partial-product slots
  int task;            // ticket (trace)
};
// trace: all waits of the current task are over (slot 1)
__device__ __forceinline__ void ts_ready(const TSCtx& X) {
  if (X.S->trace && threadIdx.x == 0) X.S->trace[4LL * X.task + 1] = gtimer();
}

__device__ __forceinline__ double* ts_pslot(const TSCtx& X, const TFront& F, int f, int t, int k) {
  return X.part + X.S->pbase[f] + ((long long)t * F.nbp + k) * TBS;
}
__device__ __forceinline__ double* ts_qslot(const TSCtx& X, const TFront& F, int f, int k, int src) {
  return X.part + X.S->pbase[f] + (long long)F.nt * F.nbp * TBS + ((long long)k * F.nt + src) * TBS;
}

__device__ __forceinline__ void ts_wait(const int* c, int target) {
  if (threadIdx.x == 0) {
    while (ld_volatile(c) < target) { __nanosleep(TS_SLEEP); }
    fence_acq_rel();
  }
  __syncthreads();
}
__device__ __forceinline__ void ts_publish(int* c, int v) {
  __syncthreads();
  if (threadIdx.x == 0) st_release(c, v);   // release: cumulative over the barrier
}
__device__ __forceinline__ void ts_publish_add(int* c) {
  __syncthreads();
  if (threadIdx.x == 0) red_release_add(c, 1);
}

// r (64, shared) -= A (swizzled tile) x (64, shared): 4 threads per row, 16 columns each
__device__ __forceinline__ void ts_gemv_n(double* r, const double* A, const double* x) {
  const int row = threadIdx.x >> 2, q = threadIdx.x & 3;
  double acc = 0.0;
#pragma unroll
  for (int c = 0; c < 16; c++) {
    const int col = q * 16 + c;
    acc = fma(A[tsw(row, col)], x[col], acc);
  }
  acc += __shfl_xor_sync(0xffffffffu, acc, 1);
  acc += __shfl_xor_sync(0xffffffffu, acc, 2);
  __syncthreads();
  if (q == 0) r[row] -= acc;
  __syncthreads();
}
// z (64, shared) -= A^T x: 4 threads per column, 16 rows each
__device__ __forceinline__ void ts_gemv_t(double* z, const double* A, const double* x) {
  const int col = threadIdx.x >> 2, q = threadIdx.x & 3;
  double acc = 0.0;
#pragma unroll
  for (int c = 0; c < 16; c++) {
    const int row = q * 16 + c;
    acc = fma(A[tsw(row, col)], x[row], acc);
  }
  acc += __shfl_xor_sync(0xffffffffu, acc, 1);
  acc += __shfl_xor_sync(0xffffffffu, acc, 2);
  __syncthreads();
  if (q == 0) z[col] -= acc;
  __syncthreads();
}
// y = L^-1 r for a 64 x 64 lower-triangular swizzled tile with inverse pivots di (shared): warp 0,
// lane = row, two 32-row halves (substitution) with a 32 x 32 product between them
__device__ __forceinline__ void ts_lsolve(double* v, const double* L, const double* di, int nb) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp == 0) {
#pragma unroll
    for (int h = 0; h < 2; h++) {
      const int row = 32 * h + lane;
      double a = v[row];
      if (h == 1) {
        double acc = 0.0;
#pragma unroll 8
        for (int c = 0; c < 32; c++) acc = fma(L[tsw(row, c)], v[c], acc);
        a -= acc;
      }
      const double dr = di[row];
#pragma unroll
      for (int c = 0; c < 32; c++) {
        const double yc = __shfl_sync(0xffffffffu, a * dr, c);
        if (lane == c) a = yc;
        else if (lane > c) a = fma(-L[tsw(row, 32 * h + c)], yc, a);
      }
      v[row] = (row < nb) ? a : 0.0;
      __syncwarp();
    }
  }
  __syncthreads();
}
// x = L^-T z (same tile), warp 0, lane = column, halves 1 then 0
__device__ __forceinline__ void ts_ltsolve(double* v, const double* L, const double* di, int nb) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (warp == 0) {
#pragma unroll
    for (int h = 1; h >= 0; h--) {
      const int col = 32 * h + lane;
      double a = v[col];
      if (h == 0) {
        double acc = 0.0;
#pragma unroll 8
        for (int r = 32; r < 64; r++) acc = fma(L[tsw(r, col)], v[r], acc);
        a -= acc;
      }
      const double dc = di[col];
#pragma unroll
      for (int k = 31; k >= 0; k--) {
        const double xk = __shfl_sync(0xffffffffu, a * dc, k);
        if (lane == k) a = xk;
        else if (lane < k) a = fma(-L[tsw(32 * h + k, col)], xk, a);
      }
      v[col] = (col < nb) ? a : 0.0;
      __syncwarp();
    }
  }
  __syncthreads();
}

__device__ __forceinline__ const double* ts_tile(const TSCtx& X, const TFront& F, int i, int j) {
  return X.pool + F.tbase + (long long)tlin(i, j, F.nt) * TBD;
}

// FG(f, t): gather of row block t (children in fixed order) -> the block's working vector; gf = 1.
// A huge child's update entries are finalised here: u_e = v_e - sum_k P_child[t_c][k] (k ascending)
// once the child's blocks t_c covering them have all their partial products (no separate task).
// Latency: everything that does not depend on the huge children's flags -- the right-hand side
// through perm, every child's record, cut and row map, the final u entries of non-huge children
// -- is loaded before the wait, one warp per child, into a per-child table in shared memory
// (child q's entries land on distinct rows); after the wait only the huge children's u entries
// and partials remain, then the table is summed into the block child by child (q ascending:
// the same order and operations as the per-child loop, bitwise the same result).
constexpr int TS_GMAX = 160;   // children staged per gather (more: per-child loop)
__device__ void ts_gather(const TSCtx& X, const TFront& F, int f, int t, double* sv) {
  const DevPlan& P = *X.P;
  const SnInfo I = P.sn[F.s];
  const int r0 = trow0(F, t), nr = tsize(F, t);
  const int nch = F.nch;
  if (nch <= TS_GMAX) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    double* cval = sv + 64;                                           // [nch][64]
    int* crow = reinterpret_cast<int*>(cval + (long long)nch * 64);   // [nch][64] target row or -1
    int4* cmeta = reinterpret_cast<int4*>(crow + nch * 64);           // [nch] {hc, a, b, uvp}
    __syncthreads();  // the previous task's shared-memory reads are done
    if (threadIdx.x < TBS)
      sv[threadIdx.x] = (t < F.nbp && threadIdx.x < nr) ? __ldg(X.rhs + __ldg(P.perm + I.f0 + r0 + threadIdx.x)) : 0.0;
    for (int q = warp; q < nch; q += TILE_THREADS / 32) {
      const int2 cr = X.T->tch[F.ch0 + q];
      const int* cut = X.T->tcut + cr.y;
      const int a = __ldg(cut + t), b = __ldg(cut + t + 1);
      const int hc = __ldg(X.T->hidx + cr.x);
      int uvp = 0;
      if (b > a) {
        const SnInfo C = P.sn[cr.x];
        uvp = C.uvp;
        const int* rel = P.sn_rel + C.rp0 + C.w;
        const double* u = X.uvb + C.uvp;
        for (int e0 = 0; e0 < b - a; e0 += 32) {
          const int e = a + e0 + lane;
          if (e < b) {
            crow[q * 64 + e0 + lane] = __ldg(rel + e) - r0;
            if (hc < 0) cval[q * 64 + e0 + lane] = __ldcg(u + e);
          }
        }
      }
      if (lane == 0) cmeta[q] = make_int4(hc, a, b, uvp);
    }
    if (threadIdx.x < nch) {  // huge children: the blocks feeding this one must be complete
      const int2 cr = X.T->tch[F.ch0 + threadIdx.x];
      const int hc = __ldg(X.T->hidx + cr.x);
      const int* cut = X.T->tcut + cr.y;
      const int a = __ldg(cut + t), b = __ldg(cut + t + 1);
      if (hc >= 0 && b > a) {
        const TFront C = X.T->fr[hc];
        for (int tc = C.nbp + (a >> 6); tc <= C.nbp + ((b - 1) >> 6); tc++) {
          const int* g = ts_gf(*X.S, X.cnt, C, hc, tc);
          const int* pc = ts_pc(*X.S, X.cnt, C, hc, tc);
          while (ld_volatile(g) < 1) { __nanosleep(TS_SLEEP); }
          while (ld_volatile(pc) < C.nbp) { __nanosleep(TS_SLEEP); }
        }
        fence_acq_rel();
      }
    }
    __syncthreads();
    ts_ready(X);
    for (int q = warp; q < nch; q += TILE_THREADS / 32) {
      const int4 m = cmeta[q];
      if (m.x < 0 || m.z <= m.y) continue;
      const TFront Cf = X.T->fr[m.x];
      const double* u = X.uvb + m.w;
      for (int e0 = 0; e0 < m.z - m.y; e0 += 32) {
        const int e = m.y + e0 + lane;
        if (e < m.z) {
          double val = __ldcg(u + e);
          const double* p0 = X.part + X.S->pbase[m.x] + ((long long)(Cf.nbp + (e >> 6)) * Cf.nbp) * TBS + (e & 63);
#pragma unroll 8
          for (int k = 0; k < Cf.nbp; k++) val -= __ldcg(p0 + (long long)k * TBS);
          cval[q * 64 + e0 + lane] = val;
        }
      }
    }
    __syncthreads();
    if (warp == 0) {  // child by child, q ascending
      for (int q = 0; q < nch; q++) {
        const int4 m = cmeta[q];
        for (int e = lane; e < m.z - m.y; e += 32) sv[crow[q * 64 + e]] += cval[q * 64 + e];
        __syncwarp();
      }
    }
    __syncthreads();
    double* v = ts_vec(F, I, X.Y, X.uvb, t);
    if (threadIdx.x < nr) v[threadIdx.x] = sv[threadIdx.x];
    ts_publish(ts_gf(*X.S, X.cnt, F, f, t), 1);
    return;
  }
  if (threadIdx.x < F.nch) {  // huge children: the blocks feeding this one must be complete
    const int2 cr = X.T->tch[F.ch0 + threadIdx.x];
    const int hc = __ldg(X.T->hidx + cr.x);
    const int* cut = X.T->tcut + cr.y;
    const int a = __ldg(cut + t), b = __ldg(cut + t + 1);
    if (hc >= 0 && b > a) {
      const TFront C = X.T->fr[hc];
      for (int tc = C.nbp + (a >> 6); tc <= C.nbp + ((b - 1) >> 6); tc++) {
        const int* g = ts_gf(*X.S, X.cnt, C, hc, tc);
        const int* pc = ts_pc(*X.S, X.cnt, C, hc, tc);
        while (ld_volatile(g) < 1) { __nanosleep(TS_SLEEP); }
        while (ld_volatile(pc) < C.nbp) { __nanosleep(TS_SLEEP); }
      }
      fence_acq_rel();
    }
  }
  __syncthreads();
  ts_ready(X);
  if (threadIdx.x < TBS)
    sv[threadIdx.x] = (t < F.nbp && threadIdx.x < nr) ? __ldg(X.rhs + __ldg(P.perm + I.f0 + r0 + threadIdx.x)) : 0.0;
  for (int q = 0; q < F.nch; q++) {
    const int2 cr = X.T->tch[F.ch0 + q];
    const int* cut = X.T->tcut + cr.y;
    const int a = __ldg(cut + t), b = __ldg(cut + t + 1);
    __syncthreads();
    if (b > a) {
      const SnInfo C = P.sn[cr.x];
      const int* rel = P.sn_rel + C.rp0 + C.w;
      const double* u = X.uvb + C.uvp;
      const int hc = __ldg(X.T->hidx + cr.x);
      if (hc >= 0) {
        const TFront Cf = X.T->fr[hc];
        for (int e = a + threadIdx.x; e < b; e += TILE_THREADS) {
          double val = __ldcg(u + e);
          const double* p0 = X.part + X.S->pbase[hc] + ((long long)(Cf.nbp + (e >> 6)) * Cf.nbp) * TBS + (e & 63);
#pragma unroll 8
          for (int k = 0; k < Cf.nbp; k++) val -= __ldcg(p0 + (long long)k * TBS);
          sv[__ldg(rel + e) - r0] += val;
        }
      } else {
        for (int e = a + threadIdx.x; e < b; e += TILE_THREADS) sv[__ldg(rel + e) - r0] += __ldcg(u + e);
      }
    }
  }
  __syncthreads();
  double* v = ts_vec(F, I, X.Y, X.uvb, t);
  if (threadIdx.x < nr) v[threadIdx.x] = sv[threadIdx.x];
  ts_publish(ts_gf(*X.S, X.cnt, F, f, t), 1);
}

// r (64, shared) = v_t - sum_{k < nk} P[t][k] in fixed order (k ascending)
__device__ __forceinline__ void ts_sum_partials(const TSCtx& X, const TFront& F, int f, int t, int nk, const double* v,
                                                double* r) {
  if (threadIdx.x < TBS) {
    double a = v[threadIdx.x];
    const double* p0 = ts_pslot(X, F, f, t, 0) + threadIdx.x;
#pragma unroll 8
    for (int k = 0; k < nk; k++) a -= __ldcg(p0 + (long long)k * TBS);   // loads in flight, fixed order
    r[threadIdx.x] = a;
  }
  __syncthreads();
}

// FU(f, i, k): partial P[i][k] = L_ik y_k (no ordering among the producers of one block)
__device__ void ts_fupdate(const TSCtx& X, const TFront& F, int f, int i, int k, double* sm) {
  const SnInfo I = X.P->sn[F.s];
  double *A = sm, *yv = sm + 3 * TBD, *pv = yv + 64;
  tile_load_async(A, ts_tile(X, F, i, k));
  ts_wait(ts_yf(*X.S, X.cnt, F, f, k), 1);
  ts_ready(X);
  const int nk = tsize(F, k);
  if (threadIdx.x < TBS) { yv[threadIdx.x] = threadIdx.x < nk ? __ldcg(X.Y + I.f0 + k * TBS + threadIdx.x) : 0.0; pv[threadIdx.x] = 0.0; }
  cp_async_wait_all();
  __syncthreads();
  ts_gemv_n(pv, A, yv);                                   // pv = -L_ik y_k
  if (threadIdx.x < TBS) ts_pslot(X, F, f, i, k)[threadIdx.x] = -pv[threadIdx.x];
  ts_publish_add(ts_pc(*X.S, X.cnt, F, f, i));
}

// FC(f, k): chain step -- r_k = v_k - sum_j P[k][j], y_k = L_kk^-1 r_k (inverse tile), publish;
// then the partial P[k+1][k] = L_{k+1,k} y_k for the next block
__device__ void ts_fchain(const TSCtx& X, const TFront& F, int f, int k, double* sm) {
  const SnInfo I = X.P->sn[F.s];
  double *Xi = sm, *Lo = sm + TBD, *r = sm + 3 * TBD, *w = r + 64, *v = w + 64;
  tile_load_async(Xi, X.inv + X.T->ibase[f] + (long long)k * TBD);   // (L_kk^-1)^T
  if (k + 1 < F.nt) tile_load_async(Lo, ts_tile(X, F, k + 1, k));
  const int nk = tsize(F, k);
  if (threadIdx.x == 0) {  // the block's gather and its k partial products, one wait
    const int* g = ts_gf(*X.S, X.cnt, F, f, k);
    const int* pc = ts_pc(*X.S, X.cnt, F, f, k);
    while (ld_volatile(g) < 1 || ld_volatile(pc) < k) { __nanosleep(TS_SLEEP); }
    fence_acq_rel();
  }
  __syncthreads();
  ts_ready(X);
  double* y = X.Y + I.f0 + k * TBS;
  if (threadIdx.x < TBS) {  // r = v_k - sum_j P[k][j] (j ascending): all loads in one round trip
    double a = threadIdx.x < nk ? __ldcg(y + threadIdx.x) : 0.0;
    const double* p0 = ts_pslot(X, F, f, k, 0) + threadIdx.x;
#pragma unroll 8
    for (int j = 0; j < k; j++) a -= __ldcg(p0 + (long long)j * TBS);
    r[threadIdx.x] = a;
    v[threadIdx.x] = 0.0;
    w[threadIdx.x] = 0.0;
  }
  cp_async_wait_all();
  __syncthreads();
  ts_gemv_t(v, Xi, r);                              // v = -(L_kk^-1 r): y = -v
  if (threadIdx.x < TBS) v[threadIdx.x] = -v[threadIdx.x];
  __syncthreads();
  if (threadIdx.x < nk) y[threadIdx.x] = v[threadIdx.x];
  if (k + 1 < F.nt) {  // the next block's partial first: one fence publishes both (chain latency)
    ts_gemv_n(w, Lo, v);                            // w = -L_{k+1,k} y_k
    if (threadIdx.x < TBS) ts_pslot(X, F, f, k + 1, k)[threadIdx.x] = -w[threadIdx.x];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    fence_acq_rel();   // one release fence for both flags
    st_relaxed(ts_yf(*X.S, X.cnt, F, f, k), 1);
    if (k + 1 < F.nt) red_relaxed_add(ts_pc(*X.S, X.cnt, F, f, k + 1), 1);
  }
}

// UF(f, t), t >= nbp: u_t = v_t - sum_k P[t][k] (k ascending) -> the front's u vector; ufin++
__device__ void ts_ufinal(const TSCtx& X, const TFront& F, int f, int t, double* sm) {
  const SnInfo I = X.P->sn[F.s];
  double *v = sm + 3 * TBD, *r = v + 64;
  ts_wait(ts_gf(*X.S, X.cnt, F, f, t), 1);
  ts_wait(ts_pc(*X.S, X.cnt, F, f, t), F.nbp);
  ts_ready(X);
  double* u = ts_vec(F, I, X.Y, X.uvb, t);
  const int nr = tsize(F, t);
  if (threadIdx.x < TBS) v[threadIdx.x] = threadIdx.x < nr ? __ldcg(u + threadIdx.x) : 0.0;
  __syncthreads();
  ts_sum_partials(X, F, f, t, F.nbp, v, r);
  if (threadIdx.x < nr) u[threadIdx.x] = r[threadIdx.x];
  ts_publish_add(ts_ufin(*X.S, X.cnt, F, f));
}

// backward: x of row r of front f's update rows (ancestor columns, final after the parent)
__device__ __forceinline__ double ts_xanc(const TSCtx& X, const SnInfo& I, const TFront& F, int row) {
  return __ldcg(X.Xp + __ldg(X.P->sn_rows + I.rp0 + row));
}

// BU(f, k, i): backward partial Q[k][s] = L_ik^T x_i.  i >= nbp: one task for all update rows
// (i descending nt-1..nbp, tiles double-buffered; slot s = nbp) once the parent's backward is
// done; i < nbp: one panel row block (after x_i; slot s = i)
__device__ void ts_bupdate(const TSCtx& X, const TFront& F, int f, int k, int i, double* sm) {
  const SnInfo I = X.P->sn[F.s];
  double *A0 = sm, *A1 = sm + TBD, *xv = sm + 3 * TBD, *zv = xv + 2 * 64;
  const bool urows = (i >= F.nbp);
  const int chunk = urows ? (i - F.nbp) / TS_UCHUNK : 0;
  const int i_lo = urows ? F.nbp + chunk * TS_UCHUNK : i;
  const int i_hi = urows ? min(F.nt - 1, i_lo + TS_UCHUNK - 1) : i;
  static_assert(TS_UCHUNK <= 2, "ts_bupdate stages at most two tiles");
  // every tile of the chunk and the row indices of its x entries are fetched before the wait;
  // after it only the x values remain (one round trip)
  tile_load_async(A0, ts_tile(X, F, i_hi, k));
  if (i_hi > i_lo) tile_load_async(A1, ts_tile(X, F, i_lo, k));
  const int tq = threadIdx.x & 63, which = threadIdx.x >> 6;   // (entry, tile of the chunk)
  const int ii_x = i_hi - which;
  int xidx = -1;
  if (which <= i_hi - i_lo && tq < tsize(F, ii_x)) {
    const int row = trow0(F, ii_x) + tq;
    xidx = urows ? __ldg(X.P->sn_rows + I.rp0 + row) : I.f0 + row;
  }
  if (urows) {
    if (I.par >= 0) {
      const int hp = __ldg(X.T->hidx + I.par);
      const TFront Pf = X.T->fr[hp];
      ts_wait(ts_xdone(*X.S, X.cnt, Pf, hp), Pf.nbp);
    }
  } else {
    ts_wait(ts_xf(*X.S, X.cnt, F, f, i), 1);
  }
  ts_ready(X);
  if (which <= i_hi - i_lo) xv[which * 64 + tq] = xidx >= 0 ? __ldcg(X.Xp + xidx) : 0.0;
  if (threadIdx.x < TBS) zv[threadIdx.x] = 0.0;
  cp_async_wait_all();
  __syncthreads();
  for (int ii = i_hi; ii >= i_lo; ii--)
    ts_gemv_t(zv, ii == i_hi ? A0 : A1, xv + (i_hi - ii) * 64);   // zv -= L^T x (ii descending)
  if (threadIdx.x < TBS) ts_qslot(X, F, f, k, urows ? F.nbp + chunk : i)[threadIdx.x] = -zv[threadIdx.x];
  ts_publish_add(ts_qc(*X.S, X.cnt, F, f, k));
}

// BC(f, k): chain step -- z_k = y_k - Q[k][U] - sum_{i = nbp-1 .. k+2} Q[k][i] - L_{k+1,k}^T x_{k+1}
// (that fixed order), x_k = L_kk^-T z_k (inverse tile), written to Xp and xout
__device__ void ts_bchain(const TSCtx& X, const TFront& F, int f, int k, double* sm) {
  const DevPlan& P = *X.P;
  const SnInfo I = P.sn[F.s];
  double *Xi = sm, *Lo = sm + TBD, *v = sm + 3 * TBD, *xn = v + 64, *o = xn + 64;
  tile_load_async(Xi, X.inv + X.T->ibase[f] + (long long)k * TBD);   // (L_kk^-1)^T
  const int own = (k + 1 < F.nbp) ? 1 : 0;
  if (own) tile_load_async(Lo, ts_tile(X, F, k + 1, k));
  const int nk = tsize(F, k);
  const int nchunk = (F.nt - F.nbp + TS_UCHUNK - 1) / TS_UCHUNK;
  const int npanel = max(F.nbp - k - 2, 0);
  ts_wait(ts_yf(*X.S, X.cnt, F, f, k), 1);
  if (own) {
    ts_wait(ts_xf(*X.S, X.cnt, F, f, k + 1), 1);
    if (threadIdx.x < TBS)
      xn[threadIdx.x] = threadIdx.x < tsize(F, k + 1) ? __ldcg(X.Xp + I.f0 + (k + 1) * TBS + threadIdx.x) : 0.0;
  }
  ts_wait(ts_qc(*X.S, X.cnt, F, f, k), nchunk + npanel);
  ts_ready(X);
  if (threadIdx.x < TBS) {
    double a = threadIdx.x < nk ? __ldcg(X.Y + I.f0 + k * TBS + threadIdx.x) : 0.0;
    const double* q0 = ts_qslot(X, F, f, k, 0) + threadIdx.x;
#pragma unroll 8
    for (int c = nchunk - 1; c >= 0; c--) a -= __ldcg(q0 + (long long)(F.nbp + c) * TBS);
#pragma unroll 8
    for (int i = F.nbp - 1; i >= k + 2; i--) a -= __ldcg(q0 + (long long)i * TBS);
    v[threadIdx.x] = a;
  }
  cp_async_wait_all();
  __syncthreads();
  if (own) ts_gemv_t(v, Lo, xn);
  if (threadIdx.x < TBS) o[threadIdx.x] = 0.0;
  __syncthreads();
  ts_gemv_n(o, Xi, v);                              // o = -(L_kk^-T z)
  if (threadIdx.x < TBS) v[threadIdx.x] = -o[threadIdx.x];
  __syncthreads();
  if (threadIdx.x < nk) {
    const int c = I.f0 + k * TBS + threadIdx.x;
    X.Xp[c] = v[threadIdx.x];
    X.xout[__ldg(P.perm + c)] = v[threadIdx.x];
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // one fence publishes x_k and the front's done count
    fence_acq_rel();
    st_relaxed(ts_xf(*X.S, X.cnt, F, f, k), 1);
    red_relaxed_add(ts_xdone(*X.S, X.cnt, F, f), 1);
  }
}

// Products with a linear (column-major, unswizzled) 64 x 64 tile in shared memory, two warps
// per tile: gemv_n gives row h * 32 + lane of A x (consecutive rows across the lanes:
// conflict-free), gemv_t column h * 32 + lane of A^T x with the rows visited from r = lane on
// (banks spread).  Two partial sums (even / odd steps) added at the end.
__device__ __forceinline__ double ts_gemv_n_half(const double* A, const double* x, int h, int lane) {
  double a = 0.0, b = 0.0;
  const double* Ar = A + h * 32 + lane;
#pragma unroll 8
  for (int c = 0; c < 64; c += 2) {
    a = fma(Ar[c * 64], x[c], a);
    b = fma(Ar[(c + 1) * 64], x[c + 1], b);
  }
  return a + b;
}
__device__ __forceinline__ double ts_gemv_t_half(const double* A, const double* x, int h, int lane) {
  double a = 0.0, b = 0.0;
  const double* Ac = A + (h * 32 + lane) * 64;
#pragma unroll 8
  for (int s = 0; s < 64; s += 2) {
    const int r0 = (s + lane) & 63, r1 = (s + 1 + lane) & 63;
    a = fma(Ac[r0], x[r0], a);
    b = fma(Ac[r1], x[r1], b);
  }
  return a + b;
}

// Ring of TS_RING tile slots filled by TMA bulk copies (32 KB each); ph = parity bit per slot,
// kept identical by every thread (each fill completes its slot's mbarrier phase once).
struct TsRing {
  double* slot;        // [TS_RING][TBD]
  uint64_t* bar;       // [TS_RING] mbarriers
};
__device__ __forceinline__ void ts_ring_issue(const TsRing& R, int q, const double* g) {  // one thread
  uint64_t* b = R.bar + (q % TS_RING);
  fence_proxy_async_smem();
  mbar_arrive_expect_tx(b, TBD * 8);
  bulk_g2s(R.slot + (q % TS_RING) * TBD, g, TBD * 8, b);
}
__device__ __forceinline__ void ts_ring_wait(const TsRing& R, int q, uint32_t ph) {
  mbar_wait(R.bar + (q % TS_RING), (ph >> (q % TS_RING)) & 1u);
}

// FCH(f): forward through the front's panel on one CTA, right-looking over the panel's column
// blocks: y_j = L_jj^-1 a_j (the stored inverse tile (L_jj^-1)^T, transposed product on warp
// 0), then a_k -= L_kj y_j for every panel row block k > j (one warp per tile); tiles streamed
// in that order (Xi_j, L_{j+1,j}, ..., L_{nbp-1,j}, Xi_{j+1}, ...).  y_j is published per block
// (the update-row FU tasks consume it).  Waits only on the front's gathers: deadlock-free.
__device__ void ts_fchain_front(const TSCtx& X, const TFront& F, int f, double* sm, const TsRing& R, uint32_t& ph) {
  const SnInfo I = X.P->sn[F.s];
  const int nbp = F.nbp, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* av = sm + TS_RING * TBD;     // [nbp][64]
  double* yv = av + TS_NBP_MAX * 64;   // [nbp][64], zero-padded
  const int ntile = nbp + nbp * (nbp - 1) / 2;
  auto src = [&](int q) -> const double* {  // q-th tile of the stream
    int j = 0, c = q;
    while (c >= nbp - j) { c -= nbp - j; j++; }
    return c == 0 ? X.inv + X.T->ibase[f] + (long long)j * TBD : ts_tile(X, F, j + c, j);
  };
  __syncthreads();  // the previous task's shared-memory reads are done
  if (threadIdx.x == 0)
    for (int q = 0; q < min(TS_RING, ntile); q++) ts_ring_issue(R, q, src(q));
  if (threadIdx.x < nbp) {  // every panel block gathered (one flag per thread: polled in parallel)
    while (ld_volatile(ts_gf(*X.S, X.cnt, F, f, threadIdx.x)) < 1) { __nanosleep(TS_SLEEP); }
    fence_acq_rel();
  }
  __syncthreads();
  ts_ready(X);
  for (int q = threadIdx.x; q < nbp * 64; q += TILE_THREADS) {
    const int t = q >> 6, e = q & 63;
    av[q] = e < tsize(F, t) ? __ldcg(X.Y + I.f0 + t * TBS + e) : 0.0;
  }
  __syncthreads();
  int q = 0;  // consume cursor
  for (int j = 0; j < nbp; j++) {
    const int nk = tsize(F, j);
    if (warp < 2) {  // y_j = (Xi_j)^T a_j, column halves on warps 0 and 1
      ts_ring_wait(R, q, ph);
      const int e = warp * 32 + lane;
      const double o = ts_gemv_t_half(R.slot + (q % TS_RING) * TBD, av + j * 64, warp, lane);
      yv[j * 64 + e] = e < nk ? o : 0.0;
      if (e < nk) X.Y[I.f0 + j * TBS + e] = o;
    }
    __syncthreads();
    ph ^= 1u << (q % TS_RING);
    if (threadIdx.x == 0) {
      if (q + TS_RING < ntile) ts_ring_issue(R, q + TS_RING, src(q + TS_RING));
      st_release(ts_yf(*X.S, X.cnt, F, f, j), 1);   // cumulative over the barrier
    }
    q++;
    const int wv = X.S->wave;
    for (int k0 = j + 1; k0 < nbp; k0 += wv) {  // waves of at most wv tiles (the ring holds the next ones)
      const int nw = min(wv, nbp - k0);
      if ((warp >> 1) < nw) {  // two warps per tile (row halves)
        const int t = warp >> 1, hh = warp & 1, qq = q + t, k = k0 + t;
        ts_ring_wait(R, qq, ph);
        av[k * 64 + hh * 32 + lane] -= ts_gemv_n_half(R.slot + (qq % TS_RING) * TBD, yv + j * 64, hh, lane);
      }
      __syncthreads();
      for (int u = 0; u < nw; u++) ph ^= 1u << ((q + u) % TS_RING);
      if (threadIdx.x == 0)
        for (int u = 0; u < nw; u++)
          if (q + u + TS_RING < ntile) ts_ring_issue(R, q + u + TS_RING, src(q + u + TS_RING));
      q += nw;
    }
  }
}

// BCH(f): backward through the panel on one CTA: a_k = y_k - (update-row chunks, last first),
// then for i = nbp-1 .. 0: x_i = L_ii^-T a_i (inverse tile, warp 0), a_k -= L_ik^T x_i for
// k < i (one warp per tile); tiles streamed as Xi_i, L_{i,i-1}, ..., L_{i,0}, Xi_{i-1}, ...
__device__ void ts_bchain_front(const TSCtx& X, const TFront& F, int f, double* sm, const TsRing& R, uint32_t& ph) {
  const DevPlan& P = *X.P;
  const SnInfo I = P.sn[F.s];
  const int nbp = F.nbp, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* av = sm + TS_RING * TBD;
  double* xs = av + TS_NBP_MAX * 64;
  const int nchunk = (F.nt - F.nbp + TS_UCHUNK - 1) / TS_UCHUNK;
  const int ntile = nbp + nbp * (nbp - 1) / 2;
  auto src = [&](int q) -> const double* {  // q-th tile: row block i from the top, Xi_i then L(i, i-1 .. 0)
    int i = nbp - 1, c = q;
    while (c >= i + 1) { c -= i + 1; i--; }
    return c == 0 ? X.inv + X.T->ibase[f] + (long long)i * TBD : ts_tile(X, F, i, i - c);
  };
  __syncthreads();
  if (threadIdx.x == 0)
    for (int q = 0; q < min(TS_RING, ntile); q++) ts_ring_issue(R, q, src(q));
  if (threadIdx.x < nbp) {  // the forward chain done, every update-row chunk product present
    while (ld_volatile(ts_yf(*X.S, X.cnt, F, f, threadIdx.x)) < 1) { __nanosleep(TS_SLEEP); }
    while (ld_volatile(ts_qc(*X.S, X.cnt, F, f, threadIdx.x)) < nchunk) { __nanosleep(TS_SLEEP); }
    fence_acq_rel();
  }
  __syncthreads();
  ts_ready(X);
  for (int q = threadIdx.x; q < nbp * 64; q += TILE_THREADS) {
    const int t = q >> 6, e = q & 63;
    double a = e < tsize(F, t) ? __ldcg(X.Y + I.f0 + t * TBS + e) : 0.0;
    const double* q0 = ts_qslot(X, F, f, t, 0) + e;
#pragma unroll 4
    for (int c = nchunk - 1; c >= 0; c--) a -= __ldcg(q0 + (long long)(F.nbp + c) * TBS);
    av[q] = a;
  }
  __syncthreads();
  int q = 0;
  for (int i = nbp - 1; i >= 0; i--) {
    const int nk = tsize(F, i);
    if (warp < 2) {  // x_i = Xi_i a_i, row halves on warps 0 and 1
      ts_ring_wait(R, q, ph);
      const int e = warp * 32 + lane;
      const double o = ts_gemv_n_half(R.slot + (q % TS_RING) * TBD, av + i * 64, warp, lane);
      xs[i * 64 + e] = e < nk ? o : 0.0;
      if (e < nk) {
        const int c = I.f0 + i * TBS + e;
        X.Xp[c] = o;
        X.xout[__ldg(P.perm + c)] = o;
      }
    }
    __syncthreads();
    ph ^= 1u << (q % TS_RING);
    if (threadIdx.x == 0) {
      if (q + TS_RING < ntile) ts_ring_issue(R, q + TS_RING, src(q + TS_RING));
      fence_acq_rel();
      st_relaxed(ts_xf(*X.S, X.cnt, F, f, i), 1);
      red_relaxed_add(ts_xdone(*X.S, X.cnt, F, f), 1);
    }
    q++;
    const int wv = X.S->wave;
    for (int c0 = 0; c0 < i; c0 += wv) {  // tiles L(i, i-1-c), waves of at most wv
      const int nw = min(wv, i - c0);
      if ((warp >> 1) < nw) {  // two warps per tile (column halves)
        const int t = warp >> 1, hh = warp & 1, qq = q + t, k = i - 1 - (c0 + t);
        ts_ring_wait(R, qq, ph);
        av[k * 64 + hh * 32 + lane] -= ts_gemv_t_half(R.slot + (qq % TS_RING) * TBD, xs + i * 64, hh, lane);
      }
      __syncthreads();
      for (int u = 0; u < nw; u++) ph ^= 1u << ((q + u) % TS_RING);
      if (threadIdx.x == 0)
        for (int u = 0; u < nw; u++)
          if (q + u + TS_RING < ntile) ts_ring_issue(R, q + u + TS_RING, src(q + u + TS_RING));
      q += nw;
    }
  }
}

__global__ void __launch_bounds__(TILE_THREADS, 1) tile_solve_kernel(DevPlan P, TilePlan T, TSolvePlan S,
                                                                   const double* __restrict__ Dv_all,
                                                                   const double* __restrict__ rhs, long long rs,
                                                                   double* Y_all, double* uv_all, double* Xp_all,
                                                                   double* xout, long long xs,
                                                                   const int* __restrict__ done) {
  extern __shared__ __align__(16) double tsm[];
  __shared__ int s_task;
  __shared__ __align__(8) uint64_t s_bar[TS_RING];
  if (done && done[P.batch] == 0) return;  // every instance has finished refining (grid-uniform)
  if (threadIdx.x < TS_RING) mbar_init(s_bar + threadIdx.x, 1);
  __syncthreads();
  const TsRing ring{tsm, s_bar};
  uint32_t ph = 0;
  int* ticket = S.cnt + (long long)P.batch * S.ncnt;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_task = atomicAdd(ticket, 1);
    __syncthreads();
    const int t = s_task;
    if (t >= S.ntask) break;
    const int4 tk = S.tasks[t];
    const int type = tk.x & 15, b = tk.x >> 4;
    if (done && done[b]) continue;   // finished instance: all its tasks skip (no dependents run)
    if (S.trace && threadIdx.x == 0) S.trace[4LL * t] = gtimer();
    TSCtx X;
    X.P = &P; X.T = &T; X.S = &S;
    X.pool = T.pool + (long long)b * T.pool_doubles;
    X.inv = T.inv + (long long)b * T.inv_doubles;
    X.Dv = Dv_all + (long long)b * P.n;
    X.rhs = rhs + (long long)b * rs;
    X.Y = Y_all + (long long)b * P.n;
    X.uvb = uv_all + (long long)b * P.uvec_doubles;
    X.Xp = Xp_all + (long long)b * P.n;
    X.xout = xout + (long long)b * xs;
    X.cnt = S.cnt + (long long)b * S.ncnt;
    X.part = S.part + (long long)b * S.part_doubles;
    X.task = t;
    const TFront F = T.fr[tk.y];
    switch (type) {
      case TS_GATHER: ts_gather(X, F, tk.y, tk.z, tsm); break;
      case TS_FU: ts_fupdate(X, F, tk.y, tk.z, tk.w, tsm); break;
      case TS_FC: ts_fchain(X, F, tk.y, tk.w, tsm); break;
      case TS_BU: ts_bupdate(X, F, tk.y, tk.w, tk.z, tsm); break;
      case TS_UF: ts_ufinal(X, F, tk.y, tk.z, tsm); break;
      case TS_FCH: ts_fchain_front(X, F, tk.y, tsm, ring, ph); break;
      case TS_BCH: ts_bchain_front(X, F, tk.y, tsm, ring, ph); break;
      default: ts_bchain(X, F, tk.y, tk.w, tsm); break;
    }
    if (S.trace) {
      __syncthreads();
      if (threadIdx.x == 0) S.trace[4LL * t + 2] = gtimer();
    }
  }
}

}  // namespace kkt
