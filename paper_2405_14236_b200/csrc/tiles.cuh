// tiles.cuh -- factorisation of the large fronts ("huge": beyond one CTA's shared memory) as a
// task DAG over 64 x 64 tiles executed by a persistent grid of CTA workers (the
// pivot-free Cholesky of the condensed matrix, the FP64-tensor-core share).
//
// Front of huge supernode s (r rows, w pivot columns, R = r - w): rows/columns are cut into
// tiles of 64 that restart at w (tile rows 0..nbp-1 cover the pivot columns, nbp..nt-1 the update
// rows), so a tile is either part of the panel L or of the update matrix U.  The front lives in a
// tile pool in HBM (tile (i, j), i >= j, 64 x 64 column-major, zero-padded), i.e. contiguous 32 KB
// blocks that are staged into shared memory with cp.async (16-byte chunks, all in flight at once,
// XOR-swizzled so that the DMMA fragment loads are conflict-free).
//
// Tasks (one CTA each; 8 warps):
//   ASM(f, i, jt)   assemble tile (i, jt) in shared memory: K entries, then the rectangle of every
//                   child's update matrix that lands in it (children in fixed order: deterministic)
//   POTRF0(f)       Cholesky of tile (0, 0)
//   TRSM(f, i, k)   L_ik = A_ik L_kk^-T                                      (i >= k + 2)
//   CRIT(f, k)      the critical path of step k in one task: TRSM(k+1, k) (published at once),
//                   A_{k+1,k+1} -= L_{k+1,k} L_{k+1,k}^T, Cholesky of tile (k+1, k+1)
//   UPD(f, i, j, k) A_ij -= L_ik L_jk^T on DMMA (mma.sync m8n8k4 f64), k < nbp, j > k
// Dependencies are per-tile counters in HBM: cnt(i, j) = 1 once the tile is assembled, 1 + the
// number of updates applied (k) after that, and k + 2 once panel tile (i, k) is final (a U tile
// is final at nbp + 1; the parent's assembly waits for exactly the child tiles it reads).  Tasks
// are taken in a static order (a list schedule simulated at bind, tile_plan.cpp) with a global
// ticket; every dependency of a task precedes it in that order, so with all workers resident
// (cooperative launch) a worker spinning on a dependency always waits for a running task:
// deadlock-free.  Final L tiles are also written to the supernodal panel layout (r x w,
// column-major) that the triangular solves read.
#pragma once
#ifndef TILE_SLEEP
#define TILE_SLEEP 32   // spin back-off (ns) of the dependency waits
#endif
#include "dense.cuh"
#include "ldlt.cuh"

namespace kkt {

constexpr int TBS = 64;            // tile edge
constexpr int TBD = TBS * TBS;     // doubles per tile
constexpr int TASK_ASM = 0, TASK_POTRF0 = 1, TASK_TRSM = 2, TASK_CRIT = 3, TASK_UPD = 4, TASK_INV = 5;
constexpr int TILE_THREADS = 256;
// shared memory of tile_factor_kernel: three swizzled tiles + 64 inverse pivots + scratch
constexpr int TILE_SMEM_BYTES = (3 * TBD + 64 + 32 * 32 + 64) * 8 + 64;  // + 64 pivot signs (LDL^T)

// One huge front (device view).
struct alignas(16) TFront {
  int s, r, w, nbp;    // supernode, rows, width, panel tile count
  int nt, cbase, nU, ch0;  // tile count per dimension, counter base, U tile count, first child record
  long long tbase;     // tile pool offset (doubles, per instance)
  int nch, pad2;       // child records [ch0, ch0 + nch)
};
static_assert(sizeof(TFront) == 48, "TFront layout");

struct TilePlan {
  const TFront* fr;    // [nf]
  const int4* tasks;   // [ntask]: x = type | (instance << 4), y = front, z = i | (j << 16), w = k
  const int* hidx;     // [ns] huge-front index of a supernode or -1
  const int2* tch;     // child records {child supernode, offset of its cut array in tcut}
  const int* tcut;     // per child record [nt + 1]: first child row/column whose parent index is
                       // >= the start of parent tile t (rel is increasing), t = 0..nt
  const int* tkptr;    // [ncnt + 1] range of the K entries of each tile in tkidx (counter indexing)
  const int* tkidx;    // K entry indices grouped by tile
  int nf, ntask, ncnt;
  long long pool_doubles;  // per instance
  double* pool;        // [batch][pool_doubles]
  int* cnt;            // [batch][ncnt] (zeroed before the launch) ; cnt[batch * ncnt] = ticket
  long long* trace;    // optional [ntask][4]: start, dependencies met, end (globaltimer ns), SM id
  double* inv;         // [batch][inv_doubles]: (L_kk^-1)^T of every diagonal panel tile (solves)
  long long inv_doubles;
  const long long* ibase;  // [nf] offset of a front's nbp inverse tiles
  int panel;           // 1: also write final L tiles to the supernodal panel layout (read by the CTA-view
                       // and level solves); 0 when the tile solve reads the pool (no copy on the chain)
};

__device__ __forceinline__ int tlin(int i, int j, int nt) { return j * nt - j * (j - 1) / 2 + (i - j); }
__device__ __forceinline__ int trow0(const TFront& F, int t) { return t < F.nbp ? t * TBS : F.w + (t - F.nbp) * TBS; }
__device__ __forceinline__ int tsize(const TFront& F, int t) {
  return t < F.nbp ? min(TBS, F.w - t * TBS) : min(TBS, F.r - F.w - (t - F.nbp) * TBS);
}
__device__ __forceinline__ int trow_of(const TFront& F, int x) { return x < F.w ? x / TBS : F.nbp + (x - F.w) / TBS; }
// swizzled shared-memory index of (row, col) of a 64 x 64 column-major tile: the XOR on row bits
// 3-4 spreads the 4 columns a DMMA fragment load touches over all banks (16-byte chunks intact)
__device__ __forceinline__ int tsw(int row, int col) { return col * TBS + (row ^ ((col & 3) << 3)); }

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}
// 64 x 64 tile (global, column-major ld 64) -> shared (swizzled); 2048 16-byte chunks, 8 per thread
__device__ __forceinline__ void tile_load_async(double* s, const double* g) {
  for (int q = threadIdx.x; q < TBD / 2; q += TILE_THREADS) {
    const int col = q >> 5, row = (q & 31) << 1;
    cp_async16(s + tsw(row, col), g + col * TBS + row);
  }
}
// shared (swizzled) -> global tile, 16-byte stores
__device__ __forceinline__ void tile_store(double* g, const double* s) {
  for (int q = threadIdx.x; q < TBD / 2; q += TILE_THREADS) {
    const int col = q >> 5, row = (q & 31) << 1;
    *reinterpret_cast<double2*>(g + col * TBS + row) = *reinterpret_cast<const double2*>(s + tsw(row, col));
  }
}
// non-volatile DMMA (lets the compiler hoist the fragment loads of later k-steps)
__device__ __forceinline__ void dmma_nv(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

__device__ __forceinline__ void wait_cnt(const int* c, int target) {
  if (threadIdx.x == 0) {
    while (ld_volatile(c) < target) { __nanosleep(TILE_SLEEP); }
    fence_acq_rel();
  }
  __syncthreads();
}
// publish: every thread's global writes -> barrier -> one gpu-scope release by thread 0
__device__ __forceinline__ void publish_cnt(int* c, int value) {
  __syncthreads();
  if (threadIdx.x == 0) st_release(c, value);   // release: cumulative over the barrier
}

// Final panel tile (i, k) -> supernodal panel layout Lx (r x w column-major); diagonal tiles
// store zeros above the diagonal (the panel's upper part is read as zero by the solves).
__device__ __forceinline__ void tile_to_panel(const TFront& F, const double* s, double* Lp, int i, int k) {
  const int r0 = trow0(F, i), nr = tsize(F, i), c0 = k * TBS, nc = tsize(F, k);
  const bool dg = (i == k);
  for (int q = threadIdx.x; q < TBD; q += TILE_THREADS) {
    const int col = q >> 6, row = q & 63;
    if (row < nr && col < nc) Lp[(long long)(c0 + col) * F.r + r0 + row] = (dg && row < col) ? 0.0 : s[tsw(row, col)];
  }
}

// C (64 x 64, in global memory) -= A B^T with A, B swizzled 64 x 64 tiles in shared memory;
// warp w owns rows 16 (w >> 1) .. +16, columns 32 (w & 1) .. +32 (2 x 4 DMMA blocks).  The
// read-modify-write of C is issued before the k-loop so its latency hides under the MMAs.
template <bool SG = false>
__device__ __forceinline__ void tile_gemm_nt_global(double* C, const double* A, const double* B, const double* ssg = nullptr) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, lr = lane >> 2, lc = lane & 3;
  const int rb = (warp >> 1) * 16, cb = (warp & 1) * 32;
  double acc[2][4][2], cv[2][4][2];
#pragma unroll
  for (int m = 0; m < 2; m++)
#pragma unroll
    for (int n = 0; n < 4; n++)
#pragma unroll
      for (int e = 0; e < 2; e++) {  // C in flight during the k-loop
        cv[m][n][e] = __ldcg(C + (cb + 8 * n + 2 * lc + e) * TBS + rb + 8 * m + lr);
        acc[m][n][e] = 0.0;
      }
#pragma unroll 4
  for (int ks = 0; ks < TBS / 4; ks++) {
    const int kk = 4 * ks + lc;
    double a[2], b[4];
#pragma unroll
    for (int m = 0; m < 2; m++) a[m] = SG ? A[tsw(rb + 8 * m + lr, kk)] * ssg[kk] : A[tsw(rb + 8 * m + lr, kk)];
#pragma unroll
    for (int n = 0; n < 4; n++) b[n] = B[tsw(cb + 8 * n + lr, kk)];
#pragma unroll
    for (int m = 0; m < 2; m++)
#pragma unroll
      for (int n = 0; n < 4; n++) dmma_nv(acc[m][n][0], acc[m][n][1], a[m], b[n]);
  }
#pragma unroll
  for (int m = 0; m < 2; m++)
#pragma unroll
    for (int n = 0; n < 4; n++)
#pragma unroll
      for (int e = 0; e < 2; e++) {
        const int row = rb + 8 * m + lr, col = cb + 8 * n + 2 * lc + e;
        C[col * TBS + row] = cv[m][n][e] - acc[m][n][e];
      }
}

// Same product into a swizzled shared-memory C (the diagonal update inside CRIT).
template <bool SG = false>
__device__ __forceinline__ void tile_gemm_nt_smem(double* C, const double* A, const double* B, const double* ssg = nullptr) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, lr = lane >> 2, lc = lane & 3;
  const int rb = (warp >> 1) * 16, cb = (warp & 1) * 32;
  double acc[2][4][2];
#pragma unroll
  for (int m = 0; m < 2; m++)
#pragma unroll
    for (int n = 0; n < 4; n++) acc[m][n][0] = acc[m][n][1] = 0.0;
#pragma unroll 4
  for (int ks = 0; ks < TBS / 4; ks++) {
    const int kk = 4 * ks + lc;
    double a[2], b[4];
#pragma unroll
    for (int m = 0; m < 2; m++) a[m] = SG ? A[tsw(rb + 8 * m + lr, kk)] * ssg[kk] : A[tsw(rb + 8 * m + lr, kk)];
#pragma unroll
    for (int n = 0; n < 4; n++) b[n] = B[tsw(cb + 8 * n + lr, kk)];
#pragma unroll
    for (int m = 0; m < 2; m++)
#pragma unroll
      for (int n = 0; n < 4; n++) dmma_nv(acc[m][n][0], acc[m][n][1], a[m], b[n]);
  }
  __syncthreads();
#pragma unroll
  for (int m = 0; m < 2; m++)
#pragma unroll
    for (int n = 0; n < 4; n++)
#pragma unroll
      for (int e = 0; e < 2; e++) {
        const int row = rb + 8 * m + lr, col = cb + 8 * n + 2 * lc + e;
        C[tsw(row, col)] -= acc[m][n][e];
      }
  __syncthreads();
}

// Cholesky of the 32 x 32 diagonal block at (c0, c0) of a swizzled tile by one warp (lane =
// row; rows/columns beyond kb padded with the identity), the software-pipelined pivot chain of
// dense.cuh ll_diag_warp: fma -> shuffle -> rsqrt -> mul per column, column broadcasts through the
// 32 x 32 scratch L11s.  Writes L into T (zeros above the diagonal), the inverse pivots into
// sinv[c0 ..] and dinv[c0 ..] and the first failing column (tile-local) into *fail_k.
// PUB: also publish each finished column to another warp (tile_syrk_potrf64's row solve
// follower): inverse pivot into sinv, then *pflag = c + 1 after the column is in L11s.
template <int c0, bool PUB = false>
__device__ __forceinline__ void tile_diag32(double* T, int kb, int lane, double* dinv, double* sinv,
                                            double* L11s, int* fail_k, volatile int* pflag = nullptr) {
  const int row = c0 + lane;
  double a[32];
#pragma unroll
  for (int c = 0; c < 32; c++)
    a[c] = (lane < kb && c < kb && c <= lane) ? T[tsw(row, c0 + c)] : (c == lane ? 1.0 : 0.0);
  double myinv = 0.0;
  unsigned bad = 0;
  double d = shfl_idx_d(a[0], 0);
  double inv = rsqrt_fast(d);
#pragma unroll
  for (int c = 0; c < 32; c++) {
    const bool b_ = pivot_bad(d);
    bad |= (b_ ? 1u : 0u) << c;
    const double iv = inv;  // a bad pivot already gives a non-finite rsqrt (R6): the check stays off the chain
    if (lane == c) myinv = iv;
    if (PUB && lane == c) sinv[c0 + c] = (c < kb) ? iv : 0.0;
    const double l = (lane > c) ? a[c] * iv : (lane == c ? d * iv : 0.0);
    a[c] = l;
    L11s[c * 32 + lane] = l;
    if (c + 1 < 32) {
      d = shfl_idx_d(fma(-l, l, a[c + 1]), c + 1);
      inv = rsqrt_fast(d);
    }
    warp_bar();
    if (PUB && lane == 0) { __threadfence_block(); *pflag = c + 1; }
    const double2* col2 = reinterpret_cast<const double2*>(L11s + c * 32);
    if ((c + 1) & 1) a[c + 1] = fma(-l, L11s[c * 32 + c + 1], a[c + 1]);
#pragma unroll
    for (int q = (c + 2) / 2; q < 16; q++) {
      const double2 l2 = col2[q];
      a[2 * q] = fma(-l, l2.x, a[2 * q]);
      a[2 * q + 1] = fma(-l, l2.y, a[2 * q + 1]);
    }
    asm volatile("" ::: "memory");  // keep each column's broadcasts in its step (register pressure)
  }
  bad &= (kb < 32) ? ((1u << kb) - 1u) : 0xffffffffu;
#pragma unroll
  for (int c = 0; c < 32; c++)
    if (c < kb) T[tsw(row, c0 + c)] = (lane < kb && c <= lane) ? a[c] : 0.0;
  if (lane < kb) { sinv[c0 + lane] = myinv; dinv[c0 + lane] = myinv; }
  else sinv[c0 + lane] = 0.0;
  if (lane == 0 && bad && *fail_k < 0) *fail_k = c0 + __ffs(bad) - 1;
  warp_bar();
}

// Row solve of rows [r0, r0 + 32*?) handled by threads tid < nrows: x(row, c0:c0+32) against the
// lower 32 x 32 block L(c0:c0+32, c0:c0+32) of the swizzled tile L (inverse pivots sinv), in place
// in the swizzled tile X.  Column-oriented: x_c *= 1/L_cc ; x_c' -= x_c L_c'c (c' > c).
template <int c0>
__device__ __forceinline__ void tile_rowsolve32(double* X, int xrow0, int nrows, const double* L,
                                                const double* sinv) {
  const int t = threadIdx.x;
  if (t < nrows) {
    const int row = xrow0 + t;
    double x[32];
#pragma unroll
    for (int c = 0; c < 32; c++) x[c] = X[tsw(row, c0 + c)];
#pragma unroll
    for (int c = 0; c < 32; c++) {
      x[c] *= sinv[c0 + c];
#pragma unroll
      for (int cc = c + 1; cc < 32; cc++) x[cc] = fma(-x[c], L[tsw(c0 + cc, c0 + c)], x[cc]);
      asm volatile("" ::: "memory");
    }
#pragma unroll
    for (int c = 0; c < 32; c++) X[tsw(row, c0 + c)] = x[c];
  }
}

// X(rows, c1:c1+32) -= X(rows, c0:c0+32) L(c1:c1+32, c0:c0+32)^T for rows [xrow0, xrow0+nr), nr in
// {32, 64}; all threads, DMMA (8 warps: 8-row strips x 32 columns, nr / 8 strips).
template <bool SG = false>
__device__ __forceinline__ void tile_block_update(double* X, int xrow0, int nr, const double* L, int c0, int c1,
                                                  const double* ssg = nullptr) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, lr = lane >> 2, lc = lane & 3;
  const int nstrip = nr >> 3;
  for (int st = warp; st < nstrip; st += 8) {
    const int rb = xrow0 + 8 * st;
    double acc[4][2];
#pragma unroll
    for (int n = 0; n < 4; n++) acc[n][0] = acc[n][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < 8; ks++) {
      const int kk = c0 + 4 * ks + lc;
      const double a = SG ? X[tsw(rb + lr, kk)] * ssg[kk] : X[tsw(rb + lr, kk)];
#pragma unroll
      for (int n = 0; n < 4; n++) dmma_nv(acc[n][0], acc[n][1], a, L[tsw(c1 + 8 * n + lr, kk)]);
    }
#pragma unroll
    for (int n = 0; n < 4; n++)
#pragma unroll
      for (int e = 0; e < 2; e++) X[tsw(rb + lr, c1 + 8 * n + 2 * lc + e)] -= acc[n][e];
  }
}

// L_ik = A_ik L_kk^-T for a whole 64 x 64 tile X (swizzled, in place): 32-column halves with a
// DMMA update between them.  L: the final diagonal tile (k, k); sinv: its 64 inverse pivots.
// LDL^T (SG): the unsigned row solve gives Y = A L~^-T; the signed factor is L~_ik = Y S_k.
template <bool SG = false>
__device__ __forceinline__ void tile_trsm64(double* X, const double* L, const double* sinv, const double* ssg = nullptr) {
  tile_rowsolve32<0>(X, 0, 64, L, sinv);
  __syncthreads();
  tile_block_update(X, 0, 64, L, 0, 32);
  __syncthreads();
  tile_rowsolve32<32>(X, 0, 64, L, sinv);
  __syncthreads();
  if (SG) {
    for (int q = threadIdx.x; q < TBD; q += TILE_THREADS) {
      const int col = q >> 6, row = q & 63;
      X[tsw(row, col)] *= ssg[col];
    }
    __syncthreads();
  }
}

// Signed (LDL^T) Cholesky of a 32 x 32 diagonal block of a swizzled tile (ldlt.cuh rules): one
// warp, lane = row, not pipelined (the LL^T path keeps the pipelined tile_diag32).
template <int c0>
__device__ __forceinline__ void tile_diag32_signed(double* T, int kb, int lane, double* dinv, double* sinv, double* ssg,
                                                   double* L11s, int* fail_k, double* sg_out, double kjj_lane,
                                                   int* cnt3) {
  const int row = c0 + lane;
  double a[32];
#pragma unroll
  for (int c = 0; c < 32; c++)
    a[c] = (lane < kb && c < kb && c <= lane) ? T[tsw(row, c0 + c)] : (c == lane ? 1.0 : 0.0);
  double myinv = 0.0, mys = 1.0;
  unsigned bad = 0;
  int npos = 0, nneg = 0, nzero = 0;
#pragma unroll
  for (int c = 0; c < 32; c++) {
    const double d = shfl_idx_d(a[c], c);
    const double kjj = shfl_idx_d(kjj_lane, c);
    double sgn;
    bool zero, b_;
    const double ad = ldlt_pivot(d, kjj, sgn, zero, b_);
    if (c < kb) {
      bad |= (b_ ? 1u : 0u) << c;
      if (zero) nzero++; else if (sgn > 0) npos++; else nneg++;
    }
    const double inv = 1.0 / sqrt(ad);
    if (lane == c) { myinv = inv; mys = sgn; }
    const double l = (lane > c) ? a[c] * inv * sgn : (lane == c ? ad * inv : 0.0);
    a[c] = l;
    L11s[c * 32 + lane] = l;
    warp_bar();
    const double ls = l * sgn;
#pragma unroll
    for (int cc = c + 1; cc < 32; cc++) a[cc] = fma(-ls, L11s[c * 32 + cc], a[cc]);
    asm volatile("" ::: "memory");
  }
#pragma unroll
  for (int c = 0; c < 32; c++)
    if (c < kb) T[tsw(row, c0 + c)] = (lane < kb && c <= lane) ? a[c] : 0.0;
  if (lane < kb) { sinv[c0 + lane] = myinv; ssg[c0 + lane] = mys; dinv[c0 + lane] = myinv; sg_out[c0 + lane] = mys; }
  else { sinv[c0 + lane] = 0.0; ssg[c0 + lane] = 1.0; }
  bad &= (kb < 32) ? ((1u << kb) - 1u) : 0xffffffffu;
  if (lane == 0) {
    if (bad && *fail_k < 0) *fail_k = c0 + __ffs(bad) - 1;
    if (npos) atomicAdd(cnt3, npos);
    if (nneg) atomicAdd(cnt3 + 1, nneg);
    if (nzero) atomicAdd(cnt3 + 2, nzero);
  }
  warp_bar();
}

// Cholesky of a 64 x 64 diagonal tile T (swizzled, in place) with kb valid columns:
// chol(T00) -> T10 L00^-T -> T11 -= L10 L10^T -> chol(T11).  sinv[64] in shared memory.
// LDL^T variant: signed diagonal blocks, L~10 = Y10 S0 before the signed block update.
__device__ __forceinline__ void tile_potrf64_signed(double* T, int kb, double* dinv, double* sinv, double* L11s,
                                                    int* fail_k, double* ssg, double* sg_out, const double* kjj,
                                                    int* cnt3) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int kb0 = min(kb, 32), kb1 = max(kb - 32, 0);
  if (warp == 0) tile_diag32_signed<0>(T, kb0, lane, dinv, sinv, ssg, L11s, fail_k, sg_out,
                                       lane < kb0 ? kjj[lane] : 1.0, cnt3);
  __syncthreads();
  if (kb1 > 0) {
    tile_rowsolve32<0>(T, 32, 32, T, sinv);
    __syncthreads();
    if (threadIdx.x < 32) {
      for (int c = 0; c < 32; c++) T[tsw(32 + threadIdx.x, c)] *= ssg[c];
    }
    __syncthreads();
    tile_block_update<true>(T, 32, 32, T, 0, 32, ssg);
    __syncthreads();
    if (warp == 0) tile_diag32_signed<32>(T, kb1, lane, dinv, sinv, ssg, L11s, fail_k, sg_out,
                                          lane < kb1 ? kjj[32 + lane] : 1.0, cnt3);
  } else if (warp == 0) {
    for (int c = 0; c < 64; c++) T[tsw(32 + lane, c)] = 0.0;
    sinv[32 + lane] = 0.0;
    ssg[32 + lane] = 1.0;
  }
  __syncthreads();
}

__device__ __forceinline__ void tile_potrf64(double* T, int kb, double* dinv, double* sinv, double* L11s,
                                             int* fail_k) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int kb0 = min(kb, 32), kb1 = max(kb - 32, 0);
  if (warp == 0) tile_diag32<0>(T, kb0, lane, dinv, sinv, L11s, fail_k);
  __syncthreads();
  if (kb1 > 0) {
    tile_rowsolve32<0>(T, 32, 32, T, sinv);
    __syncthreads();
    tile_block_update(T, 32, 32, T, 0, 32);
    __syncthreads();
    if (warp == 0) tile_diag32<32>(T, kb1, lane, dinv, sinv, L11s, fail_k);
  } else if (warp == 0) {
    // kb <= 32: rows / columns 32..63 are padding -- keep them zero, inverse pivots zero
    for (int c = 0; c < 64; c++) T[tsw(32 + lane, c)] = 0.0;
    sinv[32 + lane] = 0.0;
  }
  __syncthreads();
}

// C(rb:rb+8, cb:cb+32) -= A(rb:rb+8, :) A(cb:cb+32, :)^T by one warp (the per-warp DMMA block of
// tile_gemm_nt_smem, same k order: the same sums)
__device__ __forceinline__ void tile_syrk_strip(double* C, const double* A, int rb, int cb) {
  const int lane = threadIdx.x & 31, lr = lane >> 2, lc = lane & 3;
  double acc[4][2];
#pragma unroll
  for (int n = 0; n < 4; n++) acc[n][0] = acc[n][1] = 0.0;
#pragma unroll 4
  for (int ks = 0; ks < TBS / 4; ks++) {
    const int kk = 4 * ks + lc;
    const double a = A[tsw(rb + lr, kk)];
    double b[4];
#pragma unroll
    for (int n = 0; n < 4; n++) b[n] = A[tsw(cb + 8 * n + lr, kk)];
#pragma unroll
    for (int n = 0; n < 4; n++) dmma_nv(acc[n][0], acc[n][1], a, b[n]);
  }
#pragma unroll
  for (int n = 0; n < 4; n++)
#pragma unroll
    for (int e = 0; e < 2; e++) C[tsw(rb + lr, cb + 8 * n + 2 * lc + e)] -= acc[n][e];
}
__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// CRIT's diagonal step (POTRF0: A1 = NULL, no update), A2 -= A1 A1^T then Cholesky of A2, with the update overlapped: warps 0-3
// update the top-left 32 x 32 block while warps 4-7 update the bottom-left one; warp 0 then
// factors the top-left block while warps 4-7 update the bottom-right one (the top-right block is
// above the diagonal: never read).  Same products and factorisation as tile_gemm_nt_smem +
// tile_potrf64.
template <bool FOLLOW = true>
__device__ __forceinline__ void tile_syrk_potrf64(double* A2, const double* A1, int kb, double* dinv, double* sinv,
                                                  double* L11s, int* fail_k) {
  __shared__ int s_col;  // columns of the top-left factor published to the row-solve follower
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int kb0 = min(kb, 32), kb1 = max(kb - 32, 0);
  if (threadIdx.x == 0) s_col = 0;
  if (A1) tile_syrk_strip(A2, A1, warp < 4 ? 8 * warp : 32 + 8 * (warp - 4), 0);
  __syncthreads();  // top-left and bottom-left blocks updated
  if (warp == 0) {
    tile_diag32<0, FOLLOW>(A2, kb0, lane, dinv, sinv, L11s, fail_k, &s_col);
  } else if (FOLLOW && warp == 1 && kb1 > 0) {
    // L21 = A21 L11^-T for rows 32..63, one column behind warp 0 (tile_rowsolve32's arithmetic,
    // L11 read from the published columns)
    const int row = 32 + lane;
    double x[32];
#pragma unroll
    for (int c = 0; c < 32; c++) x[c] = A2[tsw(row, c)];
    volatile int* vc = &s_col;
#pragma unroll
    for (int c = 0; c < 32; c++) {
      while (*vc < c + 1) { }
      __threadfence_block();
      x[c] *= sinv[c];
#pragma unroll
      for (int cc = c + 1; cc < 32; cc++) x[cc] = fma(-x[c], L11s[c * 32 + cc], x[cc]);
    }
#pragma unroll
    for (int c = 0; c < 32; c++) A2[tsw(row, c)] = x[c];
  } else if (A1 && warp >= 4 && kb1 > 0) {
    tile_syrk_strip(A2, A1, 32 + 8 * (warp - 4), 32);
  }
  __syncthreads();
  if (kb1 > 0) {
    if (!FOLLOW) {
      tile_rowsolve32<0>(A2, 32, 32, A2, sinv);
      __syncthreads();
    }
    tile_block_update(A2, 32, 32, A2, 0, 32);
    __syncthreads();
    if (warp == 0) tile_diag32<32>(A2, kb1, lane, dinv, sinv, L11s, fail_k);
  } else if (warp == 0) {
    for (int c = 0; c < 64; c++) A2[tsw(32 + lane, c)] = 0.0;
    sinv[32 + lane] = 0.0;
  }
  __syncthreads();
}

// ------------------------------------------------------------------------------ tasks
struct TileCtx {
  const DevPlan* P;
  const TilePlan* T;
  const double* Kv;   // instance values
  double* Lx;
  const double* Ub;
  double* Dv;
  double* pool;
  int* cnt;
  int* fail_all;
  int task;           // ticket of the current task (trace)
  double* inv;        // instance's inverse-diagonal-tile pool
  double* Sg;         // LDL^T: pivot signs of the instance (internal numbering)
  int* cnt3;          // LDL^T: (positive, negative, zero) pivot counts of the instance
};

__device__ __forceinline__ double* tile_ptr(const TileCtx& X, const TFront& F, int i, int j) {
  return X.pool + F.tbase + (long long)tlin(i, j, F.nt) * TBD;
}
__device__ __forceinline__ int* tile_cnt(const TileCtx& X, const TFront& F, int i, int j) {
  return X.cnt + F.cbase + tlin(i, j, F.nt);
}
__device__ __forceinline__ int* asm_cnt(const TileCtx& X, const TFront& F) {
  return X.cnt + F.cbase + F.nt * (F.nt + 1) / 2;
}
__device__ __forceinline__ int* done_cnt(const TileCtx& X, const TFront& F) { return asm_cnt(X, F) + 1; }
// trace: all dependencies of the current task are met (slot 1)
__device__ __forceinline__ void stamp_ready(const TileCtx& X) {
  if (X.T->trace && threadIdx.x == 0) X.T->trace[4LL * X.task + 1] = gtimer();
}

// ASM(f, i, jt): tile (i, jt) of front f assembled in shared memory -- zero, its K entries, then
// every child's contribution (children in fixed order; a child's rows and columns that land in
// this tile form the rectangle [cut_i, cut_i+1) x [cut_jt, cut_jt+1) of its update matrix) -- and
// written once to the tile pool; cnt(i, jt) = 1 marks it assembled.  A huge child's update tiles
// are read once final (their counter = nbp_c + 1).  All children's values are loaded in one round
// (up to 8 per thread), then added child by child (fixed order, no atomics: deterministic).
__device__ void task_asm(const TileCtx& X, const TFront& F, int i, int jt, double* sm) {
  const DevPlan& P = *X.P;
  const SnInfo I = P.sn[F.s];
  // per child: a, b, ra, rb, huge index, prefix of entries, rel offset, Rc, nbp_c, nt_c
  __shared__ int s_cut[32][10];
  __shared__ long long s_base[32];  // child update matrix (packed Up) or tile pool base
  __shared__ int s_tot;
  const int nch = min(F.nch, 31);
  if (threadIdx.x < nch) {
    const int2 cr = X.T->tch[F.ch0 + threadIdx.x];
    const int* cut = X.T->tcut + cr.y;
    const int a = __ldg(cut + jt), b = __ldg(cut + jt + 1), ra = __ldg(cut + i), rb = __ldg(cut + i + 1);
    const int hc = __ldg(X.T->hidx + cr.x);
    const SnInfo Ci = P.sn[cr.x];
    s_cut[threadIdx.x][0] = a; s_cut[threadIdx.x][1] = b; s_cut[threadIdx.x][2] = ra; s_cut[threadIdx.x][3] = rb;
    s_cut[threadIdx.x][4] = hc;
    s_cut[threadIdx.x][5] = (b > a && rb > ra) ? (b - a) * (rb - ra) : 0;
    s_cut[threadIdx.x][6] = Ci.rp0 + Ci.w;
    s_cut[threadIdx.x][7] = Ci.r - Ci.w;
    s_base[threadIdx.x] = Ci.Up;
    if (hc >= 0) {
      const TFront C = X.T->fr[hc];
      s_cut[threadIdx.x][8] = C.nbp; s_cut[threadIdx.x][9] = C.nt;
      s_base[threadIdx.x] = C.tbase;
    }
    if (hc >= 0 && b > a && rb > ra) {  // wait for the child tiles this rectangle reads
      const TFront C = X.T->fr[hc];
      for (int tj = a >> 6; tj <= (b - 1) >> 6; tj++)
        for (int ti = max(tj, ra >> 6); ti <= (rb - 1) >> 6; ti++) {
          const int* c = X.cnt + C.cbase + tlin(C.nbp + ti, C.nbp + tj, C.nt);
          while (ld_volatile(c) < C.nbp + 1) { __nanosleep(64); }
        }
      fence_acq_rel();
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int q = 0; q < nch; q++) { const int t = s_cut[q][5]; s_cut[q][5] = acc; acc += t; }
    s_cut[nch][5] = acc;
    s_tot = acc;
  }
  stamp_ready(X);
  double* T = sm;  // plain column-major 64 x 64
  for (int q = threadIdx.x; q < TBD / 2; q += TILE_THREADS) reinterpret_cast<double2*>(T)[q] = make_double2(0.0, 0.0);
  const int c_lo = trow0(F, jt), nc = tsize(F, jt), r_lo = trow0(F, i);
  // panel rows above the diagonal tile of this tile column: zero in Lx (read as zero by the solves)
  if (jt < F.nbp && i == jt) {
    double* Lp = X.Lx + I.Lp;
    for (int q = threadIdx.x; q < nc * c_lo; q += TILE_THREADS) {
      const int col = q / c_lo, row = q - col * c_lo;
      Lp[(long long)(c_lo + col) * F.r + row] = 0.0;
    }
  }
  __syncthreads();
  {  // K entries of this tile (kpos = col * r + row)
    const int t = F.cbase + tlin(i, jt, F.nt);
    const int k0 = __ldg(X.T->tkptr + t), k1 = __ldg(X.T->tkptr + t + 1);
    for (int q = k0 + threadIdx.x; q < k1; q += TILE_THREADS) {
      const int k = __ldg(X.T->tkidx + q);
      const int pos = __ldg(P.kpos + k);
      const int col = pos / F.r, row = pos - col * F.r;
      T[(col - c_lo) * TBS + (row - r_lo)] = __ldg(X.Kv + k);
    }
  }
  const int tot = s_tot;
  for (int q0 = 0; q0 < tot; q0 += TILE_THREADS * 8) {
    double v[8];
    int dst[8], chd[8];
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const int qq = q0 + u * TILE_THREADS + threadIdx.x;
      dst[u] = -1;
      chd[u] = -1;
      if (qq < tot) {
        int c = 0;
        while (s_cut[c + 1][5] <= qq) c++;
        const int a = s_cut[c][0], ra = s_cut[c][2], nrow = s_cut[c][3] - ra, hc = s_cut[c][4];
        const int off = qq - s_cut[c][5];
        const int jc = a + off / nrow, ic = ra + off % nrow;
        if (ic >= jc) {
          const int* rel = P.sn_rel + s_cut[c][6];
          if (hc >= 0) {
            const int nbpc = s_cut[c][8];
            v[u] = __ldcg(X.pool + s_base[c] + (long long)tlin(nbpc + (ic >> 6), nbpc + (jc >> 6), s_cut[c][9]) * TBD +
                          (jc & 63) * TBS + (ic & 63));
          } else {
            v[u] = __ldcg(X.Ub + s_base[c] + upk(ic, jc, s_cut[c][7]));
          }
          dst[u] = (__ldg(rel + jc) - c_lo) * TBS + (__ldg(rel + ic) - r_lo);
          chd[u] = c;
        }
      }
    }
    // children in fixed order (the K entries were placed before the first barrier)
    const int c_first = (q0 < tot) ? 0 : 0;
    for (int c = c_first; c < nch; c++) {
      if (s_cut[c + 1][5] <= q0 || s_cut[c][5] >= q0 + TILE_THREADS * 8) continue;  // child not in this chunk
      __syncthreads();
#pragma unroll
      for (int u = 0; u < 8; u++)
        if (chd[u] == c) T[dst[u]] += v[u];
    }
  }
  __syncthreads();
  double2* g = reinterpret_cast<double2*>(tile_ptr(X, F, i, jt));
  for (int q = threadIdx.x; q < TBD / 2; q += TILE_THREADS) g[q] = reinterpret_cast<const double2*>(T)[q];
  publish_cnt(tile_cnt(X, F, i, jt), 1);
}

// sinv[0..64) <- inverse pivots of panel tile k (global Dv, final once tile (k, k) is); with
// LDL^T also ssg[0..64) <- the pivot signs
template <bool SG = false>
__device__ __forceinline__ void load_sinv(const TileCtx& X, const TFront& F, int k, double* sinv, double* ssg = nullptr) {
  const SnInfo I = X.P->sn[F.s];
  if (threadIdx.x < 64) {
    const int c = k * TBS + threadIdx.x;
    const bool v = threadIdx.x < tsize(F, k);
    sinv[threadIdx.x] = v ? __ldcg(X.Dv + I.f0 + c) : 0.0;
    if (SG) ssg[threadIdx.x] = v ? __ldcg(X.Sg + I.f0 + c) : 1.0;
  }
}
// LDL^T: K_jj of the columns of panel tile k (zero-pivot threshold, ldlt.cuh)
__device__ __forceinline__ void load_kjj(const TileCtx& X, const TFront& F, int k, double* kjj) {
  const SnInfo I = X.P->sn[F.s];
  if (threadIdx.x < 64) {
    const int c = I.f0 + k * TBS + threadIdx.x;
    kjj[threadIdx.x] = (threadIdx.x < tsize(F, k)) ? __ldg(X.Kv + __ldg(X.P->Kp + c)) : 1.0;
  }
}

template <bool SG>
__device__ void task_potrf0(const TileCtx& X, const TFront& F, double* sm) {
  double *T0 = sm, *sinv = sm + 3 * TBD, *L11s = sinv + 64, *ssg = L11s + 1024;
  __shared__ int s_fail;
  __shared__ double s_kjj[64];
  if (SG) load_kjj(X, F, 0, s_kjj);
  wait_cnt(tile_cnt(X, F, 0, 0), 1);
  if (threadIdx.x == 0) s_fail = -1;
  tile_load_async(T0, tile_ptr(X, F, 0, 0));
  stamp_ready(X);
  cp_async_wait_all();
  __syncthreads();
  const SnInfo I = X.P->sn[F.s];
  if (SG) tile_potrf64_signed(T0, tsize(F, 0), X.Dv + I.f0, sinv, L11s, &s_fail, ssg, X.Sg + I.f0, s_kjj, X.cnt3);
  else tile_syrk_potrf64(T0, nullptr, tsize(F, 0), X.Dv + I.f0, sinv, L11s, &s_fail);
  tile_store(tile_ptr(X, F, 0, 0), T0);
  if (X.T->panel) tile_to_panel(F, T0, X.Lx + I.Lp, 0, 0);
  if (threadIdx.x == 0 && s_fail >= 0) atomicMin(X.fail_all, I.f0 + s_fail);
  publish_cnt(tile_cnt(X, F, 0, 0), 2);
}

template <bool SG>
__device__ void task_trsm(const TileCtx& X, const TFront& F, int i, int k, double* sm) {
  double *Lk = sm, *A = sm + TBD, *sinv = sm + 3 * TBD, *ssg = sinv + 64 + 1024;
  wait_cnt(tile_cnt(X, F, k, k), k + 2);
  tile_load_async(Lk, tile_ptr(X, F, k, k));
  wait_cnt(tile_cnt(X, F, i, k), k + 1);
  tile_load_async(A, tile_ptr(X, F, i, k));
  load_sinv<SG>(X, F, k, sinv, ssg);
  stamp_ready(X);
  cp_async_wait_all();
  __syncthreads();
  tile_trsm64<SG>(A, Lk, sinv, ssg);
  tile_store(tile_ptr(X, F, i, k), A);
  const SnInfo I = X.P->sn[F.s];
  if (X.T->panel) tile_to_panel(F, A, X.Lx + I.Lp, i, k);
  publish_cnt(tile_cnt(X, F, i, k), k + 2);
}

template <bool SG>
__device__ void task_crit(const TileCtx& X, const TFront& F, int k, double* sm) {
  double *Lk = sm, *A1 = sm + TBD, *A2 = sm + 2 * TBD, *sinv = sm + 3 * TBD, *L11s = sinv + 64, *ssg = L11s + 1024;
  __shared__ int s_fail;
  __shared__ double s_kjj[64];
  if (SG) load_kjj(X, F, k + 1, s_kjj);
  const SnInfo I = X.P->sn[F.s];
  if (threadIdx.x == 0) s_fail = -1;
  // the updated tiles are ready before the previous step's diagonal tile: stage them first
  wait_cnt(tile_cnt(X, F, k + 1, k), k + 1);
  tile_load_async(A1, tile_ptr(X, F, k + 1, k));
  wait_cnt(tile_cnt(X, F, k + 1, k + 1), k + 1);
  tile_load_async(A2, tile_ptr(X, F, k + 1, k + 1));
  wait_cnt(tile_cnt(X, F, k, k), k + 2);
  tile_load_async(Lk, tile_ptr(X, F, k, k));
  load_sinv<SG>(X, F, k, sinv, ssg);
  stamp_ready(X);
  cp_async_wait_all();
  __syncthreads();
  // TRSM(k+1, k), published at once (the other updates of step k may start)
  tile_trsm64<SG>(A1, Lk, sinv, ssg);
  tile_store(tile_ptr(X, F, k + 1, k), A1);
  if (X.T->panel) tile_to_panel(F, A1, X.Lx + I.Lp, k + 1, k);
  publish_cnt(tile_cnt(X, F, k + 1, k), k + 2);
  // A2 -= L1 L1^T, Cholesky of A2
  if (SG) {
    tile_gemm_nt_smem<SG>(A2, A1, A1, ssg);
    tile_potrf64_signed(A2, tsize(F, k + 1), X.Dv + I.f0 + (k + 1) * TBS, sinv, L11s, &s_fail, ssg,
                        X.Sg + I.f0 + (k + 1) * TBS, s_kjj, X.cnt3);
  } else {
    tile_syrk_potrf64(A2, A1, tsize(F, k + 1), X.Dv + I.f0 + (k + 1) * TBS, sinv, L11s, &s_fail);
  }
  tile_store(tile_ptr(X, F, k + 1, k + 1), A2);
  if (X.T->panel) tile_to_panel(F, A2, X.Lx + I.Lp, k + 1, k + 1);
  if (threadIdx.x == 0 && s_fail >= 0) atomicMin(X.fail_all, I.f0 + (k + 1) * TBS + s_fail);
  publish_cnt(tile_cnt(X, F, k + 1, k + 1), k + 3);
}

template <bool SG>
__device__ void task_upd(const TileCtx& X, const TFront& F, int i, int j, int k, double* sm) {
  double *A = sm, *B = sm + TBD, *sinv = sm + 3 * TBD, *ssg = sinv + 64 + 1024;
  wait_cnt(tile_cnt(X, F, i, k), k + 2);
  tile_load_async(A, tile_ptr(X, F, i, k));
  if (j != i) {
    wait_cnt(tile_cnt(X, F, j, k), k + 2);
    tile_load_async(B, tile_ptr(X, F, j, k));
  }
  wait_cnt(tile_cnt(X, F, i, j), k + 1);
  stamp_ready(X);
  if (SG) load_sinv<true>(X, F, k, sinv, ssg);
  cp_async_wait_all();
  __syncthreads();
  tile_gemm_nt_global<SG>(tile_ptr(X, F, i, j), A, j != i ? B : A, ssg);
  publish_cnt(tile_cnt(X, F, i, j), k + 2);
}

// INV(f, k): (L_kk^-1)^T of the final diagonal tile for the triangular solves (tsolve.cuh):
// the row solve of the identity, X = I L_kk^-T (tile_trsm64), off the factorisation's critical path
__device__ void task_inv(const TileCtx& X, const TFront& F, int fidx, int k, double* sm) {
  double *Lk = sm, *A = sm + TBD, *sinv = sm + 3 * TBD;
  wait_cnt(tile_cnt(X, F, k, k), k + 2);
  tile_load_async(Lk, tile_ptr(X, F, k, k));
  load_sinv<false>(X, F, k, sinv);
  for (int q = threadIdx.x; q < TBD; q += TILE_THREADS) {
    const int col = q >> 6, row = q & 63;
    A[tsw(row, col)] = (row == col) ? 1.0 : 0.0;
  }
  stamp_ready(X);
  cp_async_wait_all();
  __syncthreads();
  tile_trsm64<false>(A, Lk, sinv);
  tile_store(X.inv + X.T->ibase[fidx] + (long long)k * TBD, A);
  __syncthreads();
}

template <bool SG>
__global__ void __launch_bounds__(TILE_THREADS, 1) tile_factor_kernel(DevPlan P, TilePlan T, const double* __restrict__ Kv_all,
                                                                    double* Lx_all, const double* U_all, double* Dv_all,
                                                                    int* fail_all) {
  extern __shared__ __align__(16) double tsm[];
  __shared__ int s_task;
  int* ticket = T.cnt + (long long)P.batch * T.ncnt;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_task = atomicAdd(ticket, 1);
    __syncthreads();
    const int t = s_task;
    if (t >= T.ntask) break;
    if (T.trace && threadIdx.x == 0) {
      T.trace[4LL * t] = gtimer();
      unsigned smid;
      asm("mov.u32 %0, %%smid;" : "=r"(smid));
      T.trace[4LL * t + 3] = smid;
    }
    const int4 tk = T.tasks[t];
    const int type = tk.x & 15, b = tk.x >> 4;
    TileCtx X;
    X.P = &P; X.T = &T;
    X.Kv = Kv_all + (long long)b * P.nnzK;
    X.Lx = Lx_all + (long long)b * P.nnzL_stored;
    X.Ub = U_all + (long long)b * P.update_doubles;
    X.Dv = Dv_all + (long long)b * P.n;
    X.pool = T.pool + (long long)b * T.pool_doubles;
    X.cnt = T.cnt + (long long)b * T.ncnt;
    X.fail_all = fail_all;
    X.task = t;
    X.inv = T.inv + (long long)b * T.inv_doubles;
    X.Sg = SG ? P.Sg + (long long)b * P.n : nullptr;
    X.cnt3 = SG ? P.inert + 3 * b : nullptr;
    const TFront F = T.fr[tk.y];
    const int i = tk.z & 0xffff, j = tk.z >> 16, k = tk.w;
    switch (type) {
      case TASK_ASM: task_asm(X, F, i, j, tsm); break;
      case TASK_POTRF0: task_potrf0<SG>(X, F, tsm); break;
      case TASK_TRSM: task_trsm<SG>(X, F, i, k, tsm); break;
      case TASK_CRIT: task_crit<SG>(X, F, k, tsm); break;
      case TASK_INV: task_inv(X, F, tk.y, k, tsm); break;
      default: task_upd<SG>(X, F, i, j, k, tsm); break;
    }
    if (T.trace) {
      __syncthreads();
      if (threadIdx.x == 0) T.trace[4LL * t + 2] = gtimer();
    }
  }
}

}  // namespace kkt
