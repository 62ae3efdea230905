// huge.cuh -- whole-GPU factorisation of the top fronts ("huge": front > one CTA's shared
// memory).  Fronts are processed by levels (children before parents, one grid barrier per level);
// the fronts of one level run side by side on disjoint CTA groups.  Per front:
//
//   assemble    group-stride zero / K scatter / extend-add of every child's update matrix
//               (children in fixed order, group barrier between children: deterministic)
//   factorise   tiled right-looking Cholesky as a dataflow over WARPS: the front's lower
//               triangle is cut into 32 x 32 tiles (row/column blocks restart at w so a tile is
//               either panel or update matrix); every tile belongs to one warp of the group for
//               its whole life, so the read-modify-writes of a tile are ordered by that warp's
//               program order.  For step k (panel column block k < nb):
//                 POTRF(k)      L_kk = chol(A_kk)                (warp registers)
//                 TRSM(i,k)     L_ik = A_ik L_kk^-T              (lane = row, L_kk in smem)
//                 UPDATE(i,j,k) A_ij -= L_ik L_jk^T, j > k       (DMMA m8n8k4.f64, fragments
//                                                                  straight from L2)
//               A finished panel tile publishes a flag (batch index + 1); consumers spin on it.
//               Each warp runs its tiles in (k, column, row) order and finalises a tile of
//               column k+1 right after applying step k to it (look-ahead), so the critical path
//               per 32 columns is TRSM -> UPDATE -> POTRF plus three flag hand-offs.  Every wait
//               is on a task earlier in that global order: deadlock-free with all CTAs resident
//               (cooperative launch).
#pragma once
#include <cooperative_groups.h>

#include "dense.cuh"

namespace kkt {

#define HB 32  // tile edge of the huge path (one warp lane per tile row)

// shared memory of factor_huge_kernel: one 32 x 32 scratch tile per warp (doubles)
constexpr int HUGE_SMEM_DOUBLES_PER_WARP = HB * HB;
// warps per CTA of factor_huge_kernel, one CTA per SM (KKT_HUGE_WARPS overrides; 2 or 4 warps
// per SM did not shorten the critical path: measured)
constexpr int HUGE_WARPS = 8;

// Group of CTAs cooperating on one front (contiguous blockIdx range); a group barrier is an
// arrival counter in its own slot (targets grow with the generation), or __syncthreads for 1 CTA.
struct CtaGroup {
  int rank, size;
  int* ctr;
  int gen;
  __device__ __forceinline__ void sync() {
    __syncthreads();
    if (size > 1) {
      if (threadIdx.x == 0) {
        __threadfence();
        gen++;
        atomicAdd(ctr, 1);
        while (ld_volatile(ctr) < gen * size) { }
        __threadfence();
      }
      __syncthreads();
    }
  }
};

// Level schedule of the huge fronts (built at kkt_bind for the launch grid G):
//   lvl_ptr[L]..lvl_ptr[L+1]: entries of level L; entry e = {front s, first CTA, #CTAs, offset of
//   the front's block flags (hsolve.cuh)}; the group barrier counter of entry e is ctr[e]
// Fronts of one level are independent; a level with more fronts than CTAs is run round-robin by
// single-CTA groups (ncta = 0 marks that mode: CTA c takes entries c, c+G, ...).
struct HugeSched {
  const int* lvl_ptr;   // [nlev+1]
  const int4* ent;      // [nent]
  int nlev;
  int* ctr;             // [nent] group barrier counters (zeroed by the kernel)
  int nflag;            // flags per direction: sum over entries of the front's flag count
  int* flags;           // [2 * nflag] tile / block flags (zeroed by the kernel)
  long long* dbg;       // optional [4096][8] per-step stamps of the root front (KKT_TRACE=2)
};

// Tile geometry of one huge front: blocks 0..nb-1 cover the w pivot columns in 32s, blocks
// nb..nt-1 the R update rows/columns (restarting at w).  Tiles (i, j), i >= j, are numbered
// column-major over the lower triangle.
struct HFront {
  double* F;  // r x w panel, ld r
  double* U;  // packed lower update matrix, R x R
  int r, w, nb, nt;
  __device__ __forceinline__ int bstart(int t) const { return t < nb ? t * HB : w + (t - nb) * HB; }
  __device__ __forceinline__ int bsize(int t) const {
    return t < nb ? min(HB, w - t * HB) : min(HB, r - w - (t - nb) * HB);
  }
  __device__ __forceinline__ int lin(int i, int j) const { return j * nt - j * (j - 1) / 2 + (i - j); }
};

__device__ __forceinline__ void tile_wait(const int* f, int target) { spin_acquire(f, target); }
// The warp barrier orders every lane's tile stores before lane 0's gpu-scope release (release is
// cumulative over writes ordered before it), so consumers that acquire the flag see the tile.
__device__ __forceinline__ void tile_publish(int* f, int target, int lane) {
  __syncwarp();
  if (lane == 0) st_release(f, target);
}

// POTRF of diagonal tile k (one warp; lane = row): L_kk and the inverse pivots.  Blocked by 8:
// inside a panel of 8 columns the pivot column is broadcast by shuffles (short dependent chain);
// the panel then updates the trailing columns as a rank-8 update with the panel rows staged in
// the warp's scratch (broadcast LDS.128).  A non-positive pivot lowers *fail_col to its column.
template <int PNL>
__device__ __forceinline__ void potrf_panel(double (&a)[HB], double& myinv, int& fail_col, double* pb,
                                            int lane, int kb, int c0) {
  const unsigned full = 0xffffffffu;
#pragma unroll
  for (int c = 8 * PNL; c < 8 * PNL + 8; c++) {
    if (c < kb) {
      const double d = __shfl_sync(full, a[c], c);
      const bool bad = !(d > 0.0) || !isfinite(d);
      const double inv = bad ? nan_d() : rsqrt(d);
      double l = a[c] * inv;
      if (lane == c) {
        l = d * inv;
        myinv = inv;
        if (bad) fail_col = min(fail_col, c0 + c);
      }
      a[c] = (lane >= c) ? l : 0.0;
#pragma unroll
      for (int cc = c + 1; cc < 8 * PNL + 8; cc++) {
        const double lcc = __shfl_sync(full, l, cc);  // L[cc][c]
        if (lane > c) a[cc] = fma(-l, lcc, a[cc]);
      }
    }
  }
  if (PNL < HB / 8 - 1 && 8 * PNL + 8 < kb) {  // trailing: a[cc] -= sum_q L[lane][8P+q] L[cc][8P+q]
#pragma unroll
    for (int q = 0; q < 8; q++) pb[lane * 8 + q] = a[8 * PNL + q];
    __syncwarp();
#pragma unroll
    for (int cc = 8 * PNL + 8; cc < HB; cc++) {
#pragma unroll
      for (int q = 0; q < 8; q++) a[cc] = fma(-a[8 * PNL + q], pb[cc * 8 + q], a[cc]);
    }
    __syncwarp();
  }
}

__device__ __forceinline__ void tile_potrf(const HFront& H, int k, double* dinv, double* pb, int lane,
                                           int* fail_col) {
  // software-pipelined warp Cholesky of the diagonal tile (dense.cuh ll_diag_warp: raw shuffle +
  // branch-free rsqrt on the pivot chain, shared-memory column broadcasts); loads bypass L1
  // (the tile was produced by other SMs in this launch).  pb: the warp's 32 x 32 scratch.
  int fk = -1;
  ll_diag_warp<true>(H.F, H.r, k * HB, H.bsize(k), lane, dinv, pb, pb, &fk);
  if (lane == 0 && fk >= 0) *fail_col = min(*fail_col, fk);
  __syncwarp();  // scratch reuse
}

// TRSM of panel tile (i, k), i > k: L_ik = A_ik L_kk^-T (one warp; lane = row; L_kk staged in
// the warp's shared scratch for broadcast reads).
__device__ __forceinline__ void tile_trsm(const HFront& H, int i, int k, const double* dinv, double* Ls,
                                          int lane) {
  const int c0 = k * HB, kb = H.bsize(k);
  const int r0 = H.bstart(i), ib = H.bsize(i);
  const unsigned full = 0xffffffffu;
#pragma unroll
  for (int c = 0; c < HB; c++)
    Ls[c * HB + lane] = (c < kb && lane < kb && lane > c) ? ldcg(H.F + (long long)(c0 + c) * H.r + c0 + lane) : 0.0;
  const double di = (lane < kb) ? ldcg(dinv + c0 + lane) : 0.0;
  double x[HB];
#pragma unroll
  for (int c = 0; c < HB; c++)
    x[c] = (lane < ib && c < kb) ? ldcg(H.F + (long long)(c0 + c) * H.r + r0 + lane) : 0.0;
  __syncwarp();
#pragma unroll
  for (int c = 0; c < HB; c++) {
    if (c < kb) {
      x[c] *= __shfl_sync(full, di, c);
#pragma unroll
      for (int t = c + 1; t < HB; t++) x[t] = fma(-x[c], Ls[c * HB + t], x[t]);
    }
  }
#pragma unroll
  for (int c = 0; c < HB; c++)
    if (lane < ib && c < kb) H.F[(long long)(c0 + c) * H.r + r0 + lane] = x[c];
  __syncwarp();  // scratch reuse
}

// UPDATE of tile (i, j) by panel column block k: A_ij -= L_ik L_jk^T on DMMA (one warp).
// m8n8k4 fragments come straight from L2: for k-step ks the lane reads
// L[8m + lane/4][4 ks + lane%4] of row block i (A operand) and of row block j (B operand).
__device__ __forceinline__ void tile_update(const HFront& H, int i, int j, int k, int lane) {
  const int c0 = k * HB, kb = H.bsize(k);
  const int ri = H.bstart(i), ni = H.bsize(i), rj = H.bstart(j), nj = H.bsize(j);
  const bool dg = (i == j);
  const int lr = lane >> 2, lc = lane & 3;
  double c0v[4][4], c1v[4][4];
#pragma unroll
  for (int m = 0; m < 4; m++)
#pragma unroll
    for (int n = 0; n < 4; n++) { c0v[m][n] = 0.0; c1v[m][n] = 0.0; }
#pragma unroll
  for (int ks = 0; ks < HB / 4; ks++) {
    if (ks * 4 < kb) {
      const int kk = ks * 4 + lc;
      const bool kv = kk < kb;
      const double* col = H.F + (long long)(c0 + kk) * H.r;
      double fa[4], fb[4];
#pragma unroll
      for (int m = 0; m < 4; m++) fa[m] = (kv && 8 * m + lr < ni) ? ldcg(col + ri + 8 * m + lr) : 0.0;
#pragma unroll
      for (int n = 0; n < 4; n++)
        fb[n] = dg ? fa[n] : ((kv && 8 * n + lr < nj) ? ldcg(col + rj + 8 * n + lr) : 0.0);
#pragma unroll
      for (int m = 0; m < 4; m++)
#pragma unroll
        for (int n = 0; n < 4; n++)
          if (!dg || n <= m) dmma8x8x4(c0v[m][n], c1v[m][n], fa[m], fb[n]);
    }
  }
  // read-modify-write of the tile, two row halves: all loads of a half before its stores
#pragma unroll
  for (int h = 0; h < 2; h++) {
    double* pp[16];
    double old[16];
#pragma unroll
    for (int mm = 0; mm < 2; mm++)
#pragma unroll
      for (int n = 0; n < 4; n++)
#pragma unroll
        for (int e = 0; e < 2; e++) {
          const int a = 8 * (2 * h + mm) + lr, b = 8 * n + 2 * lc + e;
          const bool v = (a < ni) && (b < nj) && (!dg || a >= b);
          pp[(mm * 4 + n) * 2 + e] = v ? front_at(H.F, H.U, H.r, H.w, ri + a, rj + b) : nullptr;
        }
#pragma unroll
    for (int q = 0; q < 16; q++) old[q] = pp[q] ? ldcg(pp[q]) : 0.0;
#pragma unroll
    for (int mm = 0; mm < 2; mm++)
#pragma unroll
      for (int n = 0; n < 4; n++) {
        const int q = (mm * 4 + n) * 2;
        if (pp[q]) *pp[q] = old[q] - c0v[2 * h + mm][n];
        if (pp[q + 1]) *pp[q + 1] = old[q + 1] - c1v[2 * h + mm][n];
      }
  }
}

__global__ void __launch_bounds__(256, 1) factor_huge_kernel(DevPlan P, const double* __restrict__ Kv_all,
                                                             double* Lx_all, double* U_all, double* Dv_all,
                                                             int* cnt_all, int* fail_all, HugeSched H) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double sm[];
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  double* ws = sm + warp * HB * HB;  // this warp's scratch tile
  for (int q = blockIdx.x * nt + tid; q < H.lvl_ptr[H.nlev]; q += gridDim.x * nt) H.ctr[q] = 0;
  for (int q = blockIdx.x * nt + tid; q < H.nflag; q += gridDim.x * nt) H.flags[q] = 0;
  grid.sync();
  for (int L = 0; L < H.nlev; L++) {
   const int e0 = H.lvl_ptr[L], e1 = H.lvl_ptr[L + 1];
   const bool rr = (H.ent[e0].z == 0);  // round-robin singletons
   for (int e = rr ? e0 + (int)blockIdx.x : e0; e < e1; e += rr ? (int)gridDim.x : 1) {
    const int4 E = H.ent[e];
    CtaGroup G;
    if (rr) { G.rank = 0; G.size = 1; }
    else {
      if ((int)blockIdx.x < E.y || (int)blockIdx.x >= E.y + E.z) continue;
      G.rank = blockIdx.x - E.y; G.size = E.z;
    }
    G.ctr = H.ctr + e; G.gen = 0;
    const long long gtid = (long long)G.rank * nt + tid, gnt = (long long)G.size * nt;
    const int s = E.x;
    const SnInfo I = P.sn[s];
    const int r = I.r, w = I.w, R = r - w;
    const long long pw = (long long)r * w;
    const long long usz = I.par >= 0 ? (long long)R * (R + 1) / 2 : 0;
    for (int b = 0; b < P.batch; b++) {
      if (gtid == 0) trace_stamp(P, 0, s, b, 0);
      double* F = Lx_all + (long long)b * P.nnzL_stored + I.Lp;
      double* U = U_all + (long long)b * P.update_doubles + I.Up;
      const double* Ub = U_all + (long long)b * P.update_doubles;
      const double* Kv = Kv_all + (long long)b * P.nnzK;
      double* dinv = Dv_all + (long long)b * P.n + I.f0;
      if (gtid == 0) cnt_all[(long long)b * P.ns + s] = 0;  // children are complete
      // ---------------- assemble ----------------
      for (long long q = gtid; q < pw; q += gnt) F[q] = 0.0;
      for (long long q = gtid; q < usz; q += gnt) U[q] = 0.0;
      G.sync();
      for (long long k = I.k0 + gtid; k < I.k1; k += gnt) F[__ldg(P.kpos + k)] = __ldg(Kv + k);
      for (int ci = I.c0; ci < I.c1; ci++) {
        const SnInfo C = P.chinfo[ci];
        const int Rc = C.r - C.w;
        const int* rel = P.sn_rel + C.rp0 + C.w;
        const double* Uc = Ub + C.Up;
        const long long tot = (long long)Rc * (Rc + 1) / 2;
        G.sync();
        for (long long q0 = gtid; q0 < tot; q0 += gnt * 8) {
          // 8 entries per thread per round: all loads (child values, relative indices, old
          // front values) are issued before the stores
          double* dst[8];
          double val[8];
#pragma unroll
          for (int u = 0; u < 8; u++) {
            const long long q = q0 + (long long)u * gnt;
            dst[u] = nullptr;
            if (q < tot) {
              // decode packed (column-major lower) index q -> (ic, jc)
              const double tR = 2.0 * Rc + 1.0;
              int jc = (int)((tR - sqrt(tR * tR - 8.0 * (double)q)) * 0.5);
              if (jc < 0) jc = 0;
              if (jc > Rc - 1) jc = Rc - 1;
              while (jc > 0 && upk(jc, jc, Rc) > q) jc--;
              while (jc + 1 < Rc && upk(jc + 1, jc + 1, Rc) <= q) jc++;
              const int ic = jc + (int)(q - upk(jc, jc, Rc));
              const int pj = __ldg(rel + jc), pi = __ldg(rel + ic);
              val[u] = ldcg(Uc + q);
              dst[u] = (pj < w) ? F + (long long)pj * r + pi : U + upk(pi - w, pj - w, R);
            }
          }
          double old[8];
#pragma unroll
          for (int u = 0; u < 8; u++) old[u] = dst[u] ? ldcg(dst[u]) : 0.0;  // L1 is not coherent
#pragma unroll
          for (int u = 0; u < 8; u++)
            if (dst[u]) *dst[u] = old[u] + val[u];
        }
      }
      G.sync();
      if (gtid == 0) trace_stamp(P, 0, s, b, 2);
      // ---------------- tile dataflow factorisation ----------------
      {
        HFront Hf;
        Hf.F = F; Hf.U = U; Hf.r = r; Hf.w = w;
        Hf.nb = (w + HB - 1) / HB;
        Hf.nt = Hf.nb + (R + HB - 1) / HB;
        int* tf = H.flags + E.w;
        const int tgt = b + 1;
        const int wpc = nt >> 5;  // warps per CTA
        const int me = G.rank * wpc + warp, NW = G.size * wpc;
        int fail_col = INT_MAX;
        // finalise panel tile (i, kk): POTRF if diagonal, else TRSM once L_kk is published
        long long* dbg = (H.dbg && s == P.ns - 1 && b == 0) ? H.dbg : nullptr;
        auto stamp = [&](int kk, int ev) { if (dbg && lane == 0 && kk < 4096) dbg[kk * 8 + ev] = gtimer(); };
        auto finalise = [&](int i, int kk) {
          if (i == kk) {
            stamp(kk, 0);
            tile_potrf(Hf, kk, dinv, ws, lane, &fail_col);
            stamp(kk, 1);
            if (lane == 0 && (kk == 1 || kk == 2 || kk == Hf.nb - 1)) trace_stamp(P, 0, s, b, kk == 1 ? 3 : kk == 2 ? 4 : 5);
          } else {
            if (i == kk + 1) stamp(kk, 7);
            tile_wait(tf + Hf.lin(kk, kk), tgt);
            if (i == kk + 1) stamp(kk, 2);
            tile_trsm(Hf, i, kk, dinv, ws, lane);
            if (i == kk + 1) stamp(kk, 3);
          }
          tile_publish(tf + Hf.lin(i, kk), tgt, lane);
        };
        for (int k = 0; k < Hf.nb; k++) {
          // this warp's tiles with column >= k, column-major (tile t is owned by warp t mod NW)
          const int l0 = Hf.lin(k, k);
          int q = ((me - l0) % NW + NW) % NW;  // offset of the first owned tile from (k, k)
          int j = k;
          while (j < Hf.nt && q >= Hf.nt - j) { q -= Hf.nt - j; j++; }
          while (j < Hf.nt) {
            const int i = j + q;
            if (j == k) {
              if (k == 0) finalise(i, 0);  // columns k > 0 were finalised one step early
            } else {
              const bool crit = (i == k + 1 && j == k + 1);
              if (crit) stamp(k, 6);
              tile_wait(tf + Hf.lin(i, k), tgt);
              tile_wait(tf + Hf.lin(j, k), tgt);
              if (crit) stamp(k, 4);
              tile_update(Hf, i, j, k, lane);
              if (crit) stamp(k, 5);
              if (j == k + 1 && j < Hf.nb) finalise(i, j);  // look-ahead
            }
            q += NW;
            while (j < Hf.nt && q >= Hf.nt - j) { q -= Hf.nt - j; j++; }
          }
        }
        fail_col = __reduce_min_sync(0xffffffffu, fail_col);
        if (lane == 0 && fail_col != INT_MAX) atomicMin(fail_all, I.f0 + fail_col);
      }
      if (lane == 0) trace_max(P, 0, s, b, 1);
    }
   }
   grid.sync();  // level done: the next level's fronts may read these update matrices
  }
}

}  // namespace kkt
