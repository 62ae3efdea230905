// huge.cuh -- whole-GPU factorisation of the top fronts ("huge": front > one CTA's shared
// memory), one front at a time in topological order, by a cooperative persistent kernel:
//
//   assemble    grid-stride zero / K scatter / extend-add of every child's update matrix
//               (children in fixed order, grid barrier between children: deterministic)
//   for each column block [k0, k0+kb), kb <= 32:
//     a. every CTA factors the kb x kb diagonal block in one warp's registers (redundantly,
//        saving a barrier); CTA 0 writes L_kk and the inverse pivots
//     b. TRSM: rows below the block, one thread per row, column-oriented sweep
//     -- grid barrier --
//     c. trailing update of the lower triangle of rows/cols [k0+kb, r) in 64 x 64 tiles over
//        all CTAs: operands staged in shared memory, 8 warps x 8 DMMA (m8n8k4.f64) tiles
//     -- grid barrier --
#pragma once
#include <cooperative_groups.h>

#include "dense.cuh"

namespace kkt {

#define HB 32          // column block of the huge path (diagonal block held in registers)
#define HT 64          // trailing-update tile edge
#define HT_LD (HT + 1) // padded leading dimension of staged operands (bank spread)

// shared memory layout of factor_huge_kernel (doubles)
constexpr int HUGE_SMEM_DOUBLES = HB * HB + HB + 2 * HB * HT_LD;

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
  int nflag;            // sum over entries of ceil(w / 32) (solve block flags per direction)
};

__global__ void __launch_bounds__(256) factor_huge_kernel(DevPlan P, const double* __restrict__ Kv_all,
                                                          double* Lx_all, double* U_all, double* Dv_all,
                                                          int* cnt_all, int* fail_all, HugeSched H) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double sm[];
  double* Dg = sm;                  // [HB][HB] diagonal block, column-major (ld HB)
  double* dsh = Dg + HB * HB;       // [HB] inverse pivots
  double* As = dsh + HB;            // [HB][HT_LD] rows of tile i (k-major)
  double* Bs = As + HB * HT_LD;     // [HB][HT_LD] rows of tile j
  __shared__ int s_fail;
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;

  for (int e = blockIdx.x; e < H.lvl_ptr[H.nlev]; e += gridDim.x) H.ctr[e] = 0;
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
      // ---------------- blocked factorisation ----------------
      if (tid == 0) s_fail = -1;
      for (int k0 = 0; k0 < w; k0 += HB) {
        const int kb = (w - k0) < HB ? (w - k0) : HB;
        // a. diagonal block in warp 0's registers (every CTA)
        if (warp == 0) {
          double a[HB];
          const int row = k0 + lane;
#pragma unroll
          for (int c = 0; c < HB; c++)
            a[c] = (lane < kb && c < kb && c <= lane) ? ldcg(F + (long long)(k0 + c) * r + row) : 0.0;
#pragma unroll
          for (int c = 0; c < HB; c++) {
            if (c < kb) {
              __syncwarp();
              double lc[HB];
#pragma unroll
              for (int cc = 0; cc < HB; cc++) lc[cc] = __shfl_sync(0xffffffffu, a[c], cc);
              const double d = lc[c];
              const bool bad = !(d > 0.0) || !isfinite(d);
              const double inv = bad ? nan_d() : rsqrt(d);
              if (lane == 0) {
                dsh[c] = inv;
                if (bad && s_fail < 0) s_fail = k0 + c;
              }
              if (lane > c) {
                const double l = a[c] * inv;
                a[c] = l;
#pragma unroll
                for (int cc = c + 1; cc < HB; cc++) a[cc] = fma(-l, lc[cc] * inv, a[cc]);
              } else if (lane == c) {
                a[c] = d * inv;
              }
            }
          }
#pragma unroll
          for (int c = 0; c < HB; c++) Dg[c * HB + lane] = (c <= lane && lane < kb && c < kb) ? a[c] : 0.0;
        }
        __syncthreads();
        if (gtid == 0 && k0 == 0) trace_stamp(P, 0, s, b, 3);
        // b. TRSM: rows i in [k0+kb, r), x = f L_kk^-T, column-oriented sweep per row
        for (long long i = k0 + kb + gtid; i < r; i += gnt) {
          double x[HB];
#pragma unroll
          for (int c = 0; c < HB; c++) x[c] = (c < kb) ? ldcg(F + (long long)(k0 + c) * r + i) : 0.0;
#pragma unroll
          for (int c = 0; c < HB; c++) {
            if (c < kb) {
              x[c] *= dsh[c];
#pragma unroll
              for (int t = c + 1; t < HB; t++) x[t] = fma(-x[c], Dg[c * HB + t], x[t]);
            }
          }
#pragma unroll
          for (int c = 0; c < HB; c++)
            if (c < kb) F[(long long)(k0 + c) * r + i] = x[c];
        }
        G.sync();
        if (gtid == 0 && k0 == 0) trace_stamp(P, 0, s, b, 4);
        // every CTA has finished reading the unfactored diagonal block: CTA 0 stores L_kk
        if (G.rank == 0) {
          for (int q = tid; q < kb * kb; q += nt) {
            const int c = q / kb, i = q % kb;
            if (i >= c) F[(long long)(k0 + c) * r + k0 + i] = Dg[c * HB + i];
          }
          for (int q = tid; q < kb; q += nt) dinv[k0 + q] = dsh[q];
        }
        // c. trailing update in HT x HT tiles
        const int j0 = k0 + kb, m = r - j0;
        if (m > 0) {
          const int ntl = (m + HT - 1) / HT;
          const long long ntiles = (long long)ntl * (ntl + 1) / 2;
          for (long long t = G.rank; t < ntiles; t += G.size) {
            int tj = 0;
            long long rem = t;
            while (rem >= ntl - tj) { rem -= ntl - tj; tj++; }
            const int ti = tj + (int)rem;
            const int i0 = j0 + ti * HT, jj0 = j0 + tj * HT;
            __syncthreads();
            {  // stage the two 32 x 64 operand panels: all loads in flight before the stores
              constexpr int PER = (HB * HT) / 256;  // 8 elements of each panel per thread
              double va[PER], vb[PER];
#pragma unroll
              for (int u = 0; u < PER; u++) {
                const int q = tid + u * 256, k = q / HT, i = q % HT;
                const bool kin = k < kb;
                va[u] = (kin && i0 + i < r) ? ldcg(F + (long long)(k0 + k) * r + i0 + i) : 0.0;
                vb[u] = (kin && jj0 + i < r) ? ldcg(F + (long long)(k0 + k) * r + jj0 + i) : 0.0;
              }
#pragma unroll
              for (int u = 0; u < PER; u++) {
                const int q = tid + u * 256, k = q / HT, i = q % HT;
                As[k * HT_LD + i] = va[u];
                Bs[k * HT_LD + i] = vb[u];
              }
            }
            __syncthreads();
            // 64 x 64 = 8 x 8 DMMA tiles; warp w owns tile row w x all 8 tile columns
            double c0[8], c1[8];
#pragma unroll
            for (int y = 0; y < 8; y++) { c0[y] = 0.0; c1[y] = 0.0; }
            __syncwarp();
            for (int kk = 0; kk < kb; kk += 4) {
              const int k = kk + (lane & 3);
              const double a = As[k * HT_LD + warp * 8 + (lane >> 2)];
              double bb[8];
#pragma unroll
              for (int y = 0; y < 8; y++) bb[y] = Bs[k * HT_LD + y * 8 + (lane >> 2)];
#pragma unroll
              for (int y = 0; y < 8; y++) dmma8x8x4(c0[y], c1[y], a, bb[y]);
            }
            const int i = i0 + warp * 8 + (lane >> 2);
            // read-modify-write of the 16 outputs: all 16 loads issued before the stores
            double* pp[16];
            double old[16];
#pragma unroll
            for (int y = 0; y < 8; y++) {
              const int jb = jj0 + y * 8 + (lane & 3) * 2;
              pp[2 * y] = (i < r && jb <= i) ? front_at(F, U, r, w, i, jb) : nullptr;
              pp[2 * y + 1] = (i < r && jb + 1 <= i) ? front_at(F, U, r, w, i, jb + 1) : nullptr;
            }
#pragma unroll
            for (int e = 0; e < 16; e++) old[e] = pp[e] ? ldcg(pp[e]) : 0.0;
#pragma unroll
            for (int y = 0; y < 8; y++) {
              if (pp[2 * y]) *pp[2 * y] = old[2 * y] - c0[y];
              if (pp[2 * y + 1]) *pp[2 * y + 1] = old[2 * y + 1] - c1[y];
            }
          }
        }
        G.sync();
        if (gtid == 0 && k0 == 0) trace_stamp(P, 0, s, b, 5);
        if (gtid == 0 && k0 == HB) trace_stamp(P, 0, s, b, 6);
      }
      if (tid == 0 && s_fail >= 0) atomicMin(fail_all, I.f0 + s_fail);
      if (gtid == 0) trace_stamp(P, 0, s, b, 1);
    }
   }
   grid.sync();  // level done: the next level's fronts may read these update matrices
  }
}

}  // namespace kkt
