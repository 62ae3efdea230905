// sblock.h -- subtree blocks of the small supernodes for the triangular solves (sblock.cuh).
//
// A subtree block is a whole etree subtree of small (warp-class) supernodes whose panels and
// solve vectors fit one CTA's shared memory.  In the internal (postorder) numbering such a
// subtree is a contiguous supernode range [s_lo, s_hi] (s_hi = its root), so everything the
// solve reads for it -- the L panels, the SnInfo records, the row / relative-index maps, the
// children lists, the inverse pivots, the permutation and y -- is a handful of contiguous
// global ranges: one CTA stages them with TMA bulk copies and then runs the subtree level by
// level out of shared memory (one warp per supernode, a CTA barrier per level), with no
// global dependency counters or memory round trips between the subtree's supernodes.
// Small supernodes outside every block (their subtree exceeds the budget) keep the per-node
// warp path; they are few (< 1 % on the ACOPF shapes) and lie just below the big phase.
#pragma once
#include <vector>

#include "plan.h"

namespace kkt {

struct alignas(16) SBlk {
  int s_lo, s_hi, nlev, m0;      // supernode range (s_hi = root), levels, offset into meta
  int F0, ncol, RP0, nr;         // column range [F0, F0+ncol); sn_rows range [RP0, RP0+nr)
  int CP0, nch, Rroot, pad;      // sn_ch range [CP0, CP0+nch); update rows of the root
  long long L0, nL;              // panel range [L0, L0+nL) of Lx (doubles)
};
static_assert(sizeof(SBlk) == 64, "SBlk layout");

// Shared-memory layout of one block (doubles; every section starts 16-byte aligned).  The same
// function sizes the block on the host and carves the buffer on the device.
struct SBLayout {
  int L, v, bcol, D, sn, rel, ch, meta, perm, xa, q, total;
};
#ifndef __CUDACC__
#define SB_HD inline
#else
#define SB_HD __host__ __device__ __forceinline__
#endif
// CTA sizes of the tree kernels: 256 threads for latency-bound trees, 128 (more CTAs per SM,
// smaller blocks) for throughput-bound ones; the layout's per-warp scratch depends on it
SB_HD int sb_al(int d) { return (d + 1) & ~1; }            // doubles -> 16-byte multiple
SB_HD int sb_ai(int i) { return ((i + 3) & ~3) / 2; }      // ints -> doubles, 16-byte multiple
// fwd: L | v (sum r) | bcol (ncol) | D | sn | rel | ch | meta
// bwd: L | xl (ncol + Rroot) | xa (per warp 64) | D | sn | lrow (= rel slot) | ch | perm | meta
// both: q = the block's ready queue and per-supernode pending-children counts (ints)
// The TMA-filled sections (L, D, sn, rel, ch, perm, meta) hold the copied range rounded out to
// 16 bytes; the generic-written ones (v / xl, bcol / xa) never share a 16-byte chunk with them.
SB_HD SBLayout sb_layout(int nn, int nlev, long long nL, int ncol, int nr, int nch, int Rroot, int nw) {
  SBLayout o;
  int p = 0;
  o.L = p;    p += sb_al((int)nL + 2);
  o.v = p;    p += sb_al(nr > ncol + Rroot ? nr : ncol + Rroot);   // fwd v buffers / bwd xl (generic writes only)
  o.bcol = p; p += sb_al(ncol > nw * 64 ? ncol : nw * 64);         // fwd bcol / bwd xa
  o.D = p;    p += sb_al(ncol + 2);
  o.sn = p;   p += nn * 8;
  o.rel = p;  p += sb_ai(nr + 4);
  o.ch = p;   p += sb_ai(nch + 4);
  o.perm = p; p += sb_ai(ncol + 4);
  o.meta = p; p += sb_ai(nlev + 1 + nn + 4);
  o.q = p;    p += sb_ai(2 * nn + 4);                                // ready queue + pending counts
  o.xa = o.bcol;
  o.total = p;
  return o;
}

// Factorisation blocks (fblock.cuh): the same subtree partition with the factor's budget --
// fronts F (r x w, the panel layout of Lx) and update matrices U (packed, the layout of Ub) of
// every supernode of the subtree, plus the staged K values and their panel positions.
struct alignas(16) FBlk {
  int s_lo, s_hi, nlev, m0;
  int K0, nK, RP0, nr;           // K entries [K0, K0+nK) of the block's columns; sn_rows range
  int CP0, nch, nL, nU;          // sn_ch range; panel and update-matrix sizes (doubles)
  long long L0, U0;              // panel / update-matrix offsets of the first supernode
};
static_assert(sizeof(FBlk) == 64, "FBlk layout");
struct FBLayout {
  int F, U, K, kpos, sn, rel, ch, meta, q, total;
};
SB_HD FBLayout fb_layout(int nn, int nlev, int nL, int nU, int nK, int nr, int nch) {
  FBLayout o;
  int p = 0;
  o.F = p;    p += sb_al(nL);
  o.U = p;    p += sb_al(nU);
  o.K = p;    p += sb_al(nK + 2);
  o.kpos = p; p += sb_ai(nK + 4);
  o.sn = p;   p += nn * 8;
  o.rel = p;  p += sb_ai(nr + 4);
  o.ch = p;   p += sb_ai(nch + 4);
  o.meta = p; p += sb_ai(nlev + 1 + nn + 4);
  o.q = p;    p += sb_ai(2 * nn + 4);
  o.total = p;
  return o;
}
struct FBlockHost {
  std::vector<FBlk> blk;
  std::vector<int> meta;
  std::vector<int> up_init;  // small supernodes outside the blocks without children (none in practice)
  int n_single = 0, max_smem = 0, nodes_in_blocks = 0;
};
void build_fblocks(const Plan& P, int cap, FBlockHost& out);

struct SBlockHost {
  std::vector<SBlk> blk;     // blocks in increasing root order
  std::vector<int> blk_of;   // [ns] block index if s is a block root, -2 inside a block, -1 otherwise
  std::vector<int> meta;     // per block: nlev + 1 level offsets, then the level-ordered local node ids
  std::vector<int> lrow;     // parallel to sn_rows: backward index into the block's xl (block nodes)
  int n_single = 0;          // small supernodes outside every block
  int max_smem = 0;          // largest block layout (doubles)
  int nodes_in_blocks = 0;
};

// Partition the small supernodes into maximal subtrees whose layout fits `cap` doubles.
void build_sblocks(const Plan& P, int cap, int nw, SBlockHost& out);

}  // namespace kkt
