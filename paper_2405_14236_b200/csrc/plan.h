// plan.h -- host analysis plan of the condensed-KKT solve (internal to libkkt.so).
//
// Built once per sparsity pattern by analyze() (analysis.cpp), uploaded once to the device
// by kkt_bind (kkt_api.cu).  Numbering conventions:
//   "orig"      the caller's variable indices
//   "md"        MD-exact-v1 elimination order (exported by kkt_get_symbolic; bit-exact contract)
//   "internal"  the etree postorder of the md order (equivalent ordering: same fill, same
//               etree shape) used for supernodes so that every supernode is a contiguous
//               column range and siblings' subtrees are contiguous.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "devplan.h"

namespace kkt {

struct Plan {
  int n = 0, m = 0, m_eq = 0, nnzW = 0, nnzJ = 0, batch = 1;

  // ---- ordering / symbolic (md numbering, exported) ----
  std::vector<int> perm_md;      // md -> orig
  std::vector<int> etree_md;     // parent in md numbering, -1 root
  std::vector<int> colcount_md;  // nnz of column j of L (incl. diagonal)

  // ---- internal numbering ----
  std::vector<int> perm;         // internal -> orig
  std::vector<int> iperm;        // orig -> internal

  // ---- K pattern, internal numbering, lower CSC (rows sorted, diagonal first) ----
  std::vector<int> Kp, Ki;
  // K entry k (internal CSC order) -> original (row, col) for export
  // condensation gather map (R16: deterministic, no atomics)
  std::vector<int> kw;           // W_vals index or -1
  std::vector<int> kdiag;        // orig variable index if diagonal entry else -1
  std::vector<int> pptr;         // [nnzK+1] products per K entry
  std::vector<int> pa, pb;       // J_vals indices of the two factors (pa == pb on the diagonal)
  std::vector<int> jrow;         // J row of each J nonzero

  // ---- supernodes (internal numbering) ----
  int ns = 0;
  std::vector<int> sn_first;     // [ns+1] first column
  std::vector<int> sn_rp;        // [ns+1] offsets into sn_rows
  std::vector<int> sn_rows;      // row structure R_s (sorted; first w_s entries = own columns)
  std::vector<int> sn_rel;       // parallel to sn_rows: for t >= w_s, position of R_s[t] in R_parent
  std::vector<long long> sn_Lp;  // [ns+1] panel offsets (r_s x w_s column-major, ld = r_s)
  std::vector<long long> sn_Up;  // [ns+1] packed lower update-matrix offsets, (R)(R+1)/2, R = r-w
  std::vector<long long> sn_uvp; // [ns+1] forward-solve update-vector offsets (length R)
  std::vector<long long> sn_Lip; // [ns] offset of L11^-1 (w x w, col-major) of big non-huge supernodes, -1 otherwise
  std::vector<int> sn_parent;    // -1 root
  std::vector<int> sn_cp, sn_ch; // children lists (CSR)
  std::vector<int> sn_level;     // 0 = leaf
  std::vector<int> order;        // task order: (level, s) ascending
  std::vector<int> order_s, order_b;  // small / big supernodes (devplan.h KKT_SCAP), level order
  int max_r_small = 0;
  // Ready lists (spin-free scheduling, see factor.cuh):
  //   up_s: small leaves (phase-1 bottom-up start);  up_b: big supernodes with no big child
  //   dn_b: big non-huge roots + big non-huge children of huge (top-down start after the huge
  //         phase);                                  dn_s: small roots + small children of big
  std::vector<int> up_s, up_b, dn_b, dn_s;
  std::vector<int> up_bf, order_h;  // big non-huge supernodes with no big non-huge child; huge list
  std::vector<SnInfo> sn;
  std::vector<SnInfo> chinfo;    // parallel to sn_ch: SnInfo of each child (one hop less)
  std::vector<int> sn_hsub;      // subtree height
  std::vector<int> kpos;         // per K entry: offset inside its supernode's panel
  std::vector<int> col_sn;       // internal column -> supernode
  int height = 0, max_front = 0;

  // ---- residual operator maps (orig numbering) ----
  std::vector<int> Wf_p, Wf_c, Wf_k;   // full (both triangles) W: CSR with W_vals index
  std::vector<int> Jt_p, Jt_r, Jt_k;   // J^T CSR: per column the (row, J_vals index)
  std::vector<int> Gt_end;             // per column: end of the rows < m_eq inside Jt (G^T prefix)

  // ---- stats ----
  long long nnzL = 0, nnzL_stored = 0, nprod = 0, update_doubles = 0, uvec_doubles = 0, linv_doubles = 0;
  double flops = 0.0, analyze_ms = 0.0, order_ms = 0.0;
  double flops_huge = 0.0;   // sum over huge supernodes of sum_t (r - t)^2, t < w (stored structure)
  int factor_kind = 0;       // 0 LL^T, 1 pivot-free LDL^T (signed Cholesky, ldlt.cuh)
  int n_huge = 0;
};

struct Options {
  int ordering = 0;
  int factor_kind = 0;   // 1: LDL^T (every supernode on the CTA / tile paths, ldlt.cuh)
  int relax_small = 4;
  int relax_big = 64;
  double relax_zero_frac = 0.05;
  int batch = 1;
};

// Returns empty string on success, else an error message.  code: 1 = arg, 2 = pattern.
std::string analyze(int n, int m, int m_eq, const int* Wp, const int* Wc, const int* Jp,
                    const int* Jc, const Options& opt, Plan& plan, int* code);

// MD-exact-v1 on a symmetric adjacency (no diagonal), quotient graph with exact degrees.
void md_exact_v1(int n, const std::vector<int>& adjp, const std::vector<int>& adji,
                 std::vector<int>& perm);

}  // namespace kkt
