// devplan.h -- device-side view of the analysis plan and of the per-handle numeric state.
#pragma once
#include <cstdint>

namespace kkt {

// Per-warp front capacity (doubles) of the warp-per-supernode kernels.  A supernode is
// "small" when every front in its subtree needs <= KKT_SCAP doubles (panel r*w plus packed
// update matrix R(R+1)/2); small subtrees run one warp per supernode, the remaining top of the
// tree ("big" supernodes) runs one CTA per supernode.  Small is closed under descendants, so
// the small phase never waits on the big phase (bottom-up) and vice versa (top-down).
constexpr int KKT_SCAP = 2048;
constexpr int KKT_WPB = 4;      // warps per CTA in the warp-per-supernode kernels
constexpr int KKT_BNT = 256;    // threads per CTA in the big-supernode kernels
// Fronts needing more than KKT_HCAP doubles (and their ancestors) are factorised by the
// whole-GPU cooperative kernel (huge.cuh); the rest of the big ones by one CTA in shared memory.
constexpr int KKT_HCAP = 25600;

// Per-supernode metadata packed in 64 bytes so one broadcast load fetches it.
struct alignas(16) SnInfo {
  int f0, w, r, rp0;     // first column, width, front rows, offset into sn_rows
  int par, c0, c1, big;  // parent (-1 root), children [c0,c1) in sn_ch, 1 = CTA phase
  int k0, k1, uvp, huge; // K entries of the supernode's columns [k0, k1); update-vector offset;
                         // 1 = factorised by the whole-GPU kernel (huge.cuh)
  long long Lp, Up;      // panel / update-matrix offsets
};
static_assert(sizeof(SnInfo) == 64, "SnInfo must be 64 bytes");

struct DevPlan {
  int n, m, m_eq, nnzW, nnzJ, nnzK, ns, batch;
  int max_front;
  int ns_s, ns_b, ns_bn;       // small / big / big non-huge supernode counts
  int max_r_small;             // largest front among small supernodes
  int max_rw_small;            // largest panel (r*w) among small supernodes (solve staging)
  long long nnzL_stored, update_doubles, uvec_doubles, nprod;
  const int *perm, *iperm;
  const int *Kp, *Ki, *kw, *kdiag, *pptr, *pa, *pb, *jrow, *kpos;
  const int *sn_first, *sn_rp, *sn_rows, *sn_rel, *sn_parent, *sn_cp, *sn_ch, *order;
  const int *order_s, *order_b;  // level order restricted to small / big supernodes
  const SnInfo* sn;              // [ns]
  const SnInfo* chinfo;          // parallel to sn_ch
  // ready lists of the spin-free schedulers
  const int *up_s, *up_b, *dn_b, *dn_s;   // see plan.h
  long long* trace;              // optional [3][ns][2] globaltimer stamps (KKT_TRACE=1), else NULL
  int n_up_s, n_up_b, n_dn_b, n_dn_s;
  const int *up_bf, *order_h;    // big non-huge bottom-up start list; huge supernodes in order
  int solve_huge_cta;            // 1: the solve kernels treat huge supernodes as CTA (big) supernodes
  const int* sn_nbig;            // [ns] number of big (CTA-path) children
  int n_up_bf, n_h;
  const long long *sn_Lp, *sn_Up, *sn_uvp, *sn_Lip;
  long long linv_doubles;
  const int *Wf_p, *Wf_c, *Wf_k, *Jt_p, *Jt_r, *Jt_k, *Gt_end;
  const int *Jrp, *Jci;       // J CSR pattern (caller's, copied at analysis)
  int ldlt;                   // factor_kind 1: signed Cholesky K = L~ S L~^T (ldlt.cuh)
  double* Sg;                 // [batch][n] pivot signs s_j (internal numbering), LDL^T only
  int* inert;                 // [batch][3] (positive, negative, zero) pivot counts, LDL^T only
};

// Device status words (one per batch instance where noted).
struct DevStatus {
  int status;          // kkt_status of the last numeric failure (first wins)
  int fail_col;        // internal column of the first non-SPD pivot (min over instances)
};

// Per-instance refinement / CG control (arrays of length batch).
struct DevCtrl {
  int* done;                 // refinement finished (skip further work)
  int* refine_iters;         // corrections applied
  int* grow;                 // consecutive omega increases
  unsigned long long* omega; // bits of current omega (atomicMax)
  double* omega_prev;        // previous sweep's omega
  double* omega_last;        // reported omega
  double* dxprev;            // ||dx|| of the previous correction
  unsigned long long* dxn;   // bits of ||dx||_inf
  unsigned long long* xn;    // bits of ||x||_inf
  int* sweep;                // refinement sweep counter (device-side loop control)
  // CG
  int* cg_done;
  int* cg_iters;
  int* cg_iters_first;
  double* rr;                // r.r
  double* rr0;               // ||r_0||^2
  double* rr0_first;         // ||r_0||^2 of the first HyKKT pass (absolute target of corrections)
  double* pq;                // p.q
  double* alpha;
  double* beta;
  double* partial;           // [batch][2][NPART] reduction partials
  unsigned int* part_cnt;    // [batch] arrival counters for last-block reductions
  double* rs;                // CR: r.S r
  double* qq;                // CR: q.q
  // HyKKT outer refinement on the saddle system (device-side stop, R9 analogue)
  int* odone;                // [batch+1] instance finished ([batch] = instances still refining)
  unsigned long long* onrm;  // [batch][4] bits of ||ddx||, ||dx||, ||ddy||, ||dy|| (inf norms)
  double* oprev;             // [batch] previous relative correction
  int* opass;                // [batch] correction passes applied
  int* cg_runs;              // executions of the Krylov WHILE body in the last HyKKT solve
};

}  // namespace kkt
