// devplan.h -- device-side view of the analysis plan and of the per-handle numeric state.
#pragma once
#include <cstdint>

namespace kkt {

struct DevPlan {
  int n, m, m_eq, nnzW, nnzJ, nnzK, ns, batch;
  int max_front;
  long long nnzL_stored, update_doubles, uvec_doubles, nprod;
  const int *perm, *iperm;
  const int *Kp, *Ki, *kw, *kdiag, *pptr, *pa, *pb, *jrow, *kpos;
  const int *sn_first, *sn_rp, *sn_rows, *sn_rel, *sn_parent, *sn_cp, *sn_ch, *order;
  const long long *sn_Lp, *sn_Up, *sn_uvp;
  const int *Wf_p, *Wf_c, *Wf_k, *Jt_p, *Jt_r, *Jt_k, *Gt_end;
  const int *Jrp, *Jci;       // J CSR pattern (caller's, copied at analysis)
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
  unsigned long long* dxn;   // bits of ||dx||_inf
  unsigned long long* xn;    // bits of ||x||_inf
  // CG
  int* cg_done;
  int* cg_iters;
  int* cg_iters_first;
  double* rr;                // r.r
  double* rr0;               // ||r_0||^2
  double* pq;                // p.q
  double* alpha;
  double* beta;
  double* partial;           // [batch][NPART] reduction partials
  unsigned int* part_cnt;    // [batch] arrival counters for last-block reductions
};

}  // namespace kkt
