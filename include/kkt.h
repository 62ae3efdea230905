/*
 * kkt.h -- C-ABI of libkkt.so, the B200-native condensed-KKT linear solve of the
 * condensed-space interior-point methods LiftedKKT and HyKKT (arXiv 2405.14236).
 *
 * Citations: P:n = /root/reference/PAPER.md line n (section / equation named); readings
 * R1..R17 are listed in DESIGN.md §3.
 *
 * Conventions for every call
 *   - Indices are 0-based int32.  Host pointers are marked [host], device pointers
 *     [device] (cudaMalloc'd / torch CUDA memory on the device given to kkt_bind).
 *   - The caller owns every buffer it passes.  Host pattern arrays are read only during
 *     kkt_analyze.  Device value arrays must stay valid until the stream work completes.
 *   - The handle owns the analysis plan, its device copy, the factor and all scratch.
 *   - Calls never abort the process.  Argument/state errors are returned immediately;
 *     numeric failures (non-SPD pivot, CG non-convergence, non-finite values) are
 *     recorded in a device status word and surfaced by kkt_sync_info -- the only
 *     host-blocking call besides kkt_analyze/kkt_bind/kkt_destroy and the *_host calls.
 *   - Per-iteration calls (kkt_condense, kkt_factor, kkt_solve, hykkt_solve) are
 *     stream-ordered on the stream given to kkt_bind and do not synchronise the host.
 *   - One in-flight condense->factor->solve sequence per handle.  Handles are
 *     independent; use one per GPU.
 *   - Batch (options.batch = B > 1): B instances share the pattern ("same structure,
 *     different parameters").  Every value array is [B][len] contiguous:
 *     W_vals [B][nnzW], J_vals [B][nnzJ], Sigma_x [B][n], Sigma_s [B][m-m_eq],
 *     D [B][m], b/x/dx [B][n], rbar2/dy [B][m_eq].
 */
#ifndef KKT_H
#define KKT_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct kkt_plan *kkt_handle;   /* opaque */
typedef void *kkt_stream_t;            /* a cudaStream_t (NULL = legacy default stream) */

typedef enum {
  KKT_OK = 0,
  KKT_ERR_ARG = 1,            /* bad argument (null pointer, size, index out of range) */
  KKT_ERR_PATTERN = 2,        /* pattern invalid: unsorted/duplicate/out-of-range/upper entry */
  KKT_ERR_NOT_SPD = 3,        /* a pivot <= 0 or non-finite (R6); fail_col reports it     */
  KKT_ERR_NOT_CONVERGED = 4,  /* HyKKT CG reached cg_maxit before rtol (R10)              */
  KKT_ERR_NONFINITE = 5,      /* non-finite value in a solve / refinement                 */
  KKT_ERR_CUDA = 6,           /* CUDA runtime error (message via kkt_last_error)          */
  KKT_ERR_ALLOC = 7,          /* device or host allocation failed / workspace too small   */
  KKT_ERR_STATE = 8           /* call out of order (e.g. kkt_solve before kkt_factor)     */
} kkt_status;

typedef struct {
  int ordering;          /* 0 = MD-exact-v1 (default; bit-exact contract R11), 1 = natural  */
  int factor_kind;       /* 0 = LL^T (default, R5); 1 = pivot-free LDL^T with inertia (R5b):
                            every supernode on the CTA / tile paths (no warp class)          */
  int relax_small;       /* amalgamation: merge if combined width <= relax_small (perf only) */
  int relax_big;         /* amalgamation: never merge beyond this width                     */
  double relax_zero_frac;/* amalgamation: max fraction of explicit zeros added               */
  int batch;             /* instances sharing the pattern (C5), default 1                   */
} kkt_options;

typedef struct {
  long long nnzK;        /* nnz of the lower triangle of K (diagonal included)            */
  long long nnzL;        /* nnz(L) of the exact (non-amalgamated) factor, sum of colcounts */
  long long nnzL_stored; /* doubles stored in supernodal panels (amalgamated)              */
  double flops;          /* sum_j c_j^2 (SURVEY §8(d) factor work per instance)             */
  long long nprod;       /* products in the condensation map (J^T D J terms)               */
  int nsuper;            /* supernodes after amalgamation                                 */
  int tree_height;       /* height of the supernodal elimination tree (levels)            */
  int max_front;         /* largest front (rows of a supernode)                           */
  double analyze_ms;     /* host time of kkt_analyze                                      */
  double order_ms;       /* of which: MD-exact-v1 ordering                                */
  long long update_doubles; /* per-instance multifrontal update-matrix storage            */
  double flops_huge;     /* factor flops of the "large" supernodes: fronts beyond one CTA's
                            shared memory (> 25600 doubles) and their ancestors, factorised by
                            the whole-GPU DMMA kernel; sum_s sum_{t<w_s} (r_s - t)^2        */
  int nsuper_huge;       /* number of those supernodes                                     */
} kkt_analysis_info;

/* Fill *opt with defaults (MD-exact-v1, LL^T, relax 4/64/0.05, batch 1). */
kkt_status kkt_default_options(kkt_options *opt);

/*
 * kkt_analyze -- once per sparsity pattern ("analysis phase", reported
 * separately from the numeric path).  [host] inputs:
 *   n, m, m_eq     variables; rows of J; rows [0, m_eq) of J are the equalities G whose
 *                  weight is gamma (HyKKT); rows [m_eq, m) carry D_H.
 *                  LiftedKKT: m_eq = 0 and J = H_tau.
 *   W_rowptr[n+1], W_colind[nnzW]   lower triangle of the Hessian W (col <= row), sorted,
 *                  no duplicates.  The diagonal need not be present.
 *   J_rowptr[m+1], J_colind[nnzJ]   Jacobian J (m x n) CSR, sorted, no duplicates.
 * Builds pattern(K) = pattern(W) U pattern(J^T J) U diag, the MD-exact-v1
 * ordering, etree, column counts, supernodes, the condensation gather map and the
 * multifrontal update maps.  On success *handle owns the plan; *info (optional) is filled.
 * Errors: KKT_ERR_ARG (null/negative sizes), KKT_ERR_PATTERN, KKT_ERR_ALLOC.
 */
kkt_status kkt_analyze(int n, int m, int m_eq, const int *W_rowptr, const int *W_colind,
                       const int *J_rowptr, const int *J_colind, const kkt_options *opt,
                       kkt_handle *handle, kkt_analysis_info *info);

/* [host] out: perm[n] (new -> old, MD-exact-v1 order), etree[n] (parent in the permuted
 * numbering, -1 = root), colcount[n] (nnz of column j of L incl. diagonal).  Any may be NULL. */
kkt_status kkt_get_symbolic(kkt_handle h, int *perm, int *etree, int *colcount);

/* Device bytes kkt_bind needs in its caller-provided workspace (per-iteration numeric data
 * for all `batch` instances; the static plan lives in handle-owned memory). */
kkt_status kkt_workspace_size(kkt_handle h, size_t *bytes);

/* Bind the handle to a CUDA device and stream; upload the plan (one H2D copy).
 * d_workspace [device] of >= kkt_workspace_size bytes (caller-owned, e.g. a torch tensor)
 * or NULL to let the library allocate it.  Must be called before any per-iteration call. */
kkt_status kkt_bind(kkt_handle h, int device, void *d_workspace, size_t bytes, kkt_stream_t stream);

/*
 * kkt_condense -- K = W + D_x + delta_w I + J^T D J on the fixed pattern (K1;
 * P:496 K_gamma; P:556 K_tau).  [device] inputs (batch-strided):
 *   W_vals[nnzW], J_vals[nnzJ], Sigma_x[n] (= D_x = X^-1 U), Sigma_s[m - m_eq]
 *   (= D_s = S^-1 V of the inequality rows), D[m] optional override of every row weight
 *   (NULL -> D_r = gamma for r < m_eq, D_r = (Sigma_s+dw)/(1+dc(Sigma_s+dw)) otherwise).
 * The value pointers are remembered by the handle and re-read by kkt_solve / hykkt_solve
 * (the refinement residual uses the UNASSEMBLED operator, R8); keep them unchanged until
 * the next kkt_condense.  Writes K into handle storage.  Non-blocking.
 */
kkt_status kkt_condense(kkt_handle h, const double *W_vals, const double *J_vals,
                        const double *Sigma_x, const double *Sigma_s, const double *D,
                        double delta_w, double delta_c, double gamma);

/* kkt_factor -- pivot-free supernodal multifrontal Cholesky P K P^T = L L^T (P:512, P:524,
 * P:560).  A pivot <= 0 or non-finite records KKT_ERR_NOT_SPD and the failing column
 * (original index) in the device status word; the factor is then invalid.  With factor_kind = 1
 * the pivot-free LDL^T (the paper's cuDSS choice) accepts negative pivots, counts
 * the inertia (kkt_inertia) and fails (KKT_ERR_NONFINITE via kkt_sync_info) only on a
 * non-finite pivot.  Non-blocking. */
kkt_status kkt_factor(kkt_handle h);

/*
 * kkt_solve -- x = K^-1 b by forward/backward supernodal triangular solves,
 * then up to max_refine Richardson sweeps whose residual b - K x is evaluated
 * with the UNASSEMBLED operator W x + (Sigma_x+dw) x + J^T(D o (J x)) in double-double
 * (R8/R9).  Per instance the loop stops (R9) when the correction just applied was negligible
 * (||dx_k|| <= 1e-14 ||x||), when two successive corrections converge geometrically
 * (rho = ||dx_k||/||dx_k-1|| < 1/2 and rho ||dx_k||/(1-rho) <= 1e-14 ||x||), when the
 * componentwise backward error omega grew in two consecutive sweeps, when omega <= tol_bwd
 * (only if tol_bwd > 0; tol_bwd <= 0 disables this test, the default, because a small omega
 * does not bound the forward error of an ill-conditioned K), or after max_refine corrections.
 * [device] b[n], x[n] (batch-strided; may not alias).  Non-blocking.
 */
kkt_status kkt_solve(kkt_handle h, const double *b, double *x, int max_refine, double tol_bwd);

/*
 * hykkt_solve -- HyKKT on K_gamma = K + gamma G^T G, requires a
 * preceding kkt_condense with m_eq > 0 (delta_c applies to inequality rows only)
 * and kkt_factor:
 *   s = rbar1 + gamma G^T rbar2;  CG on S_gamma dy = G K_gamma^-1 s - rbar2 (eq. 14,
 *   x0 = 0, stop ||r_k||_2 <= cg_rtol ||r_0||_2, R10);  dx = K_gamma^-1 (s - G^T dy);
 * then up to max_outer_refine correction passes of refinement on the saddle system
 * [K G^T; G 0] with a double-double residual; per instance the outer loop stops
 * on the device when the relative correction max(||ddx||/||dx||, ||ddy||/||dy||) just applied
 * is <= 1e-14 or two corrections converge geometrically below it (R9 analogue).  The Krylov
 * loop and the outer loop run on the device (one CUDA graph with WHILE nodes, recorded on the
 * first call and re-used while the value pointers, gamma and delta_w are unchanged): no host
 * synchronisation.  cg_rtol <= 0 -> 1e-12; cg_maxit <= 0 -> min(m_eq, 2000).
 * [device] rbar1[n], rbar2[m_eq] in; dx[n], dy[m_eq] out.  Non-blocking;
 * KKT_ERR_NOT_CONVERGED (maxit reached) is reported through kkt_sync_info.
 */
kkt_status hykkt_solve(kkt_handle h, const double *rbar1, const double *rbar2, double *dx,
                       double *dy, double cg_rtol, int cg_maxit, int max_outer_refine);

/* hykkt_solve with the Krylov method chosen: krylov = 0 conjugate gradients (as hykkt_solve),
 * 1 conjugate residuals (CR: "Cr ... ensure a monotonic decrease in the residual
 * norm"; Hestenes-Stiefel form, one S_gamma product per iteration like CG).  Same stopping rule
 * ||r_k||_2 <= cg_rtol ||r_0||_2 (R10).  KKT_ERR_ARG for another value. */
kkt_status hykkt_solve_krylov(kkt_handle h, const double *rbar1, const double *rbar2, double *dx,
                              double *dy, double cg_rtol, int cg_maxit, int max_outer_refine,
                              int krylov);

/*
 * kkt_solve_unreduced -- Newton direction of the unreduced KKT system K3 (eq. K3) with
 * Richardson refinement on K3 itself.  Unknowns
 * d = (dx[n], ds[mi], dy[me], dz[mi], du[n], dv[mi]) with me = m_eq (rows G of J) and
 * mi = m - m_eq (rows H); X, S, U, V = diag(x, s, u, v).  Solves K3 d = f:
 *   W dx + G^T dy + H^T dz - du = f1,   dz - dv = f2,   G dx = f3,   H dx + ds = f4,
 *   U dx + X du = f5,                   V ds + S dv = f6
 * (f = -F_mu of P:306-315).  The condensed factor of the last kkt_condense/kkt_factor is the
 * preconditioner: it must be built with Sigma_x = u/x and Sigma_s = v/s (D_x = X^-1 U, D_s =
 * S^-1 V) -- delta_w, delta_c (and gamma for m_eq > 0, via the HyKKT solve) only
 * regularise the preconditioner; the iteration converges to the unregularised K3 solution.
 * Sweep 1 is the direct solve through the condensed system (recovery of P:360-362);
 * sweeps 2.. are Richardson corrections with a double-double K3 residual.  Per instance the loop
 * stops when the relative correction ||e||_inf / ||d||_inf <= tol (tol <= 0 -> 1e-14), on a
 * geometric prediction below tol, or after 1 + max_refine sweeps; kkt_sync_info's refine_iters
 * reports the corrections applied.  [device] x, u, f1, f5, dx, du [n]; s, v, f2, f4, f6, ds, dz,
 * dv [mi] (may be NULL if mi = 0); f3, dy [me] (NULL if me = 0); batch-strided; outputs are
 * overwritten.  Non-blocking for m_eq = 0; for m_eq > 0 each correction is one hykkt_solve.
 * KKT_ERR_STATE if kkt_condense was given a D override.
 */
kkt_status kkt_solve_unreduced(kkt_handle h, const double *x, const double *s, const double *u,
                               const double *v, const double *f1, const double *f2, const double *f3,
                               const double *f4, const double *f5, const double *f6, double *dx,
                               double *ds, double *dy, double *dz, double *du, double *dv,
                               int max_refine, double tol);

/*
 * kkt_inertia -- inertia of the last LDL^T factorization (factor_kind = 1; P:424-429 eq.
 * ipm:inertia: the counts of positive / negative / zero pivots d_j equal those of the eigenvalues
 * of K by Sylvester's law).  The factor is pivot-free LDL^T in signed-Cholesky form
 * (K = L~ S L~^T, D = S diag(l~)^2, ldlt.cuh); a pivot with |d_j| <= 1e-14 |K_jj| counts as zero
 * (R6) and is replaced by sign(d_j) max(1e-14 |K_jj|, 1e-300).  [host] counts[batch][3] =
 * (positive, negative, zero).  Blocking.  KKT_ERR_STATE for factor_kind 0 or before kkt_factor.
 */
kkt_status kkt_inertia(kkt_handle h, int *counts);

/*
 * kkt_factor_inertia_correct -- condense + factor with the primal regularisation delta_w chosen
 * by the inertia-correction rule of Wachter & Biegler (2006) that the paper uses (P:373-375,
 * "delta_w is chosen dynamically using the inertia information"): try delta_w = 0;
 * else delta_w = dw_first if dw_last = 0, else max(dw_min, k_minus dw_last); while the inertia of
 * the condensed matrix is not (n, 0, 0) (K SPD), multiply delta_w by k_plus_bar
 * (dw_last = 0) or k_plus, and fail (KKT_ERR_NOT_SPD) beyond dw_max.  With factor_kind = 1 the
 * test uses the LDL^T inertia counts, with factor_kind = 0 the Cholesky breakdown (K SPD iff no
 * pivot <= 0).  [device] value arrays as kkt_condense (one delta_w for the whole batch);
 * [host] params[7] = {dw_min, dw_first, dw_max, k_minus, k_plus, k_plus_bar, dw_last} or NULL
 * for {1e-20, 1e-4, 1e40, 1/3, 8, 100, 0}; out: *delta_w_out (the handle is left condensed and
 * factored with it), *tries_out (factorizations).  Blocking (one host sync per try).
 */
kkt_status kkt_factor_inertia_correct(kkt_handle h, const double *W_vals, const double *J_vals,
                                      const double *Sigma_x, const double *Sigma_s, const double *D,
                                      double delta_c, double gamma, const double *params,
                                      double *delta_w_out, int *tries_out);

/* Block the host until the handle's stream is idle; report and clear the device status.
 * Any out pointer may be NULL.  status: a kkt_status value; fail_col: original column of
 * the first non-SPD pivot or -1; refine_iters: sweeps run by the last solve (max over the
 * batch; after hykkt_solve: the outer correction passes run after the first); cg_iters: CG iterations of the first HyKKT pass (max over the batch); bwd_err:
 * componentwise backward error omega after the last solve (max over the batch). */
kkt_status kkt_sync_info(kkt_handle h, int *status, int *fail_col, int *refine_iters,
                         int *cg_iters, double *bwd_err);

/* End-to-end convenience call on HOST buffers (the e2e path of bench.py): copies the
 * values [host] W_vals, J_vals, Sigma_x, Sigma_s, (D or NULL), b to the device, runs
 * condense -> factor -> solve and copies x [host] back.  Blocking. */
kkt_status kkt_step_host(kkt_handle h, const double *W_vals, const double *J_vals,
                         const double *Sigma_x, const double *Sigma_s, const double *D,
                         double delta_w, double delta_c, double gamma, const double *b,
                         double *x, int max_refine, double tol_bwd);

/*
 * kkt_recover -- directions of the eliminated blocks after the condensed solve (P:421-423,
 * SURVEY §8(f) NEXT-1), for the inequality rows [m_eq, m) of J (= H), with the values of the
 * last kkt_condense:
 *   dz = -C r2 + D_H (H dx + r4),  ds = -(D_s + dw I)^-1 (r2 + dz),
 *   C = (I + dc (D_s + dw I))^-1,  D_H = (D_s + dw I) C.
 * [device] r2, r4 [m - m_eq] (K2 right-hand-side blocks), dx [n] (the condensed
 * solution) in; dz, ds [m - m_eq] out (batch-strided).  D overrides are not supported here
 * (KKT_ERR_STATE if kkt_condense was given D).  Non-blocking.
 */
kkt_status kkt_recover(kkt_handle h, const double *r2, const double *r4, const double *dx,
                       double *dz, double *ds);

/*
 * kkt_recover_bounds -- bound-multiplier directions:
 *   du = -X^-1 (U dx - mu e) - u   [n],   dv = -S^-1 (V ds - mu e) - v   [m - m_eq].
 * [device] x, u, dx [n]; s, v, ds [m - m_eq] in; du [n], dv [m - m_eq] out (batch-strided;
 * s/v/ds/dv may be NULL when m == m_eq).  Non-blocking.
 */
kkt_status kkt_recover_bounds(kkt_handle h, const double *x, const double *u, const double *s,
                              const double *v, double mu, const double *dx, const double *ds,
                              double *du, double *dv);

/* Test/debug export of the condensed matrix of batch instance `inst`, lower CSC in ORIGINAL
 * indices: [host] Kp[n+1], Ki[nnzK], Kv[nnzK] (any may be NULL).  Blocking. */
kkt_status kkt_get_condensed(kkt_handle h, int inst, int *Kp, int *Ki, double *Kv);

/* Supernode partition (internal postordered numbering): nsuper; and when
 * non-NULL [host] sn_first[nsuper+1] (first column), sn_nrows[nsuper] (rows of the front),
 * sn_parent[nsuper] (-1 = root).  Call with NULL arrays first to learn nsuper. */
kkt_status kkt_get_supernodes(kkt_handle h, int *nsuper, int *sn_first, int *sn_nrows,
                              int *sn_parent);

/* Subtree blocks of the small supernodes (host plan of the block kernels; test export, needs only
 * kkt_analyze).  kind 0 = the triangular solves (sblock.cuh), 1 = the block factorisation
 * (fblock.cuh); cap = shared-memory budget per block in doubles; nwarps = warps per CTA.  Outputs
 * (host, any may be NULL; call with NULLs first to learn the sizes): nblk, nmeta;
 * blk[nblk][8] = {first supernode, root, levels, offset into meta, layout doubles, 0, 0, 0};
 * blk_of[nsuper] = block index of a block root, -2 inside a block, -1 outside every block;
 * meta[nmeta] = per block nlev + 1 level offsets then the local supernode ids by level;
 * lrow[rows of all fronts] (kind 0) = backward row map; is_big[nsuper] = 1 for CTA-class
 * supernodes.  Errors: KKT_ERR_ARG. */
kkt_status kkt_get_blocks(kkt_handle h, int kind, int cap, int nwarps, int *nblk, int *nmeta, int *blk,
                          int *blk_of, int *meta, int *lrow, int *is_big);

/* Tracing (environment KKT_TRACE=1 at kkt_bind): [host] stamps[3][nsuper][8] = globaltimer
 * (ns) start, end and checkpoints 2..7 of every supernode task of instance 0 in the last factor (row 0), forward
 * (row 1) and backward (row 2) solve.  Blocking.  KKT_ERR_STATE when tracing is off. */
kkt_status kkt_get_trace(kkt_handle h, long long *stamps);

/* Device time of the last kkt_factor split by supernode class (CUDA events on the handle's
 * stream): [host] ms[0] = warp + CTA phases (small and big supernodes, incl. the L11^-1
 * products), ms[1] = whole-GPU phase of the large supernodes (0 if there are none).
 * Blocking (waits for the events).  KKT_ERR_STATE before the first kkt_factor. */
kkt_status kkt_factor_phase_ms(kkt_handle h, double *ms);

/* Number of kernel launches the last per-iteration call enqueued (evidence counter). */
kkt_status kkt_launch_count(kkt_handle h, long long *launches);

/* Work counts of the last hykkt_solve / hykkt_solve_krylov (§3.2): [host]
 * *krylov_total = Krylov iterations (graph WHILE-body executions) summed over the first pass
 * and the outer correction passes (each body = one K_gamma trsv pair for CG, one for CR);
 * *outer_passes = correction passes run after the first (max over the batch).  Either pointer
 * may be NULL.  Blocking (one stream sync).  KKT_ERR_STATE if the last solve was not HyKKT. */
kkt_status kkt_hykkt_stats(kkt_handle h, int *krylov_total, int *outer_passes);

/* Debug export (KKT_TRACE=2 at kkt_bind): copies up to n stamps [host] out[n] of the root
 * front's per-step globaltimer record of the whole-GPU factorization (8 per 32-column step).
 * Returns 0 on success, -1 when the record is off, -2 on a CUDA error.  Blocking. */
int kkt_debug_steps(kkt_handle h, long long *out, int n);

/* Tracing export of the tile-task factorisation of the large fronts: returns the task count
 * (or -1 when there is no tile plan / tracing is off, -2 on a CUDA error) and copies up to n
 * entries: [host] tasks[n][4] (type | instance << 4, front, i | j << 16, k) in issue order,
 * trace[n][4] (globaltimer ns at ticket, dependencies met, end; SM id) when KKT_TRACE=1 was set
 * at kkt_bind; *est_us = the bind-time list-schedule estimate of the makespan.  Blocking. */
int kkt_tile_trace(kkt_handle h, long long *trace, int *tasks, int n, double *est_us);
/* Same for the tile-task solve through the large fronts (last solve launch; task types: gather,
 * forward update, forward chain step, backward update, backward chain step). */
int kkt_tile_solve_trace(kkt_handle h, long long *trace, int *tasks, int n, double *est_us);

/* Last error message (static storage, thread-local). */
const char *kkt_last_error(void);

kkt_status kkt_destroy(kkt_handle h);

#ifdef __cplusplus
}
#endif
#endif /* KKT_H */
