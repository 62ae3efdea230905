// kkt_api.cu -- C-ABI of libkkt.so (include/kkt.h): plan upload, workspace carving and the
// stream-ordered launch sequences of the per-IPM-iteration hot path.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/kkt.h"
#include "cg_kernels.cuh"
#include "condense.cuh"
#include "factor.cuh"
#include "hsolve.cuh"
#include "resid.cuh"
#include "trsv.cuh"
#include "sblock.cuh"
#include "fblock.cuh"
#include "tiles.cuh"
#include "tsolve.cuh"
#include "k3.cuh"
#include "plan.h"
#include "tile_plan.h"

using namespace kkt;

static thread_local std::string g_err;

#define CUDA_TRY(x)                                                                \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      g_err = std::string(#x) + ": " + cudaGetErrorString(e_);                     \
      return e_ == cudaErrorMemoryAllocation ? KKT_ERR_ALLOC : KKT_ERR_CUDA;       \
    }                                                                              \
  } while (0)

#define LAUNCH_CHECK()                                                             \
  do {                                                                             \
    cudaError_t e_ = cudaGetLastError();                                           \
    if (e_ != cudaSuccess) {                                                       \
      g_err = std::string("launch: ") + cudaGetErrorString(e_);                    \
      return KKT_ERR_CUDA;                                                         \
    }                                                                              \
  } while (0)

#define TRY(x) do { kkt_status s_ = (x); if (s_ != KKT_OK) return s_; } while (0)

struct kkt_plan {
  Plan P;
  int device = -1;
  cudaStream_t stream = nullptr;   // caller's stream (all work is ordered on it)
  cudaStream_t ls = nullptr;       // kernel-launch stream: == stream, or the capture stream
  cudaStream_t cap = nullptr;      // private stream used only to record CUDA graphs
  bool bound = false;
  // CUDA graph of the whole refined solve (fixed internal b / x buffers)
  bool use_graph = true;
  cudaGraphExec_t solve_exec = nullptr;
  int g_max_refine = -1;
  double g_tol = -1.0, g_dw = 0.0;
  const void *g_W = nullptr, *g_J = nullptr, *g_Sx = nullptr;
  long long g_launches = 0;
  double *gb = nullptr, *gx = nullptr;
  int sms = 148;
  // device plan
  void* plan_mem = nullptr;
  DevPlan dp{};
  // workspace
  void* ws = nullptr;
  bool ws_owned = false;
  size_t ws_bytes = 0;
  double *Dv = nullptr;
  double *Kv = nullptr, *Lx = nullptr, *Ub = nullptr, *uv = nullptr, *Y = nullptr, *Xp = nullptr;
  double *Dh = nullptr, *Dl = nullptr, *A = nullptr, *res = nullptr, *dxv = nullptr, *res2 = nullptr;
  double2* T = nullptr;
  double *sg = nullptr, *zv = nullptr, *wv = nullptr, *hdx = nullptr, *hr1 = nullptr;
  double *cr = nullptr, *cp = nullptr, *cq = nullptr, *hdy = nullptr, *hr2 = nullptr;
  double *cs = nullptr;                                    // CR: s = S r
  K3Ctx k3{};                                              // unreduced-system refinement (k3.cuh)
  double* Sg = nullptr;   // LDL^T pivot signs [B][n]
  int* inert = nullptr;   // LDL^T inertia counts [B][3]
  bool ldlt = false;
  bool resid_warp = false;   // residual columns by warps (some column has > 96 terms)
  double *g_r1 = nullptr, *g_r2 = nullptr, *g_dx = nullptr, *g_dy = nullptr;  // HyKKT graph I/O
  cudaGraphExec_t hy_exec = nullptr;                       // recorded HyKKT solve
  double hy_rtol = -1, hy_gamma = 0, hy_dw = 0;
  int hy_maxit = -1, hy_outer = -1, hy_krylov = -1;
  long long hy_fixed = 0, hy_body = 0;   // launches outside / per execution of the Krylov body
  bool hy_pending = false;               // last call was a HyKKT graph (launch count unread)
  bool last_hykkt = false;               // last solve was HyKKT: kkt_sync_info reports outer passes
  const void *hy_W = nullptr, *hy_J = nullptr, *hy_Sx = nullptr;
  TaskQueue TQ{}, TQs{};  // work queues of bwd_big / bwd_small (separate: the two may overlap)
  double* Li = nullptr;   // [batch][linv_doubles] L11^-1 of the big (CTA) supernodes (solve operator)
  int *bflag = nullptr;  // [batch][ns] backward hand-off big parent -> small children (PDL overlap)
  int *fcnt = nullptr, *facnt = nullptr, *ctl = nullptr, *fail = nullptr,
      *status = nullptr;
  DevCtrl C{};
  // current values (remembered by kkt_condense for the refinement residual)
  const double *Wv = nullptr, *Jv = nullptr, *Sx = nullptr, *Ss = nullptr, *Dov = nullptr;
  double dw = 0, dc = 0, gamma = 0;
  bool condensed = false, factored = false;
  // launch configuration
  long long factor_smem_cap = 0;
  int fsmall_smem = 0, fbig_smem = 0, tsmall_smem = 0, tbig_smem = 0, pcap = 0;
  int g_fsmall = 1, g_fbig = 1, g_tsmall = 1, g_tbig = 1, g_bsmall = 1, g_bbig = 1;
  int g_huge = 1, huge_smem = 0, huge_warps = 4;
  long long launches = 0;
  // host-buffer path (kkt_step_host)
  double *hW = nullptr, *hJ = nullptr, *hSx = nullptr, *hSs = nullptr, *hD = nullptr,
         *hb = nullptr, *hx = nullptr;
  cudaStream_t hcopy = nullptr;          // copy stream: b's upload overlaps condense + factor
  cudaEvent_t hev[2] = {nullptr, nullptr};
  int* pinned_flags = nullptr;
  long long* trace_buf = nullptr;
  long long* dbg_buf = nullptr;  // KKT_TRACE=2: per-step stamps of the root front (huge path)
  void* huge_mem = nullptr;
  HugeSched hsched{}, hsched_s{};  // factor / solve grids
  void* hsolve_mem = nullptr;
  int g_hsolve = 1;
  long long g_pro = 0, g_body = 0;   // kernels in the solve graph's prologue / per correction sweep
  bool solve_while = false;          // refinement loop as a graph WHILE node (KKT_SOLVE_WHILE=1)
  bool solve_if = false;             // sweeps 2.. behind one graph IF node (KKT_SOLVE_IF=1; measured slower:
                                     // a graph with a conditional node launches ~0.2 ms slower on C1/C2)
  bool pdl = true;                   // overlap the small/big tree phases (programmatic launch)
  int pdl_mask = 7;
  bool use_linv = true;              // inverse-diagonal-block sweeps for big supernodes (KKT_NO_LINV=1: off)
  bool huge_solve_cta = true;        // solve the huge fronts with the CTA kernels (KKT_HUGE_SOLVE=1: whole-GPU kernel)
  DevPlan dps{};                     // solve-side view of the plan (huge fronts as CTA supernodes)
  void* dps_mem = nullptr;
  void* nbig_mem = nullptr;          // [ns] big-children counts
  int linv_smem = 0, g_linv = 1;
  int fsmall_occ = 1;                // factor_small variant (resident CTAs/SM the registers allow)
  bool graph_solve_pending = false;  // last call was a graph solve whose sweep count is unread
  std::vector<cudaGraphExec_t> extra_exec;  // further instantiated graphs (HyKKT loop)
  cudaEvent_t fev[3] = {nullptr, nullptr, nullptr};  // factor phase events (start, before huge, end)
  // tile-task factorisation of the huge fronts (tiles.cuh); KKT_HUGE_OLD=1: level kernel (huge.cuh)
  bool tiles = true;
  TilePlan tp{};
  void* tile_mem = nullptr;   // fronts + tasks + hidx
  void* tile_pool = nullptr;  // [batch][pool] + counters
  size_t tile_cnt_bytes = 0;
  int g_tile = 1;
  double tile_est_us = 0.0;
  long long* tile_trace = nullptr;  // KKT_TRACE: per-task stamps of the tile kernel
  // tile-task solves through the huge fronts (tsolve.cuh); KKT_TSOLVE=0: level kernel (hsolve.cuh)
  bool tsolve = false;
  bool ts_chain = false;             // panel chains on one CTA (KKT_TS_CHAIN=0: per-step tasks)
  TSolvePlan tsp{};
  void* ts_mem = nullptr;
  size_t ts_cnt_bytes = 0;
  double ts_est_us = 0.0;
  long long* ts_trace = nullptr;
  // subtree-block solves of the small supernodes (sblock.cuh); KKT_SBLOCK=0: per-node kernels
  bool sblock = false;
  SBPlan sbp{};
  void* sb_mem = nullptr;
  void* sb_mem2 = nullptr;
  // subtree-block factorisation of the small supernodes (fblock.cuh); KKT_FBLOCK=0: per-node kernel
  bool fblock = false;
  FBPlan fbp{};
  void* fb_mem = nullptr;
  int fb_smem = 0, g_ffblk = 1;
  int sb_smem = 0, g_fblk = 1, g_bblk = 1, sb_nt = 256;
  bool fev_valid = false;
};

static size_t align_up(size_t v) { return (v + 255) & ~(size_t)255; }

struct Carver {
  char* base;
  size_t off = 0;
  bool dry;
  template <class T>
  T* take(size_t count) {
    size_t o = off;
    off = align_up(off + count * sizeof(T) + 16);  // >= 16 bytes of slack (TMA ranges round out)
    return dry ? nullptr : reinterpret_cast<T*>(base + o);
  }
};

static void carve_workspace(kkt_plan* h, Carver& c) {
  const Plan& P = h->P;
  size_t B = P.batch, n = P.n, m = P.m, me = P.m_eq, ns = P.ns;
  h->Kv = c.take<double>(B * P.Kp[n]);
  h->Lx = c.take<double>(B * P.nnzL_stored);
  h->Li = c.take<double>(B * std::max(P.linv_doubles, 1LL));
  h->Ub = c.take<double>(B * P.update_doubles);
  h->uv = c.take<double>(B * P.uvec_doubles);
  h->Y = c.take<double>(B * n);
  h->Dv = c.take<double>(B * n);
  h->Xp = c.take<double>(B * n);
  h->res = c.take<double>(B * n);
  h->gb = c.take<double>(B * n);
  h->gx = c.take<double>(B * n);
  h->dxv = c.take<double>(B * n);
  h->Dh = c.take<double>(B * m);
  h->Dl = c.take<double>(B * m);
  h->A = c.take<double>(B * m);
  h->T = c.take<double2>(B * m);
  h->res2 = c.take<double>(B * me);
  h->sg = c.take<double>(B * n);
  h->zv = c.take<double>(B * n);
  h->wv = c.take<double>(B * n);
  h->hdx = c.take<double>(B * n);
  h->hr1 = c.take<double>(B * n);
  h->cr = c.take<double>(B * me);
  h->cp = c.take<double>(B * me);
  h->cq = c.take<double>(B * me);
  h->hdy = c.take<double>(B * me);
  h->hr2 = c.take<double>(B * me);
  h->fcnt = c.take<int>(B * ns);
  h->TQ.q = c.take<int>(B * ns);
  h->TQ.flag = c.take<int>(B * ns);
  h->TQs.q = c.take<int>(B * ns);
  h->TQs.flag = c.take<int>(B * ns);
  h->facnt = c.take<int>(B * ns);
  h->bflag = c.take<int>(B * ns);
  h->ctl = c.take<int>(8 * KKT_CTL);
  h->fail = c.take<int>(1);
  h->status = c.take<int>(1);
  h->C.done = c.take<int>(B + 1);  // [B] = number of instances still refining
  h->C.refine_iters = c.take<int>(B);
  h->C.grow = c.take<int>(B);
  h->C.sweep = c.take<int>(1);
  h->C.omega = c.take<unsigned long long>(B);
  h->C.omega_prev = c.take<double>(B);
  h->C.omega_last = c.take<double>(B);
  h->C.dxprev = c.take<double>(B);
  h->C.dxn = c.take<unsigned long long>(B);
  h->C.xn = c.take<unsigned long long>(B);
  h->C.cg_done = c.take<int>(B + 1);  // [B] stays 1: the solve kernels' all-done test never fires
  h->C.cg_iters = c.take<int>(B);
  h->C.cg_iters_first = c.take<int>(B);
  h->C.rr = c.take<double>(B);
  h->C.rr0 = c.take<double>(B);
  h->C.rr0_first = c.take<double>(B);
  h->C.pq = c.take<double>(B);
  h->C.alpha = c.take<double>(B);
  h->C.beta = c.take<double>(B);
  h->C.partial = c.take<double>(B * 2 * KKT_NPART);
  h->C.part_cnt = c.take<unsigned int>(B);
  h->C.rs = c.take<double>(B);
  h->C.qq = c.take<double>(B);
  h->C.odone = c.take<int>(B + 1);
  h->C.onrm = c.take<unsigned long long>(4 * B);
  h->C.oprev = c.take<double>(B);
  h->C.opass = c.take<int>(B);
  h->C.cg_runs = c.take<int>(1);
  h->Sg = c.take<double>(P.factor_kind == 1 ? B * n : 1);
  h->inert = c.take<int>(3 * B);
  h->cs = c.take<double>(B * me);
  {  // K3 refinement scratch (k3.cuh)
    const size_t mi = m - me;
    h->k3.r5 = c.take<double>(B * n); h->k3.c1 = c.take<double>(B * n); h->k3.ex = c.take<double>(B * n);
    h->k3.ey = c.take<double>(B * std::max<size_t>(me, 1)); h->k3.r3 = c.take<double>(B * std::max<size_t>(me, 1));
    h->k3.b2 = c.take<double>(B * std::max<size_t>(mi, 1)); h->k3.r4 = c.take<double>(B * std::max<size_t>(mi, 1));
    h->k3.r6 = c.take<double>(B * std::max<size_t>(mi, 1));
    h->k3.tw = c.take<double2>(B * std::max<size_t>(m, 1));
    h->k3.done = c.take<int>(B + 1); h->k3.nrm = c.take<unsigned long long>(2 * B);
    h->k3.prev = c.take<double>(B); h->k3.sweeps = c.take<int>(B);
  }
  h->g_r1 = c.take<double>(B * n);
  h->g_dx = c.take<double>(B * n);
  h->g_r2 = c.take<double>(B * me);
  h->g_dy = c.take<double>(B * me);
}

// ------------------------------------------------------------------------------ C-ABI
extern "C" {

const char* kkt_last_error(void) { return g_err.c_str(); }

kkt_status kkt_default_options(kkt_options* o) {
  if (!o) return KKT_ERR_ARG;
  o->ordering = 0;
  o->factor_kind = 0;
  o->relax_small = 4;
  o->relax_big = 64;
  o->relax_zero_frac = 0.05;
  o->batch = 1;
  return KKT_OK;
}

kkt_status kkt_analyze(int n, int m, int m_eq, const int* W_rowptr, const int* W_colind,
                       const int* J_rowptr, const int* J_colind, const kkt_options* opt,
                       kkt_handle* handle, kkt_analysis_info* info) {
  if (!handle) { g_err = "null handle"; return KKT_ERR_ARG; }
  *handle = nullptr;
  kkt_options o;
  kkt_default_options(&o);
  if (opt) o = *opt;
  if (o.factor_kind != 0 && o.factor_kind != 1) { g_err = "factor_kind must be 0 (LL^T) or 1 (LDL^T)"; return KKT_ERR_ARG; }
  if (o.batch < 1) { g_err = "batch < 1"; return KKT_ERR_ARG; }
  kkt_plan* h = new (std::nothrow) kkt_plan();
  if (!h) return KKT_ERR_ALLOC;
  Options op;
  op.ordering = o.ordering;
  op.relax_small = o.relax_small;
  op.relax_big = o.relax_big;
  op.relax_zero_frac = o.relax_zero_frac;
  op.batch = o.batch;
  op.factor_kind = o.factor_kind;
  int code = 0;
  std::string err;
  try {
    err = analyze(n, m, m_eq, W_rowptr, W_colind, J_rowptr, J_colind, op, h->P, &code);
  } catch (const std::bad_alloc&) {
    delete h;
    g_err = "host allocation failed in analysis";
    return KKT_ERR_ALLOC;
  }
  if (!err.empty()) {
    delete h;
    g_err = err;
    return code == 1 ? KKT_ERR_ARG : KKT_ERR_PATTERN;
  }
  if (info) {
    const Plan& P = h->P;
    info->nnzK = P.Kp[P.n];
    info->nnzL = P.nnzL;
    info->nnzL_stored = P.nnzL_stored;
    info->flops = P.flops;
    info->nprod = P.nprod;
    info->nsuper = P.ns;
    info->tree_height = P.height;
    info->max_front = P.max_front;
    info->analyze_ms = P.analyze_ms;
    info->order_ms = P.order_ms;
    info->update_doubles = P.update_doubles;
    info->flops_huge = P.flops_huge;
    info->nsuper_huge = P.n_huge;
  }
  *handle = h;
  return KKT_OK;
}

kkt_status kkt_get_symbolic(kkt_handle h, int* perm, int* etree, int* colcount) {
  if (!h) return KKT_ERR_ARG;
  size_t n = h->P.n;
  if (perm) std::memcpy(perm, h->P.perm_md.data(), n * sizeof(int));
  if (etree) std::memcpy(etree, h->P.etree_md.data(), n * sizeof(int));
  if (colcount) std::memcpy(colcount, h->P.colcount_md.data(), n * sizeof(int));
  return KKT_OK;
}

kkt_status kkt_workspace_size(kkt_handle h, size_t* bytes) {
  if (!h || !bytes) return KKT_ERR_ARG;
  Carver c{nullptr, 0, true};
  carve_workspace(h, c);
  *bytes = c.off;
  return KKT_OK;
}

}  // extern "C"

// J pattern is needed on the device: analysis keeps it in Plan via jrow + these vectors.
// (Rebuilt here from Jt maps to avoid storing the caller's arrays twice.)
static void rebuild_J_csr(const Plan& P, std::vector<int>& Jrp, std::vector<int>& Jci) {
  Jrp.assign(P.m + 1, 0);
  Jci.assign(P.nnzJ, 0);
  for (int p = 0; p < P.nnzJ; p++) Jrp[P.jrow[p] + 1]++;
  for (int r = 0; r < P.m; r++) Jrp[r + 1] += Jrp[r];
  for (int i = 0; i < P.n; i++)
    for (int q = P.Jt_p[i]; q < P.Jt_p[i + 1]; q++) Jci[P.Jt_k[q]] = i;
}

template <class T>
static size_t vbytes(const std::vector<T>& v) { return align_up(v.size() * sizeof(T) + 16); }  // TMA slack

// Level schedule of the huge fronts for a cooperative grid of G CTAs (see HugeSched in
// huge.cuh): one allocation holding the entries, their barrier counters, the level pointers and
// 2 x nflag block flags of the solves (hsolve.cuh).
static kkt_status build_huge_sched(kkt_plan* h, int G, bool tiles, HugeSched* out, void** mem) {
  const Plan& P = h->P;
  std::vector<int> hl(P.ns, -1);
  int nlev = 0;
  for (int s : P.order_h) {  // postorder: children first
    int l = 0;
    for (int q = P.sn_cp[s]; q < P.sn_cp[s + 1]; q++) {
      int c = P.sn_ch[q];
      if (hl[c] >= 0) l = std::max(l, hl[c] + 1);
    }
    hl[s] = l;
    nlev = std::max(nlev, l + 1);
  }
  std::vector<std::vector<int>> lv(nlev);
  for (int s : P.order_h) lv[hl[s]].push_back(s);
  std::vector<int> lptr(1, 0);
  std::vector<int4> ent;
  int nflag = 0;
  auto flag_off = [&](int s) {  // flags of front s: one per 32 x 32 tile (factor) or per block (solve)
    const int o = nflag;
    const int w = P.sn_first[s + 1] - P.sn_first[s], R = P.sn_rp[s + 1] - P.sn_rp[s] - w;
    const int nb = (w + 31) / 32, nt = nb + (R + 31) / 32;
    nflag += tiles ? nt * (nt + 1) / 2 : nb;
    return o;
  };
  for (int L = 0; L < nlev; L++) {
    const auto& F = lv[L];
    const int k = (int)F.size();
    if (k > G) {
      for (int s : F) ent.push_back(make_int4(s, 0, 0, flag_off(s)));
    } else {
      std::vector<double> wgt(k);
      double tot = 0;
      for (int i = 0; i < k; i++) {
        double r = P.sn_rp[F[i] + 1] - P.sn_rp[F[i]], w = P.sn_first[F[i] + 1] - P.sn_first[F[i]];
        wgt[i] = r * r * (w + 2.0);
        tot += wgt[i];
      }
      std::vector<int> g(k);
      int sum = 0;
      for (int i = 0; i < k; i++) { g[i] = std::max(1, (int)(G * wgt[i] / tot)); sum += g[i]; }
      while (sum > G) {  // trim the largest groups
        int im = (int)(std::max_element(g.begin(), g.end()) - g.begin());
        g[im]--; sum--;
      }
      int c0 = 0;
      for (int i = 0; i < k; i++) { ent.push_back(make_int4(F[i], c0, g[i], flag_off(F[i]))); c0 += g[i]; }
    }
    lptr.push_back((int)ent.size());
  }
  const size_t hbytes = ent.size() * sizeof(int4) * 2 + (lptr.size() + 2 * (size_t)nflag) * sizeof(int) + 256;
  CUDA_TRY(cudaMalloc(mem, hbytes));
  char* hb = (char*)*mem;
  int4* d_ent = (int4*)hb;
  CUDA_TRY(cudaMemcpy(d_ent, ent.data(), ent.size() * sizeof(int4), cudaMemcpyHostToDevice));
  int* d_ctr = (int*)(hb + ent.size() * sizeof(int4));
  int* d_lptr = (int*)(hb + ent.size() * sizeof(int4) * 2);
  CUDA_TRY(cudaMemcpy(d_lptr, lptr.data(), lptr.size() * sizeof(int), cudaMemcpyHostToDevice));
  out->lvl_ptr = d_lptr; out->ent = d_ent; out->nlev = nlev; out->ctr = d_ctr; out->nflag = nflag;
  out->flags = d_lptr + lptr.size();
  return KKT_OK;
}

// Free every device/host resource the handle holds (bound or partially bound) and return it to
// the unbound state; safe to call twice.
static void release_device(kkt_plan* h) {
  if (h->device >= 0) cudaSetDevice(h->device);
  if (h->stream || h->bound) cudaStreamSynchronize(h->stream);
  auto fr = [](auto*& p) { if (p) cudaFree((void*)p); p = nullptr; };
  fr(h->plan_mem); fr(h->dps_mem); fr(h->nbig_mem);
  if (h->ws_owned) fr(h->ws);
  h->ws = nullptr; h->ws_owned = false;
  fr(h->hW); fr(h->hJ); fr(h->hSx); fr(h->hSs); fr(h->hD); fr(h->hb); fr(h->hx);
  if (h->pinned_flags) cudaFreeHost(h->pinned_flags);
  h->pinned_flags = nullptr;
  fr(h->trace_buf); fr(h->dbg_buf); fr(h->huge_mem); fr(h->hsolve_mem);
  fr(h->tile_mem); fr(h->tile_pool); fr(h->tile_trace); fr(h->ts_mem); fr(h->ts_trace); fr(h->sb_mem); fr(h->sb_mem2); fr(h->fb_mem);
  h->fblock = false;
  h->sblock = false;
  if (h->solve_exec) cudaGraphExecDestroy(h->solve_exec);
  h->solve_exec = nullptr;
  if (h->hy_exec) cudaGraphExecDestroy(h->hy_exec);
  h->hy_exec = nullptr;
  for (auto& ge : h->extra_exec) if (ge) cudaGraphExecDestroy(ge);
  h->extra_exec.clear();
  if (h->cap) cudaStreamDestroy(h->cap);
  h->cap = nullptr;
  if (h->hcopy) cudaStreamDestroy(h->hcopy);
  h->hcopy = nullptr;
  for (auto& e : h->hev) { if (e) cudaEventDestroy(e); e = nullptr; }
  for (auto& e : h->fev) { if (e) cudaEventDestroy(e); e = nullptr; }
  h->fev_valid = false;
  h->bound = false;
  h->condensed = h->factored = false;
}

static kkt_status bind_impl(kkt_handle h, int device, void* d_workspace, size_t bytes, kkt_stream_t stream);

extern "C" kkt_status kkt_bind(kkt_handle h, int device, void* d_workspace, size_t bytes,
                               kkt_stream_t stream) {
  if (!h) return KKT_ERR_ARG;
  if (h->bound) { g_err = "already bound"; return KKT_ERR_STATE; }
  if (d_workspace) {  // size check before any allocation
    size_t need = 0;
    kkt_workspace_size(h, &need);
    if (bytes < need) { g_err = "workspace too small"; return KKT_ERR_ALLOC; }
  }
  kkt_status st = bind_impl(h, device, d_workspace, bytes, stream);
  if (st != KKT_OK) {
    const std::string msg = g_err;
    release_device(h);  // no partial allocations survive a failed bind
    g_err = msg;
  }
  return st;
}

// Factor start lists by the estimated longest path to the top of the small + big phases (the
// critical chains first): small leaves (up_s) and the first big tasks (up_bf).  Estimated
// durations (us, C4 traces): small supernode 6, big 12 + r w / 400; huge fronts belong to the
// next kernel.  Scheduling only: every supernode's arithmetic is unchanged.
static void order_factor_lists(Plan& P) {
  const int ns = P.ns;
  if (ns == 0) return;
  std::vector<double> up(ns, 0.0);
  for (int s = ns - 1; s >= 0; s--) {
    const SnInfo& I = P.sn[s];
    const double d = I.huge ? 0.0 : (I.big ? 12.0 + (double)I.r * I.w / 400.0 : 6.0);
    const int par = P.sn_parent[s];
    up[s] = d + ((par >= 0 && !P.sn[par].huge) ? up[par] : 0.0);
  }
  auto by_up = [&](int a, int b) { return up[a] != up[b] ? up[a] > up[b] : a < b; };
  std::stable_sort(P.up_s.begin(), P.up_s.end(), by_up);
  std::stable_sort(P.up_bf.begin(), P.up_bf.end(), by_up);
}

static kkt_status bind_impl(kkt_handle h, int device, void* d_workspace, size_t bytes,
                            kkt_stream_t stream) {
  CUDA_TRY(cudaSetDevice(device));
  if (!(getenv("KKT_FACTOR_ORDER") && atoi(getenv("KKT_FACTOR_ORDER")) == 0)) order_factor_lists(h->P);
  h->device = device;
  h->stream = (cudaStream_t)stream;
  h->ls = h->stream;
  CUDA_TRY(cudaStreamCreateWithFlags(&h->cap, cudaStreamNonBlocking));
  h->use_graph = !(getenv("KKT_NO_GRAPH") && atoi(getenv("KKT_NO_GRAPH")) > 0);
  h->solve_while = getenv("KKT_SOLVE_WHILE") && atoi(getenv("KKT_SOLVE_WHILE")) > 0;
  h->pdl = !(getenv("KKT_NO_PDL") && atoi(getenv("KKT_NO_PDL")) > 0);
  if (h->solve_while) h->pdl = false;  // programmatic launches are not captured into conditional bodies
  h->solve_if = getenv("KKT_SOLVE_IF") && atoi(getenv("KKT_SOLVE_IF")) > 0;
  h->pdl_mask = getenv("KKT_PDL_MASK") ? atoi(getenv("KKT_PDL_MASK")) : 7;  // 1 factor, 2 forward, 4 backward
  h->use_linv = !(getenv("KKT_NO_LINV") && atoi(getenv("KKT_NO_LINV")) > 0);

  cudaDeviceProp prop;
  CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  h->sms = prop.multiProcessorCount;
  const Plan& P = h->P;
  std::vector<int> Jrp, Jci;
  rebuild_J_csr(P, Jrp, Jci);
  // ---- plan upload (one allocation, one H2D per array) ----
  const std::vector<int>* iv[] = {&P.perm, &P.iperm, &P.Kp, &P.Ki, &P.kw, &P.kdiag, &P.pptr,
                                  &P.pa, &P.pb, &P.jrow, &P.kpos, &P.sn_first, &P.sn_rp,
                                  &P.sn_rows, &P.sn_rel, &P.sn_parent, &P.sn_cp, &P.sn_ch,
                                  &P.order, &P.order_s, &P.order_b, &P.up_s, &P.up_b,
                                  &P.dn_b, &P.dn_s, &P.up_bf, &P.order_h, &P.Wf_p, &P.Wf_c, &P.Wf_k, &P.Jt_p, &P.Jt_r,
                                  &P.Jt_k, &P.Gt_end, &Jrp, &Jci};
  const std::vector<long long>* lv[] = {&P.sn_Lp, &P.sn_Up, &P.sn_uvp, &P.sn_Lip};
  size_t tot = 0;
  for (auto* v : iv) tot += vbytes(*v);
  for (auto* v : lv) tot += vbytes(*v);
  tot += vbytes(P.sn) + vbytes(P.chinfo);
  CUDA_TRY(cudaMalloc(&h->plan_mem, tot));
  std::vector<const void*> dptr;
  size_t off = 0;
  char* base = (char*)h->plan_mem;
  for (auto* v : iv) {
    if (!v->empty()) CUDA_TRY(cudaMemcpy(base + off, v->data(), v->size() * sizeof(int), cudaMemcpyHostToDevice));
    dptr.push_back(base + off);
    off += vbytes(*v);
  }
  for (auto* v : lv) {
    if (!v->empty()) CUDA_TRY(cudaMemcpy(base + off, v->data(), v->size() * sizeof(long long), cudaMemcpyHostToDevice));
    dptr.push_back(base + off);
    off += vbytes(*v);
  }
  if (!P.sn.empty()) CUDA_TRY(cudaMemcpy(base + off, P.sn.data(), P.sn.size() * sizeof(SnInfo), cudaMemcpyHostToDevice));
  const SnInfo* d_sn = (const SnInfo*)(base + off);
  off += vbytes(P.sn);
  if (!P.chinfo.empty()) CUDA_TRY(cudaMemcpy(base + off, P.chinfo.data(), P.chinfo.size() * sizeof(SnInfo), cudaMemcpyHostToDevice));
  const SnInfo* d_ch = (const SnInfo*)(base + off);
  off += vbytes(P.chinfo);
  DevPlan& d = h->dp;
  d.n = P.n; d.m = P.m; d.m_eq = P.m_eq; d.nnzW = P.nnzW; d.nnzJ = P.nnzJ; d.nnzK = P.Kp[P.n];
  d.ns = P.ns; d.batch = P.batch; d.max_front = P.max_front;
  d.ns_s = (int)P.order_s.size(); d.ns_b = (int)P.order_b.size();
  d.ns_bn = d.ns_b - (int)P.order_h.size(); d.max_r_small = P.max_r_small;
  d.n_up_s = (int)P.up_s.size(); d.n_up_b = (int)P.up_b.size();
  d.n_dn_b = (int)P.dn_b.size(); d.n_dn_s = (int)P.dn_s.size();
  d.n_up_bf = (int)P.up_bf.size(); d.n_h = (int)P.order_h.size();
  d.nnzL_stored = P.nnzL_stored; d.update_doubles = P.update_doubles;
  d.uvec_doubles = P.uvec_doubles; d.nprod = P.nprod;
  int k = 0;
  auto I = [&](void) { return (const int*)dptr[k++]; };
  d.perm = I(); d.iperm = I(); d.Kp = I(); d.Ki = I(); d.kw = I(); d.kdiag = I(); d.pptr = I();
  d.pa = I(); d.pb = I(); d.jrow = I(); d.kpos = I(); d.sn_first = I(); d.sn_rp = I();
  d.sn_rows = I(); d.sn_rel = I(); d.sn_parent = I(); d.sn_cp = I(); d.sn_ch = I();
  d.order = I(); d.order_s = I(); d.order_b = I(); d.up_s = I(); d.up_b = I(); d.dn_b = I();
  d.dn_s = I(); d.up_bf = I(); d.order_h = I(); d.Wf_p = I(); d.Wf_c = I(); d.Wf_k = I(); d.Jt_p = I(); d.Jt_r = I();
  d.Jt_k = I(); d.Gt_end = I(); d.Jrp = I(); d.Jci = I();
  d.sn_Lp = (const long long*)dptr[k++];
  d.linv_doubles = P.linv_doubles;
  d.sn_Up = (const long long*)dptr[k++];
  d.sn_uvp = (const long long*)dptr[k++];
  d.sn_Lip = (const long long*)dptr[k++];
  d.sn = d_sn;
  d.chinfo = d_ch;
  d.trace = nullptr;
  if (getenv("KKT_TRACE") && atoi(getenv("KKT_TRACE")) > 0) {
    CUDA_TRY(cudaMalloc(&h->trace_buf, (size_t)3 * std::max(P.ns, 1) * KKT_TRACE_SLOTS * sizeof(long long)));
    CUDA_TRY(cudaMemset(h->trace_buf, 0, (size_t)3 * std::max(P.ns, 1) * KKT_TRACE_SLOTS * sizeof(long long)));
    d.trace = h->trace_buf;
    if (atoi(getenv("KKT_TRACE")) > 1) {
      CUDA_TRY(cudaMalloc(&h->dbg_buf, 4096 * 8 * sizeof(long long)));
      CUDA_TRY(cudaMemset(h->dbg_buf, 0, 4096 * 8 * sizeof(long long)));
    }
  }
  // solve-side plan view: huge fronts are solved by the CTA kernels (their fronts are only needed
  // in shared memory for the factorization); the big phase then starts from the big leaves
  // (up_b) and, top-down, from the big roots
  {
    // huge fronts up to 512 rows are solved faster by the CTA kernels (one CTA per front, no grid
    // barriers); beyond that the whole-GPU wavefront wins (measured: C3 max front 322 -> CTA,
    // C4/C6 831/1239 -> whole GPU).  KKT_HUGE_SOLVE=1 forces the whole-GPU kernel, =0 the CTA one.
    int maxr_h = 0;
    for (int s_ : P.order_h) maxr_h = std::max(maxr_h, P.sn_rp[s_ + 1] - P.sn_rp[s_]);
    // with the per-node solve kernels (KKT_SBLOCK=0) huge fronts up to 512 rows solve faster as CTA
    // supernodes; with the whole-tree kernels the tile solve wins everywhere (C3: 20.4 -> 15.2 ms)
    const bool no_sblock = getenv("KKT_SBLOCK") && atoi(getenv("KKT_SBLOCK")) == 0;
    h->huge_solve_cta = no_sblock && maxr_h <= 512;
    if (const char* e = getenv("KKT_HUGE_SOLVE")) h->huge_solve_cta = atoi(e) == 0;
    if (P.factor_kind == 1) h->huge_solve_cta = true;  // LDL^T: S applied between the CTA-path sweeps
  }
  {  // big-children counts (bottom-up hand-off into CTA parents)
    std::vector<int> nbig(std::max(P.ns, 1), 0);
    for (int s_ = 0; s_ < P.ns; s_++)
      if (P.sn_parent[s_] >= 0 && P.sn[s_].big) nbig[P.sn_parent[s_]]++;
    CUDA_TRY(cudaMalloc(&h->nbig_mem, nbig.size() * sizeof(int)));
    CUDA_TRY(cudaMemcpy(h->nbig_mem, nbig.data(), nbig.size() * sizeof(int), cudaMemcpyHostToDevice));
    d.sn_nbig = (const int*)h->nbig_mem;
  }
  h->dps = d;
  h->dps.solve_huge_cta = 0;
  if (h->huge_solve_cta && !P.order_h.empty()) {
    std::vector<int> roots;
    for (int s_ : P.order_b) if (P.sn_parent[s_] < 0) roots.push_back(s_);
    CUDA_TRY(cudaMalloc(&h->dps_mem, std::max<size_t>(roots.size(), 1) * sizeof(int)));
    if (!roots.empty()) CUDA_TRY(cudaMemcpy(h->dps_mem, roots.data(), roots.size() * sizeof(int), cudaMemcpyHostToDevice));
    h->dps.solve_huge_cta = 1;
    h->dps.up_bf = d.up_b;
    h->dps.n_up_bf = d.n_up_b;
    h->dps.dn_b = (const int*)h->dps_mem;
    h->dps.n_dn_b = (int)roots.size();
    h->dps.ns_bn = d.ns_b;
  } else {
    h->huge_solve_cta = false;
  }
  // ---- workspace ----
  size_t need;
  kkt_workspace_size(h, &need);
  if (d_workspace) {
    if (bytes < need) { g_err = "workspace too small"; return KKT_ERR_ALLOC; }
    h->ws = d_workspace;
    h->ws_owned = false;
  } else {
    CUDA_TRY(cudaMalloc(&h->ws, need));
    h->ws_owned = true;
  }
  h->ws_bytes = need;
  Carver c{(char*)h->ws, 0, false};
  carve_workspace(h, c);
  h->ldlt = (P.factor_kind == 1);
  {
    int maxc = 0;
    for (int i = 0; i < P.n; i++)
      maxc = std::max(maxc, (P.Wf_p[i + 1] - P.Wf_p[i]) + (P.Jt_p[i + 1] - P.Jt_p[i]));
    h->resid_warp = maxc > 96;
    if (const char* e = getenv("KKT_RESID_WARP")) h->resid_warp = atoi(e) > 0;
  }
  for (DevPlan* dq : {&h->dp, &h->dps}) { dq->ldlt = h->ldlt; dq->Sg = h->Sg; dq->inert = h->inert; }
  CUDA_TRY(cudaMemsetAsync(h->ws, 0, need, h->stream));
  int big = INT_MAX;
  CUDA_TRY(cudaMemcpyAsync(h->fail, &big, sizeof(int), cudaMemcpyHostToDevice, h->stream));
  // ---- launch configuration ----
  long long maxneed = 0;
  for (int s : P.order_b) {
    if (P.sn[s].huge) continue;
    long long r = P.sn_rp[s + 1] - P.sn_rp[s], w = P.sn_first[s + 1] - P.sn_first[s], R = r - w;
    long long need_s = r * w + (P.sn_parent[s] >= 0 ? R * (R + 1) / 2 : 0);
    maxneed = std::max(maxneed, need_s);
  }
  const long long cap_bytes = 200 * 1024;
  h->factor_smem_cap = std::min(maxneed, cap_bytes / 8);
  h->fbig_smem = (int)(std::max<long long>(h->factor_smem_cap, 1) * 8);
  h->fsmall_smem = KKT_WPB * KKT_SCAP * 8;
  {
    int mrw = 1;
    for (int s_ : P.order_s) mrw = std::max(mrw, (P.sn_rp[s_ + 1] - P.sn_rp[s_]) * (P.sn_first[s_ + 1] - P.sn_first[s_]));
    mrw = (mrw + 1) & ~1;  // keep the per-warp slices 16-byte aligned
    h->dp.max_rw_small = mrw;
    h->dps.max_rw_small = mrw;
  }
  h->tsmall_smem = KKT_WPB * (h->dp.max_rw_small + P.max_r_small + 1) * 8;
  long long maxpanel = 0;
  for (int s : P.order_b)
    maxpanel = std::max(maxpanel, (long long)(P.sn_rp[s + 1] - P.sn_rp[s]) * (P.sn_first[s + 1] - P.sn_first[s]));
  h->pcap = (int)std::min<long long>(maxpanel, 20000);
  h->tbig_smem = (int)((P.max_front + 8 * 32) * 8);
  CUDA_TRY(cudaFuncSetAttribute(factor_small_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, h->fsmall_smem));
  CUDA_TRY(cudaFuncSetAttribute(factor_small_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, h->fsmall_smem));
  // throughput-bound small phases (>= 50k small supernode tasks: C4, C5, C6) take the
  // occupancy-capped variant, latency-bound ones (C1, C2, C3) the spill-free one (measured)
  h->fsmall_occ = ((long long)P.order_s.size() * P.batch >= 50000) ? 3 : 1;
  if (const char* e = getenv("KKT_FSMALL_OCC")) h->fsmall_occ = atoi(e) == 3 ? 3 : 1;
  CUDA_TRY(cudaFuncSetAttribute(factor_big_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, h->fbig_smem));
  CUDA_TRY(cudaFuncSetAttribute(factor_big_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, h->fbig_smem));
  CUDA_TRY(cudaFuncSetAttribute(fwd_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, h->tsmall_smem));
  CUDA_TRY(cudaFuncSetAttribute(bwd_small_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, h->tsmall_smem));
  CUDA_TRY(cudaFuncSetAttribute(fwd_big_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, h->tbig_smem));
  CUDA_TRY(cudaFuncSetAttribute(bwd_big_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, h->tbig_smem));
  auto grid_of = [&](auto kern, int threads, int smem, long long tasks_, int per_cta, int* out) -> cudaError_t {
    int occ = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem);
    long long ctas = (tasks_ + per_cta - 1) / per_cta;
    *out = (int)std::max(1LL, std::min(ctas, (long long)std::max(occ, 1) * h->sms));
    return e;
  };
  const long long us = (long long)P.up_s.size() * P.batch, ub = (long long)P.up_b.size() * P.batch;
  const long long ts = (long long)P.order_s.size() * P.batch, tb = (long long)P.order_b.size() * P.batch;
  if (h->fsmall_occ == 3) CUDA_TRY(grid_of(factor_small_kernel<3>, KKT_WPB * 32, h->fsmall_smem, us, KKT_WPB, &h->g_fsmall));
  else CUDA_TRY(grid_of(factor_small_kernel<1>, KKT_WPB * 32, h->fsmall_smem, us, KKT_WPB, &h->g_fsmall));
  {  // leave KKT_FBIG_RESERVE SMs to the (programmatically overlapped) big kernel so that the
     // critical big chain starts while the throughput-bound small phase is still running
    const int reserve = getenv("KKT_FBIG_RESERVE") ? atoi(getenv("KKT_FBIG_RESERVE")) : 0;
    if (reserve > 0 && reserve < h->sms) {
      int occ = 0;
      if (h->fsmall_occ == 3) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, factor_small_kernel<3>, KKT_WPB * 32, h->fsmall_smem);
      else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, factor_small_kernel<1>, KKT_WPB * 32, h->fsmall_smem);
      h->g_fsmall = std::max(1, std::min(h->g_fsmall, std::max(occ, 1) * (h->sms - reserve)));
    }
  }
  CUDA_TRY(grid_of(factor_big_kernel<false>, KKT_BNT, h->fbig_smem, ub, 1, &h->g_fbig));
  CUDA_TRY(grid_of(fwd_small_kernel, KKT_WPB * 32, h->tsmall_smem, us, KKT_WPB, &h->g_tsmall));
  CUDA_TRY(grid_of(fwd_big_kernel, KKT_BNT, h->tbig_smem,
                   (long long)(h->huge_solve_cta ? P.up_b.size() : P.up_bf.size()) * P.batch, 1, &h->g_tbig));
  CUDA_TRY(grid_of(bwd_small_kernel, KKT_WPB * 32, h->tsmall_smem, ts, KKT_WPB, &h->g_bsmall));
  if (const char* e = getenv("KKT_BWD_CTAS")) h->g_bsmall = std::min(h->g_bsmall, std::max(1, atoi(e)));
  CUDA_TRY(grid_of(bwd_big_kernel, KKT_BNT, h->tbig_smem, tb, 1, &h->g_bbig));
  {
    long long maxw2 = 0;
    for (int s_ : P.order_b)
      if (P.sn_Lip[s_] >= 0) {
        const long long w_ = P.sn_first[s_ + 1] - P.sn_first[s_];
        const int nb_ = (int)std::min<long long>((w_ + 31) / 32, 64);
        const long long need_ = std::max<long long>(
            linv_packed(nb_) + (linv_resident(nb_) ? nb_ * 1024 + nb_ * 32 * 32 : 0),
            linv_wave(nb_) ? linv_wave_need(nb_) - 1024 : 0);
        maxw2 = std::max(maxw2, need_);
      }
    if (maxw2 == 0 || maxw2 + 1024 > KKT_LINV_CAP) h->use_linv = false;
    if (h->use_linv) {
      h->linv_smem = (int)((maxw2 + 32 * 32) * 8);  // packed L11 (+ X blocks) + one 32 x 32 staging block
      CUDA_TRY(cudaFuncSetAttribute(linv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, h->linv_smem));
      CUDA_TRY(grid_of(linv_kernel, KKT_BNT, h->linv_smem, (long long)P.order_b.size() * P.batch, 1, &h->g_linv));
    }
  }
  // subtree blocks of the small supernodes for the factorisation (fblock.cuh)
  h->fblock = !P.order_s.empty() && getenv("KKT_FBLOCK") && atoi(getenv("KKT_FBLOCK")) > 0;  // opt-in (slower so far)
  if (h->fblock) {
    const int cap = getenv("KKT_FB_CAP") ? std::max(KKT_SCAP, atoi(getenv("KKT_FB_CAP"))) : 6144;
    FBlockHost H;
    build_fblocks(P, cap, H);
    if (H.blk.empty()) {
      h->fblock = false;
    } else {
      const size_t b1 = align_up(H.blk.size() * sizeof(FBlk) + 16), b2 = vbytes(H.meta), b3 = vbytes(H.up_init);
      CUDA_TRY(cudaMalloc(&h->fb_mem, b1 + b2 + b3));
      char* fb = (char*)h->fb_mem;
      CUDA_TRY(cudaMemcpy(fb, H.blk.data(), H.blk.size() * sizeof(FBlk), cudaMemcpyHostToDevice));
      CUDA_TRY(cudaMemcpy(fb + b1, H.meta.data(), H.meta.size() * sizeof(int), cudaMemcpyHostToDevice));
      if (!H.up_init.empty())
        CUDA_TRY(cudaMemcpy(fb + b1 + b2, H.up_init.data(), H.up_init.size() * sizeof(int), cudaMemcpyHostToDevice));
      FBPlan& F = h->fbp;
      F.blk = (const FBlk*)fb;
      F.nblk = (int)H.blk.size();
      F.meta = (const int*)(fb + b1);
      F.up_init = (const int*)(fb + b1 + b2);
      F.n_up_init = (int)H.up_init.size();
      F.smem_doubles = std::max(H.max_smem, KKT_SCAP);
      h->fb_smem = F.smem_doubles * 8;
      CUDA_TRY(cudaFuncSetAttribute(factor_block_kernel<FB_MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, h->fb_smem));
      CUDA_TRY(grid_of(factor_block_kernel<FB_MINB>, FB_NT, h->fb_smem, (long long)(F.nblk + F.n_up_init) * P.batch, 1, &h->g_ffblk));
    }
  }
  // subtree blocks of the small supernodes (sblock.cuh): the solves' small phase
  h->sblock = !P.order_s.empty() && !(getenv("KKT_SBLOCK") && atoi(getenv("KKT_SBLOCK")) == 0);
  if (h->sblock) {
    // CTA size: 256 threads for latency-bound trees, 128 (6 CTAs per SM, smaller blocks) when
    // the small phase is throughput-bound (>= 50k small supernode tasks: C4, C5, C6; measured)
    h->sb_nt = ((long long)P.order_s.size() * P.batch >= 50000) ? 128 : 256;
    if (const char* e = getenv("KKT_SB_NT")) h->sb_nt = atoi(e) == 128 ? 128 : 256;
    // measured: 256-thread trees (C1-C3) best at 12288-double blocks, 128-thread ones at 4096
    const int cap = getenv("KKT_SB_CAP") ? std::max(1024, atoi(getenv("KKT_SB_CAP"))) : (h->sb_nt == 128 ? 4096 : 12288);
    SBlockHost H;
    build_sblocks(P, cap, h->sb_nt / 32, H);
    if (H.blk.empty()) {
      h->sblock = false;
    } else {
      const size_t b1 = align_up(H.blk.size() * sizeof(SBlk) + 16), b2 = vbytes(H.blk_of),
                   b3 = vbytes(H.meta), b4 = vbytes(H.lrow);
      CUDA_TRY(cudaMalloc(&h->sb_mem, b1 + b2 + b3 + b4));
      char* sb = (char*)h->sb_mem;
      CUDA_TRY(cudaMemcpy(sb, H.blk.data(), H.blk.size() * sizeof(SBlk), cudaMemcpyHostToDevice));
      CUDA_TRY(cudaMemcpy(sb + b1, H.blk_of.data(), H.blk_of.size() * sizeof(int), cudaMemcpyHostToDevice));
      CUDA_TRY(cudaMemcpy(sb + b1 + b2, H.meta.data(), H.meta.size() * sizeof(int), cudaMemcpyHostToDevice));
      CUDA_TRY(cudaMemcpy(sb + b1 + b2 + b3, H.lrow.data(), H.lrow.size() * sizeof(int), cudaMemcpyHostToDevice));
      SBPlan& S = h->sbp;
      S.blk = (const SBlk*)sb;
      S.nblk = (int)H.blk.size();
      S.blk_of = (const int*)(sb + b1);
      S.meta = (const int*)(sb + b1 + b2);
      S.lrow = (const int*)(sb + b1 + b2 + b3);
      // whole-tree schedules for the solve-side plan view: supernodes in the tree kernels are
      // every non-huge one, or all of them when the view solves the huge fronts as CTA nodes.
      // Estimated task durations (us, measured on C4 traces): block 8, single small supernode
      // 4 + 0.3 w, big supernode 6 + r w / 1200.
      const bool vcta = h->huge_solve_cta;
      const int ns = P.ns;
      auto intree = [&](int s_) { return s_ >= 0 && (!P.sn[s_].huge || vcta); };
      std::vector<double> dur(ns, 0.0), up(ns, 0.0), start(ns, 0.0);
      for (int s_ = 0; s_ < ns; s_++) {
        const SnInfo& I = P.sn[s_];
        dur[s_] = I.big ? 6.0 + (double)I.r * I.w / 1200.0 : (H.blk_of[s_] >= 0 ? 8.0 : 4.0 + 0.3 * I.w);
      }
      for (int s_ = ns - 1; s_ >= 0; s_--) {  // parents first (postorder)
        const int par = P.sn_parent[s_];
        const bool pin = intree(par) && H.blk_of[s_] != -2;
        up[s_] = dur[s_] + (pin ? up[par] : 0.0);              // forward: path to the top
        start[s_] = pin ? start[par] + dur[par] : 0.0;        // backward: estimated start
      }
      std::vector<int> ford;
      std::vector<double> fpri;
      for (size_t q = 0; q < H.blk.size(); q++) { ford.push_back((int)q); fpri.push_back(up[H.blk[q].s_hi]); }
      std::vector<int2> bord;
      for (int s_ = 0; s_ < ns; s_++) {
        if (!intree(s_) || H.blk_of[s_] == -2) continue;
        if (P.sn[s_].big && P.sn_cp[s_ + 1] == P.sn_cp[s_]) { ford.push_back(-s_ - 1); fpri.push_back(up[s_]); }
        const int par = P.sn_parent[s_];
        bord.push_back(make_int2(s_, intree(par) ? par : -1));
      }
      std::vector<int> fidx(ford.size());
      for (size_t q = 0; q < fidx.size(); q++) fidx[q] = (int)q;
      std::stable_sort(fidx.begin(), fidx.end(), [&](int a_, int b_) { return fpri[a_] > fpri[b_]; });
      std::vector<int> fsorted(ford.size());
      for (size_t q = 0; q < fidx.size(); q++) fsorted[q] = ford[fidx[q]];
      std::stable_sort(bord.begin(), bord.end(), [&](const int2& a_, const int2& b_) {
        return start[a_.x] != start[b_.x] ? start[a_.x] < start[b_.x] : up[a_.x] > up[b_.x];
      });
      const size_t b5 = vbytes(fsorted), b6 = align_up(bord.size() * sizeof(int2) + 16);
      CUDA_TRY(cudaMalloc(&h->sb_mem2, b5 + b6));
      CUDA_TRY(cudaMemcpy(h->sb_mem2, fsorted.data(), fsorted.size() * sizeof(int), cudaMemcpyHostToDevice));
      if (!bord.empty()) CUDA_TRY(cudaMemcpy((char*)h->sb_mem2 + b5, bord.data(), bord.size() * sizeof(int2), cudaMemcpyHostToDevice));
      S.fwd_order = (const int*)h->sb_mem2;
      S.n_fwd = (int)fsorted.size();
      S.bwd_order = (const int2*)((char*)h->sb_mem2 + b5);
      S.n_bwd = (int)bord.size();
      S.smem_doubles = std::max({H.max_smem, h->dp.max_rw_small + P.max_r_small + 2, P.max_front + 8 * 32 + 32 * 33 + 2});
      h->sb_smem = S.smem_doubles * 8;
      // supernodes without L11^-1 (the CTA view of the large fronts, or KKT_NO_LINV) take the
      // register-light blocked sweeps (sblock.cuh cta_fwd_lite / cta_bwd_lite)
      auto fk = h->sb_nt == 128 ? tree_fwd_kernel<false, 128> : tree_fwd_kernel<false, 256>;
      auto bk = h->sb_nt == 128 ? tree_bwd_kernel<false, 128> : tree_bwd_kernel<false, 256>;
      CUDA_TRY(cudaFuncSetAttribute(fk, cudaFuncAttributeMaxDynamicSharedMemorySize, h->sb_smem));
      CUDA_TRY(cudaFuncSetAttribute(bk, cudaFuncAttributeMaxDynamicSharedMemorySize, h->sb_smem));
      CUDA_TRY(grid_of(fk, h->sb_nt, h->sb_smem, (long long)S.n_fwd * P.batch, 1, &h->g_fblk));
      CUDA_TRY(grid_of(bk, h->sb_nt, h->sb_smem, (long long)S.n_bwd * P.batch, 1, &h->g_bblk));
    }
  }

  {
    const long long ubf = (long long)P.up_bf.size() * P.batch;
    CUDA_TRY(grid_of(factor_big_kernel<false>, KKT_BNT, h->fbig_smem, ubf, 1, &h->g_fbig));
    h->huge_warps = HUGE_WARPS;
    if (const char* e = getenv("KKT_HUGE_WARPS")) h->huge_warps = std::min(8, std::max(1, atoi(e)));
    h->huge_smem = HUGE_SMEM_DOUBLES_PER_WARP * 8 * h->huge_warps;
    CUDA_TRY(cudaFuncSetAttribute(factor_huge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, h->huge_smem));
    int occ = 0;
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, factor_huge_kernel, 32 * h->huge_warps, h->huge_smem));
    h->g_huge = (occ >= 1 ? 1 : 0) * h->sms;  // one CTA per SM (see HUGE_WARPS)
    if (h->g_huge == 0) { g_err = "factor_huge_kernel does not fit on an SM"; return KKT_ERR_CUDA; }
    int occ_s = 0;
    CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_s, solve_huge_kernel, 256, 0));
    h->g_hsolve = std::max(1, occ_s) * h->sms;
    if (!P.order_h.empty()) {
      TRY(build_huge_sched(h, h->g_huge, true, &h->hsched, &h->huge_mem));
      h->hsched.dbg = h->dbg_buf;
      TRY(build_huge_sched(h, h->g_hsolve, false, &h->hsched_s, &h->hsolve_mem));
    }
    h->tiles = !(getenv("KKT_HUGE_OLD") && atoi(getenv("KKT_HUGE_OLD")) > 0);
    if (!P.order_h.empty() && h->tiles) {
      CUDA_TRY(cudaFuncSetAttribute(tile_factor_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, TILE_SMEM_BYTES));
      CUDA_TRY(cudaFuncSetAttribute(tile_factor_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, TILE_SMEM_BYTES));
      int occ_t = 0, occ_t2 = 0;
      CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_t, tile_factor_kernel<false>, TILE_THREADS, TILE_SMEM_BYTES));
      CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_t2, tile_factor_kernel<true>, TILE_THREADS, TILE_SMEM_BYTES));
      occ_t = std::min(occ_t, occ_t2);
      if (occ_t < 1) { g_err = "tile_factor_kernel does not fit on an SM"; return KKT_ERR_CUDA; }
      h->g_tile = occ_t * h->sms;
      TilePlanHost tph;
      build_tile_plan(P, h->g_tile, tph);
      h->tile_est_us = tph.est_us;
      if (!tph.ok) h->tiles = false;  // fall back to the level kernel (huge.cuh)
      if (!h->tiles && P.factor_kind == 1) { g_err = "LDL^T needs the tile-task path for the large fronts"; return KKT_ERR_ARG; }
    }
    if (!P.order_h.empty() && h->tiles) {
      TilePlanHost tph;
      build_tile_plan(P, h->g_tile, tph);
      const size_t B = P.batch;
      std::vector<TTask> tasks;
      tasks.reserve(tph.tasks.size() * B);
      for (const TTask& t : tph.tasks)   // instances interleaved: topological per instance
        for (size_t b = 0; b < B; b++) tasks.push_back(TTask{t.x | (int)(b << 4), t.y, t.z, t.w});
      const size_t fb = align_up(tph.fr.size() * sizeof(TFrontHost)), tkb = align_up(tasks.size() * sizeof(TTask));
      const size_t hb = align_up(tph.hidx.size() * sizeof(int));
      const size_t chb = align_up(tph.tch.size() * sizeof(int)), cub = align_up(tph.tcut.size() * sizeof(int));
      const size_t kpb = align_up(tph.tkptr.size() * sizeof(int)), kib = align_up(tph.tkidx.size() * sizeof(int));
      const size_t ibb = align_up(tph.ibase.size() * sizeof(long long));
      CUDA_TRY(cudaMalloc(&h->tile_mem, fb + tkb + hb + chb + cub + kpb + kib + ibb));
      char* base = (char*)h->tile_mem;
      CUDA_TRY(cudaMemcpy(base, tph.fr.data(), tph.fr.size() * sizeof(TFrontHost), cudaMemcpyHostToDevice));
      CUDA_TRY(cudaMemcpy(base + fb, tasks.data(), tasks.size() * sizeof(TTask), cudaMemcpyHostToDevice));
      CUDA_TRY(cudaMemcpy(base + fb + tkb, tph.hidx.data(), tph.hidx.size() * sizeof(int), cudaMemcpyHostToDevice));
      CUDA_TRY(cudaMemcpy(base + fb + tkb + hb, tph.tch.data(), tph.tch.size() * sizeof(int), cudaMemcpyHostToDevice));
      CUDA_TRY(cudaMemcpy(base + fb + tkb + hb + chb, tph.tcut.data(), tph.tcut.size() * sizeof(int), cudaMemcpyHostToDevice));
      char* kb_ = base + fb + tkb + hb + chb + cub;
      CUDA_TRY(cudaMemcpy(kb_, tph.tkptr.data(), tph.tkptr.size() * sizeof(int), cudaMemcpyHostToDevice));
      CUDA_TRY(cudaMemcpy(kb_ + kpb, tph.tkidx.data(), tph.tkidx.size() * sizeof(int), cudaMemcpyHostToDevice));
      CUDA_TRY(cudaMemcpy(kb_ + kpb + kib, tph.ibase.data(), tph.ibase.size() * sizeof(long long), cudaMemcpyHostToDevice));
      const size_t poolb = align_up(B * (size_t)tph.pool_doubles * sizeof(double));
      const size_t invb = align_up(B * (size_t)tph.inv_doubles * sizeof(double));
      h->tile_cnt_bytes = align_up((B * (size_t)tph.ncnt + 1) * sizeof(int));
      CUDA_TRY(cudaMalloc(&h->tile_pool, poolb + invb + h->tile_cnt_bytes));
      TilePlan& T = h->tp;
      T.panel = 1;
      T.fr = (const TFront*)base;
      T.tasks = (const int4*)(base + fb);
      T.hidx = (const int*)(base + fb + tkb);
      T.tch = (const int2*)(base + fb + tkb + hb);
      T.tcut = (const int*)(base + fb + tkb + hb + chb);
      T.tkptr = (const int*)kb_;
      T.tkidx = (const int*)(kb_ + kpb);
      T.nf = (int)tph.fr.size();
      T.ntask = (int)tasks.size();
      T.ncnt = tph.ncnt;
      T.pool_doubles = tph.pool_doubles;
      T.pool = (double*)h->tile_pool;
      T.inv = (double*)((char*)h->tile_pool + poolb);
      T.inv_doubles = tph.inv_doubles;
      T.ibase = (const long long*)(kb_ + kpb + kib);
      T.cnt = (int*)((char*)h->tile_pool + poolb + invb);
      T.trace = nullptr;
      h->tsolve = !h->huge_solve_cta && !(getenv("KKT_TSOLVE") && atoi(getenv("KKT_TSOLVE")) == 0);
      // the tile solve reads L from the tile pool: the factorisation skips the panel copies
      h->tp.panel = h->tsolve ? 0 : 1;
      if (getenv("KKT_TILE_PANEL") && atoi(getenv("KKT_TILE_PANEL")) > 0) h->tp.panel = 1;
      if (h->tsolve) {
        TSolvePlanHost tsh;
        // chain tasks (one CTA per front panel, tsolve.cuh FCH / BCH) unless a panel is too tall
        int maxnbp = 0;
        for (const auto& fr_ : tph.fr) maxnbp = std::max(maxnbp, fr_.nbp);
        // measured: C4 solve 5.31 -> 4.73 ms, C3 15.8 -> 15.0 ms (KKT_TS_CHAIN=0: per-step tasks)
        h->ts_chain = maxnbp <= TS_NBP_MAX && !(getenv("KKT_TS_CHAIN") && atoi(getenv("KKT_TS_CHAIN")) == 0);
        build_tile_solve_plan(P, tph, h->g_tile, h->ts_chain, tsh);
        h->tsp.wave = 4;  // measured C4 8.69 / 8.73 / 8.76 ms at 4 / 3 / 2
        if (const char* e = getenv("KKT_TS_WAVE")) h->tsp.wave = std::min(std::min(TS_RING, TILE_THREADS / 64), std::max(1, atoi(e)));
        h->ts_est_us = tsh.est_us;
        std::vector<TTask> st;
        st.reserve(tsh.tasks.size() * B);
        for (const TTask& t : tsh.tasks)
          for (size_t b = 0; b < B; b++) st.push_back(TTask{t.x | (int)(b << 4), t.y, t.z, t.w});
        const size_t sb = align_up(st.size() * sizeof(TTask)), cbb = align_up(tsh.cbase2.size() * sizeof(int));
        const size_t pbb = align_up(tsh.pbase.size() * sizeof(long long));
        const size_t partb = align_up(B * (size_t)tsh.part_doubles * sizeof(double));
        h->ts_cnt_bytes = align_up((B * (size_t)tsh.ncnt + 1) * sizeof(int));
        CUDA_TRY(cudaMalloc(&h->ts_mem, sb + cbb + pbb + partb + h->ts_cnt_bytes));
        char* tb_ = (char*)h->ts_mem;
        CUDA_TRY(cudaMemcpy(tb_, st.data(), st.size() * sizeof(TTask), cudaMemcpyHostToDevice));
        CUDA_TRY(cudaMemcpy(tb_ + sb, tsh.cbase2.data(), tsh.cbase2.size() * sizeof(int), cudaMemcpyHostToDevice));
        CUDA_TRY(cudaMemcpy(tb_ + sb + cbb, tsh.pbase.data(), tsh.pbase.size() * sizeof(long long), cudaMemcpyHostToDevice));
        h->tsp.pbase = (const long long*)(tb_ + sb + cbb);
        h->tsp.part = (double*)(tb_ + sb + cbb + pbb);
        h->tsp.part_doubles = tsh.part_doubles;
        h->tsp.tasks = (const int4*)tb_;
        h->tsp.ntask = (int)st.size();
        h->tsp.ncnt = tsh.ncnt;
        h->tsp.cbase2 = (const int*)(tb_ + sb);
        h->tsp.cnt = (int*)(tb_ + sb + cbb + pbb + partb);
        if (h->sblock) {  // zeroed by tree_fwd_kernel, the kernel before the tile solve
          h->sbp.zbuf = h->tsp.cnt;
          h->sbp.zn = (int)(h->ts_cnt_bytes / sizeof(int));
        }
        h->tsp.trace = nullptr;
        CUDA_TRY(cudaFuncSetAttribute(tile_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, TS_SMEM_BYTES));
      }
      if (h->tsolve && getenv("KKT_TRACE") && atoi(getenv("KKT_TRACE")) > 0) {
        CUDA_TRY(cudaMalloc(&h->ts_trace, (size_t)h->tsp.ntask * 4 * sizeof(long long)));
        CUDA_TRY(cudaMemset(h->ts_trace, 0, (size_t)h->tsp.ntask * 4 * sizeof(long long)));
        h->tsp.trace = h->ts_trace;
      }
      if (getenv("KKT_TRACE") && atoi(getenv("KKT_TRACE")) > 0) {
        CUDA_TRY(cudaMalloc(&h->tile_trace, (size_t)T.ntask * 4 * sizeof(long long)));
        CUDA_TRY(cudaMemset(h->tile_trace, 0, (size_t)T.ntask * 4 * sizeof(long long)));
        T.trace = h->tile_trace;
      }
    }
  }
  CUDA_TRY(cudaHostAlloc(&h->pinned_flags, 64 * sizeof(int) + (size_t)P.batch * sizeof(int), cudaHostAllocDefault));
  for (auto& e : h->fev) CUDA_TRY(cudaEventCreate(&e));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  h->bound = true;
  return KKT_OK;
}

// Launch `kern` as a programmatic dependent of the previous kernel in the stream: it may start
// as soon as every CTA of that kernel has executed griddepcontrol.launch_dependents, and orders
// itself against the producer through device flags instead of kernel completion (the small/big
// phase boundary of the tree kernels).  Set KKT_NO_PDL=1 to serialise instead.
template <class... KArgs, class... Args>
static cudaError_t launch_pdl(bool pdl, void (*kern)(KArgs...), int grid, int block, int smem,
                              cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

static int grid_for(long long total, int threads, int sms) {
  long long g = (total + threads - 1) / threads;
  return (int)std::max(1LL, std::min(g, (long long)sms * 16));
}

// (blocks per instance, batch) grid of 256-thread blocks for the per-instance reductions
static dim3 grid_2d(long long n, int batch, int sms) {
  long long gx = (n + 255) / 256;
  const long long cap = std::max(1LL, (long long)sms * 8 / std::max(1, batch));
  return dim3((unsigned)std::max(1LL, std::min(gx, cap)), (unsigned)batch);
}

extern "C" kkt_status kkt_condense(kkt_handle h, const double* W_vals, const double* J_vals,
                                   const double* Sigma_x, const double* Sigma_s, const double* D,
                                   double delta_w, double delta_c, double gamma) {
  if (!h) return KKT_ERR_ARG;
  if (!h->bound) { g_err = "kkt_bind first"; return KKT_ERR_STATE; }
  const Plan& P = h->P;
  if ((!W_vals && P.nnzW) || (!J_vals && P.nnzJ) || !Sigma_x || (!Sigma_s && !D && P.m > P.m_eq)) {
    g_err = "null value pointer";
    return KKT_ERR_ARG;
  }
  h->Wv = W_vals; h->Jv = J_vals; h->Sx = Sigma_x; h->Ss = Sigma_s; h->Dov = D;
  h->dw = delta_w; h->dc = delta_c; h->gamma = gamma;
  h->launches = 0;
  h->graph_solve_pending = false;
  h->hy_pending = false;
  if (P.m > 0) {
    dweights_kernel<<<grid_for((long long)P.batch * P.m, 256, h->sms), 256, 0, h->ls>>>(
        h->dp, Sigma_s, D, delta_w, delta_c, gamma, h->Dh, h->Dl);
    LAUNCH_CHECK();
    h->launches++;
  }
  long long tot = (long long)P.batch * P.Kp[P.n];
  condense_kernel<<<grid_for(tot, 256, h->sms), 256, 0, h->ls>>>(h->dp, W_vals, J_vals, Sigma_x,
                                                                     h->Dh, delta_w, h->Kv);
  LAUNCH_CHECK();
  h->launches++;
  h->condensed = true;
  h->factored = false;
  return KKT_OK;
}

extern "C" kkt_status kkt_factor(kkt_handle h) {
  if (!h) return KKT_ERR_ARG;
  if (!h->condensed) { g_err = "kkt_condense first"; return KKT_ERR_STATE; }
  const Plan& P = h->P;
  const bool ev = h->ls == h->stream;  // not while recording a graph
  if (ev) CUDA_TRY(cudaEventRecord(h->fev[0], h->ls));
  if (h->ldlt) CUDA_TRY(cudaMemsetAsync(h->inert, 0, 3 * sizeof(int) * P.batch, h->ls));
  if (!P.order_s.empty() && h->fblock) {
    factor_block_kernel<FB_MINB><<<h->g_ffblk, FB_NT, h->fb_smem, h->ls>>>(
        h->dp, h->fbp, h->Kv, h->Lx, h->Ub, h->Dv, h->facnt, h->ctl + 0 * KKT_CTL, h->fail);
    LAUNCH_CHECK();
    h->launches++;
  } else if (!P.order_s.empty()) {
    if (h->fsmall_occ == 3)
      factor_small_kernel<3><<<h->g_fsmall, KKT_WPB * 32, h->fsmall_smem, h->ls>>>(
        h->dp, h->Kv, h->Lx, h->Ub, h->Dv, h->facnt, h->ctl + 0 * KKT_CTL, h->fail);
    else
      factor_small_kernel<1><<<h->g_fsmall, KKT_WPB * 32, h->fsmall_smem, h->ls>>>(
        h->dp, h->Kv, h->Lx, h->Ub, h->Dv, h->facnt, h->ctl + 0 * KKT_CTL, h->fail);
    LAUNCH_CHECK();
    h->launches++;
  }
  if (!P.up_bf.empty()) {
    CUDA_TRY(launch_pdl(h->pdl && (h->pdl_mask & 1) && !P.order_s.empty(), h->ldlt ? factor_big_kernel<true> : factor_big_kernel<false>, h->g_fbig, KKT_BNT, h->fbig_smem, h->ls,
                        h->dp, (const double*)h->Kv, h->Lx, h->Ub, h->Dv, h->facnt, h->ctl + 1 * KKT_CTL, h->fail,
                        (long long)h->factor_smem_cap));
    h->launches++;
  }
  if (h->use_linv) {  // L11^-1 of the big supernodes for the solve sweeps (parallel, off the tree path)
    linv_kernel<<<h->g_linv, KKT_BNT, h->linv_smem, h->ls>>>(h->dp, h->Lx, h->Dv, h->Li);
    LAUNCH_CHECK();
    h->launches++;
  }
  if (ev) CUDA_TRY(cudaEventRecord(h->fev[1], h->ls));
  if (!P.order_h.empty() && h->tiles) {
    CUDA_TRY(cudaMemsetAsync(h->tp.cnt, 0, h->tile_cnt_bytes, h->ls));
    DevPlan dp = h->dp;
    TilePlan tp = h->tp;
    const double* kv = h->Kv;
    double *lx = h->Lx, *dv = h->Dv;
    const double* ub = h->Ub;
    int* fail = h->fail;
    void* args[] = {&dp, &tp, &kv, &lx, &ub, &dv, &fail};
    CUDA_TRY(cudaLaunchCooperativeKernel(h->ldlt ? (const void*)tile_factor_kernel<true> : (const void*)tile_factor_kernel<false>,
                                         dim3(h->g_tile), dim3(TILE_THREADS), args,
                                         (size_t)TILE_SMEM_BYTES, h->ls));
    h->launches++;
  } else if (!P.order_h.empty()) {
    DevPlan dp = h->dp;
    const double* kv = h->Kv;
    double *lx = h->Lx, *ub = h->Ub, *dv = h->Dv;
    int *cnt = h->facnt, *fail = h->fail;
    HugeSched hs = h->hsched;
    void* args[] = {&dp, &kv, &lx, &ub, &dv, &cnt, &fail, &hs};
    CUDA_TRY(cudaLaunchCooperativeKernel((const void*)factor_huge_kernel, dim3(h->g_huge), dim3(32 * h->huge_warps), args,
                                         (size_t)h->huge_smem, h->ls));
    h->launches++;
  }
  if (ev) CUDA_TRY(cudaEventRecord(h->fev[2], h->ls));
  h->fev_valid = ev;
  h->factored = true;
  return KKT_OK;
}

extern "C" kkt_status kkt_factor_phase_ms(kkt_handle h, double* ms) {
  if (!h || !ms) return KKT_ERR_ARG;
  if (!h->fev_valid) { g_err = "no timed kkt_factor yet"; return KKT_ERR_STATE; }
  float a = 0.f, b = 0.f;
  CUDA_TRY(cudaEventSynchronize(h->fev[2]));
  CUDA_TRY(cudaEventElapsedTime(&a, h->fev[0], h->fev[1]));
  CUDA_TRY(cudaEventElapsedTime(&b, h->fev[1], h->fev[2]));
  ms[0] = a;
  ms[1] = b;
  return KKT_OK;
}

// forward + backward through the huge fronts (tile-task solve or the level kernel); nothing
// when the solve-side plan view treats them as CTA supernodes
static kkt_status launch_huge_solve(kkt_plan* h, const double* rhs, long long rs, double* xout,
                                    long long xs, const int* done) {
  const Plan& P = h->P;
  const bool cta_huge = h->huge_solve_cta;
  if (!P.order_h.empty() && !cta_huge && h->tsolve) {
    if (!(h->sblock && h->sbp.zbuf)) CUDA_TRY(cudaMemsetAsync(h->tsp.cnt, 0, h->ts_cnt_bytes, h->ls));
    DevPlan dp = h->dp;
    TilePlan tp = h->tp;
    TSolvePlan sp = h->tsp;
    const double *dv = h->Dv, *rh = rhs;
    double *y = h->Y, *uv = h->uv, *xp = h->Xp, *xo = xout;
    long long rs_ = rs, xs_ = xs;
    const int* dn = done;
    void* args[] = {&dp, &tp, &sp, &dv, &rh, &rs_, &y, &uv, &xp, &xo, &xs_, &dn};
    CUDA_TRY(cudaLaunchCooperativeKernel((const void*)tile_solve_kernel, dim3(h->g_tile), dim3(TILE_THREADS), args,
                                         (size_t)TS_SMEM_BYTES, h->ls));
    h->launches++;
  } else if (!P.order_h.empty() && !cta_huge) {
    DevPlan dp = h->dp;
    const double *lx = h->Lx, *dv = h->Dv, *rh = rhs;
    double *y = h->Y, *uv = h->uv, *xp = h->Xp, *xo = xout;
    long long rs_ = rs, xs_ = xs;
    const int* dn = done;
    HugeSched hs = h->hsched_s;
    void* args[] = {&dp, &lx, &dv, &rh, &rs_, &y, &uv, &xp, &xo, &xs_, &dn, &hs};
    CUDA_TRY(cudaLaunchCooperativeKernel((const void*)solve_huge_kernel, dim3(h->g_hsolve), dim3(256), args, 0,
                                         h->ls));
    h->launches++;
  }
  return KKT_OK;
}

// forward + backward solve of all batch instances: xout = K^-1 rhs
static kkt_status launch_solve(kkt_plan* h, const double* rhs, long long rs, double* xout,
                               long long xs, const int* done) {
  const Plan& P = h->P;
  const DevPlan& dq = h->huge_solve_cta ? h->dps : h->dp;  // solve-side plan view
  const bool cta_huge = h->huge_solve_cta;
  if (h->sblock) {  // whole-tree kernels around the huge fronts' tile solve
    const double* li = h->use_linv ? h->Li : nullptr;
    (h->sb_nt == 128 ? tree_fwd_kernel<false, 128> : tree_fwd_kernel<false, 256>)<<<h->g_fblk, h->sb_nt, h->sb_smem, h->ls>>>(
        dq, h->sbp, h->Lx, h->Dv, rhs, rs, h->Y, h->uv, h->fcnt, h->ctl + 2 * KKT_CTL, done, li);
    LAUNCH_CHECK();
    h->launches++;
    TRY(launch_huge_solve(h, rhs, rs, xout, xs, done));
    (h->sb_nt == 128 ? tree_bwd_kernel<false, 128> : tree_bwd_kernel<false, 256>)<<<h->g_bblk, h->sb_nt, h->sb_smem, h->ls>>>(
        dq, h->sbp, h->Lx, h->Dv, h->Y, h->Xp, xout, xs, h->bflag, h->ctl + 5 * KKT_CTL, done, li);
    LAUNCH_CHECK();
    h->launches++;
    return KKT_OK;
  }
  if (!P.order_s.empty()) {
    fwd_small_kernel<<<h->g_tsmall, KKT_WPB * 32, h->tsmall_smem, h->ls>>>(
        dq, h->Lx, h->Dv, rhs, rs, h->Y, h->uv, h->fcnt, h->ctl + 2 * KKT_CTL, done);
    LAUNCH_CHECK();
    h->launches++;
  }
  if (!P.order_b.empty()) {
    if (cta_huge ? !P.up_b.empty() : !P.up_bf.empty()) {
      CUDA_TRY(launch_pdl(h->pdl && (h->pdl_mask & 2) && !P.order_s.empty(), fwd_big_kernel, h->g_tbig, KKT_BNT, h->tbig_smem, h->ls,
                          dq, (const double*)h->Lx, (const double*)h->Dv, rhs, rs, h->Y, h->uv, h->fcnt,
                          h->ctl + 3 * KKT_CTL, done, h->pcap, (const double*)(h->use_linv ? h->Li : nullptr)));
      h->launches++;
    }
    TRY(launch_huge_solve(h, rhs, rs, xout, xs, done));
    if (h->ldlt) {  // K^-1 = L~^-T S L~^-1: y <- S y before the backward sweep
      ldlt_sign_kernel<<<grid_for((long long)P.batch * P.n, 256, h->sms), 256, 0, h->ls>>>((long long)P.batch * P.n, h->Y, h->Sg);
      LAUNCH_CHECK();
      h->launches++;
    }
    if (cta_huge || P.order_b.size() > P.order_h.size()) {
      bwd_big_kernel<<<h->g_bbig, KKT_BNT, h->tbig_smem, h->ls>>>(
          dq, h->Lx, h->Dv, h->Y, h->Xp, xout, xs, h->TQ, h->ctl + 4 * KKT_CTL, done, h->pcap, h->bflag,
          h->use_linv ? h->Li : nullptr);
      LAUNCH_CHECK();
      h->launches++;
    }
  }
  if (!P.order_s.empty()) {
    // overlapped with bwd_big only when bwd_big is the kernel right before it
    const bool after_big = (cta_huge ? !P.order_b.empty() : P.order_b.size() > P.order_h.size()) && (h->pdl_mask & 4);
    CUDA_TRY(launch_pdl(h->pdl && after_big, bwd_small_kernel, h->g_bsmall, KKT_WPB * 32, h->tsmall_smem, h->ls,
                          dq, (const double*)h->Lx, (const double*)h->Dv, (const double*)h->Y, h->Xp, xout, xs,
                          h->TQs, h->ctl + 5 * KKT_CTL, done, h->bflag, (int)(h->pdl && after_big)));
    h->launches++;
  }
  return KKT_OK;
}

static kkt_status launch_resid(kkt_plan* h, const double* x, const double* rhs, int mode,
                               const double* dy, const double* rb2, double* res,
                               unsigned long long* omega, const int* done) {
  const Plan& P = h->P;
  if (P.m > 0) {
    resid_rows_kernel<<<grid_for((long long)P.batch * P.m, 256, h->sms), 256, 0, h->ls>>>(
        h->dp, h->Jv, h->Dh, h->Dl, x, P.n, mode, dy, rb2, h->res2, h->T, h->A, done);
    LAUNCH_CHECK();
    h->launches++;
  }
  if (h->resid_warp) {  // long columns (dense W): one warp per column
    dim3 g = grid_2d(((long long)P.n + 7) / 8 * 256, P.batch, h->sms);
    resid_cols_warp_kernel<<<g, 256, 0, h->ls>>>(
        h->dp, h->Wv, h->Jv, h->Sx, h->dw, x, P.n, rhs, P.n, h->T, h->A, res, omega, done);
    LAUNCH_CHECK();
    h->launches++;
    return KKT_OK;
  }
  resid_cols_kernel<<<grid_2d(P.n, P.batch, h->sms), 256, 0, h->ls>>>(
      h->dp, h->Wv, h->Jv, h->Sx, h->dw, x, P.n, rhs, P.n, h->T, h->A, res, omega, done);
  LAUNCH_CHECK();
  h->launches++;
  return KKT_OK;
}


// One refinement sweep's tail: residual of x, per-instance stop decision, sweep counter (and
// the WHILE condition when recorded into the solve graph).
static kkt_status enqueue_check(kkt_plan* h, const double* b, double* x, int max_refine, double tol_bwd,
                                cudaGraphConditionalHandle hc, int use_handle) {
  const Plan& P = h->P;
  const int gb = (P.batch + 127) / 128;
  TRY(launch_resid(h, x, b, 0, nullptr, nullptr, h->res, h->C.omega, h->C.done));
  refine_decide_kernel<<<gb, 128, 0, h->ls>>>(P.batch, h->C, tol_bwd, max_refine);
  LAUNCH_CHECK();
  refine_cond_kernel<<<1, 1, 0, h->ls>>>(P.batch, h->C, hc, use_handle);
  LAUNCH_CHECK();
  h->launches += 2;
  return KKT_OK;
}

static kkt_status enqueue_correction(kkt_plan* h, double* x) {
  const Plan& P = h->P;
  TRY(launch_solve(h, h->res, P.n, h->dxv, P.n, h->C.done));
  refine_update_kernel<<<grid_2d(P.n, P.batch, h->sms), 256, 0, h->ls>>>(
      P.batch, P.n, x, h->dxv, h->C);
  LAUNCH_CHECK();
  h->launches++;
  return KKT_OK;
}

static kkt_status enqueue_prologue(kkt_plan* h, const double* b, double* x) {
  const Plan& P = h->P;
  refine_init_kernel<<<(P.batch + 127) / 128, 128, 0, h->ls>>>(P.batch, h->C);
  LAUNCH_CHECK();
  h->launches++;
  return launch_solve(h, b, P.n, x, P.n, nullptr);
}

// stream-ordered refined solve (no graph): host loop over the sweeps, finished instances and
// finished sweeps early-exit on device
static kkt_status enqueue_solve(kkt_plan* h, const double* b, double* x, int max_refine, double tol_bwd) {
  TRY(enqueue_prologue(h, b, x));
  for (int k = 0; k <= max_refine; k++) {
    TRY(enqueue_check(h, b, x, max_refine, tol_bwd, 0, 0));
    if (k == max_refine) break;
    TRY(enqueue_correction(h, x));
  }
  return KKT_OK;
}

// Record the refined solve as one graph: prologue (first solve + residual + decision, first
// correction sweep), then a WHILE node whose body is one correction sweep; the body runs only
// while some instance is still refining, so converged solves launch no idle sweeps.
static kkt_status record_solve_graph(kkt_plan* h, int max_refine, double tol_bwd, cudaGraph_t* out,
                                     long long* n_pro, long long* n_body) {
  cudaGraph_t g = nullptr;
  if (h->solve_if && !h->solve_while && max_refine >= 2) {
    // prologue + first correction sweep recorded directly (with programmatic overlap); the
    // remaining sweeps 2..max_refine sit in the body of one IF node taken only when some instance
    // is still refining after the first correction -- converged solves skip them entirely
    CUDA_TRY(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle hc;
    cudaError_t e = cudaGraphConditionalHandleCreate(&hc, g, 0, 0);
    if (e != cudaSuccess) { cudaGraphDestroy(g); g_err = std::string("conditional handle: ") + cudaGetErrorString(e); return KKT_ERR_CUDA; }
    auto capture_into = [&](cudaGraph_t into, auto&& body) -> kkt_status {
      h->ls = h->cap;
      cudaError_t ce = cudaStreamBeginCaptureToGraph(h->cap, into, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
      if (ce != cudaSuccess) { h->ls = h->stream; g_err = std::string("capture: ") + cudaGetErrorString(ce); return KKT_ERR_CUDA; }
      kkt_status st = body();
      cudaGraph_t got = nullptr;
      ce = cudaStreamEndCapture(h->cap, &got);
      h->ls = h->stream;
      if (st != KKT_OK) return st;
      if (ce != cudaSuccess) { g_err = std::string("capture: ") + cudaGetErrorString(ce); return KKT_ERR_CUDA; }
      return KKT_OK;
    };
    h->launches = 0;
    kkt_status st = capture_into(g, [&] {
      TRY(enqueue_prologue(h, h->gb, h->gx));
      TRY(enqueue_check(h, h->gb, h->gx, max_refine, tol_bwd, hc, 1));
      TRY(enqueue_correction(h, h->gx));
      return enqueue_check(h, h->gb, h->gx, max_refine, tol_bwd, hc, 1);
    });
    if (st != KKT_OK) { cudaGraphDestroy(g); return st; }
    *n_pro = h->launches;
    size_t nn = 0, ne = 0;
    CUDA_TRY(cudaGraphGetNodes(g, nullptr, &nn));
    CUDA_TRY(cudaGraphGetEdges_v2(g, nullptr, nullptr, nullptr, &ne));  // v2: programmatic edges
    std::vector<cudaGraphNode_t> nodes(nn), from(ne), to(ne);
    std::vector<cudaGraphEdgeData> edata(ne);
    CUDA_TRY(cudaGraphGetNodes(g, nodes.data(), &nn));
    if (ne) CUDA_TRY(cudaGraphGetEdges_v2(g, from.data(), to.data(), edata.data(), &ne));
    std::vector<cudaGraphNode_t> leaves;
    for (auto nd : nodes)
      if (std::find(from.begin(), from.end(), nd) == from.end()) leaves.push_back(nd);
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = hc;
    cp.conditional.type = cudaGraphCondTypeIf;
    cp.conditional.size = 1;
    cudaGraphNode_t ifn;
    e = cudaGraphAddNode(&ifn, g, leaves.data(), leaves.size(), &cp);
    if (e != cudaSuccess) { cudaGraphDestroy(g); g_err = std::string("if node: ") + cudaGetErrorString(e); return KKT_ERR_CUDA; }
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    const bool pdl_saved = h->pdl;
    h->pdl = false;  // programmatic launches are not captured into conditional bodies
    h->launches = 0;
    st = capture_into(body, [&] {
      for (int k = 2; k <= max_refine; k++) {
        TRY(enqueue_correction(h, h->gx));
        TRY(enqueue_check(h, h->gb, h->gx, max_refine, tol_bwd, hc, 0));
      }
      return KKT_OK;
    });
    h->pdl = pdl_saved;
    if (st != KKT_OK) { cudaGraphDestroy(g); return st; }
    *n_body = h->launches;
    *out = g;
    return KKT_OK;
  }
  if (!h->solve_while) {  // all sweeps recorded; idle ones exit at once on the all-done count
    h->ls = h->cap;
    CUDA_TRY(cudaStreamBeginCapture(h->cap, cudaStreamCaptureModeThreadLocal));
    h->launches = 0;
    kkt_status st = enqueue_solve(h, h->gb, h->gx, max_refine, tol_bwd);
    cudaError_t e = cudaStreamEndCapture(h->cap, &g);
    h->ls = h->stream;
    if (st != KKT_OK) { if (g) cudaGraphDestroy(g); return st; }
    if (e != cudaSuccess) { g_err = std::string("graph capture: ") + cudaGetErrorString(e); return KKT_ERR_CUDA; }
    *n_pro = h->launches;
    *n_body = 0;
    *out = g;
    return KKT_OK;
  }
  CUDA_TRY(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle hc;
  cudaError_t e = cudaGraphConditionalHandleCreate(&hc, g, 0, 0);
  if (e != cudaSuccess) { cudaGraphDestroy(g); g_err = std::string("conditional handle: ") + cudaGetErrorString(e); return KKT_ERR_CUDA; }
  auto capture = [&](cudaGraph_t into, auto&& body) -> kkt_status {
    h->ls = h->cap;
    cudaError_t ce = cudaStreamBeginCaptureToGraph(h->cap, into, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
    if (ce != cudaSuccess) { h->ls = h->stream; g_err = std::string("capture: ") + cudaGetErrorString(ce); return KKT_ERR_CUDA; }
    kkt_status st = body();
    cudaGraph_t got = nullptr;
    ce = cudaStreamEndCapture(h->cap, &got);
    h->ls = h->stream;
    if (st != KKT_OK) return st;
    if (ce != cudaSuccess) { g_err = std::string("capture: ") + cudaGetErrorString(ce); return KKT_ERR_CUDA; }
    return KKT_OK;
  };
  h->launches = 0;
  // the first correction sweep is recorded unconditionally (its kernels exit at once when every
  // instance has already converged): the WHILE body -- a device-launched graph, measurably
  // slower to start -- then only runs for systems that need two or more corrections
  kkt_status st = capture(g, [&] {
    TRY(enqueue_prologue(h, h->gb, h->gx));
    TRY(enqueue_check(h, h->gb, h->gx, max_refine, tol_bwd, hc, 1));
    if (max_refine < 1) return KKT_OK;
    TRY(enqueue_correction(h, h->gx));
    return enqueue_check(h, h->gb, h->gx, max_refine, tol_bwd, hc, 1);
  });
  if (st != KKT_OK) { cudaGraphDestroy(g); return st; }
  *n_pro = h->launches;
  // leaves of the prologue: nodes without outgoing edges
  size_t nn = 0, ne = 0;
  CUDA_TRY(cudaGraphGetNodes(g, nullptr, &nn));
  CUDA_TRY(cudaGraphGetEdges(g, nullptr, nullptr, &ne));
  std::vector<cudaGraphNode_t> nodes(nn), from(ne), to(ne);
  CUDA_TRY(cudaGraphGetNodes(g, nodes.data(), &nn));
  if (ne) CUDA_TRY(cudaGraphGetEdges(g, from.data(), to.data(), &ne));
  std::vector<cudaGraphNode_t> leaves;
  for (auto nd : nodes)
    if (std::find(from.begin(), from.end(), nd) == from.end()) leaves.push_back(nd);
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = hc;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t wn;
  e = cudaGraphAddNode(&wn, g, leaves.data(), leaves.size(), &cp);
  if (e != cudaSuccess) { cudaGraphDestroy(g); g_err = std::string("while node: ") + cudaGetErrorString(e); return KKT_ERR_CUDA; }
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  h->launches = 0;
  st = capture(body, [&] {
    TRY(enqueue_correction(h, h->gx));
    return enqueue_check(h, h->gb, h->gx, max_refine, tol_bwd, hc, 1);
  });
  if (st != KKT_OK) { cudaGraphDestroy(g); return st; }
  *n_body = h->launches;
  *out = g;
  return KKT_OK;
}

extern "C" kkt_status kkt_solve(kkt_handle h, const double* b, double* x, int max_refine, double tol_bwd) {
  if (!h || !b || !x) return KKT_ERR_ARG;
  if (!h->factored) { g_err = "kkt_factor first"; return KKT_ERR_STATE; }
  const Plan& P = h->P;
  if (tol_bwd < 0) tol_bwd = 0;  // 0 disables the backward-error stop (R9)
  max_refine = std::max(0, max_refine);
  h->launches = 0;
  h->graph_solve_pending = false;
  h->hy_pending = false;
  h->last_hykkt = false;
  if (!h->use_graph) return enqueue_solve(h, b, x, max_refine, tol_bwd);
  // one CUDA graph per (max_refine, tol, value pointers, delta_w), recorded on a private stream
  const bool stale = !h->solve_exec || h->g_max_refine != max_refine || h->g_tol != tol_bwd ||
                     h->g_W != h->Wv || h->g_J != h->Jv || h->g_Sx != h->Sx || h->g_dw != h->dw;
  if (stale) {
    if (h->solve_exec) { cudaGraphExecDestroy(h->solve_exec); h->solve_exec = nullptr; }
    cudaGraph_t g = nullptr;
    TRY(record_solve_graph(h, max_refine, tol_bwd, &g, &h->g_pro, &h->g_body));
    cudaError_t e = cudaGraphInstantiate(&h->solve_exec, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) { g_err = std::string("graph instantiate: ") + cudaGetErrorString(e); return KKT_ERR_CUDA; }
    h->g_max_refine = max_refine; h->g_tol = tol_bwd; h->g_W = h->Wv; h->g_J = h->Jv;
    h->g_Sx = h->Sx; h->g_dw = h->dw;
  }
  const size_t bytes = (size_t)P.batch * P.n * sizeof(double);
  CUDA_TRY(cudaMemcpyAsync(h->gb, b, bytes, cudaMemcpyDeviceToDevice, h->stream));
  CUDA_TRY(cudaGraphLaunch(h->solve_exec, h->stream));
  CUDA_TRY(cudaMemcpyAsync(x, h->gx, bytes, cudaMemcpyDeviceToDevice, h->stream));
  h->launches = h->g_pro;
  h->graph_solve_pending = true;  // body executions known once the stream has drained
  return KKT_OK;
}

static kkt_status graph_leaves(cudaGraph_t g, std::vector<cudaGraphNode_t>& leaves);

// Record `body` on the capture stream into graph `into` after everything already in it (the
// captured nodes depend on the graph's current leaves); kernels go to h->ls = h->cap.
template <class F>
static kkt_status capture_into_graph(kkt_plan* h, cudaGraph_t into, F&& body) {
  std::vector<cudaGraphNode_t> deps;
  TRY(graph_leaves(into, deps));
  h->ls = h->cap;
  cudaError_t ce = cudaStreamBeginCaptureToGraph(h->cap, into, deps.empty() ? nullptr : deps.data(), nullptr,
                                                 deps.size(), cudaStreamCaptureModeThreadLocal);
  if (ce != cudaSuccess) { h->ls = h->stream; g_err = std::string("capture: ") + cudaGetErrorString(ce); return KKT_ERR_CUDA; }
  kkt_status st = body();
  cudaGraph_t got = nullptr;
  ce = cudaStreamEndCapture(h->cap, &got);
  h->ls = h->stream;
  if (st != KKT_OK) return st;
  if (ce != cudaSuccess) { g_err = std::string("capture: ") + cudaGetErrorString(ce); return KKT_ERR_CUDA; }
  return KKT_OK;
}

// Nodes of g without outgoing edges (the current tail of a recorded sequence).
static kkt_status graph_leaves(cudaGraph_t g, std::vector<cudaGraphNode_t>& leaves) {
  size_t nn = 0, ne = 0;
  CUDA_TRY(cudaGraphGetNodes(g, nullptr, &nn));
  CUDA_TRY(cudaGraphGetEdges_v2(g, nullptr, nullptr, nullptr, &ne));
  std::vector<cudaGraphNode_t> nodes(nn), from(ne), to(ne);
  std::vector<cudaGraphEdgeData> ed(ne);
  CUDA_TRY(cudaGraphGetNodes(g, nodes.data(), &nn));
  if (ne) CUDA_TRY(cudaGraphGetEdges_v2(g, from.data(), to.data(), ed.data(), &ne));
  leaves.clear();
  for (auto nd : nodes)
    if (std::find(from.begin(), from.end(), nd) == from.end()) leaves.push_back(nd);
  return KKT_OK;
}

// Append to graph g a WHILE node (after the current leaves) whose body is recorded by `body`;
// the body's last kernel sets the condition through `hc`.
template <class F>
static kkt_status append_while(kkt_plan* h, cudaGraph_t g, cudaGraphConditionalHandle hc, F&& body) {
  std::vector<cudaGraphNode_t> leaves;
  TRY(graph_leaves(g, leaves));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = hc;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t wn;
  CUDA_TRY(cudaGraphAddNode(&wn, g, leaves.data(), leaves.size(), &cp));
  const bool pdl_saved = h->pdl;
  h->pdl = false;  // programmatic launches are not captured into conditional bodies
  kkt_status st = capture_into_graph(h, cp.conditional.phGraph_out[0], body);
  h->pdl = pdl_saved;
  return st;
}

// One HyKKT pass (eq. 14) for right-hand side (r1, r2) -> (dxo, dyo), recorded into
// graph g (segments between WHILE nodes are captured in turn):
//   s = r1 + gamma G^T r2 ;  z = K_gamma^-1 s ;  r = G z - r2 ;  p = r ; dy = 0
//   Krylov loop on S_gamma dy = r (S_gamma = G K_gamma^-1 G^T), one graph WHILE node:
//     CG (krylov 0):  q = S p ; alpha = r.r / p.q ; dy += alpha p ; r -= alpha q ; p = r + beta p
//     CR (krylov 1, Hestenes-Stiefel conjugate residuals): with s = S r, q = S p,
//                     alpha = r.s / q.q ; dy += alpha p ; r -= alpha q ; s = S r ;
//                     beta = r.s_new / r.s_old ; p = r + beta p ; q = s + beta q
//   dx = K_gamma^-1 (s - G^T dy)
// Instances whose outer refinement has finished (skip != nullptr, C.odone) skip the whole pass.
static kkt_status hykkt_pass(kkt_plan* h, cudaGraph_t g, cudaGraphConditionalHandle hc,
                             const double* r1, const double* r2, double* dxo, double* dyo,
                             double rtol, int maxit, bool first, int krylov) {
  const Plan& P = h->P;
  const int gs = grid_for((long long)P.batch * P.n, 256, h->sms);
  const int* skip = first ? nullptr : h->C.odone;
  dim3 gg(KKT_NPART, P.batch);
  TRY(capture_into_graph(h, g, [&]() -> kkt_status {
    cg_init_kernel<<<1, 256, 0, h->ls>>>(P.batch, h->C, first ? 0 : 1);
    gt_kernel<<<gs, 256, 0, h->ls>>>(h->dp, h->Jv, r2, h->gamma, r1, h->sg, skip);
    LAUNCH_CHECK();
    TRY(launch_solve(h, h->sg, P.n, h->zv, P.n, skip));
    g_kernel<<<gg, KKT_CGT, 0, h->ls>>>(h->dp, h->Jv, h->zv, r2, h->cr, h->cp, dyo, h->C, 0, first ? 1 : 0, nullptr);
    LAUNCH_CHECK();
    h->launches += 3;
    if (krylov == 1) {  // s0 = q0 = S r0 (p0 = r0)
      gt_kernel<<<gs, 256, 0, h->ls>>>(h->dp, h->Jv, h->cp, 1.0, nullptr, h->wv, h->C.cg_done);
      LAUNCH_CHECK();
      TRY(launch_solve(h, h->wv, P.n, h->zv, P.n, h->C.cg_done));
      g_kernel<<<gg, KKT_CGT, 0, h->ls>>>(h->dp, h->Jv, h->zv, nullptr, h->cs, h->cp, nullptr, h->C, 2, 0, h->cq);
      LAUNCH_CHECK();
      h->launches += 2;
    }
    cg_cond_kernel<<<1, 1, 0, h->ls>>>(P.batch, h->C, hc, 0);  // loop entry condition
    LAUNCH_CHECK();
    h->launches += 1;
    return KKT_OK;
  }));
  const long long l0 = h->launches;
  TRY(append_while(h, g, hc, [&]() -> kkt_status {
    if (krylov == 0) {
      gt_kernel<<<gs, 256, 0, h->ls>>>(h->dp, h->Jv, h->cp, 1.0, nullptr, h->wv, h->C.cg_done);
      LAUNCH_CHECK();
      TRY(launch_solve(h, h->wv, P.n, h->zv, P.n, h->C.cg_done));
      g_kernel<<<gg, KKT_CGT, 0, h->ls>>>(h->dp, h->Jv, h->zv, nullptr, h->cq, h->cp, nullptr, h->C, 1, 0, nullptr);
      LAUNCH_CHECK();
      cg_update_kernel<<<gg, KKT_CGT, 0, h->ls>>>(P.batch, P.m_eq, dyo, h->cr, h->cp, h->cq, h->C,
                                               rtol, h->status, first ? 1 : 0, maxit);
      LAUNCH_CHECK();
      cg_p_kernel<<<dim3(std::max(1, std::min((P.m_eq + 255) / 256, 64)), P.batch), 256, 0, h->ls>>>(
          P.batch, P.m_eq, h->cp, h->cr, h->C);
      LAUNCH_CHECK();
    } else {
      cg_update_kernel<<<gg, KKT_CGT, 0, h->ls>>>(P.batch, P.m_eq, dyo, h->cr, h->cp, h->cq, h->C,
                                               rtol, h->status, first ? 1 : 0, maxit);
      LAUNCH_CHECK();
      gt_kernel<<<gs, 256, 0, h->ls>>>(h->dp, h->Jv, h->cr, 1.0, nullptr, h->wv, h->C.cg_done);
      LAUNCH_CHECK();
      TRY(launch_solve(h, h->wv, P.n, h->zv, P.n, h->C.cg_done));
      g_kernel<<<gg, KKT_CGT, 0, h->ls>>>(h->dp, h->Jv, h->zv, h->cr, h->cs, nullptr, nullptr, h->C, 3, 0, nullptr);
      LAUNCH_CHECK();
      cr_pq_kernel<<<gg, KKT_CGT, 0, h->ls>>>(P.batch, P.m_eq, h->cp, h->cq, h->cr, h->cs, h->C);
      LAUNCH_CHECK();
    }
    cg_cond_kernel<<<1, 1, 0, h->ls>>>(P.batch, h->C, hc, 1);
    LAUNCH_CHECK();
    h->launches += 5;
    return KKT_OK;
  }));
  h->hy_body = h->launches - l0;
  return capture_into_graph(h, g, [&]() -> kkt_status {
    cg_finish_kernel<<<(P.batch + 127) / 128, 128, 0, h->ls>>>(P.batch, h->C, first ? 1 : 0, h->status);
    LAUNCH_CHECK();
    // dx = K_gamma^-1 (s - G^T dy)
    gt_kernel<<<gs, 256, 0, h->ls>>>(h->dp, h->Jv, dyo, -1.0, h->sg, h->wv, skip);
    LAUNCH_CHECK();
    TRY(launch_solve(h, h->wv, P.n, dxo, P.n, skip));
    h->launches += 2;
    return KKT_OK;
  });
}

// The whole HyKKT solve as one graph: first pass, then max_outer_refine correction passes on
// the saddle system [K_gamma-part G^T; G 0] with a double-double residual; the outer loop stops
// per instance on the device (outer_decide_kernel), later passes skip finished instances.
static kkt_status record_hykkt_graph(kkt_plan* h, double rtol, int maxit, int max_outer, int krylov,
                                     cudaGraph_t* out) {
  const Plan& P = h->P;
  cudaGraph_t g = nullptr;
  CUDA_TRY(cudaGraphCreate(&g, 0));
  auto fail = [&](kkt_status st) { cudaGraphDestroy(g); return st; };
  h->launches = 0;
  kkt_status st = capture_into_graph(h, g, [&]() -> kkt_status {
    outer_init_kernel<<<(P.batch + 127) / 128, 128, 0, h->ls>>>(P.batch, h->C);
    LAUNCH_CHECK();
    return KKT_OK;
  });
  if (st != KKT_OK) return fail(st);
  const long long mm = P.m_eq;
  for (int k = 0; k <= max_outer; k++) {
    cudaGraphConditionalHandle hc;
    cudaError_t e = cudaGraphConditionalHandleCreate(&hc, g, 0, cudaGraphCondAssignDefault);
    if (e != cudaSuccess) { g_err = std::string("conditional handle: ") + cudaGetErrorString(e); return fail(KKT_ERR_CUDA); }
    if (k == 0) {
      st = hykkt_pass(h, g, hc, h->g_r1, h->g_r2, h->g_dx, h->g_dy, rtol, maxit, true, krylov);
    } else {
      // rho1 = rbar1 - K dx - G^T dy ; rho2 = rbar2 - G dx (double-double, K without gamma rows)
      st = capture_into_graph(h, g, [&]() -> kkt_status {
        return launch_resid(h, h->g_dx, h->g_r1, 1, h->g_dy, h->g_r2, h->hr1, nullptr, h->C.odone);
      });
      if (st == KKT_OK)
        st = hykkt_pass(h, g, hc, h->hr1, h->res2, h->hdx, h->hdy, rtol, maxit, false, krylov);
      if (st == KKT_OK)
        st = capture_into_graph(h, g, [&]() -> kkt_status {
          outer_update_kernel<<<grid_2d(P.n, P.batch, h->sms), 256, 0, h->ls>>>(P.batch, P.n, h->g_dx, h->hdx, h->C, 0);
          LAUNCH_CHECK();
          outer_update_kernel<<<grid_2d(mm, P.batch, h->sms), 256, 0, h->ls>>>(P.batch, mm, h->g_dy, h->hdy, h->C, 2);
          LAUNCH_CHECK();
          outer_decide_kernel<<<(P.batch + 127) / 128, 128, 0, h->ls>>>(P.batch, h->C);
          LAUNCH_CHECK();
          h->launches += 3;
          return KKT_OK;
        });
    }
    if (st != KKT_OK) return fail(st);
  }
  h->hy_fixed = h->launches - (long long)(max_outer + 1) * h->hy_body;
  *out = g;
  return KKT_OK;
}

extern "C" kkt_status hykkt_solve_krylov(kkt_handle h, const double* rbar1, const double* rbar2, double* dx,
                                         double* dy, double cg_rtol, int cg_maxit, int max_outer_refine,
                                         int krylov) {
  if (!h || !rbar1 || !dx) return KKT_ERR_ARG;
  if (krylov != 0 && krylov != 1) { g_err = "krylov must be 0 (CG) or 1 (CR)"; return KKT_ERR_ARG; }
  const Plan& P = h->P;
  if (P.m_eq > 0 && (!rbar2 || !dy)) return KKT_ERR_ARG;
  if (!h->factored) { g_err = "kkt_factor first"; return KKT_ERR_STATE; }
  if (cg_rtol <= 0) cg_rtol = 1e-12;
  if (cg_maxit <= 0) cg_maxit = std::max(1, std::min(P.m_eq, 2000));
  max_outer_refine = std::max(0, max_outer_refine);
  h->launches = 0;
  h->graph_solve_pending = false;
  h->hy_pending = false;
  h->last_hykkt = false;
  if (P.m_eq == 0) return kkt_solve(h, rbar1, dx, max_outer_refine, 0.0);
  const bool stale = !h->hy_exec || h->hy_rtol != cg_rtol || h->hy_maxit != cg_maxit ||
                     h->hy_outer != max_outer_refine || h->hy_krylov != krylov || h->hy_W != h->Wv ||
                     h->hy_J != h->Jv || h->hy_Sx != h->Sx || h->hy_gamma != h->gamma || h->hy_dw != h->dw;
  if (stale) {
    if (h->hy_exec) { cudaGraphExecDestroy(h->hy_exec); h->hy_exec = nullptr; }
    cudaGraph_t g = nullptr;
    TRY(record_hykkt_graph(h, cg_rtol, cg_maxit, max_outer_refine, krylov, &g));
    cudaError_t e = cudaGraphInstantiate(&h->hy_exec, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) { g_err = std::string("hykkt graph instantiate: ") + cudaGetErrorString(e); return KKT_ERR_CUDA; }
    h->hy_rtol = cg_rtol; h->hy_maxit = cg_maxit; h->hy_outer = max_outer_refine; h->hy_krylov = krylov;
    h->hy_W = h->Wv; h->hy_J = h->Jv; h->hy_Sx = h->Sx; h->hy_gamma = h->gamma; h->hy_dw = h->dw;
  }
  const size_t nb = (size_t)P.batch * P.n * sizeof(double), mb = (size_t)P.batch * P.m_eq * sizeof(double);
  CUDA_TRY(cudaMemcpyAsync(h->g_r1, rbar1, nb, cudaMemcpyDeviceToDevice, h->stream));
  CUDA_TRY(cudaMemcpyAsync(h->g_r2, rbar2, mb, cudaMemcpyDeviceToDevice, h->stream));
  CUDA_TRY(cudaGraphLaunch(h->hy_exec, h->stream));
  CUDA_TRY(cudaMemcpyAsync(dx, h->g_dx, nb, cudaMemcpyDeviceToDevice, h->stream));
  CUDA_TRY(cudaMemcpyAsync(dy, h->g_dy, mb, cudaMemcpyDeviceToDevice, h->stream));
  h->launches = h->hy_fixed;
  h->hy_pending = true;
  h->last_hykkt = true;
  return KKT_OK;
}

extern "C" kkt_status kkt_solve_unreduced(kkt_handle h, const double* x, const double* s, const double* u,
                                          const double* v, const double* f1, const double* f2, const double* f3,
                                          const double* f4, const double* f5, const double* f6, double* dx,
                                          double* ds, double* dy, double* dz, double* du, double* dv,
                                          int max_refine, double tol) {
  if (!h || !x || !u || !f1 || !f5 || !dx || !du) return KKT_ERR_ARG;
  if (!h->factored) { g_err = "kkt_factor first"; return KKT_ERR_STATE; }
  if (h->Dov) { g_err = "kkt_solve_unreduced needs the Sigma_s form of kkt_condense (no D override)"; return KKT_ERR_STATE; }
  const Plan& P = h->P;
  const int me = P.m_eq, mi = P.m - P.m_eq;
  if (mi > 0 && (!s || !v || !f2 || !f4 || !f6 || !ds || !dz || !dv)) return KKT_ERR_ARG;
  if (me > 0 && (!f3 || !dy)) return KKT_ERR_ARG;
  max_refine = std::max(0, max_refine);
  if (tol <= 0) tol = 1e-14;
  const size_t B = P.batch;
  K3Ctx& K = h->k3;
  K.x = x; K.s = s; K.u = u; K.v = v;
  K.f1 = f1; K.f2 = f2; K.f3 = f3; K.f4 = f4; K.f5 = f5; K.f6 = f6;
  K.dx = dx; K.ds = ds; K.dy = dy; K.dz = dz; K.du = du; K.dv = dv;
  K.dw = h->dw; K.dc = h->dc; K.Ss = h->Ss;
  cudaStream_t st = h->stream;
  CUDA_TRY(cudaMemsetAsync(dx, 0, B * P.n * 8, st));
  CUDA_TRY(cudaMemsetAsync(du, 0, B * P.n * 8, st));
  if (mi > 0) {
    CUDA_TRY(cudaMemsetAsync(ds, 0, B * mi * 8, st));
    CUDA_TRY(cudaMemsetAsync(dz, 0, B * mi * 8, st));
    CUDA_TRY(cudaMemsetAsync(dv, 0, B * mi * 8, st));
  }
  if (me > 0) CUDA_TRY(cudaMemsetAsync(dy, 0, B * me * 8, st));
  long long launches = 0;
  k3_init_kernel<<<(P.batch + 127) / 128, 128, 0, h->ls>>>(P.batch, K);
  LAUNCH_CHECK();
  launches++;
  for (int sw = 0; sw <= max_refine; sw++) {
    if (P.m > 0) {
      k3_rows_kernel<<<grid_for((long long)P.batch * P.m, 256, h->sms), 256, 0, h->ls>>>(h->dp, h->Jv, K);
      LAUNCH_CHECK();
      launches++;
    }
    k3_cols_kernel<<<grid_for((long long)P.batch * P.n, 256, h->sms), 256, 0, h->ls>>>(h->dp, h->Wv, h->Jv, K);
    LAUNCH_CHECK();
    launches++;
    if (me == 0) {
      h->launches = 0;
      TRY(launch_solve(h, K.c1, P.n, K.ex, P.n, K.done));
      launches += h->launches;
    } else {
      TRY(hykkt_solve_krylov(h, K.c1, K.r3, K.ex, K.ey, 1e-12, 0, 2, 0));
      long long nl = 0;
      kkt_launch_count(h, &nl);   // (blocking for the HyKKT graph count; K3 on HyKKT is host-synchronous)
      launches += nl;
    }
    k3_update_rows_kernel<<<grid_2d(std::max(P.m, 1), P.batch, h->sms), 256, 0, h->ls>>>(h->dp, h->Jv, K);
    LAUNCH_CHECK();
    k3_update_cols_kernel<<<grid_2d(P.n, P.batch, h->sms), 256, 0, h->ls>>>(h->dp, K);
    LAUNCH_CHECK();
    k3_decide_kernel<<<(P.batch + 127) / 128, 128, 0, h->ls>>>(P.batch, K, tol, max_refine + 1, h->status);
    LAUNCH_CHECK();
    launches += 3;
  }
  k3_finish_kernel<<<(P.batch + 127) / 128, 128, 0, h->ls>>>(P.batch, K, h->C.refine_iters);
  LAUNCH_CHECK();
  h->launches = launches + 1;
  h->graph_solve_pending = false;
  h->hy_pending = false;
  h->last_hykkt = false;
  return KKT_OK;
}

extern "C" kkt_status hykkt_solve(kkt_handle h, const double* rbar1, const double* rbar2, double* dx,
                                  double* dy, double cg_rtol, int cg_maxit, int max_outer_refine) {
  return hykkt_solve_krylov(h, rbar1, rbar2, dx, dy, cg_rtol, cg_maxit, max_outer_refine, 0);
}

extern "C" kkt_status kkt_sync_info(kkt_handle h, int* status, int* fail_col, int* refine_iters,
                                    int* cg_iters, double* bwd_err) {
  if (!h) return KKT_ERR_ARG;
  if (!h->bound) { g_err = "not bound"; return KKT_ERR_STATE; }
  const Plan& P = h->P;
  int st = 0, fl = INT_MAX;
  std::vector<int> it(P.batch), cg(P.batch);
  std::vector<double> om(P.batch);
  CUDA_TRY(cudaMemcpyAsync(&st, h->status, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(cudaMemcpyAsync(&fl, h->fail, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(cudaMemcpyAsync(it.data(), h->last_hykkt ? h->C.opass : h->C.refine_iters, P.batch * sizeof(int),
                           cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(cudaMemcpyAsync(cg.data(), h->C.cg_iters_first, P.batch * sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(cudaMemcpyAsync(om.data(), h->C.omega_last, P.batch * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  int zero = 0, big = INT_MAX;
  CUDA_TRY(cudaMemcpyAsync(h->status, &zero, sizeof(int), cudaMemcpyHostToDevice, h->stream));
  CUDA_TRY(cudaMemcpyAsync(h->fail, &big, sizeof(int), cudaMemcpyHostToDevice, h->stream));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  if (fl != INT_MAX && st == 0) st = h->ldlt ? KKT_ERR_NONFINITE : KKT_ERR_NOT_SPD;
  if (status) *status = st;
  if (fail_col) *fail_col = (fl != INT_MAX) ? P.perm[fl] : -1;
  if (refine_iters) *refine_iters = *std::max_element(it.begin(), it.end());
  if (cg_iters) *cg_iters = *std::max_element(cg.begin(), cg.end());
  if (bwd_err) *bwd_err = *std::max_element(om.begin(), om.end());
  return KKT_OK;
}

extern "C" kkt_status kkt_inertia(kkt_handle h, int* counts) {
  if (!h || !counts) return KKT_ERR_ARG;
  if (!h->ldlt) { g_err = "kkt_inertia needs factor_kind = 1 (LDL^T)"; return KKT_ERR_STATE; }
  if (!h->factored) { g_err = "kkt_factor first"; return KKT_ERR_STATE; }
  CUDA_TRY(cudaMemcpyAsync(counts, h->inert, 3 * sizeof(int) * h->P.batch, cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  return KKT_OK;
}

extern "C" kkt_status kkt_factor_inertia_correct(kkt_handle h, const double* W_vals, const double* J_vals,
                                                 const double* Sigma_x, const double* Sigma_s, const double* D,
                                                 double delta_c, double gamma, const double* params,
                                                 double* delta_w_out, int* tries_out) {
  if (!h || !delta_w_out) return KKT_ERR_ARG;
  if (!h->bound) { g_err = "kkt_bind first"; return KKT_ERR_STATE; }
  // Wachter & Biegler (2006) inertia correction, primal part: defaults of IPOPT
  double dw_min = 1e-20, dw_first = 1e-4, dw_max = 1e40, k_minus = 1.0 / 3.0, k_plus = 8.0, k_plus_bar = 100.0;
  double dw_last = 0.0;
  if (params) {
    dw_min = params[0]; dw_first = params[1]; dw_max = params[2];
    k_minus = params[3]; k_plus = params[4]; k_plus_bar = params[5]; dw_last = params[6];
  }
  const Plan& P = h->P;
  std::vector<int> cnt(3 * P.batch);
  auto correct = [&](bool* ok) -> kkt_status {  // target inertia of the condensed matrix: (n, 0, 0)
    int st = 0, fc = -1;
    TRY(kkt_sync_info(h, &st, &fc, nullptr, nullptr, nullptr));
    if (h->ldlt) {
      TRY(kkt_inertia(h, cnt.data()));
      bool good = (st == 0);
      for (int b = 0; b < P.batch; b++) good = good && cnt[3 * b] == P.n && cnt[3 * b + 1] == 0 && cnt[3 * b + 2] == 0;
      *ok = good;
    } else {
      if (st != 0 && st != KKT_ERR_NOT_SPD) return (kkt_status)st;
      *ok = (st == 0);   // LL^T: K is SPD iff no pivot failed
    }
    return KKT_OK;
  };
  int tries = 0;
  double dw = 0.0;
  bool ok = false;
  TRY(kkt_condense(h, W_vals, J_vals, Sigma_x, Sigma_s, D, 0.0, delta_c, gamma));  // IC-1: delta_w = 0
  TRY(kkt_factor(h));
  tries++;
  TRY(correct(&ok));
  if (!ok) {
    dw = (dw_last == 0.0) ? dw_first : std::max(dw_min, k_minus * dw_last);       // IC-3
    for (;;) {
      TRY(kkt_condense(h, W_vals, J_vals, Sigma_x, Sigma_s, D, dw, delta_c, gamma));  // IC-4
      TRY(kkt_factor(h));
      tries++;
      TRY(correct(&ok));
      if (ok) break;
      dw = (dw_last == 0.0) ? k_plus_bar * dw : k_plus * dw;                         // IC-5
      if (dw > dw_max) { *delta_w_out = dw; if (tries_out) *tries_out = tries; g_err = "inertia correction: delta_w > max"; return KKT_ERR_NOT_SPD; }
    }
  }
  *delta_w_out = dw;
  if (tries_out) *tries_out = tries;
  return KKT_OK;
}

extern "C" kkt_status kkt_step_host(kkt_handle h, const double* W_vals, const double* J_vals,
                                    const double* Sigma_x, const double* Sigma_s, const double* D,
                                    double delta_w, double delta_c, double gamma, const double* b,
                                    double* x, int max_refine, double tol_bwd) {
  if (!h || !b || !x || !Sigma_x) return KKT_ERR_ARG;
  if (!h->bound) { g_err = "kkt_bind first"; return KKT_ERR_STATE; }
  const Plan& P = h->P;
  size_t B = P.batch;
  if (!h->hb) {
    CUDA_TRY(cudaMalloc(&h->hW, std::max<size_t>(1, B * P.nnzW) * 8));
    CUDA_TRY(cudaMalloc(&h->hJ, std::max<size_t>(1, B * P.nnzJ) * 8));
    CUDA_TRY(cudaMalloc(&h->hSx, B * P.n * 8));
    CUDA_TRY(cudaMalloc(&h->hSs, std::max<size_t>(1, B * (P.m - P.m_eq)) * 8));
    CUDA_TRY(cudaMalloc(&h->hD, std::max<size_t>(1, B * P.m) * 8));
    CUDA_TRY(cudaMalloc(&h->hb, B * P.n * 8));
    CUDA_TRY(cudaMalloc(&h->hx, B * P.n * 8));
  }
  if (!h->hcopy) {
    CUDA_TRY(cudaStreamCreateWithFlags(&h->hcopy, cudaStreamNonBlocking));
    for (auto& e : h->hev) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  cudaStream_t s = h->stream;
  if (P.nnzW) CUDA_TRY(cudaMemcpyAsync(h->hW, W_vals, B * P.nnzW * 8, cudaMemcpyHostToDevice, s));
  if (P.nnzJ) CUDA_TRY(cudaMemcpyAsync(h->hJ, J_vals, B * P.nnzJ * 8, cudaMemcpyHostToDevice, s));
  CUDA_TRY(cudaMemcpyAsync(h->hSx, Sigma_x, B * P.n * 8, cudaMemcpyHostToDevice, s));
  if (Sigma_s && P.m > P.m_eq)
    CUDA_TRY(cudaMemcpyAsync(h->hSs, Sigma_s, B * (P.m - P.m_eq) * 8, cudaMemcpyHostToDevice, s));
  if (D && P.m) CUDA_TRY(cudaMemcpyAsync(h->hD, D, B * P.m * 8, cudaMemcpyHostToDevice, s));
  // b is needed only by the solve: its upload runs on the copy stream while the handle's stream
  // condenses and factorises (after the matrix uploads, so it does not share the link with them)
  CUDA_TRY(cudaEventRecord(h->hev[0], s));
  CUDA_TRY(cudaStreamWaitEvent(h->hcopy, h->hev[0], 0));
  CUDA_TRY(cudaMemcpyAsync(h->hb, b, B * P.n * 8, cudaMemcpyHostToDevice, h->hcopy));
  CUDA_TRY(cudaEventRecord(h->hev[1], h->hcopy));
  TRY(kkt_condense(h, h->hW, h->hJ, h->hSx, Sigma_s ? h->hSs : nullptr, D ? h->hD : nullptr, delta_w, delta_c, gamma));
  TRY(kkt_factor(h));
  CUDA_TRY(cudaStreamWaitEvent(s, h->hev[1], 0));
  TRY(kkt_solve(h, h->hb, h->hx, max_refine, tol_bwd));
  CUDA_TRY(cudaMemcpyAsync(x, h->hx, B * P.n * 8, cudaMemcpyDeviceToHost, s));
  CUDA_TRY(cudaStreamSynchronize(s));
  return KKT_OK;
}

extern "C" kkt_status kkt_recover(kkt_handle h, const double* r2, const double* r4, const double* dx,
                                   double* dz, double* ds) {
  if (!h || !dx) return KKT_ERR_ARG;
  if (!h->condensed) { g_err = "kkt_condense first"; return KKT_ERR_STATE; }
  if (h->Dov) { g_err = "kkt_recover needs the Sigma_s form of kkt_condense (no D override)"; return KKT_ERR_STATE; }
  const Plan& P = h->P;
  const long long tot = (long long)P.batch * (P.m - P.m_eq);
  if (tot == 0) return KKT_OK;
  if (!r2 || !r4 || !dz || !ds) return KKT_ERR_ARG;
  recover_kernel<<<grid_for(tot, 256, h->sms), 256, 0, h->ls>>>(h->dp, h->Jv, h->Ss, h->dw, h->dc, r2, r4,
                                                                  dx, dz, ds);
  LAUNCH_CHECK();
  h->launches = 1;
  return KKT_OK;
}

extern "C" kkt_status kkt_recover_bounds(kkt_handle h, const double* x, const double* u, const double* s,
                                          const double* v, double mu, const double* dx, const double* ds,
                                          double* du, double* dv) {
  if (!h || !x || !u || !dx || !du) return KKT_ERR_ARG;
  if (!h->bound) { g_err = "kkt_bind first"; return KKT_ERR_STATE; }
  const Plan& P = h->P;
  const long long nx = (long long)P.batch * P.n, ns = (long long)P.batch * (P.m - P.m_eq);
  if (ns > 0 && (!s || !v || !ds || !dv)) return KKT_ERR_ARG;
  recover_bounds_kernel<<<grid_for(nx + ns, 256, h->sms), 256, 0, h->ls>>>(nx, ns, x, u, s, v, mu, dx, ds,
                                                                            du, dv);
  LAUNCH_CHECK();
  h->launches = 1;
  return KKT_OK;
}

extern "C" kkt_status kkt_get_condensed(kkt_handle h, int inst, int* Kp, int* Ki, double* Kv) {
  if (!h) return KKT_ERR_ARG;
  const Plan& P = h->P;
  if (inst < 0 || inst >= P.batch) return KKT_ERR_ARG;
  const int n = P.n, nnz = P.Kp[n];
  std::vector<double> v(nnz);
  if (Kv) {
    if (!h->condensed) { g_err = "kkt_condense first"; return KKT_ERR_STATE; }
    CUDA_TRY(cudaMemcpyAsync(v.data(), h->Kv + (size_t)inst * nnz, nnz * sizeof(double),
                             cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(cudaStreamSynchronize(h->stream));
  }
  // internal (i, j) -> original lower (max, min), CSC sorted
  std::vector<int> cnt(n + 1, 0);
  for (int j = 0; j < n; j++)
    for (int p = P.Kp[j]; p < P.Kp[j + 1]; p++) {
      int a = P.perm[P.Ki[p]], c = P.perm[j];
      cnt[std::min(a, c) + 1]++;
    }
  for (int j = 0; j < n; j++) cnt[j + 1] += cnt[j];
  std::vector<std::pair<int, int>> ent(nnz);  // (row, internal p) per orig column slot
  std::vector<int> f(cnt.begin(), cnt.end() - 1);
  for (int j = 0; j < n; j++)
    for (int p = P.Kp[j]; p < P.Kp[j + 1]; p++) {
      int a = P.perm[P.Ki[p]], c = P.perm[j];
      ent[f[std::min(a, c)]++] = {std::max(a, c), p};
    }
  for (int j = 0; j < n; j++) std::sort(ent.begin() + cnt[j], ent.begin() + cnt[j + 1]);
  if (Kp) std::memcpy(Kp, cnt.data(), (n + 1) * sizeof(int));
  for (int q = 0; q < nnz; q++) {
    if (Ki) Ki[q] = ent[q].first;
    if (Kv) Kv[q] = v[ent[q].second];
  }
  return KKT_OK;
}

extern "C" kkt_status kkt_get_supernodes(kkt_handle h, int* nsuper, int* sn_first, int* sn_nrows,
                                         int* sn_parent) {
  if (!h) return KKT_ERR_ARG;
  const Plan& P = h->P;
  if (nsuper) *nsuper = P.ns;
  for (int s = 0; s < P.ns; s++) {
    if (sn_first) sn_first[s] = P.sn_first[s];
    if (sn_nrows) sn_nrows[s] = P.sn_rp[s + 1] - P.sn_rp[s];
    if (sn_parent) sn_parent[s] = P.sn_parent[s];
  }
  if (sn_first) sn_first[P.ns] = P.n;
  return KKT_OK;
}

extern "C" kkt_status kkt_get_blocks(kkt_handle h, int kind, int cap, int nwarps, int* nblk, int* nmeta,
                                     int* blk, int* blk_of, int* meta, int* lrow, int* is_big) {
  if (!h || (kind != 0 && kind != 1) || cap <= 0 || nwarps <= 0) return KKT_ERR_ARG;
  const Plan& P = h->P;
  if (is_big)
    for (int s = 0; s < P.ns; s++) is_big[s] = P.sn[s].big;
  if (kind == 0) {
    SBlockHost H;
    build_sblocks(P, cap, nwarps, H);
    if (nblk) *nblk = (int)H.blk.size();
    if (nmeta) *nmeta = (int)H.meta.size();
    for (size_t q = 0; blk && q < H.blk.size(); q++) {
      const SBlk& B = H.blk[q];
      const int v[8] = {B.s_lo, B.s_hi, B.nlev, B.m0, sb_layout(B.s_hi - B.s_lo + 1, B.nlev, B.nL, B.ncol, B.nr,
                                                               B.nch, B.Rroot, nwarps).total, 0, 0, 0};
      std::copy(v, v + 8, blk + 8 * q);
    }
    if (blk_of) std::copy(H.blk_of.begin(), H.blk_of.end(), blk_of);
    if (meta) std::copy(H.meta.begin(), H.meta.end(), meta);
    if (lrow) std::copy(H.lrow.begin(), H.lrow.end(), lrow);
  } else {
    FBlockHost H;
    build_fblocks(P, cap, H);
    if (nblk) *nblk = (int)H.blk.size();
    if (nmeta) *nmeta = (int)H.meta.size();
    for (size_t q = 0; blk && q < H.blk.size(); q++) {
      const FBlk& B = H.blk[q];
      const int v[8] = {B.s_lo, B.s_hi, B.nlev, B.m0, fb_layout(B.s_hi - B.s_lo + 1, B.nlev, B.nL, B.nU, B.nK, B.nr,
                                                               B.nch).total, 0, 0, 0};
      std::copy(v, v + 8, blk + 8 * q);
    }
    if (blk_of) {
      std::fill(blk_of, blk_of + P.ns, -1);
      for (size_t q = 0; q < H.blk.size(); q++) {
        for (int t = H.blk[q].s_lo; t < H.blk[q].s_hi; t++) blk_of[t] = -2;
        blk_of[H.blk[q].s_hi] = (int)q;
      }
    }
    if (meta) std::copy(H.meta.begin(), H.meta.end(), meta);
  }
  return KKT_OK;
}

extern "C" kkt_status kkt_get_trace(kkt_handle h, long long* stamps) {
  if (!h || !stamps) return KKT_ERR_ARG;
  if (!h->trace_buf) { g_err = "tracing disabled: set KKT_TRACE=1 before kkt_bind"; return KKT_ERR_STATE; }
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  CUDA_TRY(cudaMemcpy(stamps, h->trace_buf, (size_t)3 * h->P.ns * KKT_TRACE_SLOTS * sizeof(long long), cudaMemcpyDeviceToHost));
  return KKT_OK;
}

extern "C" kkt_status kkt_launch_count(kkt_handle h, long long* launches) {
  if (!h || !launches) return KKT_ERR_ARG;
  if (h->graph_solve_pending && h->g_body > 0) {  // a graph solve: add its executed conditional body
    int sw = 0;
    CUDA_TRY(cudaStreamSynchronize(h->stream));
    CUDA_TRY(cudaMemcpy(&sw, h->C.sweep, sizeof(int), cudaMemcpyDeviceToHost));
    if (h->solve_while) h->launches = h->g_pro + h->g_body * std::max(0, sw - (h->g_max_refine >= 1 ? 2 : 1));
    else h->launches = h->g_pro + (sw > 2 ? h->g_body : 0);  // IF body: all of sweeps 2.. or none
    h->graph_solve_pending = false;
  }
  if (h->hy_pending) {  // HyKKT graph: add the executed Krylov bodies
    int runs = 0;
    CUDA_TRY(cudaStreamSynchronize(h->stream));
    CUDA_TRY(cudaMemcpy(&runs, h->C.cg_runs, sizeof(int), cudaMemcpyDeviceToHost));
    h->launches = h->hy_fixed + h->hy_body * runs;
    h->hy_pending = false;
  }
  *launches = h->launches;
  return KKT_OK;
}

extern "C" kkt_status kkt_hykkt_stats(kkt_handle h, int* krylov_total, int* outer_passes) {
  if (!h) return KKT_ERR_ARG;
  if (!h->last_hykkt) { g_err = "the last solve was not hykkt_solve"; return KKT_ERR_STATE; }
  const Plan& P = h->P;
  int runs = 0;
  std::vector<int> op(P.batch);
  CUDA_TRY(cudaMemcpyAsync(&runs, h->C.cg_runs, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(cudaMemcpyAsync(op.data(), h->C.opass, P.batch * sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  CUDA_TRY(cudaStreamSynchronize(h->stream));
  if (krylov_total) *krylov_total = runs;
  if (outer_passes) *outer_passes = *std::max_element(op.begin(), op.end());
  return KKT_OK;
}

extern "C" kkt_status kkt_destroy(kkt_handle h) {
  if (!h) return KKT_ERR_ARG;
  release_device(h);
  delete h;
  return KKT_OK;
}

// tracing aid: per-task stamps of the tile-task factorisation (KKT_TRACE=1 at kkt_bind)
extern "C" int kkt_tile_trace(kkt_handle h, long long* trace, int* tasks, int n, double* est_us) {
  if (!h || !h->tiles || !h->tile_mem) return -1;
  if (est_us) *est_us = h->tile_est_us;
  const int nt = h->tp.ntask;
  n = std::min(n, nt);
  if (cudaStreamSynchronize(h->stream) != cudaSuccess) return -2;
  if (tasks && n > 0 && cudaMemcpy(tasks, h->tp.tasks, (size_t)n * 16, cudaMemcpyDeviceToHost) != cudaSuccess) return -2;
  if (trace && n > 0) {
    if (!h->tile_trace) return -1;
    if (cudaMemcpy(trace, h->tile_trace, (size_t)n * 32, cudaMemcpyDeviceToHost) != cudaSuccess) return -2;
  }
  return nt;
}

// tracing aid: the same for the tile-task solve of the last solve launch (which = 1)
extern "C" int kkt_tile_solve_trace(kkt_handle h, long long* trace, int* tasks, int n, double* est_us) {
  if (!h || !h->tsolve || !h->ts_mem) return -1;
  if (est_us) *est_us = h->ts_est_us;
  const int nt = h->tsp.ntask;
  n = std::min(n, nt);
  if (cudaStreamSynchronize(h->stream) != cudaSuccess) return -2;
  if (tasks && n > 0 && cudaMemcpy(tasks, h->tsp.tasks, (size_t)n * 16, cudaMemcpyDeviceToHost) != cudaSuccess) return -2;
  if (trace && n > 0) {
    if (!h->ts_trace) return -1;
    if (cudaMemcpy(trace, h->ts_trace, (size_t)n * 32, cudaMemcpyDeviceToHost) != cudaSuccess) return -2;
  }
  return nt;
}

// debugging aid (not part of the public header): per-step stamps of the root front, KKT_TRACE=2
extern "C" int kkt_debug_steps(kkt_handle h, long long* out, int n) {
  if (!h || !h->dbg_buf) return -1;
  n = std::min(n, 4096 * 8);
  return cudaMemcpy(out, h->dbg_buf, (size_t)n * sizeof(long long), cudaMemcpyDeviceToHost) == cudaSuccess ? 0 : -2;
}
