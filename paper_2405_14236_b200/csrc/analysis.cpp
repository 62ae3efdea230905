// analysis.cpp -- once-per-pattern host analysis ("analysis phase"; reported
// separately from the timed numeric path).
//
//   1. pattern(K) = pattern(W) U pattern(J^T J) U diag
//   2. MD-exact-v1 ordering (R11): quotient graph with elements, exact degrees,
//      mass elimination only of provably indistinguishable vertices (see md_exact_v1)
//   3. etree (Liu's ancestor algorithm) and column counts (row-subtree traversal)
//   4. etree postorder -> internal numbering; fundamental supernodes + relaxed amalgamation
//   5. supernode row structures, multifrontal relative-index maps, level schedule
//   6. condensation gather map (products of J^T D J per K entry; deterministic, R16)
//   7. operator maps for the double-double residual (full W, J^T, G^T)
#include "plan.h"

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <queue>
#include <tuple>

namespace kkt {

// =====================================================================================
// MD-exact-v1.  Rule (R11): repeatedly eliminate the vertex v minimising (deg(v), v), where
// deg(v) = number of uneliminated vertices adjacent to v in the current elimination graph.
//
// Representation: quotient graph of supervariables (sets of vertices proven to have equal
// closed neighbourhoods) and elements (eliminated cliques).  For a supervariable i:
//   Reach(i) = (avar[i] U  U_{e in aelm[i]} le[e]) \ {i},
//   deg(i)   = nv[i] - 1 + sum_{j in Reach(i)} nv[j]          (exact, per member vertex)
// The chosen vertex is the smallest-index member of the supervariable minimising
// (deg, minidx).  After eliminating v the only vertices of degree deg(v)-1 are those
// indistinguishable from v, so the rule eliminates v's whole indistinguishable class S* next,
// in increasing index order.  At selection time S* is completed exactly: every supervariable
// q in Reach(p) with deg(q) = deg(p) and Reach(q) subset of Reach(p) U {p} joins p.  Hence mass
// elimination reproduces the one-vertex-at-a-time rule exactly.  Supervariable detection
// after each step (identical quotient adjacency) is sound and only saves work.
// =====================================================================================
void md_exact_v1(int n, const std::vector<int>& adjp, const std::vector<int>& adji,
                 std::vector<int>& perm) {
  perm.clear();
  perm.reserve(n);
  std::vector<std::vector<int>> avar(n), aelm(n), le(n), mem(n);
  std::vector<int> nv(n, 1), minidx(n), deg(n);
  std::vector<char> valive(n, 1), ealive(n, 0);
  std::vector<int> mark(n, 0), mark2(n, 0);
  int stamp = 0, stamp2 = 0;
  for (int v = 0; v < n; v++) {
    avar[v].assign(adji.begin() + adjp[v], adji.begin() + adjp[v + 1]);
    deg[v] = (int)avar[v].size();
    minidx[v] = v;
    mem[v].push_back(v);
  }
  typedef std::tuple<int, int, int> Key;  // (deg, minidx, rep)
  std::priority_queue<Key, std::vector<Key>, std::greater<Key>> heap;
  for (int v = 0; v < n; v++) heap.emplace(deg[v], minidx[v], v);

  auto reach_scan = [&](int i, auto&& f) {
    for (int x : avar[i])
      if (valive[x] && x != i) f(x);
    for (int e : aelm[i]) {
      if (!ealive[e]) continue;
      auto& L = le[e];
      // compact dead variables in place (dead is permanent)
      size_t w = 0;
      for (size_t t = 0; t < L.size(); t++)
        if (valive[L[t]]) L[w++] = L[t];
      L.resize(w);
      for (int x : L)
        if (x != i) f(x);
    }
  };

  std::vector<int> R, Lp, members;
  std::vector<std::pair<long long, int>> hashes;
  int eliminated = 0;
  while (eliminated < n) {
    Key k = heap.top();
    heap.pop();
    int p = std::get<2>(k);
    if (!valive[p] || deg[p] != std::get<0>(k) || minidx[p] != std::get<1>(k)) continue;

    // ---- Reach(p) ----
    ++stamp;
    R.clear();
    mark[p] = stamp;
    reach_scan(p, [&](int x) {
      if (mark[x] != stamp) { mark[x] = stamp; R.push_back(x); }
    });
    // ---- complete the indistinguishable class S* ----
    std::vector<int> absorbed_elems(aelm[p].begin(), aelm[p].end());
    for (int q : R) {
      if (!valive[q] || deg[q] != deg[p]) continue;
      bool ok = true;
      reach_scan(q, [&](int x) {
        if (ok && x != p && mark[x] != stamp) ok = false;
      });
      if (!ok) continue;
      // q is indistinguishable from p: merge
      valive[q] = 0;
      nv[p] += nv[q];
      minidx[p] = std::min(minidx[p], minidx[q]);
      mem[p].insert(mem[p].end(), mem[q].begin(), mem[q].end());
      for (int e : aelm[q]) absorbed_elems.push_back(e);
      std::vector<int>().swap(mem[q]);
      std::vector<int>().swap(avar[q]);
      std::vector<int>().swap(aelm[q]);
    }
    // ---- emit the class in increasing index order ----
    members = mem[p];
    std::sort(members.begin(), members.end());
    for (int v : members) perm.push_back(v);
    eliminated += (int)members.size();
    // ---- new element e = p with le[p] = alive part of R ----
    Lp.clear();
    for (int x : R)
      if (valive[x]) Lp.push_back(x);
    valive[p] = 0;
    for (int e : absorbed_elems)
      if (e != p) { ealive[e] = 0; std::vector<int>().swap(le[e]); }
    std::vector<int>().swap(avar[p]);
    std::vector<int>().swap(aelm[p]);
    std::vector<int>().swap(mem[p]);
    le[p] = Lp;
    ealive[p] = 1;
    // ---- prune adjacency of the variables in Lp ----
    ++stamp2;
    for (int x : Lp) mark2[x] = stamp2;
    for (int i : Lp) {
      auto& A = avar[i];
      size_t w = 0;
      for (size_t t = 0; t < A.size(); t++) {
        int x = A[t];
        if (valive[x] && mark2[x] != stamp2) A[w++] = x;  // vars in Lp are covered by element p
      }
      A.resize(w);
      auto& E = aelm[i];
      w = 0;
      for (size_t t = 0; t < E.size(); t++)
        if (ealive[E[t]]) E[w++] = E[t];
      E.resize(w);
      E.push_back(p);
    }
    // ---- sound supervariable detection among Lp (identical quotient adjacency) ----
    if (Lp.size() > 1) {
      hashes.clear();
      for (int i : Lp) {
        std::sort(avar[i].begin(), avar[i].end());
        std::sort(aelm[i].begin(), aelm[i].end());
        long long h = (long long)avar[i].size() * 1000003LL + (long long)aelm[i].size();
        for (int x : avar[i]) h = h * 31 + x;
        for (int e : aelm[i]) h = h * 37 + e;
        hashes.emplace_back(h, i);
      }
      std::sort(hashes.begin(), hashes.end());
      for (size_t a = 0; a < hashes.size();) {
        size_t b = a;
        while (b < hashes.size() && hashes[b].first == hashes[a].first) b++;
        for (size_t s = a; s < b; s++) {
          int i = hashes[s].second;
          if (!valive[i]) continue;
          for (size_t t = s + 1; t < b; t++) {
            int j = hashes[t].second;
            if (!valive[j]) continue;
            if (avar[i] == avar[j] && aelm[i] == aelm[j]) {
              valive[j] = 0;
              nv[i] += nv[j];
              minidx[i] = std::min(minidx[i], minidx[j]);
              mem[i].insert(mem[i].end(), mem[j].begin(), mem[j].end());
              std::vector<int>().swap(mem[j]);
              std::vector<int>().swap(avar[j]);
              std::vector<int>().swap(aelm[j]);
            }
          }
        }
        a = b;
      }
    }
    // ---- exact degrees of the variables in Lp ----
    for (int i : Lp) {
      if (!valive[i]) continue;
      ++stamp;
      mark[i] = stamp;
      long long d = nv[i] - 1;
      reach_scan(i, [&](int x) {
        if (mark[x] != stamp) { mark[x] = stamp; d += nv[x]; }
      });
      deg[i] = (int)d;
      heap.emplace(deg[i], minidx[i], i);
    }
  }
}

// =====================================================================================
namespace {

double now_ms() {
  return std::chrono::duration<double, std::milli>(
             std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

std::string analyze(int n, int m, int m_eq, const int* Wp, const int* Wc, const int* Jp,
                    const int* Jc, const Options& opt, Plan& P, int* code) {
  double t0 = now_ms();
  *code = 1;
  if (n < 0 || m < 0 || m_eq < 0 || m_eq > m) return "bad sizes";
  if (!Wp || (!Jp && m > 0)) return "null pattern pointer";
  *code = 2;
  P = Plan();
  P.n = n; P.m = m; P.m_eq = m_eq; P.batch = std::max(1, opt.batch);
  P.factor_kind = opt.factor_kind;
  P.nnzW = Wp[n];
  P.nnzJ = m ? Jp[m] : 0;
  if (Wp[0] != 0 || (m && Jp[0] != 0)) return "rowptr[0] != 0";
  for (int i = 0; i < n; i++) {
    if (Wp[i + 1] < Wp[i]) return "W rowptr not monotone";
    for (int p = Wp[i]; p < Wp[i + 1]; p++) {
      int j = Wc[p];
      if (j < 0 || j > i) return "W entry outside lower triangle";
      if (p > Wp[i] && Wc[p - 1] >= j) return "W columns unsorted or duplicate";
    }
  }
  for (int r = 0; r < m; r++) {
    if (Jp[r + 1] < Jp[r]) return "J rowptr not monotone";
    for (int p = Jp[r]; p < Jp[r + 1]; p++) {
      int j = Jc[p];
      if (j < 0 || j >= n) return "J column out of range";
      if (p > Jp[r] && Jc[p - 1] >= j) return "J columns unsorted or duplicate";
    }
  }
  *code = 0;

  // ---------------- 1. symmetric adjacency of pattern(K) (orig numbering) -------------
  // off-diagonal pairs from W and from every J row clique
  std::vector<std::vector<int>> adj(n);
  for (int i = 0; i < n; i++)
    for (int p = Wp[i]; p < Wp[i + 1]; p++)
      if (Wc[p] != i) { adj[i].push_back(Wc[p]); adj[Wc[p]].push_back(i); }
  for (int r = 0; r < m; r++)
    for (int a = Jp[r]; a < Jp[r + 1]; a++)
      for (int b = a + 1; b < Jp[r + 1]; b++) {
        adj[Jc[a]].push_back(Jc[b]);
        adj[Jc[b]].push_back(Jc[a]);
      }
  std::vector<int> adjp(n + 1, 0), adji;
  for (int v = 0; v < n; v++) {
    auto& A = adj[v];
    std::sort(A.begin(), A.end());
    A.erase(std::unique(A.begin(), A.end()), A.end());
    adjp[v + 1] = adjp[v] + (int)A.size();
  }
  adji.resize(adjp[n]);
  for (int v = 0; v < n; v++) {
    std::copy(adj[v].begin(), adj[v].end(), adji.begin() + adjp[v]);
    std::vector<int>().swap(adj[v]);
  }

  // ---------------- 2. ordering -------------------------------------------------------
  double t1 = now_ms();
  if (opt.ordering == 1) {
    P.perm_md.resize(n);
    std::iota(P.perm_md.begin(), P.perm_md.end(), 0);
  } else {
    md_exact_v1(n, adjp, adji, P.perm_md);
  }
  P.order_ms = now_ms() - t1;
  std::vector<int> ipmd(n);
  for (int k = 0; k < n; k++) ipmd[P.perm_md[k]] = k;

  // ---------------- 3. etree (Liu) + column counts (row subtrees), md numbering -------
  // "upper" neighbours of md column k: md indices i < k adjacent to k
  std::vector<int> parent(n, -1), anc(n, -1);
  for (int k = 0; k < n; k++) {
    int v = P.perm_md[k];
    for (int p = adjp[v]; p < adjp[v + 1]; p++) {
      int i = ipmd[adji[p]];
      if (i >= k) continue;
      // climb from i to the root of its current subtree with path compression
      while (i != -1 && i != k) {
        int nx = anc[i];
        anc[i] = k;
        if (nx == -1) { parent[i] = k; break; }
        i = nx;
      }
    }
  }
  std::vector<int> cc(n, 0), rmark(n, -1);
  for (int i = 0; i < n; i++) {
    int v = P.perm_md[i];
    rmark[i] = i;
    cc[i] += 1;  // diagonal
    for (int p = adjp[v]; p < adjp[v + 1]; p++) {
      int k = ipmd[adji[p]];
      if (k >= i) continue;
      while (rmark[k] != i) {  // L_ik != 0 for every k on the path to the marked subtree
        cc[k] += 1;
        rmark[k] = i;
        k = parent[k];
      }
    }
  }
  P.etree_md = parent;
  P.colcount_md = cc;
  P.nnzL = 0;
  P.flops = 0;
  for (int j = 0; j < n; j++) { P.nnzL += cc[j]; P.flops += (double)cc[j] * cc[j]; }

  // ---------------- 4. postorder -> internal numbering --------------------------------
  std::vector<int> chp(n + 1, 0), chl(n);
  for (int j = 0; j < n; j++) if (parent[j] >= 0) chp[parent[j] + 1]++;
  for (int j = 0; j < n; j++) chp[j + 1] += chp[j];
  {
    std::vector<int> f(chp.begin(), chp.end() - 1);
    for (int j = 0; j < n; j++) if (parent[j] >= 0) chl[f[parent[j]]++] = j;  // increasing
  }
  std::vector<int> post(n), stack;  // post[md] = internal
  {
    int cnt = 0;
    std::vector<int> it(n);
    for (int r = 0; r < n; r++) {
      if (parent[r] != -1) continue;
      stack.push_back(r);
      it[r] = chp[r];
      while (!stack.empty()) {
        int v = stack.back();
        if (it[v] < chp[v + 1]) {
          int c = chl[it[v]++];
          it[c] = chp[c];
          stack.push_back(c);
        } else {
          post[v] = cnt++;
          stack.pop_back();
        }
      }
    }
  }
  P.perm.resize(n);
  P.iperm.resize(n);
  std::vector<int> par(n, -1), cnt(n);
  for (int j = 0; j < n; j++) {
    P.perm[post[j]] = P.perm_md[j];
    par[post[j]] = parent[j] < 0 ? -1 : post[parent[j]];
    cnt[post[j]] = cc[j];
  }
  for (int k = 0; k < n; k++) P.iperm[P.perm[k]] = k;

  // ---------------- 5. fundamental supernodes + relaxed amalgamation -----------------
  std::vector<int> nchild(n, 0);
  for (int j = 0; j < n; j++) if (par[j] >= 0) nchild[par[j]]++;
  std::vector<int> sfirst;  // fundamental supernode starts
  for (int j = 0; j < n; j++) {
    bool cont = j > 0 && par[j - 1] == j && cnt[j - 1] == cnt[j] + 1 && nchild[j] == 1;
    if (!cont) sfirst.push_back(j);
  }
  sfirst.push_back(n);
  int nf = (int)sfirst.size() - 1;
  // supernode data for amalgamation: width, count of first column, parent supernode
  std::vector<int> fcol_sn(n);
  for (int s = 0; s < nf; s++)
    for (int j = sfirst[s]; j < sfirst[s + 1]; j++) fcol_sn[j] = s;
  // merge child s into parent p when s's last column + 1 == p's first column (postorder:
  // s is p's last child).  Greedy in increasing s (children before parents).
  std::vector<int> g_first(sfirst.begin(), sfirst.end() - 1), g_width(nf), g_cnt0(nf);
  std::vector<long long> g_zeros(nf, 0);
  std::vector<int> rep(nf);
  for (int s = 0; s < nf; s++) {
    g_width[s] = sfirst[s + 1] - sfirst[s];
    g_cnt0[s] = cnt[sfirst[s]];  // rows of the first column = r_s
    rep[s] = s;
  }
  auto find = [&](int s) { while (rep[s] != s) s = rep[s] = rep[rep[s]]; return s; };
  for (int s = 0; s < nf; s++) {
    int last = sfirst[s + 1] - 1;
    int pj = par[last];
    if (pj < 0 || pj != last + 1) continue;
    int a = find(s), b = find(fcol_sn[pj]);
    if (a == b) continue;
    // merged group: columns of a then b; rows = cols(a) U R_b
    int wa = g_width[a], wb = g_width[b];
    int rb = g_cnt0[b];
    int newr = wa + rb;
    // zeros added: each column t of a had count (g_cnt0[a]-t), now (newr - t)
    long long add = (long long)wa * (newr - g_cnt0[a]);
    long long tot = (long long)(wa + wb) * newr;
    long long zeros = g_zeros[a] + g_zeros[b] + add;
    int W = wa + wb;
    bool ok = W <= opt.relax_small ||
              (W <= opt.relax_big && (double)zeros <= opt.relax_zero_frac * (double)tot);
    if (!ok) continue;
    rep[b] = a;  // keep a as representative
    g_width[a] = W;
    g_cnt0[a] = newr;
    g_zeros[a] = zeros;
    // g_first[a] unchanged (a precedes b)
  }
  std::vector<int> snf;
  for (int s = 0; s < nf; s++)
    if (find(s) == s) snf.push_back(g_first[s]);
  // groups are contiguous column ranges in postorder; collect their starts in order
  std::sort(snf.begin(), snf.end());
  snf.push_back(n);
  P.ns = (int)snf.size() - 1;
  const int ns = P.ns;
  P.sn_first = snf;
  P.col_sn.resize(n);
  for (int s = 0; s < ns; s++)
    for (int j = snf[s]; j < snf[s + 1]; j++) P.col_sn[j] = s;
  P.sn_parent.assign(ns, -1);
  for (int s = 0; s < ns; s++) {
    int last = snf[s + 1] - 1;
    P.sn_parent[s] = par[last] < 0 ? -1 : P.col_sn[par[last]];
  }

  // ---------------- K pattern in internal numbering (lower CSC) ----------------------
  {
    std::vector<int> colcnt(n + 1, 0);
    for (int v = 0; v < n; v++) {
      int j = P.iperm[v];
      colcnt[j + 1]++;  // diagonal
      for (int p = adjp[v]; p < adjp[v + 1]; p++)
        if (P.iperm[adji[p]] > j) colcnt[j + 1]++;
    }
    P.Kp.assign(n + 1, 0);
    for (int j = 0; j < n; j++) P.Kp[j + 1] = P.Kp[j] + colcnt[j + 1];
    P.Ki.resize(P.Kp[n]);
    std::vector<int> f(P.Kp.begin(), P.Kp.end() - 1);
    for (int v = 0; v < n; v++) {
      int j = P.iperm[v];
      P.Ki[f[j]++] = j;
      for (int p = adjp[v]; p < adjp[v + 1]; p++) {
        int i = P.iperm[adji[p]];
        if (i > j) P.Ki[f[j]++] = i;
      }
    }
    for (int j = 0; j < n; j++) std::sort(P.Ki.begin() + P.Kp[j], P.Ki.begin() + P.Kp[j + 1]);
  }

  // ---------------- supernode row structures --------------------------------------
  P.sn_cp.assign(ns + 1, 0);
  for (int s = 0; s < ns; s++) if (P.sn_parent[s] >= 0) P.sn_cp[P.sn_parent[s] + 1]++;
  for (int s = 0; s < ns; s++) P.sn_cp[s + 1] += P.sn_cp[s];
  P.sn_ch.resize(P.sn_cp[ns]);
  {
    std::vector<int> f(P.sn_cp.begin(), P.sn_cp.end() - 1);
    for (int s = 0; s < ns; s++) if (P.sn_parent[s] >= 0) P.sn_ch[f[P.sn_parent[s]]++] = s;
  }
  // children ordered by subtree height (descending): the top-down solve continues with the
  // child on the longest remaining chain and queues the others (critical path first)
  {
    std::vector<int> hsub(ns, 0);
    for (int s = 0; s < ns; s++)
      if (P.sn_parent[s] >= 0) hsub[P.sn_parent[s]] = std::max(hsub[P.sn_parent[s]], hsub[s] + 1);
    for (int s = 0; s < ns; s++)
      std::sort(P.sn_ch.begin() + P.sn_cp[s], P.sn_ch.begin() + P.sn_cp[s + 1], [&](int a, int b) {
        return hsub[a] != hsub[b] ? hsub[a] > hsub[b] : a < b;
      });
    P.sn_hsub = hsub;
  }
  std::vector<std::vector<int>> rows(ns);
  std::vector<int> smark(n, -1);
  P.max_front = 0;
  for (int s = 0; s < ns; s++) {  // children precede parents in postorder
    int f0 = snf[s], f1 = snf[s + 1];
    auto& R = rows[s];
    for (int j = f0; j < f1; j++) { R.push_back(j); smark[j] = s; }
    for (int j = f0; j < f1; j++)
      for (int p = P.Kp[j]; p < P.Kp[j + 1]; p++) {
        int i = P.Ki[p];
        if (smark[i] != s) { smark[i] = s; R.push_back(i); }
      }
    for (int t = P.sn_cp[s]; t < P.sn_cp[s + 1]; t++) {
      int c = P.sn_ch[t];
      int wc = snf[c + 1] - snf[c];
      for (size_t q = wc; q < rows[c].size(); q++) {
        int i = rows[c][q];
        if (smark[i] != s) { smark[i] = s; R.push_back(i); }
      }
    }
    std::sort(R.begin() + (f1 - f0), R.end());
    P.max_front = std::max(P.max_front, (int)R.size());
  }
  P.sn_rp.assign(ns + 1, 0);
  P.sn_Lp.assign(ns + 1, 0);
  P.sn_Up.assign(ns + 1, 0);
  P.sn_uvp.assign(ns + 1, 0);
  for (int s = 0; s < ns; s++) {
    long long r = (long long)rows[s].size(), w = snf[s + 1] - snf[s], R = r - w;
    P.sn_rp[s + 1] = P.sn_rp[s] + (int)r;
    P.sn_Lp[s + 1] = P.sn_Lp[s] + r * w;
    P.sn_Up[s + 1] = P.sn_Up[s] + (P.sn_parent[s] >= 0 ? R * (R + 1) / 2 : 0);
    P.sn_uvp[s + 1] = P.sn_uvp[s] + R;
  }
  if (P.sn_uvp[ns] >= (1LL << 31)) { *code = 2; return "update vectors exceed int32 offsets"; }
  P.nnzL_stored = P.sn_Lp[ns];
  P.update_doubles = P.sn_Up[ns];
  P.uvec_doubles = P.sn_uvp[ns];
  P.sn_rows.resize(P.sn_rp[ns]);
  P.sn_rel.assign(P.sn_rp[ns], -1);
  for (int s = 0; s < ns; s++)
    std::copy(rows[s].begin(), rows[s].end(), P.sn_rows.begin() + P.sn_rp[s]);
  {
    std::vector<int> pos(n, -1);
    for (int p = 0; p < ns; p++) {
      const int* Rp = &P.sn_rows[P.sn_rp[p]];
      int rp = P.sn_rp[p + 1] - P.sn_rp[p];
      for (int t = 0; t < rp; t++) pos[Rp[t]] = t;
      for (int q = P.sn_cp[p]; q < P.sn_cp[p + 1]; q++) {
        int c = P.sn_ch[q];
        int wc = snf[c + 1] - snf[c];
        for (int t = P.sn_rp[c] + wc; t < P.sn_rp[c + 1]; t++) {
          int pp = pos[P.sn_rows[t]];
          if (pp < 0) { *code = 2; return "internal: child row not in parent structure"; }
          P.sn_rel[t] = pp;
        }
      }
      for (int t = 0; t < rp; t++) pos[Rp[t]] = -1;
    }
    // K entry -> panel offset
    P.kpos.resize(P.Kp[n]);
    for (int s = 0; s < ns; s++) {
      const int* Rs = &P.sn_rows[P.sn_rp[s]];
      int r = P.sn_rp[s + 1] - P.sn_rp[s];
      for (int t = 0; t < r; t++) pos[Rs[t]] = t;
      for (int j = snf[s]; j < snf[s + 1]; j++)
        for (int p = P.Kp[j]; p < P.Kp[j + 1]; p++)
          P.kpos[p] = (j - snf[s]) * r + pos[P.Ki[p]];
      for (int t = 0; t < r; t++) pos[Rs[t]] = -1;
    }
  }
  // ---------------- level schedule -------------------------------------------------
  P.sn_level.assign(ns, 0);
  for (int s = 0; s < ns; s++)
    if (P.sn_parent[s] >= 0)
      P.sn_level[P.sn_parent[s]] = std::max(P.sn_level[P.sn_parent[s]], P.sn_level[s] + 1);
  P.height = 0;
  for (int s = 0; s < ns; s++) P.height = std::max(P.height, P.sn_level[s] + 1);
  P.order.resize(ns);
  std::iota(P.order.begin(), P.order.end(), 0);
  std::stable_sort(P.order.begin(), P.order.end(),
                   [&](int a, int b) { return P.sn_level[a] < P.sn_level[b]; });

  // small (warp) / big (CTA) split, closed under descendants
  {
    std::vector<char> big(ns, 0);
    // warp-per-supernode class threshold (<= KKT_SCAP, the per-warp shared-memory slice);
    // KKT_SCLASS=<doubles> overrides it (tuning hook)
    long long sclass = KKT_SCAP;
    if (const char* e = getenv("KKT_SCLASS")) sclass = std::min<long long>(KKT_SCAP, std::max(0LL, atoll(e)));
    if (opt.factor_kind == 1) sclass = -1;  // LDL^T: no warp class (every supernode on a signed CTA / tile path)
    for (int s = 0; s < ns; s++) {
      long long r = P.sn_rp[s + 1] - P.sn_rp[s], w = snf[s + 1] - snf[s], R = r - w;
      long long need = r * w + (P.sn_parent[s] >= 0 ? R * (R + 1) / 2 : 0);
      if (need > sclass) big[s] = 1;
    }
    for (int s = 0; s < ns; s++)  // children precede parents
      if (big[s] && P.sn_parent[s] >= 0) big[P.sn_parent[s]] = 1;
    P.order_s.clear(); P.order_b.clear(); P.max_r_small = 0;
    P.up_s.clear(); P.up_b.clear(); P.dn_b.clear(); P.dn_s.clear();
    std::vector<int> nbigch(ns, 0);
    for (int s = 0; s < ns; s++)
      if (big[s] && P.sn_parent[s] >= 0) nbigch[P.sn_parent[s]]++;
    for (int s = 0; s < ns; s++) {
      int par = P.sn_parent[s];
      bool leaf = P.sn_cp[s + 1] == P.sn_cp[s];
      if (!big[s] && leaf) P.up_s.push_back(s);
      if (big[s] && nbigch[s] == 0) P.up_b.push_back(s);
      if (!big[s] && (par < 0 || big[par])) P.dn_s.push_back(s);
    }
    auto by_height = [&](int a, int b) {
      return P.sn_hsub[a] != P.sn_hsub[b] ? P.sn_hsub[a] > P.sn_hsub[b] : a < b;
    };
    std::sort(P.dn_s.begin(), P.dn_s.end(), by_height);
    std::sort(P.up_s.begin(), P.up_s.end(), [&](int a, int b) {  // deepest chains first
      int ha = 0, hb = 0;
      for (int x = a; x >= 0 && !big[x]; x = P.sn_parent[x]) ha++;
      for (int x = b; x >= 0 && !big[x]; x = P.sn_parent[x]) hb++;
      return ha != hb ? ha > hb : a < b;
    });
    // huge: fronts beyond one CTA's shared memory (KKT_HCAP doubles), closed upward
    std::vector<char> huge(ns, 0);
    long long hcap = KKT_HCAP;  // test hook: KKT_HCAP=<doubles> moves smaller fronts to the GPU-wide path
    if (const char* e = getenv("KKT_HCAP")) hcap = std::min<long long>(hcap, std::max(0LL, atoll(e)));
    for (int s = 0; s < ns; s++) {
      long long r = P.sn_rp[s + 1] - P.sn_rp[s], w = snf[s + 1] - snf[s], R = r - w;
      long long need = r * w + (P.sn_parent[s] >= 0 ? R * (R + 1) / 2 : 0);
      if (need > hcap && big[s]) huge[s] = 1;
    }
    for (int s = 0; s < ns; s++)
      if (huge[s] && P.sn_parent[s] >= 0) huge[P.sn_parent[s]] = 1;
    P.up_bf.clear(); P.order_h.clear();
    {
      std::vector<int> nbn(ns, 0);  // big non-huge children
      for (int s = 0; s < ns; s++)
        if (big[s] && !huge[s] && P.sn_parent[s] >= 0) nbn[P.sn_parent[s]]++;
      for (int s = 0; s < ns; s++) {
        const int par = P.sn_parent[s];
        if (big[s] && !huge[s] && nbn[s] == 0) P.up_bf.push_back(s);
        if (big[s] && !huge[s] && (par < 0 || huge[par])) P.dn_b.push_back(s);
        if (huge[s]) P.order_h.push_back(s);  // postorder = topological
      }
      P.flops_huge = 0.0;
      P.n_huge = (int)P.order_h.size();
      for (int s : P.order_h) {
        const double r = P.sn_rp[s + 1] - P.sn_rp[s], w = snf[s + 1] - snf[s];
        for (int t = 0; t < (int)w; t++) P.flops_huge += (r - t) * (r - t);
      }
      std::sort(P.dn_b.begin(), P.dn_b.end(), by_height);
    }
    P.sn.resize(ns);
    for (int s = 0; s < ns; s++) {
      SnInfo& I = P.sn[s];
      std::memset(&I, 0, sizeof(I));
      I.f0 = snf[s]; I.w = snf[s + 1] - snf[s];
      I.rp0 = P.sn_rp[s]; I.r = P.sn_rp[s + 1] - P.sn_rp[s];
      I.par = P.sn_parent[s]; I.c0 = P.sn_cp[s]; I.c1 = P.sn_cp[s + 1]; I.big = big[s];
      I.k0 = P.Kp[snf[s]]; I.k1 = P.Kp[snf[s + 1]];
      I.Lp = P.sn_Lp[s]; I.Up = P.sn_Up[s]; I.uvp = (int)P.sn_uvp[s]; I.huge = huge[s];
    }
    P.sn_Lip.assign(ns, -1);
    P.linv_doubles = 0;
    for (int s = 0; s < ns; s++)
      if (big[s] && !huge[s]) {
        const long long w = snf[s + 1] - snf[s];
        P.sn_Lip[s] = P.linv_doubles;
        P.linv_doubles += w * w;
      }
    P.chinfo.resize(P.sn_ch.size());
    for (size_t t = 0; t < P.sn_ch.size(); t++) P.chinfo[t] = P.sn[P.sn_ch[t]];
    for (int s : P.order) {
      if (big[s]) P.order_b.push_back(s);
      else {
        P.order_s.push_back(s);
        P.max_r_small = std::max(P.max_r_small, P.sn_rp[s + 1] - P.sn_rp[s]);
      }
    }
  }

  // ---------------- 6. condensation gather map ------------------------------------
  P.kw.assign(P.Kp[n], -1);
  P.kdiag.assign(P.Kp[n], -1);
  for (int j = 0; j < n; j++) P.kdiag[P.Kp[j]] = P.perm[j];
  auto kfind = [&](int i, int j) {  // internal (i >= j)
    auto b = P.Ki.begin() + P.Kp[j], e = P.Ki.begin() + P.Kp[j + 1];
    auto it = std::lower_bound(b, e, i);
    return (int)(it - P.Ki.begin());
  };
  for (int i = 0; i < n; i++)
    for (int p = Wp[i]; p < Wp[i + 1]; p++) {
      int a = P.iperm[i], b = P.iperm[Wc[p]];
      P.kw[kfind(std::max(a, b), std::min(a, b))] = p;
    }
  P.jrow.resize(P.nnzJ);
  for (int r = 0; r < m; r++)
    for (int p = Jp[r]; p < Jp[r + 1]; p++) P.jrow[p] = r;
  {
    std::vector<int> cntp(P.Kp[n] + 1, 0);
    std::vector<std::tuple<int, int, int>> prods;  // (k, pa, pb)
    prods.reserve(64);
    long long np = 0;
    for (int r = 0; r < m; r++)
      for (int a = Jp[r]; a < Jp[r + 1]; a++)
        for (int b = a; b < Jp[r + 1]; b++) np++;
    std::vector<int> pk(np), pa(np), pb(np);
    long long t = 0;
    for (int r = 0; r < m; r++)
      for (int a = Jp[r]; a < Jp[r + 1]; a++)
        for (int b = a; b < Jp[r + 1]; b++) {
          int ia = P.iperm[Jc[a]], ib = P.iperm[Jc[b]];
          int k = kfind(std::max(ia, ib), std::min(ia, ib));
          pk[t] = k; pa[t] = a; pb[t] = b; cntp[k + 1]++; t++;
        }
    P.pptr.assign(P.Kp[n] + 1, 0);
    for (int k = 0; k < P.Kp[n]; k++) P.pptr[k + 1] = P.pptr[k] + cntp[k + 1];
    P.pa.resize(np); P.pb.resize(np);
    std::vector<int> f(P.pptr.begin(), P.pptr.end() - 1);
    for (long long q = 0; q < np; q++) {  // rows in increasing order: deterministic sum order
      int k = pk[q];
      P.pa[f[k]] = pa[q]; P.pb[f[k]] = pb[q]; f[k]++;
    }
    P.nprod = np;
  }

  // ---------------- 7. residual operator maps (orig numbering) ---------------------
  {
    std::vector<int> c(n + 1, 0);
    for (int i = 0; i < n; i++)
      for (int p = Wp[i]; p < Wp[i + 1]; p++) {
        c[i + 1]++;
        if (Wc[p] != i) c[Wc[p] + 1]++;
      }
    P.Wf_p.assign(n + 1, 0);
    for (int i = 0; i < n; i++) P.Wf_p[i + 1] = P.Wf_p[i] + c[i + 1];
    P.Wf_c.resize(P.Wf_p[n]); P.Wf_k.resize(P.Wf_p[n]);
    std::vector<int> f(P.Wf_p.begin(), P.Wf_p.end() - 1);
    for (int i = 0; i < n; i++)
      for (int p = Wp[i]; p < Wp[i + 1]; p++) {
        int j = Wc[p];
        P.Wf_c[f[i]] = j; P.Wf_k[f[i]] = p; f[i]++;
        if (j != i) { P.Wf_c[f[j]] = i; P.Wf_k[f[j]] = p; f[j]++; }
      }
    std::vector<int> jc(n + 1, 0);
    for (int p = 0; p < P.nnzJ; p++) jc[Jc[p] + 1]++;
    P.Jt_p.assign(n + 1, 0);
    for (int i = 0; i < n; i++) P.Jt_p[i + 1] = P.Jt_p[i] + jc[i + 1];
    P.Jt_r.resize(P.nnzJ); P.Jt_k.resize(P.nnzJ);
    std::vector<int> g(P.Jt_p.begin(), P.Jt_p.end() - 1);
    for (int r = 0; r < m; r++)  // rows ascending -> G rows form a prefix of every column
      for (int p = Jp[r]; p < Jp[r + 1]; p++) {
        int i = Jc[p];
        P.Jt_r[g[i]] = r; P.Jt_k[g[i]] = p; g[i]++;
      }
    P.Gt_end.resize(n);
    for (int i = 0; i < n; i++) {
      int e = P.Jt_p[i];
      while (e < P.Jt_p[i + 1] && P.Jt_r[e] < m_eq) e++;
      P.Gt_end[i] = e;
    }
  }
  P.analyze_ms = now_ms() - t0;
  return "";
}

}  // namespace kkt
