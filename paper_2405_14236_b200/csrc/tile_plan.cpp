// tile_plan.cpp -- host scheduler of the tile-task factorisation of the large fronts (tiles.cuh).
//
// Builds the task DAG of every huge front (ASM / POTRF0 / TRSM / CRIT / UPD over 64 x 64 tiles,
// see tiles.cuh for the dependency rules), then orders it by a list-scheduling simulation on
// `workers` identical workers: tasks are prioritised by their bottom level (longest remaining
// path, estimated durations) and issued to the earliest free worker as soon as their
// predecessors finish.  The resulting start order is a topological order, which is what the
// device ticket protocol needs for deadlock freedom; the priorities put the per-front critical
// chains (POTRF -> TRSM -> UPDATE of the diagonal) ahead of the bulk Schur updates.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <functional>
#include <queue>
#include <vector>

#include "tile_plan.h"

namespace kkt {

namespace {
constexpr int TB = 64;
constexpr int TS_G = 0, TS_U = 1, TS_C = 2, TS_BU_ = 3, TS_BC_ = 4, TS_UF = 5, TS_FCH_ = 6, TS_BCH_ = 7;  // tsolve.cuh task types

struct Task {
  int type, f, i, j, k;
  double dur;
};

int tl(int i, int j, int nt) { return j * nt - j * (j - 1) / 2 + (i - j); }
}  // namespace

// List-scheduling simulation: bottom-level priorities, earliest free worker; returns the
// simulated makespan and the start order (a topological order of the DAG).
template <class TaskT>
static double list_schedule(const std::vector<TaskT>& tasks, const std::vector<std::vector<int>>& pred,
                            int workers, std::vector<int>& order) {
  const int N = (int)tasks.size();
  std::vector<std::vector<int>> succ(N);
  for (int t = 0; t < N; t++)
    for (int p : pred[t]) succ[p].push_back(t);
  std::vector<double> blev(N, 0.0);
  for (int t = N - 1; t >= 0; t--) {
    double m = 0.0;
    for (int q : succ[t]) m = std::max(m, blev[q]);
    blev[t] = tasks[t].dur + m;
  }
  std::vector<int> npred(N);
  std::vector<double> ready_at(N, 0.0), fin(N, 0.0);
  for (int t = 0; t < N; t++) npred[t] = (int)pred[t].size();
  using PQ = std::pair<double, int>;
  auto cmp_prio = [&](int a, int b) { return blev[a] != blev[b] ? blev[a] < blev[b] : a > b; };
  std::priority_queue<int, std::vector<int>, decltype(cmp_prio)> avail(cmp_prio);
  std::priority_queue<PQ, std::vector<PQ>, std::greater<PQ>> pending, running;
  for (int t = 0; t < N; t++)
    if (npred[t] == 0) pending.push({0.0, t});
  int free_w = std::max(1, workers);
  double now = 0.0;
  order.clear();
  order.reserve(N);
  while ((int)order.size() < N) {
    while (!pending.empty() && pending.top().first <= now) { avail.push(pending.top().second); pending.pop(); }
    if (free_w > 0 && !avail.empty()) {
      const int t = avail.top();
      avail.pop();
      fin[t] = now + tasks[t].dur;
      running.push({fin[t], t});
      order.push_back(t);
      free_w--;
      continue;
    }
    double nxt = 1e300;
    if (!running.empty()) nxt = running.top().first;
    if (free_w > 0 && !pending.empty()) nxt = std::min(nxt, pending.top().first);
    now = std::max(now, nxt);
    while (!running.empty() && running.top().first <= now) {
      const int t = running.top().second;
      running.pop();
      free_w++;
      for (int q : succ[t]) {
        ready_at[q] = std::max(ready_at[q], fin[t]);
        if (--npred[q] == 0) pending.push({ready_at[q], q});
      }
    }
  }
  double mk = 0.0;
  for (int t = 0; t < N; t++) mk = std::max(mk, fin[t]);
  return mk;
}

void build_tile_plan(const Plan& P, int workers, TilePlanHost& out) {
  out = TilePlanHost();
  const int ns = P.ns;
  out.hidx.assign(std::max(ns, 1), -1);
  for (int s : P.order_h) {  // postorder: children first
    TFrontHost F;
    std::memset(&F, 0, sizeof(F));
    F.s = s;
    F.r = P.sn_rp[s + 1] - P.sn_rp[s];
    F.w = P.sn_first[s + 1] - P.sn_first[s];
    F.nbp = (F.w + TB - 1) / TB;
    const int nbu = (F.r - F.w + TB - 1) / TB;
    F.nt = F.nbp + nbu;
    F.nU = nbu * (nbu + 1) / 2;
    out.hidx[s] = (int)out.fr.size();
    out.fr.push_back(F);
  }
  long long tb = 0;
  int cb = 0;
  for (auto& F : out.fr) {
    F.tbase = tb;
    F.cbase = cb;
    const int T = F.nt * (F.nt + 1) / 2;
    tb += (long long)T * TB * TB;
    cb += T + 2;  // tile counters, asm count, done count
    // child records: for every child, cut[t] = first child update row/column whose parent front
    // row is >= the first row of parent tile t (the relative-index map rel is increasing)
    F.ch0 = (int)out.tch.size() / 2;
    F.nch = P.sn_cp[F.s + 1] - P.sn_cp[F.s];
    if (F.nch > 31) out.ok = false;  // tiles.cuh task_asm keeps <= 31 child records in shared memory
    for (int q = P.sn_cp[F.s]; q < P.sn_cp[F.s + 1]; q++) {
      const int c = P.sn_ch[q];
      const int wc = P.sn_first[c + 1] - P.sn_first[c];
      const int Rc = (P.sn_rp[c + 1] - P.sn_rp[c]) - wc;
      const int* rel = &P.sn_rel[P.sn_rp[c] + wc];
      out.tch.push_back(c);
      out.tch.push_back((int)out.tcut.size());
      for (int t = 0; t <= F.nt; t++) {
        const int start = (t < F.nbp) ? t * TB : (t < F.nt ? F.w + (t - F.nbp) * TB : F.r);
        out.tcut.push_back((int)(std::lower_bound(rel, rel + Rc, start) - rel));
      }
    }
  }
  if (out.tch.empty()) { out.tch.assign(2, 0); }
  if (out.tcut.empty()) out.tcut.assign(1, 0);
  // K entries grouped by tile (pointer array indexed like the tile counters)
  out.tkptr.assign(cb + 1, 0);
  {
    std::vector<std::vector<int>> lists(cb);
    for (const auto& F : out.fr) {
      const int f0 = P.sn_first[F.s];
      for (int k = P.Kp[f0]; k < P.Kp[f0 + F.w]; k++) {
        const int pos = P.kpos[k], col = pos / F.r, row = pos - col * F.r;
        const int ti = row < F.w ? row / TB : F.nbp + (row - F.w) / TB, tj = col / TB;
        lists[F.cbase + tl(ti, tj, F.nt)].push_back(k);
      }
    }
    for (int q = 0; q < cb; q++) {
      out.tkptr[q + 1] = out.tkptr[q] + (int)lists[q].size();
      out.tkidx.insert(out.tkidx.end(), lists[q].begin(), lists[q].end());
    }
    if (out.tkidx.empty()) out.tkidx.assign(1, 0);
  }
  out.pool_doubles = std::max<long long>(tb, 1);
  out.ncnt = std::max(cb, 1);
  {
    long long ib = 0;
    for (auto& F : out.fr) { out.ibase.push_back(ib); ib += (long long)F.nbp * TB * TB; }
    out.inv_doubles = std::max<long long>(ib, 1);
    if (out.ibase.empty()) out.ibase.push_back(0);
  }
  if (out.fr.empty()) return;

  // ---- tasks with predecessor lists (generation order is topological) ----
  // estimated durations (us) of one CTA task (B200, measured order of magnitude)
  const double d_upd = 5.0, d_trsm = 4.5, d_crit = 18.0, d_potrf = 9.0;  // measured (round 2 micro-bench)
  std::vector<Task> tasks;
  std::vector<std::vector<int>> pred;
  std::vector<std::vector<int>> final_u(out.fr.size());
  auto add = [&](int type, int f, int i, int j, int k, double dur, std::vector<int> p) {
    tasks.push_back({type, f, i, j, k, dur});
    pred.push_back(std::move(p));
    return (int)tasks.size() - 1;
  };
  for (int f = 0; f < (int)out.fr.size(); f++) {
    const TFrontHost& F = out.fr[f];
    const int s = F.s, nt = F.nt, nbp = F.nbp;
    // one assembly task per tile; it waits for the final update of the child U tiles it reads
    // (huge children) -- estimate: child entries landing in the tile at ~8 B / 4 ns
    std::vector<int> last_upd(nt * (nt + 1) / 2, -1);   // last task writing tile (i, j)
    for (int jt = 0; jt < nt; jt++)
      for (int i = jt; i < nt; i++) {
        long long ent = 0;
        std::vector<int> p;
        for (int q = 0; q < F.nch; q++) {
          const int c = out.tch[2 * (F.ch0 + q)];
          const int* cut = &out.tcut[out.tch[2 * (F.ch0 + q) + 1]];
          const int a = cut[jt], b = cut[jt + 1], ra = cut[i], rb = cut[i + 1];
          ent += (long long)std::max(0, b - a) * std::max(0, rb - ra);
          const int hc = out.hidx[c];
          if (hc >= 0 && b > a && rb > ra) {
            const TFrontHost& C = out.fr[hc];
            for (int tj = a >> 6; tj <= (b - 1) >> 6; tj++)
              for (int ti = std::max(tj, ra >> 6); ti <= (rb - 1) >> 6; ti++)
                p.push_back(final_u[hc][tl(C.nbp + ti, C.nbp + tj, C.nt) - tl(C.nbp, C.nbp, C.nt)]);
          }
        }
        last_upd[tl(i, jt, nt)] = add(0, f, i, jt, 0, 1.5 + ent * 0.004 / 4.0, p);
      }
    std::vector<int> lprod(nt, -1);                      // producer of L(i, k) for the current k
    const std::vector<int> p_asm;                        // (per-tile assembly dependencies)
    int diag_prod = add(1, f, 0, 0, 0, d_potrf, {last_upd[tl(0, 0, nt)]});  // POTRF0
    last_upd[tl(0, 0, nt)] = diag_prod;
    add(5, f, 0, 0, 0, d_trsm, {diag_prod});                                  // INV(0)
    for (int k = 0; k < nbp; k++) {
      const bool crit = (k + 1 < nbp);
      std::fill(lprod.begin(), lprod.end(), -1);
      lprod[k] = diag_prod;
      int crit_id = -1;
      if (crit) {
        std::vector<int> p = {diag_prod};
        if (last_upd[tl(k + 1, k, nt)] >= 0) p.push_back(last_upd[tl(k + 1, k, nt)]);
        if (last_upd[tl(k + 1, k + 1, nt)] >= 0) p.push_back(last_upd[tl(k + 1, k + 1, nt)]);
        if (k == 0) p.insert(p.end(), p_asm.begin(), p_asm.end());
        crit_id = add(3, f, k + 1, k + 1, k, d_crit, p);
        lprod[k + 1] = crit_id;
      }
      for (int i = crit ? k + 2 : k + 1; i < nt; i++) {
        std::vector<int> p = {diag_prod};
        if (last_upd[tl(i, k, nt)] >= 0) p.push_back(last_upd[tl(i, k, nt)]);
        if (k == 0) p.insert(p.end(), p_asm.begin(), p_asm.end());
        lprod[i] = add(2, f, i, k, k, d_trsm, p);
      }
      for (int j = k + 1; j < nt; j++)
        for (int i = j; i < nt; i++) {
          if (crit && i == k + 1 && j == k + 1) continue;  // inside CRIT(k)
          std::vector<int> p = {lprod[i]};
          if (j != i) p.push_back(lprod[j]);
          if (last_upd[tl(i, j, nt)] >= 0) p.push_back(last_upd[tl(i, j, nt)]);
          if (k == 0) p.insert(p.end(), p_asm.begin(), p_asm.end());
          const double dur = (i == j) ? d_upd * 0.75 : d_upd;
          const int id = add(4, f, i, j, k, dur, p);
          last_upd[tl(i, j, nt)] = id;
          if (j >= nbp && k == nbp - 1) {
            final_u[f].resize(F.nU, -1);
            final_u[f][tl(i, j, nt) - tl(nbp, nbp, nt)] = id;
          }
        }
      if (crit) {
        last_upd[tl(k + 1, k + 1, nt)] = crit_id;
        diag_prod = crit_id;
        add(5, f, k + 1, k + 1, k + 1, d_trsm, {crit_id});                    // INV(k + 1)
      }
    }
  }
  std::vector<int> order;
  out.est_us = list_schedule(tasks, pred, workers, order);
  const int N = (int)tasks.size();
  out.tasks.resize(N);
  for (int q = 0; q < N; q++) {
    const Task& T = tasks[order[q]];
    out.tasks[q] = TTask{T.type, T.f, T.i | (T.j << 16), T.k};
  }
  out.ntask_by_type.assign(6, 0);
  for (const Task& T : tasks) out.ntask_by_type[T.type]++;
}

}  // namespace kkt

namespace kkt {

void build_tile_solve_plan(const Plan& P, const TilePlanHost& tp, int workers, bool chains, TSolvePlanHost& out) {
  out = TSolvePlanHost();
  const int nf = (int)tp.fr.size();
  out.cbase2.resize(std::max(nf, 1));
  out.pbase.resize(std::max(nf, 1));
  int cb = 0;
  long long pb = 0;
  for (int f = 0; f < nf; f++) {
    const TFrontHost& F = tp.fr[f];
    out.cbase2[f] = cb;
    cb += 2 * F.nt + 3 * F.nbp + 2;
    out.pbase[f] = pb;
    pb += ((long long)F.nt * F.nbp + (long long)F.nbp * F.nt) * TB;
  }
  out.ncnt = std::max(cb, 1);
  out.part_doubles = std::max<long long>(pb, 1);
  if (nf == 0) return;
  struct STask { int type, f, i, k; double dur; };
  std::vector<STask> tasks;
  std::vector<std::vector<int>> pred;
  auto add = [&](int type, int f, int i, int k, double dur, std::vector<int> p) {
    tasks.push_back({type, f, i, k, dur});
    pred.push_back(std::move(p));
    return (int)tasks.size() - 1;
  };
  const double d_g = 2.0, d_u = 1.5, d_c = 2.5;
  std::vector<std::vector<std::vector<int>>> ublk(nf);   // per U block: its gather + partial producers
  std::vector<std::vector<int>> fc(nf);
  // ---- forward, fronts in postorder ----
  for (int f = 0; f < nf; f++) {
    const TFrontHost& F = tp.fr[f];
    const int nt = F.nt, nbp = F.nbp;
    std::vector<int> g(nt);
    for (int t = 0; t < nt; t++) {   // the gather waits for the child blocks feeding parent block t
      std::vector<int> chp;
      for (int q = 0; q < F.nch; q++) {
        const int hc = tp.hidx[tp.tch[2 * (F.ch0 + q)]];
        const int* cut = &tp.tcut[tp.tch[2 * (F.ch0 + q) + 1]];
        if (hc < 0 || cut[t + 1] <= cut[t]) continue;
        for (int tc = cut[t] >> 6; tc <= (cut[t + 1] - 1) >> 6; tc++)
          chp.insert(chp.end(), ublk[hc][tc].begin(), ublk[hc][tc].end());
      }
      g[t] = add(TS_G, f, t, 0, d_g, chp);
    }
    std::vector<std::vector<int>> prod(nt);     // producers of the partials P[t][.]
    fc[f].assign(nbp, -1);
    if (chains) {
      // the panel on one CTA (tsolve.cuh FCH), then the update rows' products per (t, k)
      std::vector<int> p(g.begin(), g.begin() + nbp);
      const double dch = 1.0 + 1.2 * nbp + 0.4 * nbp * (nbp - 1) / 2;
      const int c = add(TS_FCH_, f, 0, 0, dch, p);
      for (int k = 0; k < nbp; k++) fc[f][k] = c;
      for (int k = 0; k < nbp; k++)
        for (int i = nbp; i < nt; i++) prod[i].push_back(add(TS_U, f, i, k, d_u, {c}));
    } else {
      for (int k = 0; k < nbp; k++) {
        std::vector<int> p = {g[k]};
        p.insert(p.end(), prod[k].begin(), prod[k].end());
        const int c = add(TS_C, f, k + 1, k, d_c, p);
        fc[f][k] = c;
        if (k + 1 < nt) prod[k + 1].push_back(c);
        for (int i = k + 2; i < nt; i++) prod[i].push_back(add(TS_U, f, i, k, d_u, {c}));
      }
    }
    for (int t = nbp; t < nt; t++) {
      std::vector<int> p = {g[t]};
      p.insert(p.end(), prod[t].begin(), prod[t].end());
      ublk[f].push_back(p);
    }
  }
  // ---- backward, fronts top-down (reverse postorder) ----
  std::vector<int> xlast(nf, -1);
  for (int f = nf - 1; f >= 0; f--) {
    const TFrontHost& F = tp.fr[f];
    const int nt = F.nt, nbp = F.nbp;
    const int par = P.sn_parent[F.s];
    const int hp = par >= 0 ? tp.hidx[par] : -1;
    std::vector<std::vector<int>> q(nbp);       // producers of Q[k][.]
#ifndef TS_UCHUNK_N
#define TS_UCHUNK_N 1
#endif
    const int UCH = TS_UCHUNK_N;   // tsolve.cuh TS_UCHUNK
    for (int k = 0; k < nbp; k++)       // update rows in chunks of UCH tiles, parallel
      for (int c0 = nbp; c0 < nt; c0 += UCH) {
        std::vector<int> p;
        if (hp >= 0) p.push_back(xlast[hp]);
        q[k].push_back(add(TS_BU_, f, c0, k, d_u * std::min(UCH, nt - c0), p));
      }
    if (chains) {
      std::vector<int> p = {fc[f][0]};
      for (int k = 0; k < nbp; k++) p.insert(p.end(), q[k].begin(), q[k].end());
      const double dch = 1.0 + 1.2 * nbp + 0.4 * nbp * (nbp - 1) / 2;
      xlast[f] = add(TS_BCH_, f, 0, 0, dch, p);
      continue;
    }
    int xprev = -1;
    for (int k = nbp - 1; k >= 0; k--) {
      std::vector<int> p = {fc[f][k]};
      p.insert(p.end(), q[k].begin(), q[k].end());
      if (xprev >= 0) p.push_back(xprev);
      const int x = add(TS_BC_, f, k + 1, k, d_c, p);
      xprev = x;
      for (int j = k - 2; j >= 0; j--) q[j].push_back(add(TS_BU_, f, k, j, d_u, {x}));
    }
    xlast[f] = xprev;
  }
  std::vector<int> order;
  out.est_us = list_schedule(tasks, pred, workers, order);
  out.tasks.resize(tasks.size());
  for (size_t qq = 0; qq < order.size(); qq++) {
    const STask& T = tasks[order[qq]];
    out.tasks[qq] = TTask{T.type, T.f, T.i, T.k};
  }
}

}  // namespace kkt
