// sblock_plan.cpp -- host construction of the subtree blocks of the small supernodes (sblock.h).
#include "sblock.h"

#include <algorithm>

namespace kkt {

void build_sblocks(const Plan& P, int cap, int nw, SBlockHost& out) {
  const int ns = P.ns;
  out = SBlockHost{};
  out.blk_of.assign(ns, -1);
  out.lrow.assign(P.sn_rows.size(), 0);
  if (ns == 0) return;
  // subtree extents (postorder: the subtree of s is [lo[s], s]) and "all small" flags
  std::vector<int> lo(ns), hgt(ns, 0);
  std::vector<char> allsmall(ns, 1);
  for (int s = 0; s < ns; s++) lo[s] = s;
  for (int s = 0; s < ns; s++) {
    if (P.sn[s].big) allsmall[s] = 0;
    const int p = P.sn_parent[s];
    if (p >= 0) {
      lo[p] = std::min(lo[p], lo[s]);
      if (!allsmall[s]) allsmall[p] = 0;
      hgt[p] = std::max(hgt[p], hgt[s] + 1);
    }
  }
  auto layout_of = [&](int a, int s) {
    const int nn = s - a + 1;
    const long long nL = P.sn_Lp[s + 1] - P.sn_Lp[a];
    const int ncol = P.sn_first[s + 1] - P.sn_first[a];
    const int nr = P.sn_rp[s + 1] - P.sn_rp[a];
    const int nch = P.sn_cp[s + 1] - P.sn_cp[a];
    const int R = (P.sn_rp[s + 1] - P.sn_rp[s]) - (P.sn_first[s + 1] - P.sn_first[s]);
    // the level count is the subtree height + 1 (levels by height within the subtree)
    return sb_layout(nn, hgt[s] + 1, nL, ncol, nr, nch, R, nw);
  };
  std::vector<char> fits(ns, 0);
  for (int s = 0; s < ns; s++) {
    if (!allsmall[s]) continue;
    const long long nL = P.sn_Lp[s + 1] - P.sn_Lp[lo[s]];
    if (nL > cap) continue;
    fits[s] = layout_of(lo[s], s).total <= cap;
  }
  for (int s = 0; s < ns; s++) {
    if (P.sn[s].big) continue;
    const int p = P.sn_parent[s];
    if (!fits[s] || (p >= 0 && fits[p])) continue;
    // block root s: subtree [lo[s], s]
    const int a = lo[s];
    SBlk B{};
    B.s_lo = a; B.s_hi = s; B.nlev = hgt[s] + 1; B.m0 = (int)out.meta.size();
    B.F0 = P.sn_first[a]; B.ncol = P.sn_first[s + 1] - P.sn_first[a];
    B.RP0 = P.sn_rp[a]; B.nr = P.sn_rp[s + 1] - P.sn_rp[a];
    B.CP0 = P.sn_cp[a]; B.nch = P.sn_cp[s + 1] - P.sn_cp[a];
    B.Rroot = (P.sn_rp[s + 1] - P.sn_rp[s]) - (P.sn_first[s + 1] - P.sn_first[s]);
    B.L0 = P.sn_Lp[a]; B.nL = P.sn_Lp[s + 1] - P.sn_Lp[a];
    // levels by height inside the subtree: children strictly below their parent
    std::vector<int> cntl(B.nlev + 1, 0);
    for (int t = a; t <= s; t++) cntl[hgt[t] + 1]++;
    for (int l = 0; l < B.nlev; l++) cntl[l + 1] += cntl[l];
    std::vector<int> nodes(s - a + 1);
    std::vector<int> pos(cntl.begin(), cntl.end() - 1);
    for (int t = a; t <= s; t++) nodes[pos[hgt[t]]++] = t - a;
    out.meta.insert(out.meta.end(), cntl.begin(), cntl.end());
    out.meta.insert(out.meta.end(), nodes.begin(), nodes.end());
    // backward row map: own and in-block rows -> column offset; rows above the block -> slot
    // ncol + (position among the root's update rows).  Every row of a block supernode that lies
    // above the block is in the root's structure (struct(L_j) \ {j} is inside struct(L_parent)).
    const int F1 = B.F0 + B.ncol;
    const int rw = P.sn_first[s + 1] - P.sn_first[s];
    for (int t = a; t <= s; t++) {
      for (int q = P.sn_rp[t]; q < P.sn_rp[t + 1]; q++) {
        const int i = P.sn_rows[q];
        if (i < F1) {
          out.lrow[q] = i - B.F0;
        } else {
          const int* rb = P.sn_rows.data() + P.sn_rp[s] + rw;
          const int* re = P.sn_rows.data() + P.sn_rp[s + 1];
          const int* it = std::lower_bound(rb, re, i);
          out.lrow[q] = B.ncol + (int)(it - rb);
        }
      }
    }
    for (int t = a; t < s; t++) out.blk_of[t] = -2;
    out.blk_of[s] = (int)out.blk.size();
    out.max_smem = std::max(out.max_smem, layout_of(a, s).total);
    out.nodes_in_blocks += s - a + 1;
    out.blk.push_back(B);
  }
  for (int s = 0; s < ns; s++)
    if (!P.sn[s].big && out.blk_of[s] == -1) out.n_single++;
}

void build_fblocks(const Plan& P, int cap, FBlockHost& out) {
  const int ns = P.ns;
  out = FBlockHost{};
  if (ns == 0) return;
  std::vector<int> lo(ns), hgt(ns, 0);
  for (int s = 0; s < ns; s++) lo[s] = s;
  for (int s = 0; s < ns; s++) {
    const int p = P.sn_parent[s];
    if (p >= 0) { lo[p] = std::min(lo[p], lo[s]); hgt[p] = std::max(hgt[p], hgt[s] + 1); }
  }
  auto layout_of = [&](int a, int s) {
    return fb_layout(s - a + 1, hgt[s] + 1, (int)(P.sn_Lp[s + 1] - P.sn_Lp[a]), (int)(P.sn_Up[s + 1] - P.sn_Up[a]),
                     P.Kp[P.sn_first[s + 1]] - P.Kp[P.sn_first[a]], P.sn_rp[s + 1] - P.sn_rp[a],
                     P.sn_cp[s + 1] - P.sn_cp[a]);
  };
  std::vector<char> fits(ns, 0);
  for (int s = 0; s < ns; s++) {
    if (P.sn[s].big) continue;  // small is closed under descendants
    if (P.sn_Lp[s + 1] - P.sn_Lp[lo[s]] + P.sn_Up[s + 1] - P.sn_Up[lo[s]] > cap) continue;
    fits[s] = layout_of(lo[s], s).total <= cap;
  }
  std::vector<char> inblk(ns, 0);
  for (int s = 0; s < ns; s++) {
    if (P.sn[s].big) continue;
    const int p = P.sn_parent[s];
    if (!fits[s] || (p >= 0 && fits[p])) continue;
    const int a = lo[s];
    FBlk B{};
    B.s_lo = a; B.s_hi = s; B.nlev = hgt[s] + 1; B.m0 = (int)out.meta.size();
    B.K0 = P.Kp[P.sn_first[a]]; B.nK = P.Kp[P.sn_first[s + 1]] - B.K0;
    B.RP0 = P.sn_rp[a]; B.nr = P.sn_rp[s + 1] - B.RP0;
    B.CP0 = P.sn_cp[a]; B.nch = P.sn_cp[s + 1] - B.CP0;
    B.L0 = P.sn_Lp[a]; B.nL = (int)(P.sn_Lp[s + 1] - B.L0);
    B.U0 = P.sn_Up[a]; B.nU = (int)(P.sn_Up[s + 1] - B.U0);
    std::vector<int> cntl(B.nlev + 1, 0);
    for (int t = a; t <= s; t++) cntl[hgt[t] + 1]++;
    for (int l = 0; l < B.nlev; l++) cntl[l + 1] += cntl[l];
    std::vector<int> nodes(s - a + 1);
    std::vector<int> pos(cntl.begin(), cntl.end() - 1);
    for (int t = a; t <= s; t++) nodes[pos[hgt[t]]++] = t - a;
    out.meta.insert(out.meta.end(), cntl.begin(), cntl.end());
    out.meta.insert(out.meta.end(), nodes.begin(), nodes.end());
    for (int t = a; t <= s; t++) inblk[t] = 1;
    out.max_smem = std::max(out.max_smem, layout_of(a, s).total);
    out.nodes_in_blocks += s - a + 1;
    out.blk.push_back(B);
  }
  for (int s = 0; s < ns; s++)
    if (!P.sn[s].big && !inblk[s]) {
      out.n_single++;
      if (P.sn_cp[s + 1] == P.sn_cp[s]) out.up_init.push_back(s);
    }
}

}  // namespace kkt
