"""Per-task timeline of the tile-task factorisation of the large fronts (KKT_TRACE=1).

usage: python tools/tile_trace.py [C4] [--save out.npz]
Prints per task type: count, mean duration after dependencies were met (work), mean wait for
dependencies (spin), and the kernel span / worker utilisation.
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("KKT_TRACE", "1")
import numpy as np, torch
import paper_2405_14236_b200 as K
from paper_2405_14236_b200 import kkt as KK
from synth.generator import make_config

cfg = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else "C4"
SOLVE = "--solve" in sys.argv
inst = make_config(cfg)
S = K.KKTSolver.from_instance(inst).bind(0)
d = lambda a: torch.as_tensor(a, dtype=torch.float64, device="cuda:0")
W, J, Sx, Ss = d(inst.W_vals), d(inst.J_vals), d(inst.Sigma_x), d(inst.Sigma_s)
b = d(inst.b)
xs = torch.zeros_like(b)
for _ in range(3):
    S.condense(W, J, Sx, Ss, None, inst.delta_w, inst.delta_c, inst.gamma)
    S.factor()
    if SOLVE:
        S.solve(b, xs, 0, 0.0)
torch.cuda.synchronize()
print("factor phase ms (small+big, large):", S.factor_phase_ms())
tasks, tr, est = KK.kkt_tile_trace(S.h, solve=SOLVE)
tr = tr.astype(np.float64)
t0 = tr[:, 0].min()
st, rd, en = (tr[:, 0] - t0) / 1e3, (tr[:, 1] - t0) / 1e3, (tr[:, 2] - t0) / 1e3
rd = np.where(tr[:, 1] > 0, rd, st)      # no wait recorded -> ready at start
typ = tasks[:, 0] & 15
names = ["FG", "FU", "FC", "BU", "BC", "UF", "FCH", "BCH"] if SOLVE else ["ASM", "POTRF0", "TRSM", "CRIT", "UPD", "INV"]
span = en.max()
print(f"tasks {len(tasks)}  span {span:.1f} us  (list-schedule estimate {est:.1f} us)")
busy = (en - st).sum()
work = (en - rd).sum()
nw = len(np.unique(tr[:, 3]))
print(f"SMs used {nw}; sum(task time) {busy:.0f} us, sum(work after deps) {work:.0f} us, workers*span {nw*2*span:.0f} us")
for t in range(len(names)):
    m = typ == t
    if m.any():
        print(f"  {names[t]:6s} n={m.sum():6d}  work mean {np.mean(en[m]-rd[m]):7.2f} us  p90 {np.percentile(en[m]-rd[m],90):7.2f}"
              f"  wait mean {np.mean(rd[m]-st[m]):7.2f} us  total work {np.sum(en[m]-rd[m]):9.0f} us")
if "--save" in sys.argv:
    np.savez(sys.argv[sys.argv.index("--save") + 1], tasks=tasks, trace=tr, est=est)
if SOLVE and "--chains" in sys.argv:  # chain tasks in start order: front, start, ready, end (us)
    for i in np.argsort(st):
        if typ[i] in (6, 7):
            print(f"  {names[typ[i]]} front {tasks[i, 1]:4d}  start {st[i]:8.1f}  ready {rd[i]:8.1f}  end {en[i]:8.1f}"
                  f"  work {en[i] - rd[i]:6.1f}")
if SOLVE and "--all" in sys.argv:  # every task in ticket order: type, front, z, w, start, ready, end (us)
    for i in range(len(tasks)):
        print(f"  T{i:5d} {names[typ[i]]:4s} f {tasks[i, 1]:4d} z {tasks[i, 2]:3d} w {tasks[i, 3]:3d}  start {st[i]:8.1f}"
              f"  ready {rd[i]:8.1f}  end {en[i]:8.1f}  sm {int(tr[i, 3])}")
