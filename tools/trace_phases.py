"""Phase timeline of a KKT_TRACE dump: start/end of the small / big / huge classes per sweep.
usage: python tools/trace_phases.py gpurun_out/trace_raw_C6.npy C6"""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2405_14236_b200 as K
from synth.generator import make_config

raw = np.load(sys.argv[1]).astype(np.float64) / 1e3
S = K.KKTSolver.from_instance(make_config(sys.argv[2]))
f, r, p = S.supernodes()
w = np.diff(f); R = r - w; ns = len(r)
need = r * w + np.where(p >= 0, R * (R + 1) // 2, 0)
big = need > 2048
for s in range(ns):
    if big[s] and p[s] >= 0: big[p[s]] = True
huge = big & (need > 25600)
for s in range(ns):
    if huge[s] and p[s] >= 0: huge[p[s]] = True
for k, name in enumerate(["factor", "forward", "backward"]):
    st, en = raw[k, :, 0], raw[k, :, 1]
    ok = st > 0
    t0 = st[ok].min()
    st, en = st - t0, en - t0
    out = []
    for cname, m in (("small", ~big), ("big", big & ~huge), ("huge", huge)):
        m = m & ok
        if m.any():
            out.append(f"{cname}[{st[m].min():8.1f},{en[m].max():8.1f}] n={m.sum()} busy={np.sum(en[m]-st[m]):.0f}")
    print(f"{name:8s} span {en[ok].max():8.1f} us  " + "  ".join(out))
