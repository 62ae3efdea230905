"""Per-supernode timing trace of factor / forward / backward (KKT_TRACE=1).

usage: KKT_TRACE=1 python tools/trace_analyze.py [C2] [--json out.json]
Prints, for each phase, the kernel span, node-duration statistics (small vs big supernodes) and
the critical path: for every node on the longest dependency chain its duration and the gap
between the end of its last-finishing dependency and its own start (scheduling latency).
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("KKT_TRACE", "1")

import numpy as np
import torch

import paper_2405_14236_b200 as K
from synth.generator import make_config


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else "C2"
    inst = make_config(cfg) if cfg != "C5" else make_config("C5", batch=1)
    S = K.KKTSolver.from_instance(inst).bind(0)
    d = lambda a: torch.as_tensor(a, dtype=torch.float64, device="cuda:0")
    W, J, Sx, Ss, b = d(inst.W_vals), d(inst.J_vals), d(inst.Sigma_x), d(inst.Sigma_s), d(inst.b)
    x = torch.zeros_like(b)
    for _ in range(3):
        S.condense(W, J, Sx, Ss, None, inst.delta_w, inst.delta_c, inst.gamma)
        S.factor()
        S.solve(b, x, 0, 0.0)
    torch.cuda.synchronize()
    raw = S.trace()
    np.save(os.path.join(ROOT, "gpurun_out", f"trace_raw_{cfg}.npy"), raw)
    T = raw.astype(np.float64) / 1e3  # us
    base = T[T > 0].min()
    T = np.where(T > 0, T - base, -1e12)
    f, r, p = S.supernodes()
    w = np.diff(f)
    R = r - w
    need = r * w + np.where(p >= 0, R * (R + 1) // 2, 0)
    big = need > 2048
    ns = len(r)
    for s in range(ns):
        if big[s] and p[s] >= 0:
            big[p[s]] = True
    children = [[] for _ in range(ns)]
    for s in range(ns):
        if p[s] >= 0:
            children[p[s]].append(s)
    out = {}
    for kind, name in enumerate(["factor", "forward", "backward"]):
        st, en = T[kind, :, 0], T[kind, :, 1]
        t0 = st[st > -1e11].min()
        st, en = st - t0, en - t0
        dur = en - st
        span = en.max()
        # critical path by finish time
        if kind < 2:
            dep_end = np.array([max([en[c] for c in children[s]], default=0.0) for s in range(ns)])
            s = int(np.argmax(en))
            path = []
            while True:
                path.append(s)
                if not children[s]:
                    break
                s = max(children[s], key=lambda c: en[c])
        else:
            dep_end = np.array([en[p[s]] if p[s] >= 0 else 0.0 for s in range(ns)])
            s = int(np.argmax(en))
            path = []
            while s >= 0:
                path.append(s)
                s = int(p[s])
        gaps = st - dep_end
        rep = {"span_us": float(span),
               "small_dur_us_mean": float(dur[~big].mean()), "small_dur_us_max": float(dur[~big].max()),
               "big_dur_us_mean": float(dur[big].mean()) if big.any() else None,
               "big_dur_us_max": float(dur[big].max()) if big.any() else None,
               "gap_us_mean": float(gaps.mean()), "path_len": len(path),
               "path_dur_us": float(dur[path].sum()), "path_gap_us": float(np.clip(gaps[path], 0, None).sum())}
        out[name] = rep
        print(f"== {name}: span {span:.1f} us; small dur mean {rep['small_dur_us_mean']:.2f} max "
              f"{rep['small_dur_us_max']:.2f}; big dur mean {rep['big_dur_us_mean']} ; critical path "
              f"{len(path)} nodes, busy {rep['path_dur_us']:.1f} us, gaps {rep['path_gap_us']:.1f} us")
        for s in path[:40]:
            cp = T[kind, s, 2:] - t0
            cps = " ".join(f"{c - st[s]:6.2f}" for c in cp if c > -1e8)
            print(f"   s={s:6d} big={int(big[s])} r={r[s]:4d} w={w[s]:4d} nch={len(children[s])} "
                  f"start={st[s]:8.2f} dur={dur[s]:7.2f} gap={gaps[s]:6.2f}  checkpoints: {cps}")
    if "--json" in sys.argv:
        json.dump(out, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)


if __name__ == "__main__":
    main()
