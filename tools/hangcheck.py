"""C4 condense -> factor -> refined solve, 3 repetitions, reporting timing / status (hang check)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2405_14236_b200 as K
from synth.generator import make_config
cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
inst = make_config(cfg)
S = K.KKTSolver.from_instance(inst).bind(0)
d = lambda a: torch.as_tensor(a, dtype=torch.float64, device="cuda:0")
W, J, Sx, Ss, b = d(inst.W_vals), d(inst.J_vals), d(inst.Sigma_x), d(inst.Sigma_s), d(inst.b)
x = torch.zeros_like(b)
for r in range(3):
    t = time.time()
    S.condense(W, J, Sx, Ss, None, inst.delta_w, inst.delta_c, inst.gamma)
    S.factor()
    torch.cuda.synchronize(); t1 = time.time()
    S.solve(b, x, 10, 0.0)
    torch.cuda.synchronize(); t2 = time.time()
    print(r, "factor %.1f ms solve %.1f ms" % ((t1 - t) * 1e3, (t2 - t1) * 1e3), S.sync_info(), flush=True)
