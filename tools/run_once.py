"""Run condense + factor + solve of one workload a few times (profiling driver).
usage: python tools/run_once.py C6 [reps]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2405_14236_b200 as K
from synth.generator import make_config

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
inst = make_config(cfg) if cfg != "C5" else make_config("C5", batch=1)
S = K.KKTSolver.from_instance(inst).bind(0)
d = lambda a: torch.as_tensor(a, dtype=torch.float64, device="cuda:0")
W, J, Sx, Ss, b = d(inst.W_vals), d(inst.J_vals), d(inst.Sigma_x), d(inst.Sigma_s), d(inst.b)
x = torch.zeros_like(b)
for _ in range(reps):
    S.condense(W, J, Sx, Ss, None, inst.delta_w, inst.delta_c, inst.gamma)
    S.factor()
    S.solve(b, x, 1, 0.0)
torch.cuda.synchronize()
print("ok", float(x.abs().max()))
