"""One condense -> factor -> refined solve on small configs (and a HyKKT solve), for
compute-sanitizer (memcheck / racecheck / synccheck).  usage: python tools/sanitize_run.py [cases]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from synth.generator import make_config, tiny_random
from kkt_gpu import run_lifted, run_hykkt

cases = sys.argv[1].split(",") if len(sys.argv) > 1 else ["C1", "C5b2", "tiny_eq"]
for c in cases:
    if c == "C5b2":
        inst = make_config("C5", batch=2)
    elif c == "tiny_eq":
        inst = tiny_random(45, 30, 10, seed=6, Xi=1e-6, hykkt_gamma=1e5)
    else:
        inst = make_config(c)
    if inst.m_eq > 0:
        dx, dy, info, S = run_hykkt(inst)
    else:
        x, info, S = run_lifted(inst, max_refine=4)
    S.close()
    print(c, "status", info["status"], "refine", info["refine_iters"], "cg", info["cg_iters"], flush=True)
