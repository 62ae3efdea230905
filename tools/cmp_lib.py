"""Bitwise comparison of two builds of libkkt on one config (KKT_LIB selects the library).

usage: python tools/cmp_lib.py CFG other.so|other_checkout_dir   -> runs the config with the default
library and with the other library (or another checkout's binding + library) in a subprocess,
compares x (and dx, dy for HyKKT) bit for bit.
"""
import os, sys, subprocess, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
cfg = sys.argv[1]
if len(sys.argv) > 3 and sys.argv[2] == "--dump":
    import numpy as np, torch
    import paper_2405_14236_b200 as K
    from synth.generator import make_config
    inst = make_config(cfg)
    S = K.KKTSolver.from_instance(inst).bind(0)
    d = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda:0")
    S.condense(d(inst.W_vals), d(inst.J_vals), d(inst.Sigma_x), d(inst.Sigma_s), None, inst.delta_w, inst.delta_c, inst.gamma)
    S.factor()
    x = torch.zeros(inst.n, dtype=torch.float64, device="cuda:0")
    if inst.m_eq > 0:
        dy = torch.zeros(inst.m_eq, dtype=torch.float64, device="cuda:0")
        S.hykkt_solve(d(inst.rbar1), d(inst.rbar2), x, dy, 1e-12, 0, 2)
        out = torch.cat([x, dy])
    else:
        S.solve(d(inst.b), x, 10, 0.0)
        out = x
    torch.cuda.synchronize()
    np.save(sys.argv[3], out.cpu().numpy())
    print(json.dumps(S.sync_info()))
    sys.exit(0)
import numpy as np
env = dict(os.environ)
subprocess.run([sys.executable, __file__, cfg, "--dump", "/tmp/cmp_a.npy"], check=True, env=env)
other = os.path.abspath(sys.argv[2])
if os.path.isdir(other):  # another checkout (its own binding and library)
    subprocess.run([sys.executable, os.path.join(other, "tools", "cmp_lib.py"), cfg, "--dump", "/tmp/cmp_b.npy"],
                   check=True, env=env, cwd=other)
else:
    env["KKT_LIB"] = other
    subprocess.run([sys.executable, __file__, cfg, "--dump", "/tmp/cmp_b.npy"], check=True, env=env)
a, b = np.load("/tmp/cmp_a.npy"), np.load("/tmp/cmp_b.npy")
print(cfg, "bitwise equal" if np.array_equal(a, b) else f"DIFFER max {np.abs(a - b).max():.3e}")
