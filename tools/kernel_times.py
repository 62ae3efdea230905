"""Per-kernel GPU times of the solve phase from CUPTI (torch.profiler), graph launches included.

usage: python tools/kernel_times.py [C3] [--reps 5]
Condense + factor once, then profiles `reps` solves (HyKKT for configs with equality rows, else
the refined LiftedKKT solve with the bench's max_refine) and prints per kernel: launches per
solve, total / mean duration, and the solve's GPU span (first kernel start -> last kernel end).
Diagnosis only: numbers taken under a profiler are never bench values.
"""
import os, sys, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from torch.profiler import profile, ProfilerActivity
import paper_2405_14236_b200 as K
from synth.generator import make_config

cfg = sys.argv[1] if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else "C3"
reps = int(sys.argv[sys.argv.index("--reps") + 1]) if "--reps" in sys.argv else 5
inst = make_config(cfg) if cfg != "C5" else make_config("C5", batch=512)
S = K.KKTSolver.from_instance(inst).bind(0)
d = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda:0")
W, J, Sx, Ss = d(inst.W_vals), d(inst.J_vals), d(inst.Sigma_x), d(inst.Sigma_s)
hy = inst.m_eq > 0
B = inst.batch
x = torch.zeros((B, inst.n) if B > 1 else (inst.n,), dtype=torch.float64, device="cuda:0")
dy = torch.zeros(max(inst.m_eq, 1), dtype=torch.float64, device="cuda:0")
S.condense(W, J, Sx, Ss, None, inst.delta_w, inst.delta_c, inst.gamma)
S.factor()
if hy:
    r1, r2 = d(inst.rbar1), d(inst.rbar2)
    call = lambda: S.hykkt_solve(r1, r2, x, dy, 1e-12, 0, 2)
else:
    b = d(inst.b)
    call = lambda: S.solve(b, x, 10, 0.0)
for _ in range(3):
    call()
torch.cuda.synchronize()
print(cfg, "info", S.sync_info())
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(reps):
        call()
        torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
agg = collections.defaultdict(lambda: [0, 0.0])
t0 = min(e.time_range.start for e in ev); t1 = max(e.time_range.end for e in ev)
for e in ev:
    a = agg[e.name.split("(")[0][:70]]
    a[0] += 1; a[1] += e.time_range.elapsed_us()
tot = sum(a[1] for a in agg.values())
print(f"{len(ev) / reps:.0f} kernels per solve; kernel time {tot / reps:.1f} us per solve; span {(t1 - t0) / reps:.1f} us per solve (incl. host gaps)")
for n, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"  {n:70s} {c / reps:7.1f} /solve {t / reps:9.1f} us/solve {t / c:8.2f} us/launch")
