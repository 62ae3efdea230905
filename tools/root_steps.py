"""Per-step timeline of the root front's tile factorisation (KKT_TRACE=2 debugging aid)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["KKT_TRACE"] = "2"
import numpy as np, torch
import paper_2405_14236_b200 as K
from paper_2405_14236_b200 import kkt as KK
from synth.generator import make_config
cfg = sys.argv[1] if len(sys.argv) > 1 else "C6"
inst = make_config(cfg)
S = K.KKTSolver.from_instance(inst).bind(0)
d = lambda a: torch.as_tensor(a, dtype=torch.float64, device="cuda:0")
W, J, Sx, Ss = d(inst.W_vals), d(inst.J_vals), d(inst.Sigma_x), d(inst.Sigma_s)
for _ in range(2):
    S.condense(W, J, Sx, Ss, None, inst.delta_w, inst.delta_c, inst.gamma)
    S.factor()
torch.cuda.synchronize()
buf = np.zeros(4096 * 8, dtype=np.int64)
lib = KK.lib()
lib.kkt_debug_steps.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
print("rc", lib.kkt_debug_steps(S.h, buf.ctypes.data, buf.size))
T = buf.reshape(4096, 8).astype(np.float64)
nb = int(np.max(np.nonzero(T[:, 1])[0])) + 1
t0 = T[0, 0]
T = np.where(T > 0, (T - t0) / 1e3, np.nan)
print("k  potrf[beg,end]  trsm(k+1,k)[reach,go,end]  upd(k+1,k+1,k)[reach,go,end]   (us from POTRF(0) start)")
for k in range(nb):
    e = T[k]
    print(f"{k:3d}  {e[0]:8.1f} {e[1]:8.1f}   {e[7]:8.1f} {e[2]:8.1f} {e[3]:8.1f}   {e[6]:8.1f} {e[4]:8.1f} {e[5]:8.1f}")
