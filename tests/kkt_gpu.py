"""Helpers for the -m gpu tests: run an instance through the C-ABI (torch supplies device
memory and the stream).  Imports torch lazily so CPU-only collection works."""
import numpy as np

import paper_2405_14236_b200 as K


def dev(a, device):
    import torch
    if a is None:
        return None
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device=device)


def run_lifted(inst, max_refine=10, tol_bwd=0.0, solver=None, device="cuda:0", D=None):
    """condense -> factor -> solve; returns (x [batch?, n], info dict, solver)."""
    import torch
    S = solver or K.KKTSolver.from_instance(inst).bind(0)
    t = [dev(a, device) for a in (inst.W_vals, inst.J_vals if inst.nnzJ else np.zeros(1),
                                  inst.Sigma_x, inst.Sigma_s if inst.Sigma_s.size else np.zeros(1),
                                  D, inst.b)]
    W, J, Sx, Ss, Dd, b = t
    x = torch.zeros_like(b)
    S.condense(W, J, Sx, Ss, Dd, inst.delta_w, inst.delta_c, inst.gamma)
    S.factor()
    S.solve(b, x, max_refine, tol_bwd)
    info = S.sync_info()
    return x.cpu().numpy(), info, S


def run_hykkt(inst, cg_rtol=1e-12, cg_maxit=0, max_outer=2, solver=None, device="cuda:0", krylov=0):
    import torch
    S = solver or K.KKTSolver.from_instance(inst).bind(0)
    W, J, Sx, Ss, r1, r2 = [dev(a, device) for a in (inst.W_vals, inst.J_vals, inst.Sigma_x,
                                                      inst.Sigma_s if inst.Sigma_s.size else np.zeros(1),
                                                      inst.rbar1, inst.rbar2)]
    dx = torch.zeros_like(r1)
    dy = torch.zeros_like(r2)
    S.condense(W, J, Sx, Ss, None, inst.delta_w, inst.delta_c, inst.gamma)
    S.factor()
    S.hykkt_solve(r1, r2, dx, dy, cg_rtol, cg_maxit, max_outer, krylov=krylov)
    info = S.sync_info()
    return dx.cpu().numpy(), dy.cpu().numpy(), info, S


def relerr(x, xref):
    return float(np.abs(x - xref).max() / max(np.abs(xref).max(), 1e-300))
