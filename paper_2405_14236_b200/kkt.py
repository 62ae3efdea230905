"""Thin ctypes binding of libkkt.so (include/kkt.h).  Argument marshalling only: every step of
the hot path runs in the library's CUDA kernels.  There is no CPU fallback -- if libkkt.so is
missing or has no GPU to run on, calls raise.

Module-level functions carry the C names (kkt_analyze, kkt_condense, ...); `KKTSolver` bundles
them around one handle, with PyTorch supplying device memory and the stream.
"""
from __future__ import annotations

import ctypes as C
import os
import numpy as np

from . import build as _build

_lib = None

KKT_STATUS = {0: "KKT_OK", 1: "KKT_ERR_ARG", 2: "KKT_ERR_PATTERN", 3: "KKT_ERR_NOT_SPD",
              4: "KKT_ERR_NOT_CONVERGED", 5: "KKT_ERR_NONFINITE", 6: "KKT_ERR_CUDA",
              7: "KKT_ERR_ALLOC", 8: "KKT_ERR_STATE"}

EXPORTS = ["kkt_default_options", "kkt_analyze", "kkt_get_symbolic", "kkt_workspace_size",
           "kkt_bind", "kkt_condense", "kkt_factor", "kkt_solve", "hykkt_solve", "hykkt_solve_krylov",
           "kkt_sync_info", "kkt_inertia", "kkt_factor_inertia_correct", "kkt_solve_unreduced", "kkt_recover", "kkt_recover_bounds", "kkt_step_host", "kkt_get_condensed", "kkt_get_supernodes", "kkt_get_blocks", "kkt_get_trace", "kkt_launch_count", "kkt_hykkt_stats",
           "kkt_factor_phase_ms", "kkt_debug_steps", "kkt_tile_trace", "kkt_tile_solve_trace", "kkt_last_error", "kkt_destroy"]


class KKTError(RuntimeError):
    def __init__(self, code, where):
        self.code = code
        msg = lib().kkt_last_error().decode(errors="replace")
        super().__init__(f"{where}: {KKT_STATUS.get(code, code)} {msg}")


class KKTOptions(C.Structure):
    _fields_ = [("ordering", C.c_int), ("factor_kind", C.c_int), ("relax_small", C.c_int),
                ("relax_big", C.c_int), ("relax_zero_frac", C.c_double), ("batch", C.c_int)]


class KKTAnalysisInfo(C.Structure):
    _fields_ = [("nnzK", C.c_longlong), ("nnzL", C.c_longlong), ("nnzL_stored", C.c_longlong),
                ("flops", C.c_double), ("nprod", C.c_longlong), ("nsuper", C.c_int),
                ("tree_height", C.c_int), ("max_front", C.c_int), ("analyze_ms", C.c_double),
                ("order_ms", C.c_double), ("update_doubles", C.c_longlong),
                ("flops_huge", C.c_double), ("nsuper_huge", C.c_int)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


def so_path() -> str:
    # KKT_LIB: an alternative in-tree build of the same library (tuning experiments, tools/)
    return os.environ.get("KKT_LIB", _build.SO)


def lib(build_if_missing: bool = True):
    """Load libkkt.so (building it in-tree with nvcc if missing).  Raises if unavailable."""
    global _lib
    if _lib is None:
        path = so_path()
        if not os.path.exists(path):
            if not build_if_missing:
                raise OSError(f"{path} missing: run __graft_entry__.build()")
            _build.build()
        L = C.CDLL(path)
        P, I, D, S = C.c_void_p, C.c_int, C.c_double, C.c_size_t
        sig = {
            "kkt_default_options": [C.POINTER(KKTOptions)],
            "kkt_analyze": [I, I, I, P, P, P, P, C.POINTER(KKTOptions), C.POINTER(C.c_void_p),
                            C.POINTER(KKTAnalysisInfo)],
            "kkt_get_symbolic": [P, P, P, P],
            "kkt_workspace_size": [P, C.POINTER(S)],
            "kkt_bind": [P, I, P, S, P],
            "kkt_condense": [P, P, P, P, P, P, D, D, D],
            "kkt_factor": [P],
            "kkt_solve": [P, P, P, I, D],
            "hykkt_solve": [P, P, P, P, P, D, I, I],
            "hykkt_solve_krylov": [P, P, P, P, P, D, I, I, I],
            "kkt_sync_info": [P, C.POINTER(I), C.POINTER(I), C.POINTER(I), C.POINTER(I),
                              C.POINTER(D)],
            "kkt_step_host": [P, P, P, P, P, P, D, D, D, P, P, I, D],
            "kkt_get_condensed": [P, I, P, P, P],
            "kkt_recover": [P, P, P, P, P, P],
            "kkt_inertia": [P, P],
            "kkt_factor_inertia_correct": [P, P, P, P, P, P, D, D, P, C.POINTER(D), C.POINTER(I)],
            "kkt_solve_unreduced": [P] + [P] * 4 + [P] * 6 + [P] * 6 + [I, D],
            "kkt_recover_bounds": [P, P, P, P, P, D, P, P, P, P],
            "kkt_launch_count": [P, C.POINTER(C.c_longlong)],
            "kkt_hykkt_stats": [P, C.POINTER(C.c_int), C.POINTER(C.c_int)],
            "kkt_get_supernodes": [P, C.POINTER(I), P, P, P],
            "kkt_get_blocks": [P, I, I, I, P, P, P, P, P, P, P],
            "kkt_get_trace": [P, P],
            "kkt_factor_phase_ms": [P, P],
            "kkt_debug_steps": [P, P, I],
            "kkt_tile_trace": [P, P, P, I, P],
            "kkt_tile_solve_trace": [P, P, P, I, P],
            "kkt_destroy": [P],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int
        L.kkt_last_error.restype = C.c_char_p
        L.kkt_last_error.argtypes = []
        _lib = L
    return _lib


def _chk(code, where):
    if code != 0:
        raise KKTError(code, where)


def _np_i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _ptr(t):
    """Device/host pointer of a torch tensor or numpy array (None -> NULL)."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


# ------------------------------------------------------------------ C-named thin wrappers
def kkt_default_options() -> KKTOptions:
    o = KKTOptions()
    _chk(lib().kkt_default_options(C.byref(o)), "kkt_default_options")
    return o


def kkt_analyze(n, m, m_eq, W_rowptr, W_colind, J_rowptr, J_colind, options=None):
    o = options or kkt_default_options()
    h = C.c_void_p()
    info = KKTAnalysisInfo()
    arrs = [_np_i32(W_rowptr), _np_i32(W_colind), _np_i32(J_rowptr), _np_i32(J_colind)]
    _chk(lib().kkt_analyze(int(n), int(m), int(m_eq), *[a.ctypes.data for a in arrs],
                           C.byref(o), C.byref(h), C.byref(info)), "kkt_analyze")
    return h, info.as_dict()


def kkt_get_symbolic(h, n):
    perm = np.zeros(max(n, 1), np.int32); et = np.zeros(max(n, 1), np.int32)
    cc = np.zeros(max(n, 1), np.int32)
    _chk(lib().kkt_get_symbolic(h, perm.ctypes.data, et.ctypes.data, cc.ctypes.data), "kkt_get_symbolic")
    return perm[:n], et[:n], cc[:n]


def kkt_workspace_size(h):
    s = C.c_size_t()
    _chk(lib().kkt_workspace_size(h, C.byref(s)), "kkt_workspace_size")
    return s.value


def kkt_bind(h, device, workspace, nbytes, stream):
    _chk(lib().kkt_bind(h, int(device), _ptr(workspace), int(nbytes), stream), "kkt_bind")


def kkt_condense(h, W_vals, J_vals, Sigma_x, Sigma_s, D=None, delta_w=0.0, delta_c=0.0, gamma=0.0):
    _chk(lib().kkt_condense(h, _ptr(W_vals), _ptr(J_vals), _ptr(Sigma_x), _ptr(Sigma_s), _ptr(D),
                            float(delta_w), float(delta_c), float(gamma)), "kkt_condense")


def kkt_factor(h):
    _chk(lib().kkt_factor(h), "kkt_factor")


def kkt_solve(h, b, x, max_refine=10, tol_bwd=0.0):
    _chk(lib().kkt_solve(h, _ptr(b), _ptr(x), int(max_refine), float(tol_bwd)), "kkt_solve")


def hykkt_solve(h, rbar1, rbar2, dx, dy, cg_rtol=1e-12, cg_maxit=0, max_outer_refine=2):
    _chk(lib().hykkt_solve(h, _ptr(rbar1), _ptr(rbar2), _ptr(dx), _ptr(dy), float(cg_rtol),
                           int(cg_maxit), int(max_outer_refine)), "hykkt_solve")


def hykkt_solve_krylov(h, rbar1, rbar2, dx, dy, cg_rtol=1e-12, cg_maxit=0, max_outer_refine=2, krylov=0):
    _chk(lib().hykkt_solve_krylov(h, _ptr(rbar1), _ptr(rbar2), _ptr(dx), _ptr(dy), float(cg_rtol),
                                  int(cg_maxit), int(max_outer_refine), int(krylov)), "hykkt_solve_krylov")


def kkt_sync_info(h):
    st, fc, it, cg = C.c_int(), C.c_int(), C.c_int(), C.c_int()
    be = C.c_double()
    _chk(lib().kkt_sync_info(h, C.byref(st), C.byref(fc), C.byref(it), C.byref(cg), C.byref(be)),
         "kkt_sync_info")
    return dict(status=st.value, status_name=KKT_STATUS.get(st.value, str(st.value)),
                fail_col=fc.value, refine_iters=it.value, cg_iters=cg.value, bwd_err=be.value)


def kkt_solve_unreduced(h, x, s, u, v, f, d, max_refine=10, tol=0.0):
    """f = (f1..f6), d = (dx, ds, dy, dz, du, dv) device buffers (None where a block is empty)."""
    _chk(lib().kkt_solve_unreduced(h, _ptr(x), _ptr(s), _ptr(u), _ptr(v), *[_ptr(a) for a in f],
                                   *[_ptr(a) for a in d], int(max_refine), float(tol)), "kkt_solve_unreduced")


def kkt_inertia(h, batch=1):
    c = np.zeros(3 * batch, np.int32)
    _chk(lib().kkt_inertia(h, c.ctypes.data), "kkt_inertia")
    return c.reshape(batch, 3)


def kkt_factor_inertia_correct(h, W_vals, J_vals, Sigma_x, Sigma_s, D=None, delta_c=0.0, gamma=0.0,
                               params=None):
    """Returns (delta_w, tries); params = [dw_min, dw_first, dw_max, k_minus, k_plus, k_plus_bar, dw_last]."""
    dw, tr = C.c_double(0.0), C.c_int(0)
    pa = None if params is None else np.ascontiguousarray(params, dtype=np.float64)
    _chk(lib().kkt_factor_inertia_correct(h, _ptr(W_vals), _ptr(J_vals), _ptr(Sigma_x), _ptr(Sigma_s), _ptr(D),
                                          float(delta_c), float(gamma), None if pa is None else pa.ctypes.data,
                                          C.byref(dw), C.byref(tr)), "kkt_factor_inertia_correct")
    return dw.value, tr.value


def kkt_recover(h, r2, r4, dx, dz, ds):
    _chk(lib().kkt_recover(h, _ptr(r2), _ptr(r4), _ptr(dx), _ptr(dz), _ptr(ds)), "kkt_recover")


def kkt_recover_bounds(h, x, u, s, v, mu, dx, ds, du, dv):
    _chk(lib().kkt_recover_bounds(h, _ptr(x), _ptr(u), _ptr(s), _ptr(v), float(mu), _ptr(dx), _ptr(ds),
                                  _ptr(du), _ptr(dv)), "kkt_recover_bounds")


def kkt_step_host(h, W_vals, J_vals, Sigma_x, Sigma_s, D, delta_w, delta_c, gamma, b, x,
                  max_refine=10, tol_bwd=0.0):
    _chk(lib().kkt_step_host(h, _ptr(W_vals), _ptr(J_vals), _ptr(Sigma_x), _ptr(Sigma_s), _ptr(D),
                             float(delta_w), float(delta_c), float(gamma), _ptr(b), _ptr(x),
                             int(max_refine), float(tol_bwd)), "kkt_step_host")


def kkt_get_condensed(h, inst, n, nnzK, values=True):
    Kp = np.zeros(n + 1, np.int32); Ki = np.zeros(max(nnzK, 1), np.int32)
    Kv = np.zeros(max(nnzK, 1)) if values else None
    _chk(lib().kkt_get_condensed(h, int(inst), Kp.ctypes.data, Ki.ctypes.data,
                                 Kv.ctypes.data if values else None), "kkt_get_condensed")
    return Kp, Ki[:nnzK], (Kv[:nnzK] if values else None)


def kkt_get_supernodes(h):
    ns = C.c_int()
    _chk(lib().kkt_get_supernodes(h, C.byref(ns), None, None, None), "kkt_get_supernodes")
    f = np.zeros(ns.value + 1, np.int32); r = np.zeros(max(ns.value, 1), np.int32)
    p = np.zeros(max(ns.value, 1), np.int32)
    _chk(lib().kkt_get_supernodes(h, C.byref(ns), f.ctypes.data, r.ctypes.data, p.ctypes.data),
         "kkt_get_supernodes")
    return f, r[:ns.value], p[:ns.value]


def kkt_get_blocks(h, ns, nrows, kind=0, cap=6144, nwarps=8):
    """Subtree blocks of the small supernodes (host plan; test export): (blk [nblk, 8], blk_of,
    meta, lrow, is_big) -- see include/kkt.h."""
    nb, nm = C.c_int(0), C.c_int(0)
    _chk(lib().kkt_get_blocks(h, kind, cap, nwarps, C.byref(nb), C.byref(nm), None, None, None, None, None),
         "kkt_get_blocks")
    blk = np.zeros((max(nb.value, 1), 8), dtype=np.int32)
    blk_of = np.zeros(ns, dtype=np.int32)
    meta = np.zeros(max(nm.value, 1), dtype=np.int32)
    lrow = np.zeros(max(nrows, 1), dtype=np.int32)
    is_big = np.zeros(ns, dtype=np.int32)
    _chk(lib().kkt_get_blocks(h, kind, cap, nwarps, C.byref(nb), C.byref(nm), _ptr(blk), _ptr(blk_of), _ptr(meta),
                              _ptr(lrow) if kind == 0 else None, _ptr(is_big)), "kkt_get_blocks")
    return blk[:nb.value], blk_of, meta[:nm.value], lrow[:nrows], is_big


def kkt_get_trace(h, ns):
    t = np.zeros((3, max(ns, 1), 8), np.int64)
    _chk(lib().kkt_get_trace(h, t.ctypes.data), "kkt_get_trace")
    return t[:, :ns]


def kkt_hykkt_stats(h):
    kr, op = C.c_int(0), C.c_int(0)
    _chk(lib().kkt_hykkt_stats(h, C.byref(kr), C.byref(op)), "kkt_hykkt_stats")
    return {"krylov_total": kr.value, "outer_passes": op.value}


def kkt_launch_count(h):
    v = C.c_longlong()
    _chk(lib().kkt_launch_count(h, C.byref(v)), "kkt_launch_count")
    return v.value


def kkt_factor_phase_ms(h):
    ms = np.zeros(2)
    _chk(lib().kkt_factor_phase_ms(h, ms.ctypes.data), "kkt_factor_phase_ms")
    return float(ms[0]), float(ms[1])


def kkt_tile_trace(h, want_trace=True, solve=False):
    """(tasks [N, 4] int32, trace [N, 4] int64 or None, estimated makespan us) of the tile kernel
    (solve=True: of the tile-task solve)."""
    fn = lib().kkt_tile_solve_trace if solve else lib().kkt_tile_trace
    est = C.c_double(0.0)
    n = fn(h, None, None, 0, C.byref(est))
    if n < 0:
        raise KKTError(8, "kkt_tile_trace")
    tasks = np.zeros((max(n, 1), 4), np.int32)
    tr = np.zeros((max(n, 1), 4), np.int64) if want_trace else None
    rc = fn(h, tr.ctypes.data if want_trace else None, tasks.ctypes.data, n, C.byref(est))
    if rc < 0:
        raise KKTError(8, "kkt_tile_trace")
    return tasks[:n], (tr[:n] if want_trace else None), est.value


def kkt_destroy(h):
    _chk(lib().kkt_destroy(h), "kkt_destroy")


# ------------------------------------------------------------------ convenience wrapper
class KKTSolver:
    """One handle: analysis on construction; `bind()` attaches a CUDA device + torch stream."""

    def __init__(self, n, m, m_eq, W_rowptr, W_colind, J_rowptr, J_colind, batch=1, ordering=0,
                 relax_small=4, relax_big=64, relax_zero_frac=0.05, factor_kind=0):
        o = kkt_default_options()
        o.batch, o.ordering, o.factor_kind = int(batch), int(ordering), int(factor_kind)
        o.relax_small, o.relax_big, o.relax_zero_frac = relax_small, relax_big, relax_zero_frac
        self.n, self.m, self.m_eq, self.batch = n, m, m_eq, batch
        self.h, self.info = kkt_analyze(n, m, m_eq, W_rowptr, W_colind, J_rowptr, J_colind, o)
        self.ws = None
        self.device = None

    @classmethod
    def from_instance(cls, inst, **kw):
        return cls(inst.n, inst.m, inst.m_eq, inst.W_rowptr, inst.W_colind, inst.J_rowptr,
                   inst.J_colind, batch=kw.pop("batch", inst.batch), **kw)

    def symbolic(self):
        return kkt_get_symbolic(self.h, self.n)

    def bind(self, device=0, stream=None):
        import torch
        dev = torch.device("cuda", device)
        nbytes = kkt_workspace_size(self.h)
        self.ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=dev)
        s = torch.cuda.current_stream(dev) if stream is None else stream
        self.stream = s
        kkt_bind(self.h, device, self.ws, nbytes, C.c_void_p(s.cuda_stream))
        self.device = dev
        return self

    def condense(self, W_vals, J_vals, Sigma_x, Sigma_s, D=None, delta_w=0.0, delta_c=0.0, gamma=0.0):
        self._vals = (W_vals, J_vals, Sigma_x, Sigma_s, D)  # keep alive: re-read by the residual
        kkt_condense(self.h, W_vals, J_vals, Sigma_x, Sigma_s, D, delta_w, delta_c, gamma)

    def factor(self):
        kkt_factor(self.h)

    def solve(self, b, x, max_refine=10, tol_bwd=0.0):
        kkt_solve(self.h, b, x, max_refine, tol_bwd)

    def hykkt_solve(self, rbar1, rbar2, dx, dy, cg_rtol=1e-12, cg_maxit=0, max_outer_refine=2, krylov=0):
        if krylov:
            hykkt_solve_krylov(self.h, rbar1, rbar2, dx, dy, cg_rtol, cg_maxit, max_outer_refine, krylov)
        else:
            hykkt_solve(self.h, rbar1, rbar2, dx, dy, cg_rtol, cg_maxit, max_outer_refine)

    def solve_unreduced(self, x, s, u, v, f, d, max_refine=10, tol=0.0):
        kkt_solve_unreduced(self.h, x, s, u, v, f, d, max_refine, tol)

    def inertia(self):
        return kkt_inertia(self.h, self.batch)

    def factor_inertia_correct(self, W_vals, J_vals, Sigma_x, Sigma_s, D=None, delta_c=0.0, gamma=0.0, params=None):
        self._vals = (W_vals, J_vals, Sigma_x, Sigma_s, D)
        return kkt_factor_inertia_correct(self.h, W_vals, J_vals, Sigma_x, Sigma_s, D, delta_c, gamma, params)

    def recover(self, r2, r4, dx, dz, ds):
        kkt_recover(self.h, r2, r4, dx, dz, ds)

    def recover_bounds(self, x, u, s, v, mu, dx, ds, du, dv):
        kkt_recover_bounds(self.h, x, u, s, v, mu, dx, ds, du, dv)

    def sync_info(self):
        return kkt_sync_info(self.h)

    def get_condensed(self, inst=0, values=True):
        return kkt_get_condensed(self.h, inst, self.n, int(self.info["nnzK"]), values)

    def supernodes(self):
        return kkt_get_supernodes(self.h)

    def blocks(self, kind=0, cap=6144, nwarps=8):
        f, r, p = self.supernodes()
        return kkt_get_blocks(self.h, len(r), int(r.sum()), kind, cap, nwarps)

    def trace(self):
        return kkt_get_trace(self.h, int(self.info["nsuper"]))

    def launch_count(self):
        return kkt_launch_count(self.h)

    def hykkt_stats(self):
        return kkt_hykkt_stats(self.h)

    def factor_phase_ms(self):
        return kkt_factor_phase_ms(self.h)

    def close(self):
        if self.h:
            kkt_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
