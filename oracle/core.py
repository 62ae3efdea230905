"""ctypes front-end of oracle/oracle.c (plain C, __float128 accumulation).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  The shared object is built from
oracle/oracle.c alone with gcc (``build()``); nothing here touches the CUDA path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading
import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None
_lock = threading.Lock()

_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


class OracleSystem(C.Structure):
    """Mirror of `osys` in oracle.c."""
    _fields_ = [("n", C.c_int), ("m", C.c_int), ("m_eq", C.c_int),
                ("Wp", C.c_void_p), ("Wc", C.c_void_p), ("Wv", C.c_void_p),
                ("Jp", C.c_void_p), ("Jc", C.c_void_p), ("Jv", C.c_void_p),
                ("Sx", C.c_void_p), ("Ss", C.c_void_p), ("D", C.c_void_p),
                ("dw", C.c_double), ("dc", C.c_double), ("gamma", C.c_double)]


def build(force: bool = False) -> str:
    """Compile liboracle.so from oracle.c (gcc -O2, libquadmath)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-fPIC", "-shared", "-o", tmp, _SRC,
                               "-lquadmath", "-lm"])
        os.replace(tmp, _SO)
    return _SO


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = C.CDLL(build())
            P = C.c_void_p
            lib.oracle_condense.restype = C.c_long
            lib.oracle_condense.argtypes = [C.POINTER(OracleSystem), P, P, P]
            lib.oracle_md_order.argtypes = [C.c_int, P, P, P]
            lib.oracle_symbolic.restype = C.c_long
            lib.oracle_symbolic.argtypes = [C.c_int, P, P, P, P, P, P, P]
            lib.oracle_cholesky.argtypes = [C.c_int, P, P, P, P, P, P, P]
            lib.oracle_trisolve.argtypes = [C.c_int, P, P, P, P, P, P]
            lib.oracle_apply.argtypes = [C.POINTER(OracleSystem), C.c_int, P, P]
            lib.oracle_solve_refined.argtypes = [C.POINTER(OracleSystem), P, P, P, P, P, P, P,
                                                 C.c_int, C.c_double]
            lib.oracle_backward_error.restype = C.c_double
            lib.oracle_backward_error.argtypes = [C.POINTER(OracleSystem), P, P, P, P, P, P]
            lib.oracle_cg_dense.argtypes = [C.c_int, P, P, P, C.c_double, C.c_int, P]
            lib.oracle_cr_dense.argtypes = [C.c_int, P, P, P, C.c_double, C.c_int, P, P]
            lib.oracle_ldlt.argtypes = [C.c_int, P, P, P, P, P, P, P, P]
            lib.oracle_ldlt_solve.argtypes = [C.c_int, P, P, P, P, P, P]
            lib.oracle_ldlt_solve.restype = None
            lib.oracle_hykkt.argtypes = [C.POINTER(OracleSystem), P, P, P, P, P, P, P, P,
                                         C.c_double, C.c_int, C.c_int, P, P]
            _lib = lib
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


class _Sys:
    """Holds contiguous copies alive while the C struct points at them."""

    def __init__(self, inst, D=None):
        self.keep = [_i32(inst.W_rowptr), _i32(inst.W_colind), _f64(inst.W_vals),
                     _i32(inst.J_rowptr), _i32(inst.J_colind), _f64(inst.J_vals),
                     _f64(inst.Sigma_x), _f64(inst.Sigma_s) if inst.Sigma_s.size else np.zeros(1),
                     _f64(D)]
        k = self.keep
        self.s = OracleSystem(inst.n, inst.m, inst.m_eq, _p(k[0]), _p(k[1]), _p(k[2]), _p(k[3]),
                              _p(k[4]), _p(k[5]), _p(k[6]), _p(k[7]), _p(k[8]),
                              float(inst.delta_w), float(inst.delta_c), float(inst.gamma))

    def ref(self):
        return C.byref(self.s)


def condense(inst, D=None):
    """K = W + D_x + delta_w I + J^T D J, lower CSC in original indices.
    Returns (Kp, Ki, Kv); every entry is the once-rounded __float128 sum."""
    lib = _load()
    S = _Sys(inst, D)
    Kp = np.zeros(inst.n + 1, np.int32)
    nnz = lib.oracle_condense(S.ref(), _p(Kp), None, None)
    Ki = np.zeros(max(nnz, 1), np.int32)
    Kv = np.zeros(max(nnz, 1), np.float64)
    lib.oracle_condense(S.ref(), _p(Kp), _p(Ki), _p(Kv))
    return Kp, Ki[:nnz], Kv[:nnz]


def md_order(n, Kp, Ki):
    """MD-exact-v1 ordering (R11); perm[new] = old."""
    lib = _load()
    Kp, Ki = _i32(Kp), _i32(Ki)
    perm = np.zeros(max(n, 1), np.int32)
    lib.oracle_md_order(n, _p(Kp), _p(Ki), _p(perm))
    return perm[:n]


def symbolic(n, Kp, Ki, perm, want_pattern=False):
    """etree parent[], colcount[] (incl. diagonal) of P K P^T; optionally (Lp, Li)."""
    lib = _load()
    Kp, Ki, perm = _i32(Kp), _i32(Ki), _i32(perm)
    parent = np.zeros(max(n, 1), np.int32)
    cc = np.zeros(max(n, 1), np.int32)
    nnzL = lib.oracle_symbolic(n, _p(Kp), _p(Ki), _p(perm), _p(parent), _p(cc), None, None)
    if not want_pattern:
        return parent[:n], cc[:n]
    Lp = np.zeros(n + 1, np.int32)
    Li = np.zeros(max(nnzL, 1), np.int32)
    lib.oracle_symbolic(n, _p(Kp), _p(Ki), _p(perm), _p(parent), _p(cc), _p(Lp), _p(Li))
    return parent[:n], cc[:n], Lp, Li[:nnzL]


def cholesky(n, Kp, Ki, Kv, perm, Lp, Li):
    """L of P K P^T on pattern (Lp, Li).  Returns (Lx, fail) with fail = -1 or first bad column."""
    lib = _load()
    Lx = np.zeros(max(int(Lp[-1]), 1), np.float64)
    fail = lib.oracle_cholesky(n, _p(_i32(Kp)), _p(_i32(Ki)), _p(_f64(Kv)), _p(_i32(perm)),
                               _p(_i32(Lp)), _p(_i32(Li)), _p(Lx))
    return Lx[:int(Lp[-1])], fail


def trisolve(n, Lp, Li, Lx, perm, b):
    lib = _load()
    x = np.zeros(max(n, 1), np.float64)
    lib.oracle_trisolve(n, _p(_i32(Lp)), _p(_i32(Li)), _p(_f64(Lx)), _p(_i32(perm)),
                        _p(_f64(b)), _p(x))
    return x[:n]


def apply_operator(inst, x, exclude_eq=False, D=None):
    """Unassembled operator W x + (Sx+dw) x + sum_r J_r^T D_r J_r x, __float128, rounded once."""
    lib = _load()
    S = _Sys(inst, D)
    y = np.zeros(max(inst.n, 1), np.float64)
    lib.oracle_apply(S.ref(), int(exclude_eq), _p(_f64(x)), _p(y))
    return y[:inst.n]


def solve_refined(inst, Lp, Li, Lx, perm, b, max_sweeps=30, stop_rel=1e-25, D=None):
    """x_ref: Richardson with __float128 unassembled residual (R8/R9). Returns (x_hi, x_lo, sweeps)."""
    lib = _load()
    S = _Sys(inst, D)
    n = inst.n
    xh = np.zeros(max(n, 1)); xl = np.zeros(max(n, 1))
    sw = lib.oracle_solve_refined(S.ref(), _p(_i32(Lp)), _p(_i32(Li)), _p(_f64(Lx)), _p(_i32(perm)),
                                  _p(_f64(b)), _p(xh), _p(xl), int(max_sweeps), float(stop_rel))
    return xh[:n], xl[:n], sw


def backward_error(inst, K, b, x, D=None):
    """(eta, omega): normwise and componentwise backward errors (R7), residual in __float128."""
    lib = _load()
    S = _Sys(inst, D)
    Kp, Ki, Kv = K
    om = C.c_double(0.0)
    eta = lib.oracle_backward_error(S.ref(), _p(_i32(Kp)), _p(_i32(Ki)), _p(_f64(Kv)),
                                    _p(_f64(b)), _p(_f64(x)), C.byref(om))
    return eta, om.value


def cg_dense(A, b, rtol=1e-12, maxit=1000):
    """Hestenes-Stiefel CG on a dense SPD matrix.  Returns (x, status, iters)."""
    lib = _load()
    A = np.ascontiguousarray(A, dtype=np.float64)
    n = A.shape[0]
    x = np.zeros(max(n, 1))
    it = C.c_int(0)
    st = lib.oracle_cg_dense(n, _p(A), _p(_f64(b)), _p(x), float(rtol), int(maxit), C.byref(it))
    return x[:n], st, it.value


def ldlt(n, Kp, Ki, Kv, perm, Lp, Li):
    """Pivot-free LDL^T on the symbolic pattern (unit L below the diagonal slots, d_j in them).
    Returns (Lx, inertia (pos, neg, zero), first non-finite pivot or -1)."""
    lib = _load()
    Lx = np.zeros(max(int(Lp[n]), 1))
    inert = np.zeros(3, np.int32)
    fail = lib.oracle_ldlt(n, _p(_i32(Kp)), _p(_i32(Ki)), _p(_f64(Kv)), _p(_i32(perm)), _p(_i32(Lp)),
                           _p(_i32(Li)), _p(Lx), _p(inert))
    return Lx, tuple(int(v) for v in inert), fail


def ldlt_solve(n, Lp, Li, Lx, perm, b):
    lib = _load()
    x = np.zeros(max(n, 1))
    lib.oracle_ldlt_solve(n, _p(_i32(Lp)), _p(_i32(Li)), _p(_f64(Lx)), _p(_i32(perm)), _p(_f64(b)), _p(x))
    return x[:n]


def inertia_correct(inst, params=None):
    """Wachter-Biegler primal inertia correction with the oracle LDL^T:
    the delta_w sequence of kkt_factor_inertia_correct.  Returns (delta_w, tries, inertia)."""
    import copy
    dw_min, dw_first, dw_max, k_minus, k_plus, k_plus_bar, dw_last = (
        params if params is not None else (1e-20, 1e-4, 1e40, 1.0 / 3.0, 8.0, 100.0, 0.0))
    base = condense(inst)
    perm = md_order(inst.n, base[0], base[1])
    _, _, Lp, Li = symbolic(inst.n, base[0], base[1], perm, want_pattern=True)

    def inertia_at(dw):
        it = copy.copy(inst)
        it.delta_w = dw
        K = condense(it)
        _, inert, fail = ldlt(inst.n, K[0], K[1], K[2], perm, Lp, Li)
        return inert, fail

    tries = 1
    inert, fail = inertia_at(0.0)
    ok = lambda t, f: f < 0 and t == (inst.n, 0, 0)
    if ok(inert, fail):
        return 0.0, tries, inert
    dw = dw_first if dw_last == 0.0 else max(dw_min, k_minus * dw_last)
    while True:
        inert, fail = inertia_at(dw)
        tries += 1
        if ok(inert, fail):
            return dw, tries, inert
        dw = k_plus_bar * dw if dw_last == 0.0 else k_plus * dw
        if dw > dw_max:
            return dw, tries, None


def cr_dense(A, b, rtol=1e-12, maxit=1000):
    """Conjugate residuals (Hestenes-Stiefel) on a dense SPD matrix.
    Returns (x, status, iters, residual-norm history [iters + 1])."""
    lib = _load()
    A = np.ascontiguousarray(A, dtype=np.float64)
    n = A.shape[0]
    x = np.zeros(max(n, 1))
    hist = np.zeros(maxit + 1)
    it = C.c_int(0)
    st = lib.oracle_cr_dense(n, _p(A), _p(_f64(b)), _p(x), float(rtol), int(maxit), C.byref(it), _p(hist))
    return x[:n], st, it.value, hist[:it.value + 1]


def hykkt(inst, Lp, Li, Lx, perm, rbar1, rbar2, cg_rtol=1e-12, cg_maxit=2000, max_outer=30):
    """HyKKT + __float128 outer refinement on [K G^T; G 0].
    Returns (dx, dy, cg_status, cg_iters_first_pass, outer_sweeps)."""
    lib = _load()
    S = _Sys(inst)
    n, me = inst.n, inst.m_eq
    dx = np.zeros(max(n, 1)); dy = np.zeros(max(me, 1))
    it = C.c_int(0); ou = C.c_int(0)
    r2 = _f64(rbar2) if me else np.zeros(1)
    st = lib.oracle_hykkt(S.ref(), _p(_i32(Lp)), _p(_i32(Li)), _p(_f64(Lx)), _p(_i32(perm)),
                          _p(_f64(rbar1)), _p(r2), _p(dx), _p(dy), float(cg_rtol), int(cg_maxit),
                          int(max_outer), C.byref(it), C.byref(ou))
    return dx[:n], dy[:me], st, it.value, ou.value


def reference_solve(inst, b=None, D=None, max_sweeps=30):
    """Whole oracle pipeline for the condensed solve: condense -> MD -> symbolic -> Cholesky ->
    refined solve.  Returns dict with K, perm, parent, colcount, L, x (exact-input solution)."""
    b = inst.b if b is None else b
    K = condense(inst, D)
    perm = md_order(inst.n, K[0], K[1])
    parent, cc, Lp, Li = symbolic(inst.n, K[0], K[1], perm, want_pattern=True)
    Lx, fail = cholesky(inst.n, K[0], K[1], K[2], perm, Lp, Li)
    out = dict(K=K, perm=perm, parent=parent, colcount=cc, Lp=Lp, Li=Li, Lx=Lx, fail=fail)
    if fail < 0:
        xh, xl, sw = solve_refined(inst, Lp, Li, Lx, perm, b, max_sweeps=max_sweeps, D=D)
        out.update(x=xh, x_lo=xl, sweeps=sw)
    return out


def reference_hykkt(inst, cg_rtol=1e-12, cg_maxit=2000, max_outer=30):
    """Oracle HyKKT pipeline: condense K_gamma -> MD -> symbolic -> Cholesky -> HyKKT + refinement."""
    K = condense(inst)
    perm = md_order(inst.n, K[0], K[1])
    parent, cc, Lp, Li = symbolic(inst.n, K[0], K[1], perm, want_pattern=True)
    Lx, fail = cholesky(inst.n, K[0], K[1], K[2], perm, Lp, Li)
    out = dict(K=K, perm=perm, parent=parent, colcount=cc, Lp=Lp, Li=Li, Lx=Lx, fail=fail)
    if fail < 0:
        dx, dy, st, it, ou = hykkt(inst, Lp, Li, Lx, perm, inst.rbar1, inst.rbar2, cg_rtol,
                                   cg_maxit, max_outer)
        out.update(dx=dx, dy=dy, cg_status=st, cg_iters=it, outer=ou)
    return out
