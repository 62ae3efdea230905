"""Pins for oracle.cholesky, trisolve, solve_refined, backward_error -- CPU only.

Pins: numpy.linalg.cholesky (library routine) on P K P^T; reconstruction <= 1e-13 ||K||;
diagonal K -> L = sqrt(diag); first failing column on a non-SPD input (R6); exact rational
solutions (fractions Gaussian elimination) for the refined solve (R8); S:85-86 solve examples.
"""
import numpy as np
import pytest

import oracle
from oracle import dense
from synth.generator import make_config, tiny_random, KKTInstance


def _dense_lower(Kp, Ki, Kv, n):
    K = np.zeros((n, n))
    for j in range(n):
        for p in range(Kp[j], Kp[j + 1]):
            K[Ki[p], j] = Kv[p]; K[j, Ki[p]] = Kv[p]
    return K


def _Ldense(Lp, Li, Lx, n):
    L = np.zeros((n, n))
    for j in range(n):
        for p in range(Lp[j], Lp[j + 1]):
            L[Li[p], j] = Lx[p]
    return L


@pytest.mark.parametrize("cfg,Xi", [("C1", 1e-8), ("C5", 1e-2), ("C5", 1e-8)])
def test_cholesky_vs_numpy_and_reconstruction(cfg, Xi):
    """Entrywise agreement with numpy is only meaningful when K is well conditioned; at
    Xi = 1e-8 the two backward-stable factors differ by O(kappa u) and only the
    reconstruction bound is pinned."""
    inst = make_config(cfg) if cfg == "C1" else make_config("C5", batch=1, Xi=Xi)
    R = oracle.reference_solve(inst)
    n = inst.n
    K = _dense_lower(*R["K"], n)
    P = K[np.ix_(R["perm"], R["perm"])]
    L = _Ldense(R["Lp"], R["Li"], R["Lx"], n)
    assert np.abs(P - L @ L.T).max() <= 1e-13 * np.abs(K).max()
    if cfg == "C5" and Xi < 1e-4:
        return
    Lnp = np.linalg.cholesky(P)
    colscale = np.abs(Lnp).max(0)
    assert (np.abs(L - Lnp) <= 1e-11 * colscale[None, :]).all()


def test_diagonal_matrix_sqrt():
    n = 6
    rng = np.random.default_rng(3)
    d = rng.uniform(0.5, 4.0, n)
    inst = KKTInstance("diag", n, 0, 0, np.arange(n + 1, dtype=np.int32), np.arange(n, dtype=np.int32),
                       d, np.zeros(1, np.int32), np.zeros(0, np.int32), np.zeros(0), np.zeros(n),
                       np.zeros(0), b=np.arange(1.0, n + 1))
    R = oracle.reference_solve(inst)
    assert R["perm"].tolist() == list(range(n))
    assert np.array_equal(R["Lx"], np.sqrt(d))
    assert np.allclose(R["x"], np.arange(1.0, n + 1) / d, rtol=1e-16, atol=0)


def test_identity_and_diag_solves():
    """F of I, b=(1,2,3) -> (1,2,3); F of diag(2,4), b=(2,8) -> (1,2)."""
    for d, b, x in (([1.0, 1.0, 1.0], [1.0, 2.0, 3.0], [1.0, 2.0, 3.0]), ([2.0, 4.0], [2.0, 8.0], [1.0, 2.0])):
        n = len(d)
        inst = KKTInstance("d", n, 0, 0, np.arange(n + 1, dtype=np.int32), np.arange(n, dtype=np.int32),
                           np.array(d), np.zeros(1, np.int32), np.zeros(0, np.int32), np.zeros(0),
                           np.zeros(n), np.zeros(0), b=np.array(b))
        assert oracle.reference_solve(inst)["x"].tolist() == x


def test_not_spd_reports_first_column():
    """R6: LL^T fails iff a pivot <= 0; the first failing column is reported."""
    n = 3
    inst = KKTInstance("nspd", n, 0, 0, np.arange(n + 1, dtype=np.int32), np.arange(n, dtype=np.int32),
                       np.array([2.0, -3.0, 1.0]), np.zeros(1, np.int32), np.zeros(0, np.int32),
                       np.zeros(0), np.zeros(n), np.zeros(0), b=np.ones(n))
    R = oracle.reference_solve(inst)
    assert R["perm"][R["fail"]] == 1


@pytest.mark.parametrize("seed", [41, 42, 43, 44])
def test_refined_solution_is_exact_rational_solution(seed):
    """R8: x_ref equals the exact solution of the exact-input system, correctly rounded
    (tolerance 1 ulp), here with Sigma spanning 1e-6..1e6 and gamma rows."""
    inst = tiny_random(8, 6, 2, seed=seed, Xi=1e-6, hykkt_gamma=1e5, delta_w=1e-3, delta_c=1e-2)
    R = oracle.reference_solve(inst)
    xe = dense.exact_solve(dense.exact_condensed(inst), inst.b)
    xe = np.array([float(v) for v in xe])
    assert np.all(np.abs(R["x"] - xe) <= np.spacing(np.abs(xe)))


def test_backward_error_of_exact_solution_is_tiny_and_of_perturbed_is_not():
    inst = make_config("C5", batch=1)
    R = oracle.reference_solve(inst)
    eta, om = oracle.backward_error(inst, R["K"], inst.b, R["x"])
    assert eta <= 1e-16 and om <= 2.3e-16      # x rounded to double: omega <= ~u
    xp = R["x"] * (1 + 1e-9)
    eta2, om2 = oracle.backward_error(inst, R["K"], inst.b, xp)
    assert om2 > 1e-10


@pytest.mark.parametrize("seed", [51, 52])
def test_backward_error_equals_exact_rational_definition(seed):
    """R7 pinned exactly: eta = ||b - K x||_inf / (||K||_inf ||x||_inf + ||b||_inf) and
    omega = max_i |b - K x|_i / (|W||x| + |Sx+dw||x| + |J|^T |D| |J| |x| + |b|)_i, both written out
    here in exact rationals from dense matrices (both triangles of W, D of P:417-420), compared
    with the oracle's __float128 evaluation.  A dropped ||b||, a one-triangle ||K||, a missing
    W or J term in either denominator or a sign error in the residual all fail this test."""
    from fractions import Fraction as F
    inst = tiny_random(9, 7, 2, seed=seed, Xi=1e-3, hykkt_gamma=1e2, delta_w=1e-3, delta_c=1e-2)
    R = oracle.reference_solve(inst)
    rng = np.random.default_rng(seed)
    x = R["x"] * (1 + 1e-6 * rng.standard_normal(inst.n))     # residual well above rounding
    eta, om = oracle.backward_error(inst, R["K"], inst.b, x)
    n = inst.n
    Kx = dense.exact_condensed(inst)                          # exact K of the exact inputs
    xf = [F(float(v)) for v in x]
    bf = [F(float(v)) for v in inst.b]
    res = [bf[i] - sum(Kx[i][j] * xf[j] for j in range(n)) for i in range(n)]
    # ||K||_inf of the K that was passed (the oracle's correctly rounded K), both triangles
    Kp, Ki, Kv = R["K"]
    rs = [F(0)] * n
    for j in range(n):
        for p in range(Kp[j], Kp[j + 1]):
            a = abs(F(float(Kv[p])))
            rs[Ki[p]] += a
            if Ki[p] != j:
                rs[j] += a
    eta_ex = max(abs(v) for v in res) / (max(rs) * max(abs(v) for v in xf) + max(abs(v) for v in bf))
    # componentwise denominators of the unassembled operator
    W = [[F(0)] * n for _ in range(n)]
    for i in range(n):
        for p in range(inst.W_rowptr[i], inst.W_rowptr[i + 1]):
            j = int(inst.W_colind[p]); w = F(float(inst.W_vals[p]))
            W[i][j] += w
            if j != i:
                W[j][i] += w
    den = [abs(F(float(inst.Sigma_x[i])) + F(float(inst.delta_w))) * abs(xf[i]) + abs(bf[i]) +
           sum(abs(W[i][j]) * abs(xf[j]) for j in range(n)) for i in range(n)]
    for r in range(inst.m):
        if r < inst.m_eq:
            D = F(float(inst.gamma))
        else:
            t = F(float(inst.Sigma_s[r - inst.m_eq])) + F(float(inst.delta_w))
            D = t / (1 + F(float(inst.delta_c)) * t)
        cols = [(int(inst.J_colind[p]), F(float(inst.J_vals[p])))
                for p in range(inst.J_rowptr[r], inst.J_rowptr[r + 1])]
        t = abs(D) * sum(abs(v) * abs(xf[c]) for c, v in cols)
        for c, v in cols:
            den[c] += abs(v) * t
    om_ex = max(abs(res[i]) / den[i] for i in range(n))
    assert eta > 0 and om > 0
    assert abs(eta - float(eta_ex)) <= 1e-13 * float(eta_ex)
    assert abs(om - float(om_ex)) <= 1e-13 * float(om_ex)


def test_plain_fp64_solve_is_not_enough_in_stress_regime():
    """Appendix-A probe: in the 0 < l < n regime the unrefined FP64 solve misses x_ref
    by far more than 1e-8 -- the reason kkt_solve refines with a double-double residual."""
    inst = make_config("C2s")
    R = oracle.reference_solve(inst)
    x0 = oracle.trisolve(inst.n, R["Lp"], R["Li"], R["Lx"], R["perm"], inst.b)
    err = np.abs(x0 - R["x"]).max() / np.abs(R["x"]).max()
    assert err > 1e-11


def _dense_K(inst):
    Kp, Ki, Kv = oracle.condense(inst)
    n = inst.n
    A = np.zeros((n, n))
    for j in range(n):
        for p in range(Kp[j], Kp[j + 1]):
            A[Ki[p], j] = Kv[p]; A[j, Ki[p]] = Kv[p]
    return (Kp, Ki, Kv), A


def _ldlt_of(inst):
    K, A = _dense_K(inst)
    perm = oracle.md_order(inst.n, K[0], K[1])
    _, _, Lp, Li = oracle.symbolic(inst.n, K[0], K[1], perm, want_pattern=True)
    Lx, inert, fail = oracle.ldlt(inst.n, K[0], K[1], K[2], perm, Lp, Li)
    return K, A, perm, Lp, Li, Lx, inert, fail


@pytest.mark.parametrize("seed", range(6))
def test_ldlt_inertia_equals_eigenvalue_counts(seed):
    """NEXT-2 pin (Sylvester): the pivot-free LDL^T's (positive, negative, zero)
    pivot counts equal the signs of the eigenvalues of K (numpy eigvalsh) on indefinite inputs
    (W with an indefinite diagonal), and L D L^T reproduces P K P^T."""
    inst = tiny_random(24, 10, 0, seed=200 + seed, Xi=1e-2, w_psd=False)
    K, A, perm, Lp, Li, Lx, inert, fail = _ldlt_of(inst)
    assert fail < 0
    ev = np.linalg.eigvalsh(A)
    assert np.min(np.abs(ev)) > 1e-8 * np.max(np.abs(ev))      # nonsingular test matrix
    assert inert == (int((ev > 0).sum()), int((ev < 0).sum()), 0)
    n = inst.n
    L = np.eye(n); d = np.zeros(n)
    for j in range(n):
        d[j] = Lx[Lp[j]]
        for p in range(Lp[j] + 1, Lp[j + 1]):
            L[Li[p], j] = Lx[p]
    PA = A[np.ix_(perm, perm)]
    assert np.abs(L @ np.diag(d) @ L.T - PA).max() <= 1e-12 * np.abs(A).max()
    x = oracle.ldlt_solve(n, Lp, Li, Lx, perm, inst.b)
    assert np.abs(A @ x - inst.b).max() <= 1e-9 * (np.abs(A).max() * np.abs(x).max() + np.abs(inst.b).max())


def test_ldlt_textbook_and_spd_cases():
    """diag(-1, 2, -3) -> inertia (1, 2, 0); an SPD K gives d_j = (Cholesky l_jj)^2 and (n, 0, 0);
    an exactly singular K (zero row) counts one zero pivot (R6)."""
    from synth.generator import KKTInstance
    def diag_inst(dv):
        n = len(dv)
        return KKTInstance("d", n, 0, 0, np.arange(n + 1, dtype=np.int32), np.arange(n, dtype=np.int32),
                           np.array(dv, float), np.zeros(1, np.int32), np.zeros(0, np.int32), np.zeros(0),
                           np.zeros(n), np.zeros(0), b=np.ones(n))
    _, _, _, _, _, _, inert, _ = _ldlt_of(diag_inst([-1.0, 2.0, -3.0]))
    assert inert == (1, 2, 0)
    _, _, _, _, _, _, inert, _ = _ldlt_of(diag_inst([4.0, 0.0, 1.0]))
    assert inert == (2, 0, 1)
    inst = make_config("C5", batch=1, Xi=1e-2)     # well-conditioned: pivots agree to rounding
    K, A, perm, Lp, Li, Lx, inert, fail = _ldlt_of(inst)
    assert inert == (inst.n, 0, 0) and fail < 0
    Lc, f2 = oracle.cholesky(inst.n, K[0], K[1], K[2], perm, Lp, Li)
    d = np.array([Lx[Lp[j]] for j in range(inst.n)])
    lc = np.array([Lc[Lp[j]] for j in range(inst.n)])
    assert np.all(np.abs(d - lc * lc) <= 1e-11 * d)


def test_inertia_correction_rule():
    """Wachter-Biegler primal correction in the oracle: an SPD K keeps
    delta_w = 0; an indefinite W is shifted until the LDL^T inertia is (n, 0, 0), with the
    delta_w sequence 1e-4 x 100^k of the rule -- and the accepted shift exceeds -lambda_min."""
    inst = tiny_random(30, 12, 0, seed=9, Xi=1e-2)
    dw, tries, inert = oracle.inertia_correct(inst)
    assert dw == 0.0 and tries == 1 and inert == (30, 0, 0)
    bad = tiny_random(30, 12, 0, seed=9, Xi=1e-2, w_psd=False)
    dw, tries, inert = oracle.inertia_correct(bad)
    assert inert == (30, 0, 0) and tries >= 2
    assert dw == 1e-4 * 100.0 ** (tries - 2)
    _, A = _dense_K(bad)
    lam = np.linalg.eigvalsh(A).min()
    assert lam < 0 and dw > -lam
    _, A2 = _dense_K(bad)
    assert np.linalg.eigvalsh(A2 + (dw / 100.0) * np.eye(30)).min() < 0 or tries == 2
