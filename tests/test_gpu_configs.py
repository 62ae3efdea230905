"""CUDA path vs oracle on every BASELINE config at full size, plus the refinement and variant
checks the round-1 review asked for (-m gpu; B200).

Bars (BASELINE.json north_star, DESIGN.md §3 R7-R9):
  solve:     ||x - x_ref||_inf / ||x_ref||_inf <= 1e-8 (the contract) and, with refinement on,
             <= 1e-12 (R9 refines to a predicted forward error of 1e-14 ||x||);  eta <= 1e-10
  condense:  per entry |K_gpu - K_ref| <= 2 (t_ij + 1) u sum|terms| (t_ij = terms of the entry:
             W, the diagonal Sigma_x + delta_w, one product per J row touching both indices)
  HyKKT:     dx, dy relative error <= 1e-8 vs the oracle's refined saddle solution
"""
import numpy as np
import pytest

import oracle
from synth.generator import make_config, acopf

pytestmark = pytest.mark.gpu

U = 2.0 ** -53


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA not available: the -m gpu suite needs a B200 (no CPU fallback exists)")


def _terms_and_abs(inst):
    """Per K entry (oracle's lower CSC order): number of terms t_ij and sum of |terms|."""
    Kp, Ki, _ = oracle.condense(inst)
    n = inst.n
    key = {}
    for j in range(n):
        for p in range(Kp[j], Kp[j + 1]):
            key[(int(Ki[p]), j)] = p
    t = np.zeros(len(Ki))
    a = np.zeros(len(Ki))
    for i in range(n):
        for p in range(inst.W_rowptr[i], inst.W_rowptr[i + 1]):
            j = int(inst.W_colind[p])
            q = key[(max(i, j), min(i, j))]
            t[q] += 1
            a[q] += abs(inst.W_vals[p])
    for i in range(n):
        q = key[(i, i)]
        t[q] += 2
        a[q] += abs(inst.Sigma_x[i]) + abs(inst.delta_w)
    D = np.empty(inst.m)
    D[:inst.m_eq] = inst.gamma
    s = inst.Sigma_s + inst.delta_w
    D[inst.m_eq:] = s / (1 + inst.delta_c * s)
    for r in range(inst.m):
        cols = inst.J_colind[inst.J_rowptr[r]:inst.J_rowptr[r + 1]]
        vals = inst.J_vals[inst.J_rowptr[r]:inst.J_rowptr[r + 1]]
        for x_ in range(len(cols)):
            for y_ in range(x_, len(cols)):
                q = key[(max(cols[x_], cols[y_]), min(cols[x_], cols[y_]))]
                t[q] += 1
                a[q] += abs(D[r] * vals[x_] * vals[y_])
    return t, a


@pytest.mark.parametrize("case", ["C1", "C5i", "C2", "C2s"])
def test_condense_per_entry_bound(case):
    """SURVEY §8(c) condensation pin: componentwise a-priori bound per entry."""
    from kkt_gpu import run_lifted
    inst = make_config("C5", batch=1) if case == "C5i" else make_config(case)
    _, _, S = run_lifted(inst, max_refine=0)
    Kp, Ki, Kv = S.get_condensed(0)
    Op, Oi, Ov = oracle.condense(inst)
    assert np.array_equal(Kp, Op) and np.array_equal(Ki, Oi)
    t, a = _terms_and_abs(inst)
    err = np.abs(Kv - Ov)
    bound = 2 * (t + 1) * U * a
    assert np.all(err <= bound), float((err / np.maximum(bound, 1e-300)).max())
    S.close()


@pytest.mark.parametrize("case", ["C2", "C2s", "C5i"])
def test_refined_forward_error_is_tight(case):
    """R9 refines until the predicted forward error is 1e-14 ||x||: the refined x must be far
    inside the 1e-8 contract; the ill-conditioned stress case needs more than one correction
    (a stop rule that always quits after one correction fails here)."""
    from kkt_gpu import run_lifted, relerr
    inst = make_config("C5", batch=1) if case == "C5i" else make_config(case)
    R = oracle.reference_solve(inst)
    x, info, S = run_lifted(inst, max_refine=10)
    assert info["status"] == 0, info
    assert relerr(x, R["x"]) <= 1e-12, (relerr(x, R["x"]), info)
    if case == "C2s":
        x0 = oracle.trisolve(inst.n, R["Lp"], R["Li"], R["Lx"], R["perm"], inst.b)
        assert relerr(x0, R["x"]) > 1e-11          # plain FP64 is far off here (Appendix A)
        assert info["refine_iters"] >= 2, info
    S.close()


@pytest.mark.parametrize("relax_big,zero_frac", [(64, 0.05), (160, 0.3), (192, 0.5)])
def test_unrefined_linv_vs_substitution(relax_big, zero_frac, monkeypatch):
    """The L11^-1 sweeps (linv_kernel, nb = 2..6 under coarser amalgamation) without any
    refinement: on a well-conditioned instance the plain FP64 solve must match the oracle to
    1e-10 and the substitution path (KKT_NO_LINV=1) to 1e-11 -- refinement cannot hide a wrong
    inverse here."""
    import paper_2405_14236_b200 as K
    from kkt_gpu import run_lifted, relerr
    inst = make_config("C2", Xi=1e-2)
    R = oracle.reference_solve(inst)
    S = K.KKTSolver.from_instance(inst, relax_big=relax_big, relax_zero_frac=zero_frac).bind(0)
    x, info, S = run_lifted(inst, max_refine=0, solver=S)
    S.close()
    monkeypatch.setenv("KKT_NO_LINV", "1")
    S2 = K.KKTSolver.from_instance(inst, relax_big=relax_big, relax_zero_frac=zero_frac).bind(0)
    x2, info2, S2 = run_lifted(inst, max_refine=0, solver=S2)
    S2.close()
    assert info["status"] == 0 and info2["status"] == 0
    assert relerr(x, R["x"]) <= 1e-10, relerr(x, R["x"])
    assert relerr(x, x2) <= 1e-11, relerr(x, x2)


def test_c4_parity():
    """C4 (78,484-bus ACOPF, the bench headline) against the oracle's exact-input solution."""
    from kkt_gpu import run_lifted, relerr
    inst = make_config("C4")
    R = oracle.reference_solve(inst)
    x, info, S = run_lifted(inst, max_refine=10)
    assert info["status"] == 0, info
    assert relerr(x, R["x"]) <= 1e-8, (relerr(x, R["x"]), info)
    eta, _ = oracle.backward_error(inst, R["K"], inst.b, x)
    assert eta <= 1e-10, eta
    # ordering / etree exported by the GPU handle are the oracle's, bit for bit
    perm, et, cc = S.symbolic()
    assert np.array_equal(perm, R["perm"]) and np.array_equal(et, R["parent"])
    S.close()


def test_c5_full_batch_sampled_parity():
    """The full 512-instance batch (the throughput variant of the small-front kernel runs at
    this size): sampled instances against the oracle and bitwise against single-instance runs."""
    from kkt_gpu import run_lifted, relerr
    inst = make_config("C5")
    assert inst.batch == 512
    xb, info, S = run_lifted(inst, max_refine=10)
    assert info["status"] == 0, info
    xb = xb.reshape(512, -1)
    for k in (0, 1, 77, 255, 256, 400, 510, 511):
        one = inst.instance(k)
        R = oracle.reference_solve(one)
        assert relerr(xb[k], R["x"]) <= 1e-8, (k, relerr(xb[k], R["x"]))
        x1, _, S1 = run_lifted(one, max_refine=10)
        assert np.array_equal(x1, xb[k]), k
        S1.close()
    S.close()


def test_fsmall_occ3_variant(monkeypatch):
    """The occupancy-capped small-front factor kernel forced on C2: oracle parity, and the same
    bits as the default variant (identical arithmetic)."""
    from kkt_gpu import run_lifted, relerr
    inst = make_config("C2")
    R = oracle.reference_solve(inst)
    x0, _, S0 = run_lifted(inst, max_refine=10)
    S0.close()
    monkeypatch.setenv("KKT_FSMALL_OCC", "3")
    x, info, S = run_lifted(inst, max_refine=10)
    assert info["status"] == 0
    assert relerr(x, R["x"]) <= 1e-8
    assert np.array_equal(x, x0)
    S.close()


@pytest.mark.parametrize("gamma,Xi", [(1e4, None), (1e5, None), (1e6, None), (1e7, 1e-8)])
def test_hykkt_C3_gamma_sweep(gamma, Xi):
    """C3 at the north star's gamma range (Fig. 1) with Xi = 1/gamma, plus the
    stress pairing Xi = 1e-8 (SURVEY ledger 15)."""
    from kkt_gpu import run_hykkt, relerr
    kw = {} if Xi is None else {"Xi": Xi}
    inst = make_config("C3", gamma=gamma, **kw)
    R = oracle.reference_hykkt(inst)
    dx, dy, info, S = run_hykkt(inst, max_outer=3)
    assert info["status"] == 0, info
    assert relerr(dx, R["dx"]) <= 1e-8 and relerr(dy, R["dy"]) <= 1e-8, \
        (relerr(dx, R["dx"]), relerr(dy, R["dy"]), info)
    S.close()


def _dense_schur(inst):
    """Dense K_gamma (oracle condensation), G and the HyKKT right-hand side of eq. 14."""
    from oracle import dense
    Kp, Ki, Kv = oracle.condense(inst)
    n, me = inst.n, inst.m_eq
    Kg = np.zeros((n, n))
    for j in range(n):
        for p in range(Kp[j], Kp[j + 1]):
            Kg[Ki[p], j] = Kv[p]
            Kg[j, Ki[p]] = Kv[p]
    G = dense.dense_J(inst)[:me]
    s = inst.rbar1 + inst.gamma * G.T @ inst.rbar2
    Kinv_GT = np.linalg.solve(Kg, G.T)
    return G @ Kinv_GT, G @ np.linalg.solve(Kg, s) - inst.rbar2


@pytest.mark.parametrize("krylov", [0, 1])
@pytest.mark.parametrize("seed,gamma", [(1, 1e3), (2, 1e6)])
def test_hykkt_krylov_tiny_parity_and_counts(krylov, seed, gamma):
    """CG (krylov 0) and CR (krylov 1) on the device loop: solution parity with the
    oracle's refined saddle solution, and the first pass's iteration count within one of the
    oracle's cg_dense / cr_dense on the explicitly formed S_gamma = G K_gamma^-1 G^T."""
    from kkt_gpu import run_hykkt, relerr
    from synth.generator import tiny_random
    inst = tiny_random(60, 40, 15, seed=seed, Xi=1.0 / gamma, hykkt_gamma=gamma)
    R = oracle.reference_hykkt(inst)
    dx, dy, info, S = run_hykkt(inst, max_outer=3, krylov=krylov)
    assert info["status"] == 0, info
    assert relerr(dx, R["dx"]) <= 1e-8 and relerr(dy, R["dy"]) <= 1e-8
    Sg, rhs = _dense_schur(inst)
    if krylov == 0:
        _, st, it = oracle.cg_dense(Sg, rhs, rtol=1e-12, maxit=2000)
    else:
        _, st, it, _ = oracle.cr_dense(Sg, rhs, rtol=1e-12, maxit=2000)
    assert st == 0 and abs(info["cg_iters"] - it) <= 1, (info["cg_iters"], it)
    S.close()


@pytest.mark.parametrize("gamma", [1e4, 1e7])
def test_hykkt_cr_C3(gamma):
    """Conjugate residuals on C3 (HyKKT, 10k buses): parity with the oracle."""
    from kkt_gpu import run_hykkt, relerr
    inst = make_config("C3", gamma=gamma)
    R = oracle.reference_hykkt(inst)
    dx, dy, info, S = run_hykkt(inst, max_outer=3, krylov=1)
    assert info["status"] == 0, info
    assert relerr(dx, R["dx"]) <= 1e-8 and relerr(dy, R["dy"]) <= 1e-8, \
        (relerr(dx, R["dx"]), relerr(dy, R["dy"]), info)
    S.close()


def test_hykkt_is_graph_launched_without_host_sync():
    """hykkt_solve enqueues one recorded graph: a second call with the same pointers re-uses
    it, and the launch counter (read after the fact) includes the executed Krylov bodies."""
    import torch
    from kkt_gpu import run_hykkt, relerr
    inst = make_config("C3", gamma=1e6)
    dx, dy, info, S = run_hykkt(inst, max_outer=2)
    n1 = S.launch_count()
    assert n1 > 10 * max(info["cg_iters"], 1)
    # work counts: the Krylov total covers every pass (at least the first pass's count), the
    # outer passes match kkt_sync_info's report, and the launch count is consistent with them
    st = S.hykkt_stats()
    assert st["krylov_total"] >= info["cg_iters"] >= 1, (st, info)
    assert st["outer_passes"] == info["refine_iters"] and 0 <= st["outer_passes"] <= 2, (st, info)
    assert n1 >= 5 * st["krylov_total"], (n1, st)
    dx2, dy2, info2, _ = run_hykkt(inst, max_outer=2, solver=S)
    assert np.array_equal(dx, dx2) and np.array_equal(dy, dy2)     # deterministic
    S.close()


def _k3_case(n, me, mi, seed, dw=0.0, dc=0.0, gamma=0.0):
    """Tiny IPM-like K3 system: instance pattern/values plus x, s, u, v > 0 and f blocks."""
    from synth.generator import tiny_random
    from oracle import dense
    inst = tiny_random(n, mi + me, me, seed=seed, Xi=1.0, delta_w=dw, delta_c=dc,
                       hykkt_gamma=gamma if me else 0.0)
    rng = np.random.default_rng(seed + 100)
    x, u = rng.uniform(0.5, 2, n), rng.uniform(0.5, 2, n)
    s, v = rng.uniform(0.5, 2, mi), rng.uniform(0.5, 2, mi)
    f = [rng.standard_normal(k) for k in (n, mi, me, mi, n, mi)]
    J = dense.dense_J(inst)
    K3 = dense.k3_matrix(dense.dense_W(inst), J[:me], J[me:], x, s, u, v)
    dref = np.linalg.solve(K3, np.concatenate(f))
    inst.Sigma_x = u / x
    inst.Sigma_s = v / s
    return inst, (x, s, u, v), f, dense.k3_split(dref, n, me, mi)


def _run_k3(inst, xsuv, f, max_refine):
    import torch
    import paper_2405_14236_b200 as K
    from kkt_gpu import dev
    n, me, mi = inst.n, inst.m_eq, inst.m - inst.m_eq
    S = K.KKTSolver.from_instance(inst).bind(0)
    g = lambda a: dev(a, "cuda:0") if (a is not None and a.size) else None
    W, J, Sx, Ss = g(inst.W_vals), g(inst.J_vals), g(inst.Sigma_x), g(inst.Sigma_s)
    S.condense(W, J, Sx, Ss, None, inst.delta_w, inst.delta_c, inst.gamma)
    S.factor()
    d = [torch.zeros(max(k, 1), dtype=torch.float64, device="cuda:0") for k in (n, mi, me, mi, n, mi)]
    dd = [t if k else None for t, k in zip(d, (n, mi, me, mi, n, mi))]
    S.solve_unreduced(*[g(a) for a in xsuv], [g(a) for a in f], dd, max_refine)
    info = S.sync_info()
    out = [t.cpu().numpy()[:k] for t, k in zip(d, (n, mi, me, mi, n, mi))]
    S.close()
    return out, info


@pytest.mark.parametrize("me,dw,dc,gamma", [(0, 0.0, 0.0, 0.0), (0, 1e-4, 1e-6, 0.0), (8, 0.0, 0.0, 1e4),
                                           (8, 1e-5, 0.0, 1e3)])
def test_unreduced_k3_refinement(me, dw, dc, gamma):
    """NEXT-1: the direction from kkt_solve_unreduced equals the dense K3 solution
     block by block -- including with a regularised condensed factor (delta_w, delta_c)
    as the preconditioner, where only the K3 Richardson sweeps reach the unregularised solution."""
    inst, xsuv, f, ref = _k3_case(36, me, 20, seed=21 + me, dw=dw, dc=dc, gamma=gamma)
    out, info = _run_k3(inst, xsuv, f, max_refine=20)
    assert info["status"] == 0, info
    scale = max(np.abs(r).max() for r in ref if r.size)
    for a, r in zip(out, ref):
        if r.size:
            assert np.abs(a - r).max() <= 1e-10 * scale, (np.abs(a - r).max() / scale, info)
    if dw > 0:
        out0, _ = _run_k3(inst, xsuv, f, max_refine=0)
        err0 = max(np.abs(a - r).max() for a, r in zip(out0, ref) if r.size) / scale
        assert err0 > 1e-9 and info["refine_iters"] >= 1, (err0, info)


def test_elec_dense_parity():
    """NEXT-3: COPS elec shape (800 points, fully dense K), a single dense
    front factorised by the tile-task DMMA kernel, against the oracle."""
    from kkt_gpu import run_lifted, relerr
    inst = make_config("C7")
    R = oracle.reference_solve(inst)
    x, info, S = run_lifted(inst, max_refine=10)
    assert info["status"] == 0, info
    assert relerr(x, R["x"]) <= 1e-8, (relerr(x, R["x"]), info)
    eta, _ = oracle.backward_error(inst, R["K"], inst.b, x)
    assert eta <= 1e-10
    S.close()


def test_bearing_800_parity():
    """NEXT-3: COPS bearing_800 (n = 640,000) against the oracle."""
    from kkt_gpu import run_lifted, relerr
    inst = make_config("C6")
    R = oracle.reference_solve(inst)
    x, info, S = run_lifted(inst, max_refine=10)
    assert info["status"] == 0, info
    assert relerr(x, R["x"]) <= 1e-8, (relerr(x, R["x"]), info)
    S.close()


def _ldlt_solver(inst, **kw):
    import paper_2405_14236_b200 as K
    return K.KKTSolver.from_instance(inst, factor_kind=1, **kw).bind(0)


@pytest.mark.parametrize("case,hcap", [("tiny", None), ("C5i", None), ("C2", None), ("C2s", "1500"), ("C7", None)])
def test_ldlt_spd_parity(case, hcap, monkeypatch):
    """NEXT-2: factor_kind = 1 (pivot-free LDL^T, signed-Cholesky form) on SPD systems: inertia
    (n, 0, 0) and the refined solution matches the oracle; "C2s"+KKT_HCAP runs the signed tile
    kernel, C7 (dense elec) one signed dense front."""
    from kkt_gpu import run_lifted, relerr
    from synth.generator import tiny_random
    if hcap:
        monkeypatch.setenv("KKT_HCAP", hcap)
    inst = {"tiny": lambda: tiny_random(40, 30, 0, seed=5, Xi=1e-6, delta_w=1e-4, delta_c=1e-3),
            "C5i": lambda: make_config("C5", batch=1)}.get(case, lambda: make_config(case))()
    R = oracle.reference_solve(inst)
    S = _ldlt_solver(inst)
    x, info, S = run_lifted(inst, max_refine=10, solver=S)
    assert info["status"] == 0, info
    assert tuple(S.inertia()[0]) == (inst.n, 0, 0)
    assert relerr(x, R["x"]) <= 1e-8, (relerr(x, R["x"]), info)
    S.close()


def _indefinite(case, seed):
    from synth.generator import tiny_random
    if case == "tiny":
        return tiny_random(40, 16, 0, seed=seed, Xi=1e-2, w_psd=False)
    inst = make_config("C5", batch=1, Xi=1e-2)      # W - 8 I: a few dozen negative eigenvalues
    inst.W_vals = inst.W_vals.copy()
    diag = inst.W_rowptr[1:] - 1
    inst.W_vals[diag] -= 8.0
    return inst


@pytest.mark.parametrize("case,seed,hcap", [("tiny", 301, None), ("tiny", 302, None), ("C5i", 0, None),
                                            ("C5i", 0, "600")])
def test_ldlt_indefinite_inertia_and_solve(case, seed, hcap, monkeypatch):
    """NEXT-2 on indefinite K: the device inertia equals the oracle LDL^T inertia (and the dense
    eigenvalue counts for the tiny cases), and the refined solve matches a dense solve."""
    from kkt_gpu import run_lifted, relerr
    if hcap:
        monkeypatch.setenv("KKT_HCAP", hcap)
    inst = _indefinite(case, seed)
    Kp, Ki, Kv = oracle.condense(inst)
    perm = oracle.md_order(inst.n, Kp, Ki)
    _, _, Lp, Li = oracle.symbolic(inst.n, Kp, Ki, perm, want_pattern=True)
    Lx, inert, fail = oracle.ldlt(inst.n, Kp, Ki, Kv, perm, Lp, Li)
    assert fail < 0 and inert[1] > 0
    S = _ldlt_solver(inst)
    x, info, S = run_lifted(inst, max_refine=10, solver=S)
    assert info["status"] == 0, info
    assert tuple(S.inertia()[0]) == inert
    n = inst.n
    if n <= 100:
        A = np.zeros((n, n))
        for j in range(n):
            for p in range(Kp[j], Kp[j + 1]):
                A[Ki[p], j] = Kv[p]; A[j, Ki[p]] = Kv[p]
        ev = np.linalg.eigvalsh(A)
        assert inert == (int((ev > 0).sum()), int((ev < 0).sum()), 0)
        xr = np.linalg.solve(A, inst.b)
    else:
        xr = oracle.ldlt_solve(n, Lp, Li, Lx, perm, inst.b)
    assert relerr(x, xr) <= 1e-8, (relerr(x, xr), info)
    S.close()


@pytest.mark.parametrize("factor_kind", [1, 0])
def test_inertia_correction_matches_oracle(factor_kind):
    """The delta_w loop (Wachter-Biegler) on the device takes the same
    decisions as the oracle loop (LDL^T inertia counts; for LL^T the Cholesky breakdown), ends
    with the same delta_w, and the factor it leaves solves the shifted system."""
    import torch
    import paper_2405_14236_b200 as K
    from kkt_gpu import dev, relerr
    inst = _indefinite("tiny", 303)
    dw_ref, tries_ref, inert = oracle.inertia_correct(inst)
    assert inert == (inst.n, 0, 0) and tries_ref >= 2
    S = K.KKTSolver.from_instance(inst, factor_kind=factor_kind).bind(0)
    W, J, Sx, Ss, b = [dev(a, "cuda:0") for a in (inst.W_vals, inst.J_vals, inst.Sigma_x, inst.Sigma_s, inst.b)]
    dw, tries = S.factor_inertia_correct(W, J, Sx, Ss, None, inst.delta_c, inst.gamma)
    assert dw == dw_ref and tries == tries_ref, (dw, tries, dw_ref, tries_ref)
    x = torch.zeros_like(b)
    S.solve(b, x, 10, 0.0)
    info = S.sync_info()
    import copy
    shifted = copy.copy(inst)
    shifted.delta_w = dw
    R = oracle.reference_solve(shifted)
    assert info["status"] == 0 and relerr(x.cpu().numpy(), R["x"]) <= 1e-8
    S.close()


def test_warp_residual_variant(monkeypatch):
    """The warp-per-column double-double residual (chosen for long columns, e.g. dense elec)
    forced on C2s: oracle parity and deterministic (bitwise equal on a repeat)."""
    from kkt_gpu import run_lifted, relerr
    monkeypatch.setenv("KKT_RESID_WARP", "1")
    inst = make_config("C2s")
    R = oracle.reference_solve(inst)
    x, info, S = run_lifted(inst, max_refine=10)
    assert info["status"] == 0, info
    assert relerr(x, R["x"]) <= 1e-12, relerr(x, R["x"])
    x2, _, _ = run_lifted(inst, max_refine=10, solver=S)
    assert np.array_equal(x, x2)
    S.close()


SBLOCK_CASES = [("C2", {}), ("C2", {"KKT_SB_CAP": "1024", "KKT_FB_CAP": "2048"}), ("C1", {}), ("C5b8", {}),
                ("C2", {"KKT_SB_NT": "128"}), ("C5b8", {"KKT_SB_NT": "128", "KKT_SB_CAP": "2048"}),
                ("C5b8", {"KKT_SB_CAP": "1500", "KKT_FB_CAP": "3000"}), ("C2s", {"KKT_NO_PDL": "1"}),
                ("C3L", {}), ("C3L", {"KKT_HUGE_SOLVE": "0"})]


@pytest.mark.parametrize("switch", ["KKT_SBLOCK", "KKT_FBLOCK"])
@pytest.mark.parametrize("case,env", SBLOCK_CASES)
def test_subtree_block_kernels_bitwise(case, env, switch, monkeypatch):
    """Small supernodes by subtree blocks -- the whole-tree solve kernels (sblock.cuh: TMA-staged
    subtrees, big supernodes and single small ones continued in the same grid) and the block
    factorisation (fblock.cuh) -- against the per-node kernels (switch = 0): same sums in the
    same order -> bitwise the same x, and the oracle's solution.  A small budget (KKT_SB_CAP /
    KKT_FB_CAP) leaves many supernodes outside the blocks (continuation chains, single-supernode
    backward tasks, childless single leaves of the factorisation)."""
    from kkt_gpu import run_lifted, relerr
    if case == "C5b8":
        inst = make_config("C5", batch=8)
    elif case == "C3L":  # the C3 pattern as LiftedKKT: large fronts by the tile solve or (KKT_HUGE_SOLVE=0)
        # as CTA supernodes of the tree kernels without L11^-1 (cta_fwd_lite / cta_bwd_lite)
        inst = acopf(10000, 3000, name="acopf10000-lifted")
    else:
        inst = make_config(case)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    monkeypatch.setenv(switch, "0")
    x0, info0, S0 = run_lifted(inst, max_refine=10)
    S0.close()
    monkeypatch.setenv(switch, "1")
    x, info, S = run_lifted(inst, max_refine=10)
    S.close()
    assert info["status"] == 0, info
    assert info["refine_iters"] == info0["refine_iters"]
    assert np.array_equal(x, x0), float(np.abs(x - x0).max())
    if case in ("C2", "C1"):
        R = oracle.reference_solve(inst)
        assert relerr(x, R["x"]) <= 1e-8


@pytest.mark.parametrize("env", [{"KKT_TS_CHAIN": "0"}, {"KKT_TS_CHAIN": "1", "KKT_TS_WAVE": "1"},
                                 {"KKT_TS_CHAIN": "1", "KKT_TS_WAVE": "4"}])
def test_tile_solve_chain_variants(env, monkeypatch):
    """Tile solve of the large fronts: per-step chain tasks (FC / BC) and the panel chain tasks
    (FCH / BCH: TMA tile ring, two warps per tile, waves of 1 or 4 tiles) against the oracle on a
    pattern with large fronts (forced into the tile path with KKT_HUGE_SOLVE=1)."""
    from kkt_gpu import run_lifted, relerr
    monkeypatch.setenv("KKT_HUGE_SOLVE", "1")
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    inst = acopf(10000, 3000, name="acopf10000-lifted")
    R = oracle.reference_solve(inst)
    x, info, S = run_lifted(inst, max_refine=10)
    S.close()
    assert info["status"] == 0, info
    assert relerr(x, R["x"]) <= 1e-8, relerr(x, R["x"])
    eta, _ = oracle.backward_error(inst, R["K"], inst.b, x)
    assert eta <= 1e-10
