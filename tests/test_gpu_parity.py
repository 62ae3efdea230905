"""CUDA path vs oracle, element by element on the same seeded inputs (-m gpu; B200).

Bars (BASELINE.json north_star):
  condense:  |K_gpu - K_ref| <= 4 (t+2) u (|W| + |Sx+dw| + sum|D J J|)  per entry (t = #terms)
  solve:     ||x - x_ref||_inf / ||x_ref||_inf <= 1e-8 ;  eta (R7) <= 1e-10
  HyKKT:     dx, dy relative error <= 1e-8 vs the oracle's refined saddle solution
  NOT_SPD:   same failing column as the oracle
  determinism: bitwise-identical results across runs and between batch and single solves
"""
import numpy as np
import pytest

import oracle
from synth.generator import make_config, tiny_random, acopf, redraw_values

pytestmark = pytest.mark.gpu

U = 2.0 ** -53


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA not available: the -m gpu suite needs a B200 (no CPU fallback exists)")


def _abs_condensed(inst):
    """Entrywise sum of term magnitudes, via the oracle on |inputs| (tolerance only)."""
    import copy
    a = copy.copy(inst)
    a.W_vals = np.abs(inst.W_vals); a.J_vals = np.abs(inst.J_vals); a.Sigma_x = np.abs(inst.Sigma_x)
    D = np.empty(inst.m)
    D[:inst.m_eq] = inst.gamma
    t = inst.Sigma_s + inst.delta_w
    D[inst.m_eq:] = t / (1 + inst.delta_c * t)
    return oracle.condense(a, D=np.abs(D))


CASES = {
    "tiny": lambda: tiny_random(40, 30, 0, seed=5, Xi=1e-6, delta_w=1e-4, delta_c=1e-3),
    "tiny_eq": lambda: tiny_random(45, 30, 10, seed=6, Xi=1e-6, hykkt_gamma=1e5),
    "C1": lambda: make_config("C1"),
    "C5i": lambda: make_config("C5", batch=1),
    "C2": lambda: make_config("C2"),
    "C2s": lambda: make_config("C2s"),
}


@pytest.mark.parametrize("case", list(CASES))
def test_condense_parity(case):
    from kkt_gpu import run_lifted
    inst = CASES[case]()
    _, _, S = run_lifted(inst, max_refine=0)
    Kp, Ki, Kv = S.get_condensed(0)
    Op, Oi, Ov = oracle.condense(inst)
    assert np.array_equal(Kp, Op) and np.array_equal(Ki, Oi)
    _, _, Ka = _abs_condensed(inst)
    terms = np.diff(Op)  # generous per-entry term bound: column length
    tmax = max(int(terms.max()), 1) + 2 + (inst.m and int(np.diff(inst.J_rowptr).max()))
    assert np.all(np.abs(Kv - Ov) <= 4 * tmax * U * Ka)
    S.close()


@pytest.mark.parametrize("case", list(CASES))
def test_solve_parity(case):
    from kkt_gpu import run_lifted, relerr
    inst = CASES[case]()
    R = oracle.reference_solve(inst)
    x, info, S = run_lifted(inst, max_refine=10)
    assert info["status"] == 0, info
    assert relerr(x, R["x"]) <= 1e-8, (relerr(x, R["x"]), info)
    eta, om = oracle.backward_error(inst, R["K"], inst.b, x)
    assert eta <= 1e-10, (eta, info)
    assert info["bwd_err"] <= 1e-12
    S.close()


def test_unrefined_solve_is_a_valid_factorization():
    """max_refine = 0: plain FP64 supernodal solve; error bounded by the conditioning only."""
    from kkt_gpu import run_lifted, relerr
    inst = make_config("C5", batch=1, Xi=1e-2)
    R = oracle.reference_solve(inst)
    x, info, S = run_lifted(inst, max_refine=0)
    assert relerr(x, R["x"]) <= 1e-10
    S.close()


@pytest.mark.parametrize("B", [1, 3, 8])
def test_batch_parity_and_bitwise_vs_single(B):
    from kkt_gpu import run_lifted, relerr
    inst = make_config("C5", batch=B)
    xb, info, S = run_lifted(inst, max_refine=10)
    assert info["status"] == 0
    xb = xb.reshape(B, -1)
    for k in range(B):
        one = inst.instance(k)
        R = oracle.reference_solve(one)
        assert relerr(xb[k], R["x"]) <= 1e-8
        x1, _, S1 = run_lifted(one, max_refine=10)
        assert np.array_equal(x1, xb[k]), "batch result differs from single-instance result"
        S1.close()
    S.close()


def test_determinism_repeat():
    from kkt_gpu import run_lifted
    inst = make_config("C2")
    x1, _, S = run_lifted(inst)
    x2, _, _ = run_lifted(inst, solver=S)
    assert np.array_equal(x1, x2)
    S.close()


def test_value_redraw_same_pattern():
    """Successive IPM iterations: new values on the same handle (pattern fixed at analysis)."""
    from kkt_gpu import run_lifted, relerr
    inst = make_config("C2")
    _, _, S = run_lifted(inst)
    for k in range(3):
        it = redraw_values(inst, 777 + k)
        R = oracle.reference_solve(it)
        x, info, _ = run_lifted(it, solver=S)
        assert relerr(x, R["x"]) <= 1e-8, (k, relerr(x, R["x"]))
    S.close()


def test_not_spd_reports_oracle_column():
    inst = tiny_random(30, 12, 0, seed=8)
    v = 17
    d = inst.W_rowptr[v + 1] - 1           # diagonal entry of row v (last in the lower row)
    assert inst.W_colind[d] == v
    inst.W_vals = inst.W_vals.copy()
    inst.W_vals[d] = -1e6
    R = oracle.reference_solve(inst)
    assert R["fail"] >= 0
    from kkt_gpu import run_lifted
    _, info, S = run_lifted(inst, max_refine=0)
    assert info["status_name"] == "KKT_ERR_NOT_SPD"
    assert info["fail_col"] == int(R["perm"][R["fail"]]) == v
    # the handle recovers: the next (SPD) iteration solves again
    inst2 = tiny_random(30, 12, 0, seed=8)
    x, info2, _ = run_lifted(inst2, solver=S)
    assert info2["status"] == 0
    S.close()


def test_edge_sizes():
    from kkt_gpu import run_lifted, relerr
    for n, m in ((1, 0), (2, 1), (3, 0), (5, 7)):
        inst = tiny_random(n, m, 0, seed=n * 10 + m)
        R = oracle.reference_solve(inst)
        x, info, S = run_lifted(inst)
        assert info["status"] == 0 and relerr(x, R["x"]) <= 1e-12
        S.close()


@pytest.mark.parametrize("seed,gamma", [(1, 1e3), (2, 1e6)])
def test_hykkt_parity_tiny(seed, gamma):
    from kkt_gpu import run_hykkt, relerr
    inst = tiny_random(60, 40, 15, seed=seed, Xi=1.0 / gamma, hykkt_gamma=gamma)
    R = oracle.reference_hykkt(inst)
    dx, dy, info, S = run_hykkt(inst, max_outer=3)
    assert info["status"] == 0, info
    assert relerr(dx, R["dx"]) <= 1e-8 and relerr(dy, R["dy"]) <= 1e-8
    S.close()


def test_hykkt_parity_acopf_small():
    from kkt_gpu import run_hykkt, relerr
    inst = acopf(300, 3300, hykkt=True, gamma=1e6)
    R = oracle.reference_hykkt(inst)
    dx, dy, info, S = run_hykkt(inst, max_outer=3)
    assert info["status"] == 0, info
    assert relerr(dx, R["dx"]) <= 1e-8 and relerr(dy, R["dy"]) <= 1e-8, (relerr(dx, R["dx"]), relerr(dy, R["dy"]))
    S.close()


def test_step_host_matches_device_path():
    """e2e entry point (host buffers): same x as the device-buffer path, bitwise."""
    import paper_2405_14236_b200 as K
    from kkt_gpu import run_lifted
    inst = make_config("C2")
    x_dev, _, S = run_lifted(inst)
    x = np.zeros(inst.n)
    K.kkt_step_host(S.h, np.ascontiguousarray(inst.W_vals), np.ascontiguousarray(inst.J_vals),
                    np.ascontiguousarray(inst.Sigma_x), np.ascontiguousarray(inst.Sigma_s), None,
                    inst.delta_w, inst.delta_c, inst.gamma, np.ascontiguousarray(inst.b), x, 10, 0.0)
    assert np.array_equal(x, x_dev)
    S.close()


@pytest.mark.parametrize("hcap", ["1500", "4000"])
def test_gpu_wide_front_path_parity(hcap, monkeypatch):
    """Force medium fronts onto the whole-GPU cooperative path (huge.cuh) via the KKT_HCAP test
    hook and check the solve against the oracle (C2 and the C2 stress variant)."""
    from kkt_gpu import run_lifted, relerr
    monkeypatch.setenv("KKT_HCAP", hcap)
    for cfg in ("C2", "C2s"):
        inst = make_config(cfg)
        R = oracle.reference_solve(inst)
        x, info, S = run_lifted(inst, max_refine=10)
        assert info["status"] == 0, info
        assert relerr(x, R["x"]) <= 1e-8, (cfg, relerr(x, R["x"]))
        S.close()


@pytest.mark.parametrize("hcap,solve_mode", [("1500", "1"), ("4000", "1"), ("1500", "0")])
def test_gpu_huge_solve_modes_parity(hcap, solve_mode, monkeypatch):
    """Huge fronts solved by the whole-GPU wavefront kernel (KKT_HUGE_SOLVE=1, the C4/C6 path) and
    by the CTA kernels (=0, the C3 path) both match the oracle, and agree with each other to the
    refinement's accuracy."""
    from kkt_gpu import run_lifted, relerr
    monkeypatch.setenv("KKT_HCAP", hcap)
    monkeypatch.setenv("KKT_HUGE_SOLVE", solve_mode)
    inst = make_config("C2s")
    R = oracle.reference_solve(inst)
    x, info, S = run_lifted(inst, max_refine=10)
    assert info["status"] == 0, info
    assert relerr(x, R["x"]) <= 1e-8, relerr(x, R["x"])
    S.close()


@pytest.mark.parametrize("env", [{"KKT_NO_PDL": "1"}, {"KKT_NO_LINV": "1"}, {"KKT_PDL_MASK": "4"},
                                 {"KKT_NO_GRAPH": "1"}])
def test_schedule_variants_parity_and_bitwise(env, monkeypatch):
    """Serialised phases (no programmatic launch), substitution instead of L11^-1 sweeps, partial
    overlap and the graph-free solve all reproduce the oracle; the phase overlap alone never
    changes a bit (fixed summation orders, no floating-point atomics)."""
    from kkt_gpu import run_lifted, relerr
    inst = make_config("C2")
    R = oracle.reference_solve(inst)
    x0, info0, S0 = run_lifted(inst, max_refine=10)
    S0.close()
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    x, info, S = run_lifted(inst, max_refine=10)
    assert info["status"] == 0, info
    assert relerr(x, R["x"]) <= 1e-8, relerr(x, R["x"])
    if "KKT_NO_LINV" not in env:  # same operator -> same bits
        assert np.array_equal(x, x0)
    S.close()


def test_lifted_acopf10000_parity():
    """C3 pattern solved as LiftedKKT: exercises big fronts beyond one CTA's shared memory."""
    from kkt_gpu import run_lifted, relerr
    inst = acopf(10000, 3000, name="acopf10000-lifted")
    R = oracle.reference_solve(inst)
    x, info, S = run_lifted(inst, max_refine=10)
    assert info["status"] == 0, info
    assert relerr(x, R["x"]) <= 1e-8, relerr(x, R["x"])
    eta, _ = oracle.backward_error(inst, R["K"], inst.b, x)
    assert eta <= 1e-10
    S.close()


def test_hykkt_parity_C3():
    from kkt_gpu import run_hykkt, relerr
    inst = make_config("C3", gamma=1e7)
    R = oracle.reference_hykkt(inst)
    dx, dy, info, S = run_hykkt(inst, max_outer=3)
    assert info["status"] == 0, info
    assert relerr(dx, R["dx"]) <= 1e-8 and relerr(dy, R["dy"]) <= 1e-8, (relerr(dx, R["dx"]), relerr(dy, R["dy"]))
    S.close()


@pytest.mark.parametrize("seed,dw,dc", [(3, 0.0, 0.0), (4, 1e-3, 1e-2)])
def test_recover_matches_augmented_K2(seed, dw, dc):
    """NEXT-1: condensed solve on the GPU + kkt_recover reproduces the dense K2
    solution for all of dx, ds, dz; kkt_recover_bounds satisfies the K3 rows
    U dx + X du = -(X u - mu e) and V ds + S dv = -(S v - mu e)."""
    import torch
    from oracle import dense
    from kkt_gpu import dev
    import paper_2405_14236_b200 as K
    rng = np.random.default_rng(seed)
    n, mi = 24, 14
    inst = tiny_random(n, mi, 0, seed=seed, Xi=1e-2, delta_w=dw, delta_c=dc)
    Ds = rng.uniform(0.1, 10.0, mi)
    inst.Sigma_s = Ds
    H = dense.dense_J(inst)
    W = dense.dense_W(inst)
    K2 = dense.k2_matrix(W, np.zeros((0, n)), H, inst.Sigma_x, Ds, dw, dc)
    r1, r2, r4 = rng.standard_normal(n), rng.standard_normal(mi), rng.standard_normal(mi)
    sol = np.linalg.solve(K2, -np.concatenate([r1, r2, r4]))
    dx2, ds2, dz2 = sol[:n], sol[n:n + mi], sol[n + mi:]
    Cd = 1.0 / (1.0 + dc * (Ds + dw)); DH = (Ds + dw) * Cd
    rb1 = -(r1 + H.T @ (DH * r4 - Cd * r2))
    S = K.KKTSolver.from_instance(inst).bind(0)
    t = [dev(a, "cuda:0") for a in (inst.W_vals, inst.J_vals, inst.Sigma_x, Ds, rb1, r2, r4)]
    W_, J_, Sx_, Ss_, b_, r2_, r4_ = t
    x_ = torch.zeros_like(b_); dz_ = torch.zeros_like(r2_); ds_ = torch.zeros_like(r2_)
    S.condense(W_, J_, Sx_, Ss_, None, dw, dc, 0.0)
    S.factor()
    S.solve(b_, x_, 10, 0.0)
    S.recover(r2_, r4_, x_, dz_, ds_)
    info = S.sync_info()
    assert info["status"] == 0
    scale = np.abs(sol).max()
    for a, b in ((x_, dx2), (dz_, dz2), (ds_, ds2)):
        assert np.abs(a.cpu().numpy() - b).max() <= 1e-9 * scale
    # bound multipliers
    xv, uv = rng.uniform(0.5, 2, n), rng.uniform(0.5, 2, n)
    sv, vv = rng.uniform(0.5, 2, mi), rng.uniform(0.5, 2, mi)
    mu = 0.1
    du_ = torch.zeros_like(x_); dv_ = torch.zeros_like(r2_)
    S.recover_bounds(dev(xv, "cuda:0"), dev(uv, "cuda:0"), dev(sv, "cuda:0"), dev(vv, "cuda:0"), mu,
                     x_, ds_, du_, dv_)
    du, dv = du_.cpu().numpy(), dv_.cpu().numpy()
    dxv, dsv = x_.cpu().numpy(), ds_.cpu().numpy()
    assert np.abs(uv * dxv + xv * du + (xv * uv - mu)).max() <= 1e-12 * (1 + np.abs(uv * dxv).max())
    assert np.abs(vv * dsv + sv * dv + (sv * vv - mu)).max() <= 1e-12 * (1 + np.abs(vv * dsv).max())
    S.close()


def test_bearing_120_parity():
    """NEXT-3 workload family (COPS bearing) at an oracle-checkable size."""
    from kkt_gpu import run_lifted, relerr
    from synth.generator import bearing
    inst = bearing(120, 120, seed=6000)
    R = oracle.reference_solve(inst)
    x, info, S = run_lifted(inst, max_refine=10)
    assert info["status"] == 0, info
    assert relerr(x, R["x"]) <= 1e-8
    S.close()


@pytest.mark.gpu
@pytest.mark.parametrize("relax_big,zero_frac", [(160, 0.3), (192, 0.5), (256, 0.8)])
def test_wide_supernodes_linv_parity(relax_big, zero_frac):
    """Coarser amalgamation (perf-only options) widens C2's CTA-path supernodes: (160, 0.3) keeps
    every L11^-1 block resident in shared memory (w <= 128), (192, 0.5) adds w = 129..181 (packed
    resident nb = 5 and non-resident nb = 6 linv paths), (256, 0.8) has w = 256 (no linv: the
    substitution sweeps).  Every setting must match the oracle's exact-input solution."""
    from kkt_gpu import run_lifted, relerr
    import paper_2405_14236_b200 as K
    inst = make_config("C2s")
    R = oracle.reference_solve(inst)
    S = K.KKTSolver.from_instance(inst, relax_big=relax_big, relax_zero_frac=zero_frac).bind(0)
    x, info, S = run_lifted(inst, max_refine=10, solver=S)
    assert info["status"] == 0, info
    assert relerr(x, R["x"]) <= 1e-8, relerr(x, R["x"])
    S.close()
