"""Pins for oracle.cg_dense, oracle.cr_dense and oracle.hykkt -- CPU only.

Pins: CG finite termination on constructed spectra; HyKKT equals the
dense solve of the condensed saddle system with delta_c = 0; m_eq = 0 reduces to a
plain solve; Woodbury closed form of the Schur spectrum eig(S_gamma) =
1/(gamma + 1/mu_i), mu_i = eig(G K^-1 G^T); CG iterations non-increasing in gamma
(trend, P:1408-1410 / S:611; the counts themselves are parity-unpinned, R10).
"""
import numpy as np
import pytest

import oracle
from oracle import dense
from synth.generator import tiny_random, make_config, KKTInstance


def test_cg_identity_one_iteration():
    x, st, it = oracle.cg_dense(np.eye(7), np.arange(1.0, 8.0))
    assert st == 0 and it == 1 and np.allclose(x, np.arange(1.0, 8.0), rtol=0, atol=1e-15)


def test_cg_diag123():
    x, st, it = oracle.cg_dense(np.diag([1.0, 2.0, 3.0]), np.array([1.0, 2.0, 3.0]), rtol=1e-13)
    assert st == 0 and it <= 3 and np.allclose(x, 1.0, rtol=1e-12)


@pytest.mark.parametrize("seed", range(5))
def test_cg_two_distinct_eigenvalues(seed):
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(rng.standard_normal((10, 10)))
    ev = np.where(rng.random(10) < 0.5, 1.0, 7.0)
    A = (Q * ev) @ Q.T
    b = rng.standard_normal(10)
    x, st, it = oracle.cg_dense(A, b, rtol=1e-12)
    assert st == 0 and it <= 2 and np.allclose(A @ x, b, atol=1e-11)


def test_cr_identity_one_iteration():
    x, st, it, h = oracle.cr_dense(np.eye(7), np.arange(1.0, 8.0))
    assert st == 0 and it == 1 and np.allclose(x, np.arange(1.0, 8.0), rtol=0, atol=1e-15)


@pytest.mark.parametrize("seed", range(5))
def test_cr_two_distinct_eigenvalues(seed):
    rng = np.random.default_rng(seed)
    Q, _ = np.linalg.qr(rng.standard_normal((10, 10)))
    A = (Q * np.where(rng.random(10) < 0.5, 1.0, 7.0)) @ Q.T
    b = rng.standard_normal(10)
    x, st, it, h = oracle.cr_dense(A, b, rtol=1e-12)
    assert st == 0 and it <= 2 and np.allclose(A @ x, b, atol=1e-11)


@pytest.mark.parametrize("seed", range(4))
def test_cr_is_the_minimal_residual_krylov_method(seed):
    """CR decreases the residual norm monotonically.  Stronger pin: its k-th
    residual equals min over y in K_k(A, b) of ||b - A y||_2 (least squares over an explicit
    orthonormal Krylov basis), and CR and CG reach the same solution."""
    rng = np.random.default_rng(100 + seed)
    n = 30
    Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    A = (Q * np.logspace(0, 3, n)) @ Q.T
    A = (A + A.T) / 2
    b = rng.standard_normal(n)
    x, st, it, hist = oracle.cr_dense(A, b, rtol=1e-12, maxit=500)
    assert st == 0
    assert np.all(np.diff(hist) <= 1e-12 * hist[0])           # monotone
    V = np.zeros((n, 0))
    v = b.copy()
    for k in range(1, 7):
        for _ in range(2):                                       # twice-orthogonalised basis
            v = v - V @ (V.T @ v)
        V = np.column_stack([V, v / np.linalg.norm(v)])
        y, *_ = np.linalg.lstsq(A @ V, b, rcond=None)
        rmin = np.linalg.norm(b - A @ (V @ y))
        assert abs(hist[k] - rmin) <= 1e-9 * hist[0], (k, hist[k], rmin)
        v = A @ V[:, -1]
    xc, stc, itc = oracle.cg_dense(A, b, rtol=1e-12, maxit=500)
    assert np.abs(x - xc).max() <= 1e-9 * np.abs(xc).max()


def _split(inst):
    """Dense K (no gamma rows), G, from an instance with m_eq gamma rows."""
    n, me = inst.n, inst.m_eq
    J = dense.dense_J(inst)
    G, H = J[:me], J[me:]
    Ds = inst.Sigma_s
    DH = (Ds + inst.delta_w) / (1 + inst.delta_c * (Ds + inst.delta_w))
    K = dense.dense_W(inst) + np.diag(inst.Sigma_x + inst.delta_w) + H.T @ (DH[:, None] * H)
    return K, G


def _factor(inst):
    R = oracle.reference_solve(inst, b=np.zeros(inst.n))
    return R


@pytest.mark.parametrize("seed,gamma", [(1, 1e2), (2, 1e4), (3, 1e6), (4, 1e3)])
def test_hykkt_equals_saddle_solve(seed, gamma):
    inst = tiny_random(14, 9, 4, seed=seed, Xi=1e-3, hykkt_gamma=gamma, delta_w=1e-4)
    K, G = _split(inst)
    me = inst.m_eq
    S = np.block([[K, G.T], [G, np.zeros((me, me))]])
    sol = np.linalg.solve(S, np.concatenate([inst.rbar1, inst.rbar2]))
    R = _factor(inst)
    dx, dy, st, it, ou = oracle.hykkt(inst, R["Lp"], R["Li"], R["Lx"], R["perm"], inst.rbar1,
                                      inst.rbar2)
    assert st == 0
    assert np.abs(dx - sol[:inst.n]).max() <= 1e-9 * np.abs(sol).max()
    assert np.abs(dy - sol[inst.n:]).max() <= 1e-9 * np.abs(sol).max()


def test_hykkt_without_equalities_is_plain_solve():
    """m_e = 0 -> HyKKT reduces to the direct condensed solve."""
    inst = tiny_random(12, 5, 0, seed=9)
    inst.rbar1 = inst.b.copy(); inst.rbar2 = np.zeros(0)
    R = _factor(inst)
    dx, dy, st, it, ou = oracle.hykkt(inst, R["Lp"], R["Li"], R["Lx"], R["perm"], inst.rbar1, inst.rbar2)
    R2 = oracle.reference_solve(inst)
    assert np.abs(dx - R2["x"]).max() <= 1e-14 * np.abs(R2["x"]).max() and it == 0


@pytest.mark.parametrize("gamma", [1e1, 1e3, 1e5])
def test_schur_spectrum_woodbury(gamma):
    """eig(G K_gamma^-1 G^T) = 1/(gamma + 1/mu_i), mu_i = eig(G K^-1 G^T); gamma*lambda -> 1."""
    inst = tiny_random(16, 10, 5, seed=17, Xi=1e-2, hykkt_gamma=gamma)
    K, G = _split(inst)
    R = _factor(inst)
    # S_gamma column by column through the oracle's factor of K_gamma
    Sg = np.stack([G @ oracle.trisolve(inst.n, R["Lp"], R["Li"], R["Lx"], R["perm"], G[k])
                   for k in range(inst.m_eq)], axis=1)
    lam = np.sort(np.linalg.eigvalsh(0.5 * (Sg + Sg.T)))
    mu = np.linalg.eigvalsh(G @ np.linalg.solve(K, G.T))
    pred = np.sort(1.0 / (gamma + 1.0 / mu))
    assert np.allclose(lam, pred, rtol=1e-8)
    assert np.all(np.abs(gamma * lam - 1) <= np.abs(gamma * pred - 1) + 1e-8)


def test_cg_iterations_nonincreasing_in_gamma():
    its = []
    for gamma in (1e2, 1e4, 1e6, 1e8):
        inst = tiny_random(30, 20, 10, seed=23, Xi=1e-4, hykkt_gamma=gamma)
        R = _factor(inst)
        _, _, st, it, _ = oracle.hykkt(inst, R["Lp"], R["Li"], R["Lx"], R["perm"], inst.rbar1,
                                       inst.rbar2, cg_rtol=1e-10)
        its.append(it)
    assert all(a >= b for a, b in zip(its, its[1:])), its
