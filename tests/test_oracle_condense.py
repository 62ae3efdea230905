"""Pins for oracle.condense (K = W + D_x + dw I + J^T D J) -- CPU only.

Pinned against things other than the oracle's own formula:
  * the augmented system K2: condensed (K1) solution + recovery
    reproduce the dense K2 solution;
  * the inertia identity by dense eigen-counts;
  * exact rational arithmetic (fractions) -> every entry correctly rounded (R1);
  * special cases m=0 (K = W + Sx + dw I) and the two-sided LiftedKKT row (R2);
  * SPD of generated K (dense eigvalsh).
"""
import numpy as np
import pytest

import oracle
from oracle import dense
from synth.generator import tiny_random, make_config, KKTInstance


def _sub_rows(inst, rows, m_eq=0, Ss=None, gamma=0.0):
    """Instance with J restricted to `rows` (keeps values)."""
    rp, cols, vals = [0], [], []
    for r in rows:
        a, b = inst.J_rowptr[r], inst.J_rowptr[r + 1]
        cols.append(inst.J_colind[a:b]); vals.append(inst.J_vals[a:b]); rp.append(rp[-1] + b - a)
    cols = np.concatenate(cols) if cols else np.zeros(0, np.int32)
    vals = np.concatenate(vals) if vals else np.zeros(0)
    return KKTInstance("sub", inst.n, len(rows), m_eq, inst.W_rowptr, inst.W_colind, inst.W_vals,
                       np.array(rp, np.int32), cols.astype(np.int32), vals, inst.Sigma_x,
                       np.zeros(len(rows) - m_eq) if Ss is None else Ss, inst.delta_w,
                       inst.delta_c, gamma, inst.b)


def _dense_K(Kp, Ki, Kv, n):
    K = np.zeros((n, n))
    for j in range(n):
        for p in range(Kp[j], Kp[j + 1]):
            K[Ki[p], j] = Kv[p]; K[j, Ki[p]] = Kv[p]
    return K


@pytest.mark.parametrize("seed,dw,dc", [(1, 0.0, 0.0), (2, 1e-3, 1e-2), (3, 0.5, 0.3), (4, 0.0, 1e-6)])
def test_condensed_solution_equals_augmented_K2(seed, dw, dc):
    """solving K1 with the condensed K and r̄ = -(r1 + H^T(D_H r4 - C r2)), -r3 and
    recovering dz, ds gives the dense K2 solution (reading R1 of the sign)."""
    rng = np.random.default_rng(seed)
    n, me, mi = 9, 3, 5
    base = tiny_random(n, me + mi, 0, seed=seed, Xi=1e-2, delta_w=dw, delta_c=dc)
    Ds = rng.uniform(0.1, 10.0, mi)
    Hinst = _sub_rows(base, list(range(me, me + mi)), 0, Ss=Ds)
    Kp, Ki, Kv = oracle.condense(Hinst)
    K = _dense_K(Kp, Ki, Kv, n)
    J = dense.dense_J(base)
    G, H = J[:me], J[me:]
    W = dense.dense_W(base)
    K2 = dense.k2_matrix(W, G, H, base.Sigma_x, Ds, dw, dc)
    r1, r2, r3, r4 = (rng.standard_normal(k) for k in (n, mi, me, mi))
    sol = np.linalg.solve(K2, -np.concatenate([r1, r2, r3, r4]))
    dx2, ds2, dy2, dz2 = np.split(sol, [n, n + mi, n + mi + me])
    Cd = 1.0 / (1.0 + dc * (Ds + dw)); DH = (Ds + dw) * Cd
    rb1 = -(r1 + H.T @ (DH * r4 - Cd * r2)); rb2 = -r3
    K1 = np.block([[K, G.T], [G, -dc * np.eye(me)]])
    s1 = np.linalg.solve(K1, np.concatenate([rb1, rb2]))
    dx1, dy1 = s1[:n], s1[n:]
    dz1, ds1 = dense.recover_dz_ds(H, Ds, dw, dc, r2, r4, dx1)
    scale = np.abs(sol).max()
    for a, b in ((dx1, dx2), (dy1, dy2), (dz1, dz2), (ds1, ds2)):
        assert np.abs(a - b).max() <= 1e-10 * scale


@pytest.mark.parametrize("seed", [5, 6, 7, 8])
def test_inertia_identity(seed):
    """inertia(K2) = (n+mi, me+mi, 0)  <=>  inertia(K1) = (n, me, 0)."""
    rng = np.random.default_rng(seed)
    n, me, mi = 8, 2, 4
    base = tiny_random(n, me + mi, 0, seed=seed, w_psd=(seed % 2 == 0))
    Ds = rng.uniform(0.1, 5.0, mi); dw, dc = 0.05, 0.01
    Hinst = _sub_rows(base, list(range(me, me + mi)), 0, Ss=Ds)
    Hinst.delta_w, Hinst.delta_c = dw, dc
    K = _dense_K(*oracle.condense(Hinst), n)
    J = dense.dense_J(base); G, H = J[:me], J[me:]
    K2 = dense.k2_matrix(dense.dense_W(base), G, H, base.Sigma_x, Ds, dw, dc)
    K1 = np.block([[K, G.T], [G, -dc * np.eye(me)]])
    def inertia(A):
        ev = np.linalg.eigvalsh(A); tol = 1e-10 * np.abs(ev).max()
        return (int((ev > tol).sum()), int((ev < -tol).sum()), int((np.abs(ev) <= tol).sum()))
    assert (inertia(K2) == (n + mi, me + mi, 0)) == (inertia(K1) == (n, me, 0))


@pytest.mark.parametrize("seed", [11, 12, 13])
def test_entries_correctly_rounded_exact_rationals(seed):
    """R1: each K entry is the exact sum (rationals from the double inputs), rounded once."""
    inst = tiny_random(7, 6, 2, seed=seed, hykkt_gamma=1e3, delta_w=0.25, delta_c=0.125)
    Kp, Ki, Kv = oracle.condense(inst)
    Kex = dense.exact_condensed(inst)
    for j in range(inst.n):
        for p in range(Kp[j], Kp[j + 1]):
            assert Kv[p] == float(Kex[Ki[p]][j])


def test_bound_only_is_W_plus_sigma():
    """m = 0 -> K = W + D_x + delta_w I (diagonal: exact sum rounded once)."""
    from fractions import Fraction as F
    inst = make_config("C1")
    inst.delta_w = 0.5
    Kp, Ki, Kv = oracle.condense(inst)
    assert len(Kv) == inst.nnzW
    ref = {}
    for i in range(inst.n):
        for p in range(inst.W_rowptr[i], inst.W_rowptr[i + 1]):
            j = int(inst.W_colind[p])
            ref[(i, j)] = float(F(inst.W_vals[p]) + F(inst.Sigma_x[i]) + F(0.5)) if i == j \
                else inst.W_vals[p]
    for j in range(inst.n):
        for p in range(Kp[j], Kp[j + 1]):
            assert Kv[p] == ref[(int(Ki[p]), j)]


def test_two_sided_relaxation_row_equals_combined_weight():
    """R2: rows g and -g with weights D_l, D_u == one row g with D_l + D_u."""
    base = tiny_random(8, 4, 0, seed=21)
    rng = np.random.default_rng(0)
    Dl, Du = rng.uniform(1, 10, 4), rng.uniform(1, 10, 4)
    two = _sub_rows(base, [0, 1, 2, 3, 0, 1, 2, 3])
    two.J_vals = np.concatenate([base.J_vals, -base.J_vals])
    K2p, K2i, K2v = oracle.condense(two, D=np.concatenate([Dl, Du]))
    K1p, K1i, K1v = oracle.condense(base, D=Dl + Du)
    assert np.array_equal(K1p, K2p) and np.array_equal(K1i, K2i)
    assert np.allclose(K1v, K2v, rtol=4e-16, atol=0)


def test_hykkt_gamma_rows_and_deltac_zero_formula():
    """rows < m_eq weighted gamma; delta_c = 0 -> D_H = D_s + delta_w."""
    inst = tiny_random(10, 7, 3, seed=31, hykkt_gamma=1e4, delta_w=0.1, delta_c=0.0)
    D = np.concatenate([np.full(3, 1e4), inst.Sigma_s + 0.1])
    a = oracle.condense(inst)
    b = oracle.condense(inst, D=D)
    assert np.abs(a[2] - b[2]).max() <= 1e-15 * np.abs(a[2]).max()  # D rounded once vs exact


@pytest.mark.parametrize("cfg", ["C1", "C5"])
def test_generated_K_is_spd(cfg):
    """K SPD when W >= 0 and Sigma > 0 (R17): dense eigvalsh min > 0 (n <= 4,300)."""
    inst = make_config(cfg) if cfg != "C5" else make_config("C5", batch=1)
    K = _dense_K(*oracle.condense(inst), inst.n)
    assert np.linalg.eigvalsh(K).min() > 0


@pytest.mark.parametrize("seed,me", [(11, 0), (12, 4)])
def test_k3_reduces_to_k2_plus_bound_recovery(seed, me):
    """NEXT-1 oracle pin: the dense unreduced K3 solved directly equals the K2 solve
    (delta = 0, D_x = X^-1 U, D_s = S^-1 V) followed by the bound-multiplier recovery
    du = X^-1 (f5 - U dx), dv = S^-1 (f6 - V ds) (generalised right-hand side)."""
    from oracle import dense
    rng = np.random.default_rng(seed)
    n, mi = 18, 9
    inst = tiny_random(n, mi + me, me, seed=seed)
    J = dense.dense_J(inst)
    G, H = J[:me], J[me:]
    W = dense.dense_W(inst)
    x, u = rng.uniform(0.5, 2, n), rng.uniform(0.5, 2, n)
    s, v = rng.uniform(0.5, 2, mi), rng.uniform(0.5, 2, mi)
    f = [rng.standard_normal(k) for k in (n, mi, me, mi, n, mi)]
    K3 = dense.k3_matrix(W, G, H, x, s, u, v)
    d = np.linalg.solve(K3, np.concatenate(f))
    dx, ds, dy, dz, du, dv = dense.k3_split(d, n, me, mi)
    K2 = dense.k2_matrix(W, G, H, u / x, v / s, 0.0, 0.0)
    b2 = np.concatenate([f[0] + f[4] / x, f[1] + f[5] / s, f[2], f[3]])
    sol = np.linalg.solve(K2, b2)
    ex, es = sol[:n], sol[n:n + mi]
    ey, ez = sol[n + mi:n + mi + me], sol[n + mi + me:]
    scale = np.abs(d).max()
    for a, b in ((dx, ex), (ds, es), (dy, ey), (dz, ez), (du, (f[4] - u * ex) / x), (dv, (f[5] - v * es) / s)):
        assert a.size == 0 or np.abs(a - b).max() <= 1e-10 * scale
