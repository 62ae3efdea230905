"""Dense / brute-force companions of the oracle for tiny inputs (n <= ~50).

TEST INFRASTRUCTURE ONLY.  Each helper is an independent route to a quantity the C oracle
computes, used to pin the oracle (tests/test_oracle_*.py):

* dense_blocks / k2_matrix   -- the augmented system (K2), built from its blocks
* recover_dz_ds              -- P:421-423
* md_bruteforce              -- MD-exact-v1 by literal set-based elimination graphs (R11)
* symbolic_numeric_pattern   -- L pattern from numpy's dense Cholesky of a generic SPD matrix
* exact_condensed_solve      -- exact rational (fractions.Fraction) condense + Gaussian elimination
"""
from __future__ import annotations

from fractions import Fraction
import numpy as np


def dense_W(inst):
    """Symmetric dense W from its lower CSR."""
    W = np.zeros((inst.n, inst.n))
    for i in range(inst.n):
        for p in range(inst.W_rowptr[i], inst.W_rowptr[i + 1]):
            j = inst.W_colind[p]
            W[i, j] += inst.W_vals[p]
            if j != i:
                W[j, i] += inst.W_vals[p]
    return W


def dense_J(inst):
    J = np.zeros((inst.m, inst.n))
    for r in range(inst.m):
        for p in range(inst.J_rowptr[r], inst.J_rowptr[r + 1]):
            J[r, inst.J_colind[p]] += inst.J_vals[p]
    return J


def k2_matrix(W, G, H, Dx, Ds, dw, dc):
    """Augmented KKT system (K2), unknown order (dx, ds, dy, dz)."""
    n, me, mi = W.shape[0], G.shape[0], H.shape[0]
    N = n + mi + me + mi
    K = np.zeros((N, N))
    ix, is_, iy, iz = slice(0, n), slice(n, n + mi), slice(n + mi, n + mi + me), slice(n + mi + me, N)
    K[ix, ix] = W + np.diag(Dx) + dw * np.eye(n)
    K[is_, is_] = np.diag(Ds) + dw * np.eye(mi)
    K[ix, iy] = G.T; K[iy, ix] = G
    K[ix, iz] = H.T; K[iz, ix] = H
    K[is_, iz] = np.eye(mi); K[iz, is_] = np.eye(mi)
    K[iy, iy] = -dc * np.eye(me)
    K[iz, iz] = -dc * np.eye(mi)
    return K


def recover_dz_ds(H, Ds, dw, dc, r2, r4, dx):
    """dz = -C r2 + D_H (H dx + r4), ds = -(D_s + dw I)^-1 (r2 + dz)."""
    Cd = 1.0 / (1.0 + dc * (Ds + dw))
    DH = (Ds + dw) * Cd
    dz = -Cd * r2 + DH * (H @ dx + r4)
    ds = -(r2 + dz) / (Ds + dw)
    return dz, ds


def md_bruteforce(n, edges):
    """MD-exact-v1 by literally forming elimination graphs with Python sets (tiny n)."""
    adj = {v: set() for v in range(n)}
    for a, b in edges:
        if a != b:
            adj[a].add(b); adj[b].add(a)
    order = []
    alive = set(range(n))
    while alive:
        v = min(alive, key=lambda u: (len(adj[u]), u))
        nb = adj[v]
        for u in nb:
            adj[u] |= nb
            adj[u].discard(u); adj[u].discard(v)
        alive.discard(v)
        del adj[v]
        order.append(v)
    return np.array(order, dtype=np.int32)


def pattern_edges(Kp, Ki):
    e = []
    for j in range(len(Kp) - 1):
        for p in range(Kp[j], Kp[j + 1]):
            if Ki[p] != j:
                e.append((int(Ki[p]), j))
    return e


def symbolic_numeric_pattern(n, edges, perm, seed=0):
    """Pattern of L from numpy.linalg.cholesky of a generic SPD matrix with the given graph,
    symmetric-permuted by perm (new->old).  Returns (parent, colcount) of the etree."""
    rng = np.random.default_rng(seed)
    A = np.zeros((n, n))
    for a, b in edges:
        v = rng.uniform(0.5, 1.0)
        A[a, b] = A[b, a] = v
    A += np.diag(np.abs(A).sum(1) + 1.0 + rng.random(n))
    P = A[np.ix_(perm, perm)]
    L = np.linalg.cholesky(P)
    nz = np.abs(L) > 1e-300
    parent = np.full(n, -1, np.int32)
    for j in range(n):
        below = np.nonzero(nz[j + 1:, j])[0]
        if below.size:
            parent[j] = j + 1 + below[0]
    return parent, nz.sum(0).astype(np.int32)


def exact_condensed(inst):
    """K (dense, exact rationals) from the exact double inputs."""
    n = inst.n
    F = Fraction
    K = [[F(0)] * n for _ in range(n)]
    for i in range(n):
        for p in range(inst.W_rowptr[i], inst.W_rowptr[i + 1]):
            j = int(inst.W_colind[p]); w = F(float(inst.W_vals[p]))
            K[i][j] += w
            if j != i:
                K[j][i] += w
    for i in range(n):
        K[i][i] += F(float(inst.Sigma_x[i])) + F(float(inst.delta_w))
    for r in range(inst.m):
        if r < inst.m_eq:
            D = F(float(inst.gamma))
        else:
            t = F(float(inst.Sigma_s[r - inst.m_eq])) + F(float(inst.delta_w))
            D = t / (1 + F(float(inst.delta_c)) * t)
        cols = [(int(inst.J_colind[p]), F(float(inst.J_vals[p])))
                for p in range(inst.J_rowptr[r], inst.J_rowptr[r + 1])]
        for a, va in cols:
            for b, vb in cols:
                K[a][b] += D * va * vb
    return K


def exact_solve(K, b):
    """Exact rational Gaussian elimination (no pivoting needed for SPD; partial for safety)."""
    n = len(K)
    A = [row[:] + [Fraction(float(b[i]))] for i, row in enumerate(K)]
    for c in range(n):
        piv = next(r for r in range(c, n) if A[r][c] != 0)
        A[c], A[piv] = A[piv], A[c]
        for r in range(c + 1, n):
            if A[r][c] != 0:
                f = A[r][c] / A[c][c]
                A[r] = [x - f * y for x, y in zip(A[r], A[c])]
    x = [Fraction(0)] * n
    for c in range(n - 1, -1, -1):
        s = A[c][n] - sum(A[c][k] * x[k] for k in range(c + 1, n))
        x[c] = s / A[c][c]
    return x


def k3_matrix(W, G, H, x, s, u, v):
    """Dense unreduced KKT matrix K3 (eq. K3), unknown order (dx, ds, dy, dz, du, dv):
    rows  [W 0 G^T H^T -I 0; 0 0 0 I 0 -I; G 0 0 0 0 0; H I 0 0 0 0; U 0 0 0 X 0; 0 V 0 0 0 S]."""
    n, me, mi = W.shape[0], G.shape[0], H.shape[0]
    N = 2 * n + 3 * mi + me
    K = np.zeros((N, N))
    ix, is_, iy = 0, n, n + mi
    iz, iu, iv = n + mi + me, n + 2 * mi + me, 2 * n + 2 * mi + me
    K[ix:ix + n, ix:ix + n] = W
    K[ix:ix + n, iy:iy + me] = G.T
    K[ix:ix + n, iz:iz + mi] = H.T
    K[ix:ix + n, iu:iu + n] = -np.eye(n)
    K[is_:is_ + mi, iz:iz + mi] = np.eye(mi)
    K[is_:is_ + mi, iv:iv + mi] = -np.eye(mi)
    K[iy:iy + me, ix:ix + n] = G
    K[iz:iz + mi, ix:ix + n] = H
    K[iz:iz + mi, is_:is_ + mi] = np.eye(mi)
    K[iu:iu + n, ix:ix + n] = np.diag(u)
    K[iu:iu + n, iu:iu + n] = np.diag(x)
    K[iv:iv + mi, is_:is_ + mi] = np.diag(v)
    K[iv:iv + mi, iv:iv + mi] = np.diag(s)
    return K


def k3_split(d, n, me, mi):
    """(dx, ds, dy, dz, du, dv) blocks of a K3 vector."""
    o = np.cumsum([0, n, mi, me, mi, n, mi])
    return tuple(d[o[k]:o[k + 1]] for k in range(6))
