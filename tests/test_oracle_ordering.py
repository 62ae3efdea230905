"""Pins for oracle.md_order (MD-exact-v1, R11) and oracle.symbolic (etree, column
counts) -- CPU only.

Pins: hand-traced example (tests/golden/md_example_7.txt), textbook graphs (path, star,
diagonal), a set-based brute-force elimination on random tiny graphs,
the L pattern of numpy's dense Cholesky of a generic SPD matrix (library routine), and a
quality band against SciPy SuperLU's MMD_AT_PLUS_A ordering.
"""
import os
import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

import oracle
from oracle import dense
from synth.generator import make_config

GOLD = os.path.join(os.path.dirname(__file__), "golden", "md_example_7.txt")


def lower_csc(n, edges):
    cols = [[j] for j in range(n)]
    for a, b in edges:
        i, j = max(a, b), min(a, b)
        if i != j:
            cols[j].append(i)
    Kp, Ki = [0], []
    for j in range(n):
        c = sorted(set(cols[j]))
        Ki += c
        Kp.append(len(Ki))
    return np.array(Kp, np.int32), np.array(Ki, np.int32)


def read_gold():
    d = {}
    for line in open(GOLD):
        if line.startswith("#") or not line.strip():
            continue
        k, *v = line.split()
        d[k] = v
    n = int(d["n"][0])
    edges = [tuple(map(int, e.split("-"))) for e in d["edges"]]
    return n, edges, [int(x) for x in d["perm"]], [int(x) for x in d["parent"]], \
        [int(x) for x in d["colcount"]]


def test_hand_traced_example():
    n, edges, perm, parent, cc = read_gold()
    Kp, Ki = lower_csc(n, edges)
    p = oracle.md_order(n, Kp, Ki)
    assert p.tolist() == perm
    par, c = oracle.symbolic(n, Kp, Ki, p)
    assert par.tolist() == parent and c.tolist() == cc


def test_path_graph_identity_zero_fill():
    """path -> zero fill.  MD: vertex 0 (degree 1, smallest index) first, and so on."""
    n = 9
    Kp, Ki = lower_csc(n, [(i, i + 1) for i in range(n - 1)])
    p = oracle.md_order(n, Kp, Ki)
    assert p.tolist() == list(range(n))
    par, cc = oracle.symbolic(n, Kp, Ki, p)
    assert par.tolist() == list(range(1, n)) + [-1]          # path etree
    assert cc.sum() == 2 * n - 1                               # |L| = 2n - 1


def test_star_hub_last():
    """arrow/star -> leaves (degree 1) eliminated first in index order; when one leaf is
    left the hub also has degree 1 and wins the smallest-index tie.  Zero fill."""
    n = 7
    Kp, Ki = lower_csc(n, [(0, k) for k in range(1, n)])
    p = oracle.md_order(n, Kp, Ki)
    assert p.tolist() == list(range(1, n - 1)) + [0, n - 1]
    par, cc = oracle.symbolic(n, Kp, Ki, p)
    assert cc.sum() == 2 * n - 1


def test_diagonal_and_dense():
    """diagonal -> identity order, singleton forest; dense -> |L| = n(n+1)/2."""
    n = 5
    Kp, Ki = lower_csc(n, [])
    p = oracle.md_order(n, Kp, Ki)
    assert p.tolist() == list(range(n))
    par, cc = oracle.symbolic(n, Kp, Ki, p)
    assert (par == -1).all() and (cc == 1).all()
    Kp, Ki = lower_csc(3, [(0, 1), (0, 2), (1, 2)])
    par, cc = oracle.symbolic(3, Kp, Ki, oracle.md_order(3, Kp, Ki))
    assert cc.sum() == 6 and par.tolist() == [1, 2, -1]


@pytest.mark.parametrize("seed", range(40))
def test_md_matches_set_bruteforce(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 13))
    dens = rng.uniform(0.1, 0.6)
    edges = [(a, b) for a in range(n) for b in range(a) if rng.random() < dens]
    Kp, Ki = lower_csc(n, edges)
    assert oracle.md_order(n, Kp, Ki).tolist() == dense.md_bruteforce(n, edges).tolist()


@pytest.mark.parametrize("seed", range(20))
def test_symbolic_matches_numeric_cholesky_pattern(seed):
    """etree and column counts equal the nonzero structure of numpy's dense Cholesky of a
    generic SPD matrix with the same graph (no cancellation with random positive values)."""
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(3, 30))
    edges = [(a, b) for a in range(n) for b in range(a) if rng.random() < 0.15]
    Kp, Ki = lower_csc(n, edges)
    perm = rng.permutation(n).astype(np.int32) if seed % 2 else oracle.md_order(n, Kp, Ki)
    par, cc = oracle.symbolic(n, Kp, Ki, perm)
    par2, cc2 = dense.symbolic_numeric_pattern(n, edges, perm, seed)
    assert par.tolist() == par2.tolist() and cc.tolist() == cc2.tolist()


def test_fill_quality_vs_superlu_mmd():
    """Quality sanity (not parity): nnz(L) within +-25% of SuperLU MMD_AT_PLUS_A on C2."""
    inst = make_config("C2")
    Kp, Ki, Kv = oracle.condense(inst)
    perm = oracle.md_order(inst.n, Kp, Ki)
    _, cc = oracle.symbolic(inst.n, Kp, Ki, perm)
    A = sp.csc_matrix((Kv, Ki, Kp), shape=(inst.n, inst.n))
    A = (A + sp.tril(A, -1).T).tocsc()
    lu = spla.splu(A, permc_spec="MMD_AT_PLUS_A", diag_pivot_thresh=0.0,
                   options=dict(SymmetricMode=True))
    nnzL_slu = lu.L.nnz
    assert 0.75 * nnzL_slu <= cc.sum() <= 1.25 * nnzL_slu
