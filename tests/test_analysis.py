"""Host analysis of libkkt.so (kkt_analyze runs on the CPU; no GPU needed) -- `not gpu`.

* MD-exact-v1 ordering, etree and column counts are bit-exact with the oracle (R11) on the
  workload patterns and on random small patterns;
* argument / pattern validation returns status codes (never aborts);
* the library exports every symbol include/kkt.h declares.
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle
import paper_2405_14236_b200 as K
from synth.generator import make_config, tiny_random

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "kkt.h")).read()
    decl = set(re.findall(r"^(?:kkt_status|const char \*|int)\s*(\w+)\s*\(", hdr, re.M))
    assert decl, "no declarations parsed"
    L = K.lib()
    for name in decl:
        assert hasattr(L, name), name
    assert decl == set(K.EXPORTS)


@pytest.mark.parametrize("cfg", ["C1", "C2", "C5", "C3", "C4", "C7"])
def test_ordering_etree_colcounts_bitexact(cfg):
    inst = make_config(cfg) if cfg != "C5" else make_config("C5", batch=1)
    S = K.KKTSolver.from_instance(inst)
    perm, et, cc = S.symbolic()
    Kp, Ki, _ = oracle.condense(inst)
    pr = oracle.md_order(inst.n, Kp, Ki)
    par, occ = oracle.symbolic(inst.n, Kp, Ki, pr)
    assert np.array_equal(perm, pr)
    assert np.array_equal(et, par)
    assert np.array_equal(cc, occ)
    assert S.info["nnzK"] == len(Ki)
    assert S.info["nnzL"] == int(occ.sum())
    S.close()


@pytest.mark.parametrize("seed", range(60))
def test_random_patterns_bitexact(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 60))
    m = int(rng.integers(0, 40))
    inst = tiny_random(n, m, int(rng.integers(0, m + 1)) if m else 0, density=rng.uniform(0.02, 0.3),
                       seed=seed)
    S = K.KKTSolver.from_instance(inst)
    perm, et, cc = S.symbolic()
    Kp, Ki, _ = oracle.condense(inst)
    pr = oracle.md_order(inst.n, Kp, Ki)
    par, occ = oracle.symbolic(inst.n, Kp, Ki, pr)
    assert np.array_equal(perm, pr) and np.array_equal(et, par) and np.array_equal(cc, occ)
    S.close()


def test_condensed_pattern_matches_oracle():
    inst = make_config("C2")
    S = K.KKTSolver.from_instance(inst)
    Kp, Ki, _ = S.get_condensed(0, values=False)
    Op, Oi, _ = oracle.condense(inst)
    assert np.array_equal(Kp, Op) and np.array_equal(Ki, Oi)


def _analyze(n, m, me, Wp, Wc, Jp, Jc):
    h = C.c_void_p()
    o = K.kkt_default_options()
    arr = [np.ascontiguousarray(a, np.int32) for a in (Wp, Wc, Jp, Jc)]
    return K.lib().kkt_analyze(n, m, me, *[a.ctypes.data for a in arr], C.byref(o), C.byref(h), None), h


def test_pattern_errors_return_codes():
    # upper-triangle entry in W
    code, _ = _analyze(2, 0, 0, [0, 1, 2], [1, 1], [0], [0])
    assert K.KKT_STATUS[code] == "KKT_ERR_PATTERN"
    # unsorted J row
    code, _ = _analyze(3, 1, 0, [0, 1, 2, 3], [0, 1, 2], [0, 2], [2, 0])
    assert K.KKT_STATUS[code] == "KKT_ERR_PATTERN"
    # J column out of range
    code, _ = _analyze(2, 1, 0, [0, 1, 2], [0, 1], [0, 1], [5])
    assert K.KKT_STATUS[code] == "KKT_ERR_PATTERN"
    # m_eq > m
    code, _ = _analyze(2, 1, 2, [0, 1, 2], [0, 1], [0, 1], [0])
    assert K.KKT_STATUS[code] == "KKT_ERR_ARG"
    # ok (W without diagonal entries, empty J row)
    code, h = _analyze(3, 2, 0, [0, 0, 1, 1], [0], [0, 0, 2], [0, 2])
    assert code == 0
    K.kkt_destroy(h)


def test_state_errors_without_bind():
    inst = tiny_random(5, 3, 0, seed=1)
    S = K.KKTSolver.from_instance(inst)
    code = K.lib().kkt_factor(S.h)
    assert K.KKT_STATUS[code] == "KKT_ERR_STATE"
    code = K.lib().kkt_condense(S.h, None, None, None, None, None, 0.0, 0.0, 0.0)
    assert K.KKT_STATUS[code] == "KKT_ERR_STATE"


@pytest.mark.parametrize("cfg,kind,cap,nw", [("C2", 0, 6144, 8), ("C2", 0, 1024, 4), ("C5", 0, 4096, 4),
                                             ("C2", 1, 6144, 4), ("C5", 1, 2048, 4), ("C1", 0, 2048, 8)])
def test_subtree_block_plan(cfg, kind, cap, nw):
    """Host plan of the block kernels (sblock.cuh / fblock.cuh): every block is a whole subtree of
    small supernodes (a contiguous postorder range ending at its root), blocks are maximal and
    disjoint, fit the budget, their level lists put every child below its parent, and the
    backward row map sends own columns to their block-local column and every other row inside
    the block's column range or the root's update rows."""
    import paper_2405_14236_b200 as K
    inst = make_config(cfg) if cfg != "C5" else make_config("C5", batch=1)
    S = K.KKTSolver.from_instance(inst)
    f, r, par = S.supernodes()
    ns = len(r)
    w = np.diff(f)
    blk, blk_of, meta, lrow, big = S.blocks(kind, cap, nw)
    assert len(blk) > 0
    rp = np.concatenate([[0], np.cumsum(r)])
    owner = -np.ones(ns, dtype=np.int64)
    for b, (lo, hi, nlev, m0, total, *_rest) in enumerate(blk):
        assert 0 <= lo <= hi < ns and blk_of[hi] == b and total <= cap
        assert not big[lo:hi + 1].any()
        assert (owner[lo:hi + 1] == -1).all()
        owner[lo:hi + 1] = b
        # whole subtree: every member's parent is in the range (except the root's), nothing
        # outside the range has its parent inside
        for t in range(lo, hi):
            assert lo < par[t] <= hi and blk_of[t] == -2
        inside = (par >= lo) & (par <= hi)
        assert set(np.nonzero(inside)[0]) <= set(range(lo, hi + 1))
        # maximal: the root's parent is big, absent, or outside every block
        assert par[hi] < 0 or big[par[hi]] or blk_of[par[hi]] == -1
        # level lists: a permutation, children strictly below their parent
        nn = hi - lo + 1
        lv = meta[m0:m0 + nlev + 1]
        nodes = meta[m0 + nlev + 1:m0 + nlev + 1 + nn]
        assert lv[0] == 0 and lv[-1] == nn and (np.diff(lv) >= 0).all()
        assert sorted(nodes) == list(range(nn))
        level = np.empty(nn, dtype=np.int64)
        for l in range(nlev):
            level[nodes[lv[l]:lv[l + 1]]] = l
        for t in range(lo, hi):
            assert level[t - lo] < level[par[t] - lo]
        if kind == 0:  # backward row map
            F0, ncol = f[lo], f[hi + 1] - f[lo]
            Rroot = r[hi] - w[hi]
            for t in range(lo, hi + 1):
                lr = lrow[rp[t]:rp[t + 1]]
                assert (lr[:w[t]] == f[t] - F0 + np.arange(w[t])).all()
                assert ((lr >= 0) & (lr < ncol + Rroot)).all()
    # small supernodes outside the blocks are exactly the blk_of == -1 non-big ones
    assert ((owner >= 0) | big.astype(bool) | (blk_of == -1)).all()
    assert (blk_of[big.astype(bool)] == -1).all()
