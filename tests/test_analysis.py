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
