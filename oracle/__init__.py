"""CPU oracle for the condensed-KKT hot path (arXiv 2405.14236).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.  It shares no code with the CUDA path.

Functions whose parity is pinned (tests/test_oracle_*.py): condense, md_order, symbolic,
cholesky, solve_refined, backward_error, hykkt, cg_dense, cr_dense, ldlt (inertia).  Parity unpinned: none of the
numerical functions; CG iteration *counts* on generated data are reported, not compared
(R10).
"""
from .core import (OracleSystem, build, condense, md_order, symbolic, cholesky, trisolve,
                   solve_refined, backward_error, apply_operator, hykkt, cg_dense, cr_dense, ldlt, ldlt_solve, inertia_correct, reference_solve,
                   reference_hykkt)

__all__ = ["OracleSystem", "build", "condense", "md_order", "symbolic", "cholesky", "trisolve",
           "solve_refined", "backward_error", "apply_operator", "hykkt", "cg_dense", "cr_dense", "ldlt", "ldlt_solve", "inertia_correct",
           "reference_solve", "reference_hykkt"]
