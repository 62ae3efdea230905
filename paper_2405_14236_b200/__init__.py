"""B200-native condensed-KKT linear solve (LiftedKKT / HyKKT, arXiv 2405.14236).

The product is libkkt.so (C-ABI, include/kkt.h) with hand-written sm_100a kernels; this
package holds its sources (csrc/), the in-tree build (build.py) and a thin ctypes binding
(kkt.py).  No CPU fallback exists: without the library or a GPU every call raises.
"""
from .kkt import (KKTSolver, KKTError, lib, so_path, kkt_default_options, kkt_analyze,
                  kkt_get_symbolic, kkt_workspace_size, kkt_bind, kkt_condense, kkt_factor,
                  kkt_solve, hykkt_solve, hykkt_solve_krylov, kkt_sync_info, kkt_inertia, kkt_factor_inertia_correct, kkt_solve_unreduced, kkt_recover, kkt_recover_bounds, kkt_step_host, kkt_get_condensed,
                  kkt_get_supernodes, kkt_get_trace, kkt_launch_count, kkt_destroy, EXPORTS, KKT_STATUS)

__all__ = ["KKTSolver", "KKTError", "lib", "so_path", "kkt_default_options", "kkt_analyze",
           "kkt_get_symbolic", "kkt_workspace_size", "kkt_bind", "kkt_condense", "kkt_factor",
           "kkt_solve", "hykkt_solve", "hykkt_solve_krylov", "kkt_sync_info", "kkt_inertia", "kkt_factor_inertia_correct", "kkt_solve_unreduced", "kkt_recover", "kkt_recover_bounds", "kkt_step_host", "kkt_get_condensed",
           "kkt_get_supernodes", "kkt_get_trace", "kkt_launch_count", "kkt_destroy", "EXPORTS", "KKT_STATUS"]
