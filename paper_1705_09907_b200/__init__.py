"""B200-native HDG trace operator + geometric-multigrid hot path (arxiv 1705.09907).

Drop-in for the reference `hdgmg` package's hot path:
  trace.TraceSystem.matvec_free          <- hdgmg/trace.py:87-94
  multigrid.{build_hierarchy, MGLevel, p_prolongation, h_prolongation,
             attach_smoothers, v_cycle, w_cycle, solve_mg, fmg,
             mg_preconditioner, ConvergenceMonitor}  <- hdgmg/multigrid.py
All compute runs in hand-written sm_100a kernels (libhdgb200.so, C ABI in
include/hdgb200.h); importing fails loudly if the library is not built.
"""

from ._lib import HDGError, lib  # noqa: F401  (loads libhdgb200.so or raises)
from .mesh import build_cartesian, coarsen  # noqa: F401

__version__ = "0.1.0"


def __getattr__(name):
    # torch-backed modules load on first use so `import paper_1705_09907_b200` stays light
    if name in ("trace", "multigrid", "problem"):
        import importlib
        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
