"""ctypes binding of libhdgb200.so (C ABI in include/hdgb200.h).

No CPU fallback: importing the package on a machine without the built library
raises immediately, and every entry point raises HDGError on a nonzero status.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HDGB200_LIB") or os.path.join(_HERE, "libhdgb200.so")

c_double_p = ctypes.POINTER(ctypes.c_double)
c_void_p = ctypes.c_void_p
c_int = ctypes.c_int
c_int64 = ctypes.c_int64
c_int32 = ctypes.c_int32

# (name, restype, argtypes) - mirrors include/hdgb200.h exactly
SIGNATURES = [
    ("hdg_last_error", ctypes.c_char_p, []),
    ("hdg_version", c_int, []),
    ("hdg_launch_count", c_int64, []),
    ("hdg_level_create_shared", c_int, [c_int, c_int, c_int, c_void_p, ctypes.POINTER(c_void_p)]),
    ("hdg_level_create_stored", c_int, [c_int, c_int, c_int, c_void_p, ctypes.POINTER(c_void_p)]),
    ("hdg_level_create_stored_empty", c_int, [c_int, c_int, c_int, ctypes.POINTER(c_void_p)]),
    ("hdg_level_fill_stored_rows", c_int, [c_void_p, c_int, c_int, c_void_p, c_void_p]),
    ("hdg_level_destroy", c_int, [c_void_p]),
    ("hdg_level_ndof", c_int64, [c_void_p]),
    ("hdg_level_operator_bytes", c_int64, [c_void_p]),
    ("hdg_level_set_blockjacobi", c_int, [c_void_p, ctypes.c_double]),
    ("hdg_matvec", c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    ("hdg_soa_length", c_int, [c_void_p, ctypes.POINTER(c_int64)]),
    ("hdg_soa_pack", c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    ("hdg_soa_unpack", c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    ("hdg_matvec_soa", c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    ("hdg_residual", c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    ("hdg_bj_sweep", c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    ("hdg_level_set_bj_chebyshev", c_int, [c_void_p, ctypes.c_double, ctypes.c_double]),
    ("hdg_bj_sweeps", c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_void_p]),
    ("hdg_level_set_fsai", c_int, [c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_void_p,
                                   c_void_p, ctypes.c_double, ctypes.c_double, ctypes.c_double]),
    ("hdg_level_set_fsai_struct", c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int, ctypes.c_double,
                                          ctypes.c_double, c_double_p, ctypes.POINTER(c_int64), c_void_p]),
    ("hdg_level_fsai_struct_get", c_int, [c_void_p, c_void_p, c_void_p]),
    ("hdg_fsai_apply", c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    ("hdg_fsai_sweeps", c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_void_p]),
    ("hdg_transfer_create_p", c_int, [c_void_p, c_void_p, c_void_p, ctypes.POINTER(c_void_p)]),
    ("hdg_transfer_create_h", c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64,
                                      ctypes.POINTER(c_void_p)]),
    ("hdg_transfer_create_h_window", c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int, c_int,
                                             ctypes.POINTER(c_void_p)]),
    ("hdg_transfer_destroy", c_int, [c_void_p]),
    ("hdg_prolong_add", c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    ("hdg_restrict", c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    ("hdg_mg_create", c_int, [ctypes.POINTER(c_void_p), ctypes.POINTER(c_void_p), c_int,
                              ctypes.POINTER(c_void_p)]),
    ("hdg_mg_destroy", c_int, [c_void_p]),
    ("hdg_mg_set_coarse_inverse", c_int, [c_void_p, c_void_p, c_int64]),
    ("hdg_mg_set_fused_tail", c_int, [c_void_p, c_int]),
    ("hdg_mg_set_records", c_int, [c_void_p, c_int]),
    ("hdg_mg_record_levels", c_int, [c_void_p]),
    ("hdg_mg_cycle_records", c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_int,
                                     c_void_p]),
    ("hdg_fsai_rows", c_int, [c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int32,
                              ctypes.POINTER(c_int64), c_void_p]),
    ("hdg_mg_cycle", c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, c_int,
                             c_void_p]),
    ("hdg_coarse_solve", c_int, [c_void_p, c_void_p, c_void_p, c_void_p]),
    ("hdg_mg_graph_captures", c_int64, [c_void_p]),
    ("hdg_solve_mg", c_int, [c_void_p, c_void_p, c_void_p, c_int, c_int, c_int, ctypes.c_double, c_int,
                             c_double_p, ctypes.POINTER(c_int), c_void_p]),
    ("hdg_pcg", c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int, ctypes.c_double, c_int, c_int, c_int,
                        c_double_p, ctypes.POINTER(c_int), c_void_p]),
    ("hdg_dot", c_int, [c_void_p, c_void_p, c_int64, c_void_p, c_void_p]),
    ("hdg_cg_update", c_int, [c_void_p, c_void_p, c_void_p, c_void_p, ctypes.c_double, c_int64, c_void_p]),
    ("hdg_xpby", c_int, [c_void_p, ctypes.c_double, c_void_p, c_int64, c_void_p]),
    ("hdg_condense_piecewise", c_int, [c_int, c_int, c_int64] + [c_void_p] * 14),
    ("hdg_piecewise_usolve", c_int, [c_int, c_int64] + [c_void_p] * 8),
    ("hdg_gemm_nt", c_int, [c_int64, c_int, c_int, c_void_p, c_int, c_void_p, c_void_p, c_int, c_void_p, c_void_p,
                            c_void_p, c_int, ctypes.c_double, ctypes.c_double, c_void_p]),
    ("hdg_class_gemv", c_int, [c_int64, c_int, c_int, c_void_p, c_void_p, c_void_p, c_int, c_void_p, c_int,
                               ctypes.c_double, ctypes.c_double, c_void_p]),
    ("hdg_galerkin_p", c_int, [c_int64, c_int, c_int, c_void_p, c_void_p, c_void_p, c_void_p]),
    ("hdg_galerkin_h", c_int, [c_int64, c_void_p, c_void_p, c_int, c_void_p, c_void_p]),
    ("hdg_gather_elements", c_int, [c_int, c_int, c_int, c_void_p, c_void_p, c_void_p]),
    ("hdg_sum_owners", c_int, [c_int, c_int, c_int, c_void_p, c_void_p, c_void_p]),
    ("hdg_dist_init", c_int, [c_void_p, c_int, c_int, ctypes.POINTER(c_void_p)]),
    ("hdg_dist_destroy", c_int, [c_void_p]),
    ("hdg_dist_halo", c_int, [c_void_p, c_void_p, c_int, c_int, c_int, c_int, c_int, c_void_p, c_void_p]),
    ("hdg_dist_allreduce_sum", c_int, [c_void_p, c_void_p, c_int, c_void_p]),
]


class HDGError(RuntimeError):
    pass


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def check(rc):
    if rc != 0:
        raise HDGError(lib.hdg_last_error().decode() or f"hdg error {rc}")
    return rc


def exported_symbols():
    return [name for name, _, _ in SIGNATURES]
