"""ctypes binding of the C ABI (include/cyqlone_b200.h).

The product path is libcyqlone_b200.so, built in-tree for sm_100a by
`__graft_entry__.build()` (or `python -m paper_2512_09058_b200.build`).
There is no fallback: if the library is missing, or no CUDA device is
present, calls raise instead of computing anything on the CPU.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# CYQ_LIB selects another build of the same library (tools/build_debug.sh)
LIB_PATH = os.environ.get("CYQ_LIB") or os.path.join(HERE, "libcyqlone_b200.so")

CYQ_OK, CYQ_INVALID_ARG, CYQ_PIVOT_FAIL, CYQ_CUDA_ERR, CYQ_NO_DEVICE = 0, 1, 2, 3, 4
CYQ_MEM_HOST, CYQ_MEM_DEVICE = 0, 1

# cyq_ctx_set_option keys and named values (include/cyqlone_b200.h)
OPTIONS = {"panel": 0, "schur": 1, "schur_warps": 2, "schur_cluster": 3, "split": 4,
           "backsub": 5, "fused_augment": 6, "panel_warps": 7, "tail": 8, "phase_prof": 9,
           "async_status": 10, "graphs": 11, "vlen": 12}
OPTION_VALUES = {
    "panel": {"auto": 0, "warp": 1, "two_warp": 2, "cta": 3, "generic": 4, "warp_tmem": 5, "cta_tma": 6},
    "schur": {"auto": 0, "levels": 1, "scalar": 2},
    "backsub": {"auto": 0, "generic": 1},
    "tail": {"cr1": 0, "pcr": 1, "pcg": 2},
}

i64 = C.c_int64
dp = C.POINTER(C.c_double)


class CyqDims(C.Structure):
    _fields_ = [("N", i64), ("nx", i64), ("nu", i64), ("P", i64), ("batch", i64)]


class CyqOcpBatch(C.Structure):
    _fields_ = [(k, C.c_void_p) for k in ("A", "B", "R", "S", "Q", "f", "r", "q", "x_init")]


class CyqRhsBatch(C.Structure):
    _fields_ = [(k, C.c_void_p) for k in ("ru", "qx", "fd")]


class CyqSolBatch(C.Structure):
    _fields_ = [(k, C.c_void_p) for k in ("u", "x", "lam")]


class CyqUpdateReport(C.Structure):
    _fields_ = [("columns_updated", i64), ("columns_refactored", i64), ("schur_refactored", i64),
                ("schur_levels_updated", i64)]


class CyqStatus(C.Structure):
    _fields_ = [("code", C.c_int32), ("kind", C.c_int32), ("instance", i64),
                ("column_or_level", i64), ("stage", i64), ("pivot", i64)]


# exported symbols and their signatures (kept in sync with the header; the
# CPU test suite checks every declared symbol is exported)
SIGNATURES = {
    "cyq_ctx_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "cyq_ctx_destroy": (C.c_int, [C.c_void_p]),
    "cyq_ctx_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "cyq_ctx_synchronize": (C.c_int, [C.c_void_p]),
    "cyq_ctx_last_error": (C.c_char_p, [C.c_void_p]),
    "cyq_solve_problem_batch": (C.c_int, [C.c_void_p, C.POINTER(CyqDims), C.POINTER(CyqOcpBatch),
                                          C.POINTER(CyqSolBatch), C.c_void_p, C.c_int]),
    "cyq_factor_batch": (C.c_int, [C.c_void_p, C.POINTER(CyqDims), C.POINTER(CyqOcpBatch),
                                   C.c_int, C.POINTER(C.c_void_p), C.c_void_p]),
    "cyq_solve_batch": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(CyqOcpBatch),
                                  C.POINTER(CyqRhsBatch), C.POINTER(CyqSolBatch), C.c_int]),
    "cyq_factor_destroy": (C.c_int, [C.c_void_p]),
    "cyq_factor_materialize": (C.c_int, [C.c_void_p, i64, C.c_void_p, C.c_void_p, C.c_void_p,
                                         C.c_void_p]),
    "cyq_ctx_profile": (C.c_int, [C.c_void_p, C.c_int]),
    "cyq_ctx_set_option": (C.c_int, [C.c_void_p, C.c_int, i64]),
    "cyq_ctx_get_option": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(i64)]),
    "cyq_ctx_wait_status": (C.c_int, [C.c_void_p, C.c_void_p, i64]),
    "cyq_factor_materialize_schur": (C.c_int, [C.c_void_p, i64] + [C.c_void_p] * 10),
    "cyq_factor_update_batch": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, i64, C.c_void_p, C.c_void_p,
                                          C.c_void_p, i64, C.c_void_p, C.c_void_p, C.c_double, C.c_int,
                                          C.c_void_p]),
    "cyq_al_gradients_batch": (C.c_int, [C.c_void_p, C.c_void_p, i64, C.c_void_p] + [C.c_void_p] * 10
                               + [C.c_double] + [C.c_void_p] * 4),
    "cyq_ctx_profile_read": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.POINTER(i64),
                                       C.c_int]),
    "cyq_version": (C.c_char_p, []),
    "cyq_augment_hessians_batch": (C.c_int, [C.c_void_p, C.POINTER(CyqDims), i64] + [C.c_void_p] * 6
                                   + [C.c_double] + [C.c_void_p] * 3),
    "cyq_line_search_batch": (C.c_int, [C.c_void_p, i64, i64] + [C.c_void_p] * 5
                              + [C.POINTER(C.c_int32), C.c_void_p]),
    "cyq_solve_newton_batch": (C.c_int, [C.c_void_p, C.POINTER(CyqDims), C.POINTER(CyqOcpBatch), i64]
                               + [C.c_void_p] * 3 + [C.c_double, C.POINTER(CyqSolBatch), C.c_void_p]),
}

_lib = None


def load(path: str = LIB_PATH):
    """Loads libcyqlone_b200.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(
            f"{path} not built: run __graft_entry__.build() (nvcc, sm_100a). "
            "There is no CPU fallback for the KKT path.")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
