"""ctypes binding of the sm_100a C-ABI library (include/ssnal_b200.h).

There is deliberately no fallback: a missing library or a non-sm_100 device
raises CudaUnavailableError.
"""

import ctypes
import os

import numpy as np

from .errors import CudaUnavailableError, InternalError

LIB_NAME = "_ssnal_b200.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

# numpy view of ssnal_proj_state_t (checked against ssnal_proj_state_bytes())
PROJ_STATE_DTYPE = np.dtype([
    ("lo", "f8"), ("hi", "f8"), ("flo", "f8"), ("fhi", "f8"),
    ("below_max", "f8"), ("above_min", "f8"), ("in_min", "f8"), ("in_max", "f8"),
    ("in_count", "i8"), ("lam", "f8"), ("tmin", "f8"), ("tmax", "f8"),
    ("sum_v2", "f8"), ("sum_r2", "f8"), ("sum_dref2", "f8"), ("sum_a2_free", "f8"), ("sum_xv", "f8"),
    ("sum_bh", "f8"),
    ("nfree", "i8"), ("status", "i4"), ("passes", "i4"), ("ticket", "u4"), ("pad_", "u4"),
])

PROJ_SEARCH, PROJ_BRACKETED, PROJ_DONE, PROJ_APPLIED, PROJ_NEWTON = 0, 1, 2, 3, 4
PROJ_INFEASIBLE_LOW, PROJ_INFEASIBLE_HIGH = -1, -2
PHASE_RANGE, PHASE_EXACT, PHASE_APPLY = 1, 2, 4

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I = ctypes.c_int
_D = ctypes.c_double
_SZ = ctypes.c_size_t

# name -> (restype, argtypes)
_SIGNATURES = {
    "ssnal_version": (ctypes.c_char_p, []),
    "ssnal_last_error": (ctypes.c_char_p, []),
    "ssnal_launch_count": (ctypes.c_ulonglong, []),
    "ssnal_device_check": (_I, [_I]),
    "ssnal_proj_state_bytes": (_SZ, []),
    "ssnal_report_bytes": (_SZ, []),
    "ssnal_project_ws_bytes": (_SZ, [_I64, _I]),
    "ssnal_reduce_ws_bytes": (_SZ, [_I64, _I]),
    "ssnal_dense_xt_ws_bytes": (_SZ, [_I64, _I64, _I]),
    "ssnal_gram_ws_bytes": (_SZ, [_I64]),
    "ssnal_compact_ws_bytes": (_SZ, [_I64]),
    "ssnal_project": (_I, [_P, _P, _P, _P, _P, _P, _D, _D, _D, _I64, _I, _P, _P, _P, _P, _P,
                           _D, _I, _I, _I, _P]),
    "ssnal_project_ex": (_I, [_P, _P, _P, _P, _P, _P, _D, _D, _D, _I64, _I, _P, _P, _P, _P, _P,
                              _P, _D, _D, _I, _I, _I, _P]),
    "ssnal_hs_apply": (_I, [_P, _P, _P, _I64, _D, _P, _D, _P, _P, _P]),
    "ssnal_dots": (_I, [_I, _P, _P, _P, _I64, _P, _P, _P]),
    "ssnal_vec": (_I, [_I, _I64, _D, _P, _P, _P, _P, _P]),
    "ssnal_dense_xt": (_I, [_P, _I64, _I64, _I64, _P, _I, _I, _P, _P, _P, _P]),
    "ssnal_dense_x": (_I, [_P, _I64, _I64, _I64, _P, _I, _I, _P, _P, _P]),
    "ssnal_compact": (_I, [_P, _I64, _P, _P, _P, _P]),
    "ssnal_dense_gram": (_I, [_P, _I64, _I64, _I64, _P, _I, _P, _P, _I64, _P, _D, _P, _P, _P,
                              _P, _P]),
    "ssnal_chol_solve": (_I, [_P, _I64, _P, _D, _P, _P, _P]),
    "ssnal_pspace_ws_bytes": (_SZ, [_I64, _I64]),
    "ssnal_dense_newton_pspace": (_I, [_P, _I64, _I64, _I64, _P, _I, _P, _I64, _P, _P, _D, _D,
                                       _P, _P, _P, _P, _P]),
}

class CsrOperator(ctypes.Structure):
    """ssnal_csr_operator_t"""
    _fields_ = [("n", ctypes.c_int64), ("q", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("indptr", _P), ("indices", _P), ("values", _P),
                ("colptr", _P), ("rowidx", _P), ("valt", _P), ("row_sign", _P),
                ("nseg", ctypes.c_int64), ("seg_beg", _P), ("seg_end", _P), ("seg_col", _P),
                ("seg_slot", _P), ("nfold", ctypes.c_int64), ("fold_col", _P), ("fold_beg", _P),
                ("nslots", ctypes.c_int64),
                ("nhot", ctypes.c_int64), ("hot_cols", _P), ("hot_rank", _P)]


class DenseProblem(ctypes.Structure):
    """ssnal_dense_problem_t"""
    _fields_ = [("A", _P), ("n_phys", ctypes.c_int64), ("q", ctypes.c_int64),
                ("lda", ctypes.c_int64), ("row_sign", _P), ("svr_block", _I),
                ("n", ctypes.c_int64), ("c", _P), ("a", _P), ("l", _P), ("u", _P),
                ("l_const", _D), ("u_const", _D), ("d", _D), ("csr", ctypes.POINTER(CsrOperator))]


class Options(ctypes.Structure):
    """ssnal_options_t"""
    _fields_ = [("sigma0", _D), ("sigma_growth", _D), ("sigma_max", _D), ("tol_kkt", _D),
                ("lambda_min_surrogate", _D), ("max_outer", _I), ("mu", _D), ("backtrack", _D),
                ("tau", _D), ("eta", _D), ("max_inner", _I), ("direct_solve_threshold", _I),
                ("cg_max_iters", _I), ("line_search_batch", _I), ("psi_stable", _I),
                ("profile", _I)]


NOPS = 7
OP_NAMES = ("dense_xt", "dense_x", "project", "newton_system", "vector", "gram", "chol")


class Report(ctypes.Structure):
    """ssnal_report_t"""
    _fields_ = [("kkt_residual", _D), ("objective", _D), ("wall_time", _D),
                ("outer_iters", _I), ("total_inner_iters", _I),
                ("unbounded_support_count", _I), ("converged", _I),
                ("hit_max_inner_mask", _I), ("stagnated", _I), ("max_outer_reached", _I),
                ("syncs", ctypes.c_longlong), ("newton_steps", ctypes.c_longlong),
                ("projections", ctypes.c_longlong), ("launches", ctypes.c_longlong),
                ("op_seconds", _D * NOPS), ("op_calls", ctypes.c_longlong * NOPS),
                ("op_bytes", _D * NOPS), ("op_flops", _D * NOPS), ("cg_iters", ctypes.c_longlong),
                ("cg_fallbacks", ctypes.c_longlong), ("gram_builds", ctypes.c_longlong),
                ("gram_updates", ctypes.c_longlong), ("gram_rows", ctypes.c_longlong),
                ("proj_fallbacks", ctypes.c_longlong),
                ("hit_max_inner_mask64", ctypes.c_ulonglong), ("hit_max_inner_count", _I),
                ("pad_", _I)]


PROGRESS_FN = ctypes.CFUNCTYPE(None, _I, _D, _D, ctypes.c_longlong, _I, _P)

COMM_ID_BYTES = 128
ALLREDUCE_FN = ctypes.CFUNCTYPE(_I, _P, _P, _I64, _P)
ALLGATHER_FN = ctypes.CFUNCTYPE(_I, _P, _P, _P, _I64, _P)


class Comm(ctypes.Structure):
    """ssnal_comm_t (the row-sharded driver's transport)"""
    _fields_ = [("world", _I), ("rank", _I), ("allreduce_sum", ALLREDUCE_FN),
                ("allgather", ALLGATHER_FN), ("ctx", _P), ("kind", _I), ("pad_", _I)]

_SIGNATURES.update({
    "ssnal_alm_ws_bytes": (_SZ, [_I64, _I64, _I]),
    "ssnal_alm_ws_bytes_csr": (_SZ, [ctypes.POINTER(CsrOperator)]),
    "ssnal_csr_xd": (_I, [ctypes.POINTER(CsrOperator), _P, _I64, _P, _P, _P]),
    "ssnal_csr_xt": (_I, [ctypes.POINTER(CsrOperator), _P, _P, _P, _P]),
    "ssnal_csr_colsq": (_I, [ctypes.POINTER(CsrOperator), _P, _P, _P, _P]),
    "ssnal_csr_restricted_ws_bytes": (ctypes.c_size_t, [ctypes.POINTER(CsrOperator)]),
    "ssnal_csr_xt_restricted": (_I, [ctypes.POINTER(CsrOperator), _P, _P, _I64, _P, _P, _P, _P]),
    "ssnal_csr_xd_restricted": (_I, [ctypes.POINTER(CsrOperator), _P, _P, _I64, _P, _P, _P, _P]),
    "ssnal_alm_solve_dense": (_I, [ctypes.POINTER(DenseProblem), ctypes.POINTER(Options), _P, _P,
                                   _P, ctypes.POINTER(Report), _P, _SZ, PROGRESS_FN, _P, _P]),
    "ssnal_alm_ws_bytes_sharded": (_SZ, [_I64, _I64, _I, _I]),
    "ssnal_alm_ws_bytes_csr_sharded": (_SZ, [ctypes.POINTER(CsrOperator), _I]),
    "ssnal_alm_solve_sharded": (_I, [ctypes.POINTER(DenseProblem), ctypes.POINTER(Options),
                                     ctypes.POINTER(Comm), _P, _P, _P, ctypes.POINTER(Report), _P,
                                     _SZ, PROGRESS_FN, _P, _P]),
    "ssnal_nccl_unique_id": (_I, [ctypes.c_char_p]),
    "ssnal_nccl_comm_create": (_I, [_I, _I, ctypes.c_char_p, ctypes.POINTER(Comm)]),
    "ssnal_loopback_group_create": (_I, [_I, ctypes.POINTER(_P)]),
    "ssnal_loopback_comm_create": (_I, [_P, _I, ctypes.POINTER(Comm)]),
    "ssnal_loopback_group_destroy": (_I, [_P]),
    "ssnal_comm_destroy": (_I, [ctypes.POINTER(Comm)]),
    "ssnal_proj_local_ws_bytes": (_SZ, [_I64, _I]),
    "ssnal_proj_local": (_I, [_P, _P, _P, _P, _P, _P, _P, _D, _D, _I64, _I, _I, _P, _P, _P, _P,
                              _D, _P, _P, _P]),
    "ssnal_sum_slices": (_I, [_I, _I64, _P, _P, _P]),
    "ssnal_hs_apply_coef": (_I, [_P, _P, _P, _I64, _D, _P, _D, _D, _P, _P]),
    "ssnal_qspace_assemble": (_I, [_I64, _P, _D, _D, _D, _P, _P]),
    "ssnal_gradient_ws_bytes": (_SZ, [_I64, _I64]),
    "ssnal_dense_gradient": (_I, [_P, _I64, _I64, _I64, _P, _I, _P, _P, _P, _P, _P, _P, _P, _P]),
    "ssnal_dense_direction_epilogue": (_I, [_P, _I64, _I64, _I64, _P, _I, _P, _P, _P, _P, _P, _P,
                                            _D, _P, _P, _P, _P, _P, _P, _P]),
})

_lib = None


def exported_symbols():
    return tuple(_SIGNATURES)


def load():
    """Load (once) and type the library; raises CudaUnavailableError if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise CudaUnavailableError(
            f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.ssnal_proj_state_bytes() != PROJ_STATE_DTYPE.itemsize:
        raise InternalError("ssnal_proj_state_t layout mismatch between C and Python")
    if lib.ssnal_report_bytes() != ctypes.sizeof(Report):
        raise InternalError("ssnal_report_t layout mismatch between C and Python")
    _lib = lib
    return lib


def call(name, *args):
    """Invoke an entry point and raise on a nonzero status."""
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        msg = lib.ssnal_last_error().decode(errors="replace")
        raise InternalError(f"{name} failed ({rc}): {msg}")


def ptr_array(ptrs):
    """HOST array of device pointers for the const double* const* arguments."""
    arr = (ctypes.c_void_p * len(ptrs))(*[ctypes.c_void_p(p) if p else None for p in ptrs])
    return ctypes.cast(arr, ctypes.c_void_p), arr
