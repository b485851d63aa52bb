"""ctypes binding of libpk_b200.so (include/pipekrylov_b200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_1410_4054_b200/csrc``).  There is no fallback: if the library
or a CUDA device is missing, every entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libpk_b200.so"
if os.environ.get("PK_LIB_VARIANT"):  # engine experiments: libpk_b200_<variant>.so built by tools/build_variants.sh
    LIB_PATH = LIB_PATH.with_name(f"libpk_b200_{os.environ['PK_LIB_VARIANT']}.so")

PK_OK, PK_ERR_INVALID, PK_ERR_CUDA, PK_ERR_NOMEM, PK_ERR_UNSUPPORTED = 0, 1, 2, 3, 4
TERM_NAMES = {0: "converged", 1: "max_iter", 2: "breakdown", 3: "lucky_breakdown"}
KIND_NAMES = {0: None, 1: "pAp", 2: "Apr0star", 3: "AsAs", 4: "divergence", 5: "singular_R"}
METHODS = {"cg": 0, "bicgstab": 1, "gmres": 2}
DOT_INPUT, DOT_RESULT, DOT_VECTOR = 0, 1, 2
# pk_vec_update kinds (include/pipekrylov_b200.h PK_VEC_*)
VEC_AXPY, VEC_AXPY2, VEC_XPAY, VEC_SCALE, VEC_ADD_SCALED, VEC_BICG_P, VEC_COPY = range(7)
GEN = {"poisson2d": 0, "poisson3d": 1, "convdiff2d": 2, "convdiff3d": 3}
LOOP_GRAPH, LOOP_HOST = 0, 1
FMT_CSR, FMT_SELL32 = 0, 1
FLAG_PROFILE = 1


class NativeError(RuntimeError):
    """A CUDA/runtime failure inside libpk_b200 (not a numerical breakdown)."""


class PkConfig(C.Structure):
    _fields_ = [
        ("tolerance", C.c_double),
        ("max_iterations", C.c_int64),
        ("restart", C.c_int64),
        ("breakdown_tolerance", C.c_double),
        ("fixed_iterations", C.c_int64),
        ("loop_mode", C.c_int32),
        ("flags", C.c_int32),
    ]


class PkResult(C.Structure):
    _fields_ = [
        ("iterations", C.c_int64),
        ("termination", C.c_int32),
        ("breakdown_kind", C.c_int32),
        ("true_final_residual", C.c_double),
        ("loop_seconds", C.c_double),
        ("setup_launches", C.c_int64),
        ("setup_transfers", C.c_int64),
        ("launches_per_iteration", C.c_int64),
        ("transfers_per_iteration", C.c_int64),
        ("finish_launches", C.c_int64),
        ("finish_transfers", C.c_int64),
        ("total_launches", C.c_int64),
        ("total_transfers", C.c_int64),
        ("cycles", C.c_int64),
        ("check_phases", C.c_int64),
        ("kernel_seconds", C.c_double * 4),
        ("kernel_launches", C.c_int64 * 4),
    ]


DEBUG_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int32, C.c_int64, C.POINTER(C.c_double), C.POINTER(C.c_double),
                       C.c_int64, C.POINTER(C.c_double), C.c_int32)
DBG_CG_SETUP, DBG_CG_ITER, DBG_BICG_SETUP, DBG_BICG_S, DBG_BICG_XRP, DBG_GMRES_CYCLE = 1, 2, 3, 4, 5, 6

TRISOLVE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int64, C.POINTER(C.c_double), C.c_int64,
                          C.POINTER(C.c_double), C.c_double, C.POINTER(C.c_double))

_P = C.c_void_p
_DP = C.POINTER(C.c_double)
_I64P = C.POINTER(C.c_int64)

# name -> argtypes (restype is always c_int unless listed in _RESTYPES)
SIGNATURES = {
    "pk_last_error": [],
    "pk_abi_version": [],
    "pk_device_count": [C.POINTER(C.c_int)],
    "pk_ctx_create": [C.c_int, C.c_int64, C.c_int64, C.POINTER(_P)],
    "pk_ctx_destroy": [_P],
    "pk_ctx_set_stream": [_P, _P],
    "pk_ctx_set_debug": [_P, DEBUG_FN, _P],
    "pk_ctx_reset_stream": [_P],
    "pk_ctx_synchronize": [_P],
    "pk_ctx_geometry": [_P, _I64P, _I64P],
    "pk_csr_upload": [_P, C.c_int64, C.c_int64, _I64P, _I64P, _DP, C.POINTER(_P)],
    "pk_csr_generate": [_P, C.c_int32, _I64P, C.c_int32, _DP, C.c_int32, C.POINTER(_P)],
    "pk_csr_info": [_P, _I64P, _I64P, _I64P, _I64P],
    "pk_csr_download": [_P, _P, _I64P, _I64P, _DP],
    "pk_mat_destroy": [_P],
    "pk_mat_set_format": [_P, _P, C.c_int32],
    "pk_mat_get_format": [_P, C.POINTER(C.c_int32), _I64P],
    "pk_spmv": [_P, _P, _P, _P],
    "pk_spmv_fused": [_P, _P, _P, _P, C.c_int32, C.POINTER(C.c_int32), C.POINTER(_P), _P],
    "pk_reduce_stage1": [_P, C.c_int64, C.c_int32, C.POINTER(_P), _P],
    "pk_reduce_stage2": [_P, C.c_int32, _P, _P],
    "pk_dot": [_P, C.c_int64, _P, _P, _P],
    "pk_ell_upload": [_P, C.c_int64, C.c_int64, C.c_int64, _P, _P, _P],
    "pk_ell_destroy": [_P],
    "pk_spmv_ell": [_P, _P, _P, _P],
    "pk_vec_update": [_P, C.c_int32, C.c_int64, _P, _P, _P, C.c_double, C.c_double],
    "pk_cg_update": [_P, C.c_int64, _P, _P, _P, _P, C.c_double, C.c_double, _P],
    "pk_bicg_s_update": [_P, C.c_int64, _P, _P, _P, _P, C.c_double, _P, _P, _P, _P],
    "pk_bicg_xrp_update": [_P, C.c_int64, _P, _P, _P, _P, _P, _P, C.c_double, C.c_double, C.c_double, _P, _P],
    "pk_gs_stage1": [_P, C.c_int64, C.c_int32, C.POINTER(_P), _P, _P],
    "pk_gs_update": [_P, C.c_int64, _P, C.c_int32, C.POINTER(_P), _P, _P, _P],
    "pk_gs_normalize": [_P, C.c_int64, _P, _P, _P, C.c_double, _P, _P, _P],
    "pk_solve": [_P, _P, C.c_int32, _DP, _DP, C.POINTER(PkConfig), TRISOLVE_FN, _P, _DP, _DP, C.c_int64,
                 C.POINTER(PkResult)],
    "pk_solve_device": [_P, _P, C.c_int32, _P, _P, C.POINTER(PkConfig), TRISOLVE_FN, _P, _P, _DP, C.c_int64,
                        C.POINTER(PkResult)],
    "pk_solve_batch": [_P, C.c_int64, C.POINTER(_P), C.c_int32, C.POINTER(_P), C.POINTER(_P),
                       C.POINTER(PkConfig), TRISOLVE_FN, _P, C.POINTER(_P), C.POINTER(_P), C.c_int64,
                       C.POINTER(PkResult), C.c_int32],
    "pk_csr_generate_rows": [_P, C.c_int32, _I64P, C.c_int32, _DP, C.c_int32, C.c_int64, C.c_int64, C.c_int64,
                             C.c_int64, C.POINTER(_P)],
    "pk_nccl_unique_id": [_P],
    "pk_nccl_comm_create": [C.c_int, _P, C.c_int, C.c_int, C.POINTER(_P)],
    "pk_nccl_comm_destroy": [_P],
    "pk_dcg_create": [_P, C.c_int64, C.c_int64, C.c_int64, C.c_int32, C.c_int32, _P, C.c_int64, C.POINTER(_P)],
    "pk_dcg_solve": [_P, _DP, C.POINTER(PkConfig), _DP, _DP, C.c_int64, C.POINTER(PkResult)],
    "pk_dcg_destroy": [_P],
    "pk_debug_bench": [_P, _P, C.c_int, C.c_int, _DP],
    "pk_launch_floor": [_P, C.c_int32, C.c_int32, C.c_int64, _DP],
}
_RESTYPES = {"pk_last_error": C.c_char_p}

_lib = None
_lock = threading.Lock()


def lib():
    """Load (once) and return the shared library; raise if it is missing."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not LIB_PATH.exists():
                    raise NativeError(
                        f"{LIB_PATH} is missing; build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                        " (there is no CPU fallback)")
                handle = C.CDLL(os.fspath(LIB_PATH))
                for name, args in SIGNATURES.items():
                    fn = getattr(handle, name)
                    fn.argtypes = args
                    fn.restype = _RESTYPES.get(name, C.c_int)
                _lib = handle
    return _lib


def last_error() -> str:
    msg = lib().pk_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = "") -> None:
    """Map a PK_* status to the reference's exception vocabulary."""
    if rc == PK_OK:
        return
    msg = last_error()
    if what:
        msg = f"{what}: {msg}"
    if rc == PK_ERR_INVALID:
        raise ValueError(msg)
    if rc == PK_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    if rc == PK_ERR_NOMEM:
        raise MemoryError(msg)
    raise NativeError(msg)


def exported_symbols():
    return list(SIGNATURES)
