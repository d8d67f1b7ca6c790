"""ctypes binding of libriga_b200.so (include/riga_b200.h).

The library is built in-tree by ``paper_2009_08167_b200/build.py`` (or
``__graft_entry__.build()``).  There is no CPU fallback: if the library is
missing, loading fails loudly; if no CUDA device is visible, every compute
entry point raises ``RuntimeError`` (status RIGA_NO_DEVICE).
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# RIGA_LIB: load an alternative build of the same library (A/B experiments)
LIB_PATH = os.environ.get("RIGA_LIB") or os.path.join(HERE, "libriga_b200.so")

OK, ZERO_PIVOT, BAD_ARG, CUDA_ERROR, OOM, BREAKDOWN, NO_DEVICE = range(7)

_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int
_d = ctypes.c_double
_pp = ctypes.POINTER(ctypes.c_void_p)

# (name, argtypes) — every symbol declared in include/riga_b200.h
SIGNATURES = {
    "riga_version": [],
    "riga_device_count": [_p],
    "riga_mem_info": [ctypes.c_int, ctypes.c_int, _p],
    "riga_ctx_create": [_i32, _p, _p],
    "riga_ctx_destroy": [_p],
    "riga_ctx_synchronize": [_p],
    "riga_device_pool_reusable": [ctypes.c_int, _p],
    "riga_set_blocking_sync": [ctypes.c_int, ctypes.c_int],
    "riga_ctx_stream": [_p, _p],
    "riga_system_upload": [_p, _i64, _i64, _p, _p, _p, _p, _p],
    "riga_system_assemble_kron": [_p, _i32, _p, _p, _p, _p, _p, _p],
    "riga_system_set_kron": [_p, _i32, _p, _p, _p, _p, _p],
    "riga_system_assemble_quad": [_p, _i32, _i32, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p],
    "riga_system_info": [_p, _p, _p],
    "riga_system_download": [_p, _p, _p, _p, _p],
    "riga_system_device_ptrs": [_p, _p, _p, _p, _p],
    "riga_system_destroy": [_p],
    "riga_spmv": [_p, _i32, _d, _p, _p],
    "riga_csr_spmv": [_p, _i64, _p, _p, _p, _p, _p],
    "riga_spmv_many": [_p, _p, _i32, _d, _p, _i64, _i64, _p, _i64],
    "riga_separator_boxes": [_i32, _p, _i32, _p, _p, _i64, _p, _p],
    "riga_separator_emit": [_p, _i32, _p, _i64, _p, _i64, _p],
    "riga_symbolic_create": [_p, _p, _p],
    "riga_symbolic_analyze": [_i64, _p, _p, _p, _p],
    "riga_symbolic_stats": [_p, _p],
    "riga_symbolic_order": [_p, _p],
    "riga_symbolic_colcounts": [_p, _p],
    "riga_symbolic_asm_map": [_p, _p, _p, _p, _p],
    "riga_symbolic_supernodes": [_p, _p, _p, _p, _p, _p],
    "riga_symbolic_destroy": [_p],
    "riga_factor_create": [_p, _p, _d, _d, _p, _p, _p],
    "riga_factor_solve": [_p, _p, _p],
    "riga_factor_solve_many": [_p, _p, _p, _i64, _i64, _p, _i64],
    "riga_factor_time_ms": [_p, _p],
    "riga_factor_D": [_p, _p],
    "riga_factor_export": [_p, _p, _p, _p],
    "riga_factor_destroy": [_p],
    "riga_lanczos_create": [_p, _p, _i64, _i64, _p],
    "riga_lanczos_destroy": [_p],
    "riga_lanczos_reset": [_p, _p],
    "riga_lanczos_set_operator": [_p, _p],
    "riga_lanczos_k": [_p, _p],
    "riga_lanczos_set_start": [_p, _p],
    "riga_lanczos_fresh": [_p, _p, _p],
    "riga_lanczos_lock": [_p, _p, _p],
    "riga_lanczos_locked_count": [_p, _p],
    "riga_lanczos_extend": [_p, _i64, _p, _d, _p, _p, _p, _p],
    "riga_lanczos_last_extend_ms": [_p, _p],
    "riga_lanczos_step_given": [_p, _p, _p, _d, _p, _p, _p],
    "riga_lanczos_lift": [_p, _p, _i64, _p, _p],
    "riga_lanczos_restart": [_p, _p, _i64],
    "riga_lanczos_project_locked": [_p, _p, _p, _i32],
    "riga_lanczos_lock_batch": [_p, _p, _p, _i64, _i64, _p],
    "riga_lanczos_cgs_probe": [_p, _p, _i32, _p],
    "riga_lanczos_dcgs_probe": [_p, _p, _p],
    "riga_lanczos_lock_block": [_p, _p, _p, _i64, _i64, _p],
    "riga_lanczos_append_rows": [_p, _p, _p, _i64, _i64, _p, _p],
    "riga_lanczos_gram": [_p, _p],
    "riga_lanczos_basis": [_p, _p, _p, _p],
    "riga_lanczos_bytes": [_p, _p],
    "riga_residuals": [_p, _p, _p, _i64, _i64, _p, _p],
    "riga_dot": [_p, _i64, _p, _p, _p],
    "riga_tp_contract": [_p, _p, _p, _i64, _i64, _i64, _i64, _i32, _i32, _p, _p, _p, _i64],
    "riga_tp_reduce": [_p, _p, _i64, _i32, _p, _p, _p, _p, _i32, _i32, _p, _p],
    "riga_row_dots": [_p, _p, _i64, _p, _i64, _i64, _i64, _p],
    "riga_launch_count": [_p],
    "riga_set_pdl": [_i32],
    "riga_set_solve_sub_levels": [_i32],
    "riga_prof_enable": [_i32],
    "riga_prof_read": [_p, _p, _p, _i32],
    "riga_prof_reset": [],
}

_LIB = None
_LOCK = threading.Lock()


class RigaError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status


def lib():
    """Load the engine; raises ImportError when it has not been built."""
    global _LIB
    if _LIB is None:
        with _LOCK:
            if _LIB is None:
                if not os.path.exists(LIB_PATH):
                    raise ImportError(
                        f"{LIB_PATH} is missing: build it with "
                        "`python paper_2009_08167_b200/build.py` (nvcc, sm_100a). "
                        "There is no CPU fallback.")
                L = ctypes.CDLL(LIB_PATH)
                for name, args in SIGNATURES.items():
                    fn = getattr(L, name)
                    fn.argtypes = args
                    fn.restype = ctypes.c_int
                L.riga_last_error.argtypes = []
                L.riga_last_error.restype = ctypes.c_char_p
                _LIB = L
    return _LIB


def last_error() -> str:
    return lib().riga_last_error().decode(errors="replace")


def check(status: int, what: str = "") -> int:
    """Map an ABI status to the reference's exception types."""
    if status == OK or status == BREAKDOWN:
        return status
    msg = last_error()
    if what:
        msg = f"{what}: {msg}"
    if status == ZERO_PIVOT:
        from .sparsela import ZeroPivot

        raise ZeroPivot(msg)
    if status == BAD_ARG:
        raise ValueError(msg)
    raise RigaError(status, msg)


def ptr(a) -> ctypes.c_void_p:
    """Raw pointer of a numpy array (host) or torch tensor (device)."""
    if a is None:
        return ctypes.c_void_p(0)
    if isinstance(a, np.ndarray):
        return a.ctypes.data_as(ctypes.c_void_p)
    return ctypes.c_void_p(a.data_ptr())


def out_i64():
    return ctypes.c_int64(0)


def ref(x):
    return ctypes.byref(x)


def device_count() -> int:
    c = ctypes.c_int(0)
    check(lib().riga_device_count(ref(c)))
    return c.value
