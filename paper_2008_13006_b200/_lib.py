"""ctypes binding of libtw_b200.so (include/tw_b200.h).

The library is built in-tree (paper_2008_13006_b200/build.py).  There is no
fallback: if the .so is missing or fails to load, every call raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .matrix import DimensionError, FormatError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libtw_b200.so")

TW_OK, TW_ERR_DIMENSION, TW_ERR_FORMAT = 0, 1, 2
TW_F32, TW_BF16, TW_F16 = 0, 1, 2
TW_ROW_MAJOR, TW_COL_MAJOR = 0, 1
TW_PLAN_SPLIT3, TW_PLAN_F32_WEIGHTS, TW_PLAN_DENSE_PAD = 1, 2, 4

# every symbol include/tw_b200.h declares: name -> (restype, argtypes)
_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int
_pi64 = ctypes.POINTER(ctypes.c_int64)


class PlanInfo(ctypes.Structure):
    _fields_ = [("k", ctypes.c_int64), ("n", ctypes.c_int64), ("g", ctypes.c_int64),
                ("col_begin", ctypes.c_int64), ("col_end", ctypes.c_int64),
                ("n_tiles", ctypes.c_int64), ("n_live", ctypes.c_int64),
                ("n_zero_rows", ctypes.c_int64), ("kept_elems", ctypes.c_int64),
                ("union_k", ctypes.c_int64), ("sum_k", ctypes.c_int64), ("sum_n", ctypes.c_int64),
                ("block_n", ctypes.c_int64), ("wimg_bytes", ctypes.c_int64), ("in_dtype", ctypes.c_int),
                ("flags", ctypes.c_int), ("a_rows", ctypes.c_int64)]


SIGNATURES = {
    "tw_last_error": (ctypes.c_char_p, []),
    "tw_version": (_i32, []),
    "tw_pack_mask_words": (_i32, [_p, _i64, _p]),
    "tw_unpack_mask_words": (_i32, [_p, _i64, _i64, _p]),
    "tw_mask_words_to_indices": (_i32, [_p, _i64, _i64, _p, _pi64]),
    "tw_compact": (_i32, [_p, _i64, _i64, _i32, _i64, _p, _p, _p, _p, _p]),
    "tw_pruned_columns": (_i32, [_i64, _i64, _p, _p, _p, _pi64]),
    "tw_plan_create": (_i32, [_i64, _i64, _i64, _i64, _p, _p, _p, _p, _p, _i32, _i64, _i64,
                              ctypes.POINTER(ctypes.c_void_p)]),
    "tw_plan_create_ex": (_i32, [_i64, _i64, _i64, _i64, _p, _p, _p, _p, _p, _i32, _i64, _i64, _i32,
                                 ctypes.POINTER(ctypes.c_void_p)]),
    "tw_plan_build_host": (_i32, [_i64, _i64, _i64, _i64, _p, _p, _p, _p, _p, _i32, _i64, _i64,
                                  ctypes.POINTER(ctypes.c_void_p)]),
    "tw_plan_destroy": (_i32, [_p]),
    "tw_plan_get_info": (_i32, [_p, ctypes.POINTER(PlanInfo)]),
    "tw_plan_export": (_i32, [_p, _i32, _p, _pi64]),
    "tw_schedule_export": (_i32, [_p, _i64, _i32, _i32, _i32, _i32, _p, _pi64]),
    "tw_gemm": (_i32, [_p, _p, _i64, _i64, _p, _i64, _i32, _i32, _p]),
    "tw_gemm_traced": (_i32, [_p, _p, _i64, _i64, _p, _i64, _i32, _p, _p]),
    "tw_plan_kernel": (_i32, [_p, _i64, _i32, _p]),
    "tw_gemm_bias": (_i32, [_p, _p, _i64, _i64, _p, _i64, _i32, _p, _i32, _p]),
    "tw_gemm_ex": (_i32, [_p, _p, _i64, _i64, _p, _i64, _i32, _i32, _p, _i32, _p]),
    "tw_gemm_peers": (_i32, [_p, _p, _i64, _i64, _p, _i32, _i64, _i32, _p]),
    "tw_ipc_alloc": (_i32, [_i64, _p, _p]),
    "tw_ipc_free": (_i32, [_p]),
    "tw_ipc_open": (_i32, [_p, _p]),
    "tw_ipc_close": (_i32, [_p]),
    "tw_prune_col_means": (_i32, [_p, _i64, _i64, _p, _p]),
    "tw_prune_row_means": (_i32, [_p, _i64, _i64, _p, _p, _i64, _p, _p]),
    "tw_gemm_exact": (_i32, [_p, _p, _i64, _i64, _p, _i64, _p]),
    "tw_prep_activations": (_i32, [_p, _i64, _i64, _i32, _p, _i64, _i32, _p]),
    "tw_prep_activations_split": (_i32, [_p, _i64, _i64, _i32, _p, _i64, _p]),
    "tw_spmm_csc": (_i32, [_p, _i32, _i64, _i64, _i64, _i64, _p, _p, _p, _p, _i64, _i32, _i32, _p]),
    "tw_gemm_tew": (_i32, [_p, _p, _i64, _i64, _p, _p, _p, _i64, _p, _i64, _i32, _p]),
    "tw_device_sm_count": (_i32, [ctypes.POINTER(ctypes.c_int)]),
    "tw_copy_2d": (_i32, [_p, _i64, _p, _i64, _i64, _i64, _i32, _p]),
}

_lock = threading.Lock()
_lib = None


class LibraryMissing(RuntimeError):
    pass


def lib():
    """Load libtw_b200.so (once).  Raises LibraryMissing -- never falls back."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise LibraryMissing(
                    f"{LIB_PATH} is not built; run `python -m paper_2008_13006_b200.build` "
                    "(there is no CPU fallback for the TW-GEMM path)")
            L = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == TW_OK:
        return
    msg = (lib().tw_last_error() or b"").decode(errors="replace")
    if rc == TW_ERR_DIMENSION:
        raise DimensionError(msg)
    if rc == TW_ERR_FORMAT:
        raise FormatError(msg)
    raise RuntimeError(f"libtw_b200 error {rc}: {msg}")


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))
