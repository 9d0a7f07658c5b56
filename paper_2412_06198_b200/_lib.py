"""ctypes binding of the in-tree C-ABI library ``_sa_b200.so``.

The library is the product: there is no CPU fallback.  If the shared object is
missing or CUDA is unavailable, every entry point raises ``RuntimeError``.
Status codes returned by the C ABI map 1:1 onto the reference's exception
classes (include/sparseattn_b200.h; reference core.py:32-45, patterns.py:55,
search.py:47, runtime.py:35).
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# SA_B200_LIB selects a tool build (e.g. the SA_ATTN_PROF variant); default is the product .so
LIB_PATH = os.environ.get("SA_B200_LIB") or os.path.join(_HERE, "_sa_b200.so")

_lib = None
_lock = threading.Lock()

_P = ctypes.c_void_p
_I = ctypes.c_int
_F = ctypes.c_float
_LL = ctypes.c_longlong
_SZ = ctypes.c_size_t


class sa_head_index(ctypes.Structure):
    """Mirror of ``sa_head_index``."""

    _fields_ = [
        ("family", _P),
        ("tri_window", _P),
        ("tri_sinks", _P),
        ("colbits", _P),
        ("diagrev", _P),
        ("vs_words", ctypes.c_int32),
        ("blk_b", _P),
        ("blk_row_off", _P),
        ("blk_idx", _P),
        ("blk_row_stride", ctypes.c_int32),
    ]


MAX_CAND = 16  # SA_MAX_CAND (include/sparseattn_b200.h): candidates per auto selection


class sa_pattern(ctypes.Structure):
    _fields_ = [("family", ctypes.c_int32), ("p1", ctypes.c_int32), ("p2", ctypes.c_int32)]


class sa_prefill_desc(ctypes.Structure):
    _fields_ = [
        ("batch", ctypes.c_int32),
        ("heads", ctypes.c_int32),
        ("kv_heads", ctypes.c_int32),
        ("n", ctypes.c_int32),
        ("scale", ctypes.c_float),
        ("mode", ctypes.c_int32),
        ("fixed", sa_pattern),
        ("q_est", ctypes.c_int32),
        ("cal", ctypes.c_int32),
        ("ncand", ctypes.c_int32),
        ("cand", sa_pattern * MAX_CAND),
        ("full", sa_pattern * MAX_CAND),
        ("preselected", ctypes.c_int32),
        ("stage_events", ctypes.c_void_p * 6),
        ("out_ld", ctypes.c_int64),
        ("stop_after_tiles", ctypes.c_int32),
        ("check_flag", ctypes.c_void_p),
        ("cache_k", ctypes.c_void_p),
        ("cache_v", ctypes.c_void_p),
        ("cache_capacity", ctypes.c_int32),
    ]


class sa_prefill_view(ctypes.Structure):
    _fields_ = [
        ("choice", _P),
        ("family", _P),
        ("errors", _P),
        ("col_scores", _P),
        ("diag_scores", _P),
        ("col_idx", _P),
        ("diag_idx", _P),
        ("col_ld", ctypes.c_int32),
        ("diag_ld", ctypes.c_int32),
        ("index", sa_head_index),
        ("blk_head_stride", ctypes.c_int64),
        ("tile_off", _P),
        ("tile_cnt", _P),
        ("tiles", _P),
        ("nqt", ctypes.c_int32),
    ]


_IDX = ctypes.POINTER(sa_head_index)
_DESC = ctypes.POINTER(sa_prefill_desc)

# name -> (restype, argtypes); every symbol declared in include/sparseattn_b200.h
_SIGNATURES = {
    "sa_version": (ctypes.c_int, []),
    "sa_last_error": (ctypes.c_char_p, []),
    "sa_prefill_workspace_size": (_SZ, [_DESC]),
    "sa_prefill_views": (ctypes.c_int, [_DESC, _P, ctypes.POINTER(sa_prefill_view)]),
    "sa_prefill": (ctypes.c_int, [_DESC, _P, _P, _P, _P, _P, _SZ, _P]),
    "sa_prefill_select": (ctypes.c_int, [_DESC, _P, _P, _P, _SZ, _P]),
    "sa_select_windowed": (ctypes.c_int, [_I, _I, _I, _I, _I, _F, _P, _P, _I, _P, _P, _P, _P, _P,
                                          _P, _P]),
    "sa_score_tail_workspace": (_SZ, [_I, _I, _I, _I]),
    "sa_score_tail": (ctypes.c_int, [_I, _I, _I, _I, _F, _P, _P, _I, _I, _P, _P, _I, _P, _I, _P,
                                     _SZ, _P]),
    "sa_topk_stable_f32": (ctypes.c_int, [_P, _I, _I, _LL, _I, _P, _LL, _P]),
    "sa_topk_stable_rows_f32": (ctypes.c_int, [_P, _I, _LL, _P, _P, _P, _LL, _P, _P]),
    "sa_block_pool": (ctypes.c_int, [_I, _I, _I, _I, _P, _P, _P, _P]),
    "sa_block_select_workspace": (_SZ, [_I, _I, _I]),
    "sa_block_select": (ctypes.c_int, [_I, _I, _I, _I, _I, _I, _F, _P, _P, _P, _P, _P, _SZ, _P]),
    "sa_block_index_workspace": (_SZ, [_I, _I, _I, _I, _I, _I]),
    "sa_block_index_bf16": (ctypes.c_int, [_I, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P, _SZ, _P]),
    "sa_attn_weights": (ctypes.c_int, [_I, _I, _I, _I, _F, _P, _P, _P, _IDX, _P, _P]),
    "sa_block_mean_f32": (ctypes.c_int, [_P, _I, _I, _I, _P, _P]),
    "sa_build_tiles": (ctypes.c_int, [_IDX, _I, _I, _P, _P, _P, _P]),
    "sa_check_finite_bf16": (ctypes.c_int, [_P, _LL, _P, _P]),
    "sa_memcpy2d_async": (ctypes.c_int, [_P, _SZ, _P, _SZ, _SZ, _SZ, _P]),
    "sa_f32_to_bf16": (ctypes.c_int, [_P, _P, _LL, _P, _P]),
    "sa_bf16_to_f32": (ctypes.c_int, [_P, _P, _LL, _P]),
    "sa_select_family": (ctypes.c_int, [_P, ctypes.c_int64, _I, _I, _P, _P]),
    "sa_block_topk_workspace": (_SZ, [_I, _I]),
    "sa_block_topk_f32": (ctypes.c_int, [_P, _I, ctypes.c_int64, _I, _P, _P, _SZ, _P]),
    "sa_attn_sparse_work": (ctypes.c_int, [_I, _I, _I, _I, _F, _P, _P, _P, _P, _IDX, _P, _P, _P, _P, _P, _P,
                                           ctypes.c_int64, _P]),
    "sa_attn_sparse_work_peers": (ctypes.c_int, [_I, _I, _I, _I, _F, _P, _P, _P, _P, _P, _I, _IDX, _P, _P, _P,
                                                 _P, _P, _P, ctypes.c_int64, _P]),
    "sa_ipc_alloc": (ctypes.c_int, [_SZ, _P, _P]),
    "sa_ipc_free": (ctypes.c_int, [_P]),
    "sa_ipc_open": (ctypes.c_int, [_P, _P]),
    "sa_ipc_close": (ctypes.c_int, [_P]),
    "sa_peer_barrier": (ctypes.c_int, [_P, _P, ctypes.c_int, ctypes.c_int, ctypes.c_int, _P]),
    "sa_decode_workspace": (_SZ, [_I, _I, _I, _I, _I]),
    "sa_decode_attn": (ctypes.c_int, [_I, _I, _I, _I, _I, _I, _F, _P, _P, _P, _I, _P, _P, _SZ, _P]),
    "sa_order_work": (ctypes.c_int, [_P, _I, _I, _P, _P]),
    "sa_attn_sparse": (ctypes.c_int, [_I, _I, _I, _I, _F, _P, _P, _P, _P, _IDX, _P, _P, _P, _P,
                                      _P]),
}


def exported_symbols() -> list[str]:
    return sorted(_SIGNATURES)


def load():
    """Load and type the shared library (idempotent); raise if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"CUDA extension {LIB_PATH} is missing: run `make` (or __graft_entry__.build())"
            )
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, argtypes) in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = argtypes
            fn.restype = res
        _lib = lib
    return _lib


def check(status: int) -> None:
    """Raise the reference exception class that a non-zero status maps to."""
    if status == 0:
        return
    from . import errors as E

    msg = load().sa_last_error().decode(errors="replace")
    cls = {
        1: E.DimensionError,
        2: E.NonFiniteError,
        3: E.EmptyRowError,
        4: E.PatternParamError,
        5: E.SearchError,
        6: E.CacheOverflowError,
        7: E.SparseAttnError,
    }.get(status, RuntimeError)
    raise cls(msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))
