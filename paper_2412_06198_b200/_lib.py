"""ctypes binding of the in-tree C-ABI library ``_sa_b200.so``.

The library is the product: there is no CPU fallback.  If the shared object is
missing or CUDA is unavailable, every entry point raises ``RuntimeError``.
Status codes returned by the C ABI map 1:1 onto the reference's exception
classes (include/sparseattn_b200.h, core.py:32-45 of the reference).
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_sa_b200.so")

_lib = None
_lock = threading.Lock()


class sa_head_index(ctypes.Structure):
    """Mirror of ``sa_head_index`` in include/sparseattn_b200.h."""

    _fields_ = [
        ("family", ctypes.c_void_p),
        ("tri_window", ctypes.c_void_p),
        ("tri_sinks", ctypes.c_void_p),
        ("colbits", ctypes.c_void_p),
        ("diagrev", ctypes.c_void_p),
        ("vs_words", ctypes.c_int32),
        ("blk_b", ctypes.c_void_p),
        ("blk_row_off", ctypes.c_void_p),
        ("blk_idx", ctypes.c_void_p),
        ("blk_row_stride", ctypes.c_int32),
    ]


_P = ctypes.c_void_p
_I = ctypes.c_int
_F = ctypes.c_float

# name -> argtypes (restype is always c_int status unless listed in _RESTYPES)
_SIGNATURES = {
    "sa_version": [],
    "sa_last_error": [],
    "sa_build_tiles": [ctypes.POINTER(sa_head_index), _I, _I, _P, _P, _P, _P],
    "sa_attn_sparse": [_I, _I, _I, _I, _F, _P, _P, _P, _P, ctypes.POINTER(sa_head_index),
                       _P, _P, _P, _P, _P],
}
_RESTYPES = {"sa_last_error": ctypes.c_char_p}


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
        for name, argtypes in _SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = argtypes
            fn.restype = _RESTYPES.get(name, ctypes.c_int)
        _lib = lib
    return _lib


def check(status: int) -> None:
    """Raise the reference exception class that a non-zero status maps to."""
    if status == 0:
        return
    from . import errors as core

    msg = load().sa_last_error().decode(errors="replace")
    cls = {
        1: core.DimensionError,
        2: core.NonFiniteError,
        3: core.EmptyRowError,
        4: core.PatternParamError,
        5: core.SearchError,
        6: core.CacheOverflowError,
        7: core.SparseAttnError,
    }.get(status, RuntimeError)
    raise cls(msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))
