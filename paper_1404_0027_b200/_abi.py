"""ctypes declarations of libgpuar's C ABI (include/gpuar.h).  Argument marshalling only.

The library is loaded from ``paper_1404_0027_b200/lib/libgpuar.so`` (built in-tree by
``__graft_entry__.build()``).  There is no fallback: if the library is missing the
import of the binding fails loudly.
"""
from __future__ import annotations

import ctypes
import os

from . import _build

OK, EINVAL, ENOMEM, ECUDA, ENOTSET, EPROPENSITY = 0, -1, -2, -3, -4, -5
RULE_CLASSIC, RULE_ARGMIN, RULE_IT, RULE_IT_SCAN = 0, 1, 2, 3

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64
_u32 = ctypes.c_uint32
_i32 = ctypes.c_int32
_int = ctypes.c_int

# name -> (restype, argtypes); must cover every entry point of include/gpuar.h
SIGNATURES = {
    "gpuar_create": (_int, [ctypes.POINTER(_vp), _i64, _i64, _u64]),
    "gpuar_destroy": (_int, [_vp]),
    "gpuar_set_stream": (_int, [_vp, _vp]),
    "gpuar_set_propensities": (_int, [_vp, _vp, _i64, _i64]),
    "gpuar_select": (_int, [_vp, _i64, _vp, _vp, _vp]),
    "gpuar_select_epochs": (_int, [_vp, _i64, _i64, _vp, _vp, _vp]),
    "gpuar_select_host": (_int, [_vp, _vp, _i64, _i64, _i64, _vp, _vp, _vp]),
    "gpuar_set_rule": (_int, [_vp, _int, ctypes.c_float]),
    "gpuar_set_network": (_int, [_vp, _i64, _i64, _vp, _vp, _vp, _vp]),
    "gpuar_ssa_run": (_int, [_vp, _vp, _vp, _vp, _i64, _i32, ctypes.c_double]),
    "gpuar_set_selection_offset": (_int, [_vp, _i64]),
    "gpuar_set_epoch": (_int, [_vp, _u32]),
    "gpuar_get_epoch": (_int, [_vp, ctypes.POINTER(_u32)]),
    "gpuar_set_max_trials": (_int, [_vp, _u32]),
    "gpuar_get_stats": (_int, [_vp, ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_double),
                               ctypes.POINTER(ctypes.c_float)]),
    "gpuar_row_stats": (_int, [_vp, _vp, _vp]),
    "gpuar_sync": (_int, [_vp]),
    "gpuar_histogram": (_int, [_vp, _vp, _vp, _i64, _vp, _vp]),
    "gpuar_bench_philox": (_int, [_vp, _i64, _i32, _vp]),
    "gpuar_path": (_int, [_vp, ctypes.POINTER(_i32)]),
    "gpuar_last_team": (_int, [_vp, ctypes.POINTER(_i32)]),
    "gpuar_strerror": (ctypes.c_char_p, [_int]),
}

_lib = None


def library_path() -> str:
    # GPUAR_LIBRARY: an alternative in-tree build (tuning experiments); default lib/libgpuar.so
    return os.environ.get("GPUAR_LIBRARY", _build.LIBGPUAR)


def load() -> ctypes.CDLL:
    """Load libgpuar.so; raises if it has not been built (no fallback path exists)."""
    global _lib
    if _lib is None:
        path = library_path()
        if not os.path.exists(path):
            raise RuntimeError(f"libgpuar.so not built ({path}); run __graft_entry__.build()")
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


class GpuarError(RuntimeError):
    def __init__(self, status: int, where: str):
        msg = load().gpuar_strerror(status).decode()
        super().__init__(f"{where}: {msg} ({status})")
        self.status = status


def check(status: int, where: str) -> None:
    if status != OK:
        raise GpuarError(status, where)
