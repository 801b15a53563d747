"""ctypes binding of libadaptgemm_b200.so (the C-ABI in include/adaptgemm_b200.h).

The library is built in-tree by `python -m paper_1806_07060_b200.build`.
There is no fallback: every GEMM in this package runs through this library,
and a missing library raises `NativeLibraryError` on first use.
"""

import ctypes
import threading
from ctypes import POINTER, c_char_p, c_double, c_int, c_int32, c_int64, c_size_t, c_void_p
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libadaptgemm_b200.so"

AG_OK, AG_ERR_CONFIG, AG_ERR_SHAPE, AG_ERR_CUDA = 0, 1, 2, 3
AG_HOST_REGISTER = 1  # ag_gemm_host_ex flag: page-lock the caller's host buffers for the call
AG_HOST_STAGE = 2  # ag_gemm_host_ex flag: pageable buffers through the library's pinned rings
AG_FAMILY_DIRECT, AG_FAMILY_INDIRECT, AG_FAMILY_SPLITK = 0, 1, 2
AG_FAMILY_TF32, AG_FAMILY_BF16 = 3, 4
AG_FAMILY_TMA = 5
AG_FAMILY_SKINNY_N, AG_FAMILY_SKINNY_M = 6, 7
AG_FAMILY_TF32X3 = 8
AG_F32, AG_F64 = 0, 1


class NativeLibraryError(RuntimeError):
    """libadaptgemm_b200.so is missing or failed to load."""


class AgShape(ctypes.Structure):
    _fields_ = [("m", c_int64), ("n", c_int64), ("k", c_int64),
                ("alpha", c_double), ("beta", c_double),
                ("trans_a", c_int32), ("trans_b", c_int32)]


class AgConfig(ctypes.Structure):
    _fields_ = [("family", c_int32), ("bm", c_int32), ("bn", c_int32), ("bk", c_int32),
                ("tm", c_int32), ("tn", c_int32), ("uk", c_int32)]


class AgCaps(ctypes.Structure):
    _fields_ = [("tile_memory_cap", c_int64), ("register_tile_cap_direct", c_int64),
                ("register_tile_cap_indirect", c_int64), ("element_size", c_int64),
                ("max_threads", c_int64)]


_P = c_void_p
_GEMM_ARGS = [POINTER(AgShape), POINTER(AgConfig), POINTER(AgCaps), c_int,
              _P, c_int64, _P, c_int64, _P, c_int64, _P, c_int64, _P, c_size_t, _P]

# symbol -> (restype, argtypes); also the export list the CPU tests check
SIGNATURES = {
    "ag_last_error": (c_char_p, []),
    "ag_version": (c_char_p, []),
    "ag_is_legal": (c_int, [POINTER(AgConfig), POINTER(AgCaps)]),
    "ag_has_kernel": (c_int, [POINTER(AgConfig), c_int]),
    "ag_num_kernels": (c_int, []),
    "ag_workspace_bytes": (c_size_t, [POINTER(AgShape), POINTER(AgConfig), c_int]),
    "ag_gemm": (c_int, _GEMM_ARGS),
    "ag_gemm_timed": (c_int, _GEMM_ARGS + [c_int, c_int, c_int, POINTER(c_double)]),
    "ag_tune": (c_int, [POINTER(AgShape), POINTER(AgConfig), c_int, POINTER(AgCaps), c_int,
                        _P, c_int64, _P, c_int64, _P, c_int64, _P, c_int64, _P, c_size_t, _P,
                        c_int, c_int, POINTER(c_double), POINTER(c_int)]),
    "ag_tune_ex": (c_int, [POINTER(AgShape), POINTER(AgConfig), c_int, POINTER(AgCaps), c_int,
                           _P, c_int64, _P, c_int64, _P, c_int64, _P, c_int64, _P, c_size_t, _P,
                           c_int, c_int, c_int, POINTER(c_double), POINTER(c_int)]),
    "ag_gemm_reference": (c_int, [POINTER(AgShape), c_int, _P, c_int64, _P, c_int64,
                                  _P, c_int64, _P, c_int64, _P]),
    "ag_pack_padded": (c_int, [c_int, _P, c_int64, c_int64, c_int64, c_int, _P, c_int64, c_int64, _P]),
    "ag_ffma_peak": (c_int, [_P, POINTER(c_double)]),
    "ag_tree_train": (c_int, [POINTER(c_int64), POINTER(c_int64), c_int64, c_int64, c_int64,
                              POINTER(c_int32), POINTER(c_double), POINTER(c_int32), POINTER(c_int32),
                              POINTER(c_int64), POINTER(c_int64), POINTER(c_int64)]),
    "ag_best_split": (c_int, [POINTER(c_int64), POINTER(c_int64), c_int64, c_int64,
                              POINTER(c_int32), POINTER(c_double), POINTER(c_double)]),
    "ag_selector_build": (c_void_p, [POINTER(c_int32), POINTER(c_double), POINTER(c_int32),
                                     POINTER(c_int32), POINTER(c_int64), POINTER(AgConfig),
                                     c_int64, c_int64]),
    "ag_selector_build_kind": (c_void_p, [POINTER(c_int32), POINTER(c_double), POINTER(c_int32),
                                          POINTER(c_int32), POINTER(c_int64), POINTER(AgConfig),
                                          c_int64, c_int64, c_int]),
    "ag_selector_free": (None, [c_void_p]),
    "ag_selector_kind": (c_int, [c_void_p]),
    "ag_select": (c_int64, [c_void_p, c_int64, c_int64, c_int64, POINTER(AgConfig)]),
    "ag_select_many": (c_int, [c_void_p, POINTER(c_int64), c_int64, POINTER(c_int64)]),
    "ag_select_bench_ns": (c_double, [c_void_p, c_int64, c_int64, c_int64, c_int64]),
    "ag_dispatch_gemm": (c_int, [c_void_p, POINTER(AgConfig), POINTER(AgShape), POINTER(AgCaps), c_int,
                                 _P, c_int64, _P, c_int64, _P, c_int64, _P, c_int64, _P, c_size_t, _P,
                                 POINTER(AgConfig), POINTER(c_int)]),
    "ag_host_scratch_bytes": (c_size_t, [POINTER(AgShape), POINTER(AgConfig), c_int, c_int]),
    "ag_gemm_host": (c_int, _GEMM_ARGS[:-1] + [c_int, _P]),
    "ag_gemm_host_ex": (c_int, _GEMM_ARGS[:-1] + [c_int, c_int, _P, POINTER(c_double)]),
    "ag_device_scratch": (c_void_p, [c_size_t]),
    "ag_host_alloc": (c_void_p, [c_size_t]),
    "ag_host_free": (None, [c_void_p]),
    "ag_host_cache_bytes": (c_size_t, []),
    "ag_dispatch_gemm_host_ex": (c_int, [c_void_p, POINTER(AgConfig), POINTER(AgShape), POINTER(AgCaps), c_int,
                                         _P, c_int64, _P, c_int64, _P, c_int64, _P, c_int64, _P, c_size_t, c_int,
                                         c_int, _P, POINTER(AgConfig), POINTER(c_int), POINTER(c_double)]),
    "ag_dispatch_gemm_host": (c_int, [c_void_p, POINTER(AgConfig), POINTER(AgShape), POINTER(AgCaps), c_int,
                                      _P, c_int64, _P, c_int64, _P, c_int64, _P, c_int64, _P, c_size_t, c_int, _P,
                                      POINTER(AgConfig), POINTER(c_int)]),
}

_lib = None
_lock = threading.Lock()


def lib():
    """The loaded library (loaded once; raises NativeLibraryError if absent)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise NativeLibraryError(
                    f"{LIB_PATH} is not built; run `python -m paper_1806_07060_b200.build` "
                    "(there is no CPU fallback for the GEMM path)")
            try:
                handle = ctypes.CDLL(str(LIB_PATH))
            except OSError as exc:
                raise NativeLibraryError(f"cannot load {LIB_PATH}: {exc}") from exc
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


def last_error() -> str:
    msg = lib().ag_last_error()
    return msg.decode() if msg else ""
