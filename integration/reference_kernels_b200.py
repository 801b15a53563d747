"""The reference-side binding: what a maintainer adds to the reference
package (as adaptgemm/_b200.py) so its own `gemm_execute` calls run on the
B200 through the C-ABI of libadaptgemm_b200.so (include/adaptgemm_b200.h).

It replaces the body of /root/reference/pkg/src/adaptgemm/kernels.py:328-349
(gemm_execute) and keeps its contract:

  * legality first (ConfigError), then the operand checks of
    kernels.py:271-283 (ShapeError), in that order, with the same wording;
  * numpy in, numpy out; `out` written in place when given;
  * returns (out, seconds), seconds = the device time of the family path
    (the reference's perf_counter around the numba kernel, kernels.py:341-349,
    here CUDA events around the kernels, without the copies).

Dependencies are the reference's own: numpy + ctypes.  No torch: the device
scratch is the library's own (ag_device_scratch), the copies are pipelined
inside ag_gemm_host_ex and the caller's pageable arrays cross through the
library's pinned staging rings (AG_HOST_STAGE).

    import reference_kernels_b200 as b200
    b200.bind(kernels.ConfigError, kernels.ShapeError)   # the reference's classes
    out, seconds = b200.gemm_execute(shape, config, A, B, C, caps, out)
"""
import ctypes
import os
import weakref
from pathlib import Path

import numpy as np

_DEFAULT_LIB = Path(__file__).resolve().parent.parent / "paper_1806_07060_b200" / "_lib" / "libadaptgemm_b200.so"
LIB_PATH = Path(os.environ.get("ADAPTGEMM_B200_LIB", str(_DEFAULT_LIB)))


class ConfigError(ValueError):
    """Stand-in until bind() installs the reference's kernels.ConfigError."""


class ShapeError(ValueError):
    """Stand-in until bind() installs the reference's kernels.ShapeError."""


def bind(config_error, shape_error):
    """Raise the caller's exception classes (the reference's kernels module)."""
    global ConfigError, ShapeError
    ConfigError, ShapeError = config_error, shape_error


class _Shape(ctypes.Structure):
    _fields_ = [("m", ctypes.c_int64), ("n", ctypes.c_int64), ("k", ctypes.c_int64),
                ("alpha", ctypes.c_double), ("beta", ctypes.c_double),
                ("trans_a", ctypes.c_int32), ("trans_b", ctypes.c_int32)]


class _Config(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int32) for f in ("family", "bm", "bn", "bk", "tm", "tn", "uk")]


class _Caps(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int64) for f in ("tile_memory_cap", "register_tile_cap_direct",
                                              "register_tile_cap_indirect", "element_size", "max_threads")]


# include/adaptgemm_b200.h AG_FAMILY_*; the reference has the first two
_FAMILY = {"direct": 0, "indirect": 1, "splitk": 2, "tf32": 3, "bf16": 4, "tma": 5, "skinny_n": 6, "skinny_m": 7, "tf32x3": 8}
AG_HOST_STAGE = 2
_P, _I = ctypes.c_void_p, ctypes.c_int64
_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(str(LIB_PATH))
        L.ag_is_legal.argtypes = [ctypes.POINTER(_Config), ctypes.POINTER(_Caps)]
        L.ag_is_legal.restype = ctypes.c_int
        L.ag_last_error.restype = ctypes.c_char_p
        L.ag_gemm_host_ex.argtypes = [ctypes.POINTER(_Shape), ctypes.POINTER(_Config), ctypes.POINTER(_Caps),
                                      ctypes.c_int, _P, _I, _P, _I, _P, _I, _P, _I, _P, ctypes.c_size_t, ctypes.c_int,
                                      ctypes.c_int, _P, ctypes.POINTER(ctypes.c_double)]
        L.ag_gemm_host_ex.restype = ctypes.c_int
        L.ag_host_alloc.argtypes = [ctypes.c_size_t]
        L.ag_host_alloc.restype = ctypes.c_void_p
        L.ag_host_free.argtypes = [ctypes.c_void_p]
        L.ag_host_free.restype = None
        _lib = L
    return _lib


def _config(config) -> _Config:
    return _Config(_FAMILY[config.family.value], config.block_m, config.block_n, config.block_k,
                   config.tile_m, config.tile_n, config.unroll_k)


def _caps(caps) -> _Caps:
    return _Caps(caps.tile_memory_cap, caps.register_tile_cap_direct, caps.register_tile_cap_indirect,
                 caps.element_size, getattr(caps, "max_threads", 1024))


def _check_operands(shape, A, B, C):
    """kernels.py:271-283."""
    a_dims = (shape.K, shape.M) if shape.transA else (shape.M, shape.K)
    b_dims = (shape.N, shape.K) if shape.transB else (shape.K, shape.N)
    if A.ndim != 2 or A.shape != a_dims:
        raise ShapeError(f"A has shape {A.shape}, expected {a_dims}")
    if B.ndim != 2 or B.shape != b_dims:
        raise ShapeError(f"B has shape {B.shape}, expected {b_dims}")
    if C.ndim != 2 or C.shape != (shape.M, shape.N):
        raise ShapeError(f"C has shape {C.shape}, expected {(shape.M, shape.N)}")
    if not (A.dtype == B.dtype == C.dtype):
        raise ShapeError(f"mixed dtypes: {A.dtype}, {B.dtype}, {C.dtype}")
    if A.dtype not in (np.float32, np.float64):
        raise ShapeError(f"unsupported dtype {A.dtype}, want float32 or float64")


def _pinned_result(L, m, n, dtype):
    """A fresh m x n result (kernels.py:286-288) in a block of the library's
    caching pinned allocator (ag_host_alloc), so the D2H lands by DMA; the
    block goes back to the cache when the array is collected.  Small results
    (or a failed pin) are plain np.empty."""
    nbytes = m * n * np.dtype(dtype).itemsize
    p = L.ag_host_alloc(nbytes) if nbytes >= (64 << 10) else None
    if not p:
        return np.empty((m, n), dtype=dtype)
    raw = (ctypes.c_char * nbytes).from_address(p)
    weakref.finalize(raw, L.ag_host_free, p)
    return np.frombuffer(raw, dtype=dtype).reshape(m, n)


def gemm_execute(shape, config, A, B, C, caps, out=None):
    """kernels.gemm_execute (kernels.py:328-349) on the B200."""
    L = lib()
    c, k = _config(config), _caps(caps)
    if not L.ag_is_legal(ctypes.byref(c), ctypes.byref(k)):
        raise ConfigError(f"illegal config {config.canonical()} for caps {caps}")
    _check_operands(shape, A, B, C)
    A, B, C = (np.ascontiguousarray(x) for x in (A, B, C))
    if out is None:
        out = _pinned_result(L, shape.M, shape.N, A.dtype)
    elif out.shape != (shape.M, shape.N) or out.dtype != A.dtype:
        raise ShapeError("out buffer has wrong shape or dtype")
    dst = out if out.flags.c_contiguous else np.empty_like(out, order="C")
    s = _Shape(shape.M, shape.N, shape.K, shape.alpha, shape.beta, int(shape.transA), int(shape.transB))
    secs = ctypes.c_double(0.0)
    rc = L.ag_gemm_host_ex(ctypes.byref(s), ctypes.byref(c), ctypes.byref(k), 0 if A.dtype == np.float32 else 1,
                           A.ctypes.data, A.shape[1], B.ctypes.data, B.shape[1], C.ctypes.data, C.shape[1],
                           dst.ctypes.data, dst.shape[1], None, 0, 0, AG_HOST_STAGE, None, ctypes.byref(secs))
    if rc:
        msg = (L.ag_last_error() or b"").decode()
        raise (ConfigError if rc == 1 else ShapeError if rc == 2 else RuntimeError)(msg)
    if dst is not out:
        out[...] = dst
    return out, max(secs.value, 1e-9)
