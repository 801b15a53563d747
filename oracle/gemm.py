"""ctypes wrapper of liboracle_gemm.so (TEST INFRASTRUCTURE ONLY, see oracle/__init__.py).

Python-level restatement of gemm_reference / gemm_execute
(/root/reference/pkg/src/adaptgemm/kernels.py:294-349) over the C loop
nests in gemm_oracle.c.  numpy in, numpy out; no GPU.
"""

import ctypes
import subprocess
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "liboracle_gemm.so"
_lib = None

_i64, _dbl, _int, _p = ctypes.c_int64, ctypes.c_double, ctypes.c_int, ctypes.c_void_p


def build() -> Path:
    """Compile the oracle with oracle/Makefile (gcc, OpenMP, -ffp-contract=off)."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        h = ctypes.CDLL(str(LIB))
        common = [_i64, _i64, _i64, _dbl, _dbl, _int, _int, _int, _p, _i64, _p, _i64, _p, _i64, _p, _i64]
        h.oracle_reference.argtypes = common
        h.oracle_reference.restype = None
        h.oracle_direct.argtypes = common + [_int] * 5
        h.oracle_direct.restype = None
        h.oracle_indirect.argtypes = common + [_int] * 6
        h.oracle_indirect.restype = _int
        h.oracle_pack.argtypes = [_int, _p, _i64, _i64, _i64, _int, _p, _i64, _i64]
        h.oracle_pack.restype = None
        h.oracle_num_threads.restype = _int
        h.oracle_set_threads.argtypes = [_int]
        h.oracle_set_threads.restype = None
        _lib = h
    return _lib


def _dt(x):
    if x.dtype == np.float32:
        return 0
    if x.dtype == np.float64:
        return 1
    raise ValueError(f"unsupported dtype {x.dtype}")


def _args(M, N, K, alpha, beta, ta, tb, A, B, C, out):
    A, B, C = (np.ascontiguousarray(x) for x in (A, B, C))
    ptr = lambda a: a.ctypes.data_as(_p)  # noqa: E731
    return (A, B, C), (M, N, K, float(alpha), float(beta), int(bool(ta)), int(bool(tb)), _dt(A),
                       ptr(A), A.shape[1], ptr(B), B.shape[1], ptr(C), C.shape[1], ptr(out), out.shape[1])


def reference(M, N, K, alpha, beta, ta, tb, A, B, C):
    """_kernel_reference (kernels.py:184-195)."""
    out = np.empty((M, N), A.dtype)
    keep, args = _args(M, N, K, alpha, beta, ta, tb, A, B, C, out)
    lib().oracle_reference(*args)
    return out


def execute(M, N, K, alpha, beta, ta, tb, A, B, C, family, bm, bn, bk, tm, tn, uk):
    """gemm_execute's family path (kernels.py:328-349); returns (out, seconds)."""
    out = np.empty((M, N), A.dtype)
    keep, args = _args(M, N, K, alpha, beta, ta, tb, A, B, C, out)
    t0 = time.perf_counter()
    if family == "direct":
        lib().oracle_direct(*args, bm, bn, bk, tm, tn)
    else:
        if lib().oracle_indirect(*args, bm, bn, bk, tm, tn, uk):
            raise MemoryError("oracle_indirect: allocation failed")
    return out, max(time.perf_counter() - t0, 1e-9)


def pack_padded(X, rows, cols, transpose, pad_rows, pad_cols):
    """pack_padded (kernels.py:304-309)."""
    X = np.ascontiguousarray(X)
    dst = np.empty((pad_rows, pad_cols), X.dtype)
    lib().oracle_pack(_dt(X), X.ctypes.data_as(_p), X.shape[1], rows, cols, int(bool(transpose)),
                      dst.ctypes.data_as(_p), pad_rows, pad_cols)
    return dst


def num_threads() -> int:
    return int(lib().oracle_num_threads())


def set_threads(n: int) -> None:
    lib().oracle_set_threads(int(n))
