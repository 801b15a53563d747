"""GEMM problem/config types, the legal search space, and the device GEMM path.

Drop-in for `adaptgemm.kernels` (/root/reference/pkg/src/adaptgemm/
kernels.py).  Types, legality rules and enumeration order are the
reference's; execution is not: `gemm_execute` runs the family path as
sm_100a CUDA kernels from libadaptgemm_b200.so (csrc/kernels.cuh):

* direct   -- one predicated kernel on the caller's unpadded operands,
              transposes and ragged edges handled in-kernel (kernels.py:198-227);
* indirect -- pack/transpose-pad helper kernels into tile-multiple buffers,
              then the branch-free tiled core (kernels.py:230-260, 304-325).

Operands may be numpy arrays (staged to the GPU, result copied back -- the
reference's calling convention) or CUDA torch tensors (used in place).
`seconds` is the device time of the family path, measured with CUDA events
on the launching stream (helpers included, allocation and host<->device
copies excluded).  There is no CPU fallback: without a GPU or without the
built library these functions raise.
"""

import ctypes
from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from . import _device, _native, spaces


class ShapeError(ValueError):
    """Operand dimensions are inconsistent with the problem shape."""


class ConfigError(ValueError):
    """Kernel configuration is invalid or illegal for the device caps."""


class KernelFamily(str, Enum):
    """The reference's two families plus the B200 families.

    SPLITK runs the indirect core over `unroll_k` equal K slices and adds
    the slices in a fixed order (deterministic); it exists only in the B200
    profiles.  TF32 / BF16 are the tensor-core families (tcgen05.mma, TMEM
    accumulators, TMA): float32 operands packed to tf32 (round to nearest)
    or bf16, fp32 accumulation; they exist only in the "b200tc" profile.
    TMA is the indirect core's fp32 arithmetic fed by TMA from the caller's
    row-major operands (no pack passes; B200 profiles only).
    SKINNY_N / SKINNY_M stream the big operand of a GEMM whose N (resp. M)
    is small, K split over the CTAs of a cluster (csrc/skinny.cuh; B200
    profiles only).
    TF32X3 is fp32-accurate GEMM on the tensor pipe: each operand split as
    hi + lo (hi = its tf32 bits), three tf32 MMAs (hi.hi + hi.lo + lo.hi)
    into one fp32 TMEM accumulator; it meets the fp32 RF <= 1e-5 contract
    ("b200tc" profile only).
    Reference-profile spaces, tables and dispatchers are unchanged.
    """

    DIRECT = "direct"
    INDIRECT = "indirect"
    SPLITK = "splitk"
    TF32 = "tf32"
    BF16 = "bf16"
    TMA = "tma"
    SKINNY_N = "skinny_n"
    SKINNY_M = "skinny_m"
    TF32X3 = "tf32x3"


TC_FAMILIES = (KernelFamily.TF32, KernelFamily.BF16, KernelFamily.TF32X3)


REFERENCE_FAMILIES = (KernelFamily.DIRECT, KernelFamily.INDIRECT)
_FAMILY_CODE = {KernelFamily.DIRECT: _native.AG_FAMILY_DIRECT,
                KernelFamily.INDIRECT: _native.AG_FAMILY_INDIRECT,
                KernelFamily.SPLITK: _native.AG_FAMILY_SPLITK,
                KernelFamily.TF32: _native.AG_FAMILY_TF32,
                KernelFamily.BF16: _native.AG_FAMILY_BF16,
                KernelFamily.TMA: _native.AG_FAMILY_TMA,
                KernelFamily.SKINNY_N: _native.AG_FAMILY_SKINNY_N,
                KernelFamily.SKINNY_M: _native.AG_FAMILY_SKINNY_M,
                KernelFamily.TF32X3: _native.AG_FAMILY_TF32X3}
_CODE_FAMILY = {v: k for k, v in _FAMILY_CODE.items()}


@dataclass(frozen=True)
class ProblemShape:
    """One GEMM problem: C = alpha * op(A) @ op(B) + beta * C (kernels.py:37-61).

    op(A) is M x K and op(B) is K x N; transA/transB describe the stored
    layout of A and B relative to that.
    """

    M: int
    N: int
    K: int
    alpha: float = 1.0
    beta: float = 0.0
    transA: bool = False
    transB: bool = False

    def __post_init__(self):
        for name in ("M", "N", "K"):
            v = getattr(self, name)
            if isinstance(v, bool) or not isinstance(v, int) or v < 1:
                raise ShapeError(f"{name} must be a positive integer, got {v!r}")

    @property
    def mnk(self) -> tuple[int, int, int]:
        return (self.M, self.N, self.K)


@dataclass(frozen=True)
class DeviceCaps:
    """Resource limits deciding which configs are legal (kernels.py:64-82).

    The first four fields and their defaults are the reference's.  Two
    B200 fields follow: `max_threads` (threads per CTA) and `profile`, which
    selects the enumerated domains -- "reference" (144 direct / 432
    indirect) or "b200" (the reference domains plus large CTA tiles, see
    spaces.py).  `DeviceCaps.b200()` returns the B200 tuning profile.
    """

    tile_memory_cap: int = 32768
    register_tile_cap_direct: int = 8
    register_tile_cap_indirect: int = 32
    element_size: int = 4
    max_threads: int = 1024
    profile: str = spaces.PROFILE_REFERENCE

    def __post_init__(self):
        for name in ("tile_memory_cap", "register_tile_cap_direct",
                     "register_tile_cap_indirect", "element_size", "max_threads"):
            if getattr(self, name) < 1:
                raise ConfigError(f"{name} must be positive")
        if self.profile not in spaces.PROFILES:
            raise ConfigError(f"unknown caps profile {self.profile!r}")

    @classmethod
    def b200(cls, **overrides) -> "DeviceCaps":
        kw = dict(spaces.B200_CAPS)
        kw["profile"] = spaces.PROFILE_B200
        kw.update(overrides)
        return cls(**kw)

    @classmethod
    def b200_tc(cls, **overrides) -> "DeviceCaps":
        """The B200 profile plus the tensor-core families (tf32, bf16, tf32x3)."""
        kw = dict(spaces.B200_CAPS)
        kw["profile"] = spaces.PROFILE_B200_TC
        kw.update(overrides)
        return cls(**kw)

    def register_tile_cap(self, family: KernelFamily) -> int:
        if family is KernelFamily.DIRECT:
            return self.register_tile_cap_direct
        return self.register_tile_cap_indirect  # indirect and split-K

    def as_dict(self) -> dict:
        return dict(tile_memory_cap=self.tile_memory_cap,
                    register_tile_cap_direct=self.register_tile_cap_direct,
                    register_tile_cap_indirect=self.register_tile_cap_indirect,
                    element_size=self.element_size, max_threads=self.max_threads)

    def native(self) -> _native.AgCaps:
        return _native.AgCaps(self.tile_memory_cap, self.register_tile_cap_direct,
                              self.register_tile_cap_indirect, self.element_size, self.max_threads)


@dataclass(frozen=True, order=True)
class KernelConfig:
    """Family plus tuning parameters (kernels.py:85-119).

    block_m/block_n: CTA tile; block_k: K depth of one shared-memory stage;
    tile_m/tile_n: per-thread register tile; unroll_k: K steps whose register
    fragments are loaded ahead of the FMAs (indirect only; 1 for direct).
    Field order defines the canonical total order.
    """

    family: KernelFamily
    block_m: int
    block_n: int
    block_k: int
    tile_m: int
    tile_n: int
    unroll_k: int = 1

    def canonical(self) -> str:
        """Stable textual identity; equal strings mean the same class."""
        return (f"{self.family.value}:{self.block_m}-{self.block_n}-{self.block_k}"
                f"-{self.tile_m}-{self.tile_n}-{self.unroll_k}")

    def param_tuple(self) -> tuple[int, int, int, int, int, int]:
        return (self.block_m, self.block_n, self.block_k,
                self.tile_m, self.tile_n, self.unroll_k)

    @classmethod
    def from_canonical(cls, text: str) -> "KernelConfig":
        try:
            fam, params = text.split(":")
            bm, bn, bk, tm, tn, uk = (int(p) for p in params.split("-"))
            family = KernelFamily(fam)
        except ValueError as exc:
            raise ConfigError(f"bad canonical config {text!r}") from exc
        return cls(family, bm, bn, bk, tm, tn, uk)

    def native(self) -> _native.AgConfig:
        return _native.AgConfig(_FAMILY_CODE[self.family], *self.param_tuple())

    @classmethod
    def from_native(cls, c: _native.AgConfig) -> "KernelConfig":
        return cls(_CODE_FAMILY[c.family], c.bm, c.bn, c.bk, c.tm, c.tn, c.uk)

    @property
    def family_code(self) -> int:
        return _FAMILY_CODE[self.family]


# Parameter domains for exhaustive enumeration, in canonical order (kernels.py:123-138)
DIRECT_DOMAINS = spaces.DIRECT_DOMAINS
INDIRECT_DOMAINS = spaces.INDIRECT_DOMAINS


def domains_for(family: KernelFamily) -> dict[str, tuple[int, ...]]:
    if family in TC_FAMILIES:
        return {"block_m": spaces.TC_BLOCK_M, "block_n": spaces.TC_BLOCK_N,
                "block_k": (spaces.TC_BLOCK_K[family.value],), "tile_m": spaces.TC_STAGES,
                "tile_n": (1,), "unroll_k": (1,)}
    if family is KernelFamily.SPLITK:
        return {"block_m": tuple(sorted({t[0] for t in spaces.SPLITK_TILES})),
                "block_n": tuple(sorted({t[1] for t in spaces.SPLITK_TILES})),
                "block_k": spaces.SPLITK_BLOCK_K,
                "tile_m": tuple(sorted({t[2] for t in spaces.SPLITK_TILES})),
                "tile_n": tuple(sorted({t[3] for t in spaces.SPLITK_TILES})),
                "unroll_k": spaces.SPLITK_SLICES}
    if family is KernelFamily.TMA:
        return {"block_m": tuple(sorted({t[0] for t in spaces.TMA_TILES})),
                "block_n": tuple(sorted({t[1] for t in spaces.TMA_TILES})),
                "block_k": (spaces.TMA_BLOCK_K,),
                "tile_m": tuple(sorted({t[2] for t in spaces.TMA_TILES})),
                "tile_n": tuple(sorted({t[3] for t in spaces.TMA_TILES})),
                "unroll_k": (1,)}
    if family in (KernelFamily.SKINNY_N, KernelFamily.SKINNY_M):
        tuples = spaces.enumerate_tuples(family.value, spaces.B200_CAPS, spaces.PROFILE_B200)
        return {f: tuple(sorted({t[1 + i] for t in tuples})) for i, f in enumerate(
            ("block_m", "block_n", "block_k", "tile_m", "tile_n", "unroll_k"))}
    return DIRECT_DOMAINS if family is KernelFamily.DIRECT else INDIRECT_DOMAINS


def _caps_dict(caps: DeviceCaps) -> dict:
    return caps.as_dict()


def is_legal(config: KernelConfig, caps: DeviceCaps) -> bool:
    """Every configuration invariant under the given caps (kernels.py:145-158)."""
    return spaces.is_legal_tuple(config.family.value, *config.param_tuple(), _caps_dict(caps))


def enumerate_search_space(family: KernelFamily, caps: DeviceCaps = DeviceCaps()) -> list[KernelConfig]:
    """All legal configs of one family in deterministic canonical order."""
    fam = KernelFamily(family)
    return [KernelConfig(fam, *t[1:])
            for t in spaces.enumerate_tuples(fam.value, _caps_dict(caps), caps.profile)]


def full_search_space(caps: DeviceCaps = DeviceCaps()) -> list[KernelConfig]:
    """All families concatenated: direct block first, then indirect (then, in
    the B200 profiles only, split-K, TMA, skinny, and in b200tc the tensor-core
    families) -- KernelFamily order, so existing class ids keep their meaning."""
    out = []
    for fam in KernelFamily:
        out.extend(enumerate_search_space(fam, caps))
    return out


# ---------------------------------------------------------------------------
# operands


def _round_up(x: int, step: int) -> int:
    return -(-x // step) * step


def _dims(x) -> tuple:
    return tuple(int(d) for d in x.shape)


def _check_operands(shape: ProblemShape, A, B, C):
    """kernels.py:271-283, for numpy arrays and CUDA torch tensors alike."""
    a_dims = (shape.K, shape.M) if shape.transA else (shape.M, shape.K)
    b_dims = (shape.N, shape.K) if shape.transB else (shape.K, shape.N)
    if A.ndim != 2 or _dims(A) != a_dims:
        raise ShapeError(f"A has shape {_dims(A)}, expected {a_dims}")
    if B.ndim != 2 or _dims(B) != b_dims:
        raise ShapeError(f"B has shape {_dims(B)}, expected {b_dims}")
    if C.ndim != 2 or _dims(C) != (shape.M, shape.N):
        raise ShapeError(f"C has shape {_dims(C)}, expected {(shape.M, shape.N)}")
    if not (A.dtype == B.dtype == C.dtype):
        raise ShapeError(f"mixed dtypes: {A.dtype}, {B.dtype}, {C.dtype}")
    if _device.dtype_code(A.dtype) < 0:
        raise ShapeError(f"unsupported dtype {A.dtype}, want float32 or float64")


class _Operands:
    """Device views of (A, B, C, out) for one call, host or device side.

    Host operands are numpy arrays or torch CPU tensors (pinned ones move
    asynchronously).  `need_c=False` (beta == 0 with a family that never
    reads C) skips staging C; the kernel then gets `out` as a never-read C.
    """

    def __init__(self, shape: ProblemShape, A, B, C, out, need_c: bool = True):
        self.host = not any(_device.is_cuda_tensor(x) for x in (A, B, C))
        t = _device.require_cuda()
        self.code = _device.dtype_code(A.dtype)
        if self.host:
            if out is not None and (_dims(out) != (shape.M, shape.N) or _device.dtype_code(out.dtype) != self.code):
                raise ShapeError("out buffer has wrong shape or dtype")
            self.device = _device.default_device()
            self.A = _device.to_device(A, self.device)
            self.B = _device.to_device(B, self.device)
            self.out_host = out
            self.out = t.empty((shape.M, shape.N), dtype=self.A.dtype, device=self.device)
            self.C = _device.to_device(C, self.device) if need_c else self.out
        else:
            for name, x in (("A", A), ("B", B), ("C", C)):
                if not _device.is_cuda_tensor(x):
                    raise ShapeError(f"{name} must be a CUDA tensor when any operand is one")
            self.device = A.device
            if B.device != self.device or C.device != self.device:
                raise ShapeError("operands live on different devices")
            self.A = _device.row_major(A)
            self.B = _device.row_major(B)
            self.C = _device.row_major(C)
            if out is None:
                out = t.empty((shape.M, shape.N), dtype=A.dtype, device=self.device)
            elif (not _device.is_device_tensor(out) or _dims(out) != (shape.M, shape.N)
                  or out.dtype != A.dtype or out.device != self.device):
                raise ShapeError("out buffer has wrong shape, dtype or device")
            self.out_host = None
            self.out_user = out
            self.out = out if (out.stride(1) == 1 and out.stride(0) >= shape.N) else \
                t.empty((shape.M, shape.N), dtype=A.dtype, device=self.device)

    def args(self):
        ld = _device.leading_dim
        return (ctypes.c_void_p(self.A.data_ptr()), ld(self.A),
                ctypes.c_void_p(self.B.data_ptr()), ld(self.B),
                ctypes.c_void_p(self.C.data_ptr()), ld(self.C),
                ctypes.c_void_p(self.out.data_ptr()), ld(self.out))

    def result(self):
        if self.host:
            out = self.out_host
            if out is not None and _device.is_device_tensor(out):  # torch CPU (pinned: async D2H)
                out.copy_(self.out, non_blocking=bool(out.is_pinned()))
                _device.torch().cuda.current_stream(self.device).synchronize()
                return out
            res = self.out.cpu().numpy()
            if out is not None:
                out[...] = res
                return out
            return res
        if self.out is not self.out_user:
            self.out_user.copy_(self.out)
        return self.out_user


class _HostOperands:
    """Raw host views (pointer, leading dimension) of numpy / torch-CPU
    operands for the pipelined host path (ag_gemm_host / ag_dispatch_gemm_host).
    Row-major matrices (unit column stride) are used in place; anything else is
    copied to a contiguous array first.  `out` is written in place when it is
    row-major, else through a temporary copied back by result()."""

    def __init__(self, shape: ProblemShape, A, B, C, out):
        self.code = _device.dtype_code(A.dtype)
        self._keep = []
        self.A = self._view(A)
        self.B = self._view(B)
        self.C = self._view(C)
        dt = np.float32 if self.code == 0 else np.float64
        if out is None:
            self.out_user = np.empty((shape.M, shape.N), dtype=dt)
        else:
            if _dims(out) != (shape.M, shape.N) or _device.dtype_code(out.dtype) != self.code:
                raise ShapeError("out buffer has wrong shape or dtype")
            if _device.is_cuda_tensor(out):
                raise ShapeError("out must be a host buffer when the operands are host buffers")
            self.out_user = out
        view = self._view(self.out_user, writable=True)
        self.out_tmp = None
        if view is None:  # not row-major: compute into a temporary
            self.out_tmp = np.empty((shape.M, shape.N), dtype=dt)
            view = self._view(self.out_tmp, writable=True)
        self.out = view

    def _view(self, x, writable=False):
        if _device.is_device_tensor(x):
            if not (x.dim() == 2 and x.stride(1) == 1 and x.stride(0) >= max(1, x.shape[1])):
                if writable:
                    return None
                x = x.contiguous()
            self._keep.append(x)
            return ctypes.c_void_p(x.data_ptr()), max(int(x.stride(0)), int(x.shape[1]), 1)
        a = np.asarray(x)
        item = a.dtype.itemsize
        ok = a.ndim == 2 and (a.shape[1] <= 1 or a.strides[1] == item) and a.strides[0] % item == 0 \
            and (a.shape[0] <= 1 or a.strides[0] >= a.shape[1] * item)
        if not ok:
            if writable:
                return None
            a = np.ascontiguousarray(a)
        if writable and not a.flags.writeable:
            raise ShapeError("out buffer is read-only")
        self._keep.append(a)
        ld = a.strides[0] // item if a.shape[0] > 1 else a.shape[1]
        return ctypes.c_void_p(a.ctypes.data), max(int(ld), int(a.shape[1]), 1)

    def args(self):
        return (*self.A, *self.B, *self.C, *self.out)

    def result(self):
        if self.out_tmp is not None:
            if _device.is_device_tensor(self.out_user):
                self.out_user.copy_(_device.torch().from_numpy(self.out_tmp))
            else:
                self.out_user[...] = self.out_tmp
        return self.out_user


def host_scratch_bytes(shape: ProblemShape, config: KernelConfig, dtype=np.float32, panels: int = 0) -> int:
    """Device bytes the pipelined host path needs (staged operands + workspace)."""
    code = _device.dtype_code(dtype)
    return int(_native.lib().ag_host_scratch_bytes(ctypes.byref(native_shape(shape)),
                                                    ctypes.byref(config.native()), max(code, 0), int(panels)))


def _raise_for(code: int, config: "KernelConfig | None" = None):
    msg = _native.last_error()
    if code == _native.AG_ERR_CONFIG:
        raise ConfigError(msg or f"illegal config {config.canonical() if config else ''}")
    if code == _native.AG_ERR_SHAPE:
        raise ShapeError(msg)
    raise RuntimeError(f"CUDA failure in adaptgemm-b200: {msg}")


def native_shape(shape: ProblemShape) -> _native.AgShape:
    return _native.AgShape(shape.M, shape.N, shape.K, float(shape.alpha), float(shape.beta),
                           int(bool(shape.transA)), int(bool(shape.transB)))


def reads_c(shape: ProblemShape, config: KernelConfig) -> bool:
    """Whether the family path reads C: always for direct (kernels.py:227),
    only when beta != 0 for indirect / split-K / tensor-core families
    (kernels.py:318-321)."""
    return config.family is KernelFamily.DIRECT or shape.beta != 0.0


def workspace_bytes(shape: ProblemShape, config: KernelConfig, dtype=np.float32) -> int:
    """Device bytes the indirect pack buffers need (0 for direct)."""
    code = _device.dtype_code(dtype)
    return int(_native.lib().ag_workspace_bytes(ctypes.byref(native_shape(shape)),
                                                 ctypes.byref(config.native()), max(code, 0)))


# ---------------------------------------------------------------------------
# public entry points


def gemm_reference(shape: ProblemShape, A, B, C, out=None):
    """Textbook (i, j, k) GEMM with float64 accumulation; the correctness oracle.

    Runs `reference_gemm_kernel` on the GPU: the operation sequence of
    _kernel_reference (kernels.py:184-195) -- separately rounded float64
    multiply and add in k order, one rounding to the element type -- so the
    result is bit-identical to the reference's.
    """
    _check_operands(shape, A, B, C)
    ops = _Operands(shape, A, B, C, out)
    lib = _native.lib()
    a, lda, b, ldb, c, ldc, o, ldo = ops.args()
    with _device.guard(ops.device):
        rc = lib.ag_gemm_reference(ctypes.byref(native_shape(shape)), ops.code, a, lda, b, ldb, c, ldc,
                                   o, ldo, ctypes.c_void_p(_device.current_stream_handle(ops.device)))
    if rc:
        _raise_for(rc)
    return ops.result()


def pack_padded(X, rows: int, cols: int, transpose: bool, pad_rows: int, pad_cols: int):
    """Indirect-family helper pass: zero-padded copy of op(X) (kernels.py:304-309).

    Runs the device pack kernel; numpy in -> numpy out, CUDA tensor in ->
    CUDA tensor out.
    """
    t = _device.require_cuda()
    host = not _device.is_device_tensor(X)
    code = _device.dtype_code(X.dtype)
    if code < 0:
        raise ShapeError(f"unsupported dtype {X.dtype}")
    dev = _device.default_device() if host else X.device
    src = _device.to_device(X, dev) if host else _device.row_major(X)
    want = (cols, rows) if transpose else (rows, cols)
    if _dims(src) != want:
        raise ShapeError(f"X has shape {_dims(src)}, expected {want}")
    dst = t.empty((pad_rows, pad_cols), dtype=src.dtype, device=dev)
    with _device.guard(dev):
        rc = _native.lib().ag_pack_padded(code, ctypes.c_void_p(src.data_ptr()), _device.leading_dim(src),
                                          rows, cols, int(bool(transpose)), ctypes.c_void_p(dst.data_ptr()),
                                          pad_rows, pad_cols, ctypes.c_void_p(_device.current_stream_handle(dev)))
    if rc:
        _raise_for(rc)
    return dst.cpu().numpy() if host else dst


def _launch(shape: ProblemShape, config: KernelConfig, caps: DeviceCaps, ops: _Operands,
            timed: bool) -> float:
    with _device.guard(ops.device):
        return _launch_here(shape, config, caps, ops, timed)


def _launch_here(shape, config, caps, ops, timed):
    t = _device.torch()
    lib = _native.lib()
    nshape, ncfg, ncaps = native_shape(shape), config.native(), caps.native()
    ws_n = int(lib.ag_workspace_bytes(ctypes.byref(nshape), ctypes.byref(ncfg), ops.code))
    stream = t.cuda.current_stream(ops.device)
    ws = _device.workspace(ws_n, ops.device, stream.cuda_stream) if ws_n else None
    ws_ptr = ctypes.c_void_p(ws.data_ptr() if ws is not None else 0)
    a, lda, b, ldb, c, ldc, o, ldo = ops.args()
    if timed:
        e0 = t.cuda.Event(enable_timing=True)
        e1 = t.cuda.Event(enable_timing=True)
        e0.record(stream)
    rc = lib.ag_gemm(ctypes.byref(nshape), ctypes.byref(ncfg), ctypes.byref(ncaps), ops.code,
                     a, lda, b, ldb, c, ldc, o, ldo, ws_ptr, ws_n, ctypes.c_void_p(stream.cuda_stream))
    if rc:
        _raise_for(rc, config)
    if not timed:
        return 0.0
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) * 1e-3


_fp = None


def _fastpath():
    """The CPython extension for numpy operands (csrc/fastpath.c), or None
    when it is not built (the ctypes path below then serves every call)."""
    global _fp
    if _fp is None:
        try:
            from . import _fastpath as m
            m.set_errors(ConfigError, ShapeError)
            _fp = m
        except ImportError:
            _fp = False
    return _fp or None


def gemm_execute(shape: ProblemShape, config: KernelConfig, A, B, C,
                 caps: DeviceCaps = DeviceCaps(), out=None):
    """Run one config's family path end to end on the GPU (kernels.py:328-349).

    Legality is checked before the operands (ConfigError, then ShapeError).
    Returns (result, seconds); seconds is the CUDA-event device time of the
    whole family path (indirect: pack helpers + tiled core), floored at 1e-9.

    numpy operands (the reference's convention) take the compiled fast path
    once CUDA is known to be up: one C call does legality, the operand
    checks and ag_gemm_host_ex (pipelined H2D / family path / D2H with the
    host buffers page-locked for the call); `seconds` is then the device
    time of the family path's kernels.
    """
    if _device._cuda_ok and type(A) is np.ndarray and type(B) is np.ndarray and type(C) is np.ndarray and \
            (out is None or type(out) is np.ndarray):
        fp = _fastpath()
        if fp is not None:
            r = fp.execute(shape, config, A, B, C, caps, out)
            if r is not NotImplemented:
                return r
    if not is_legal(config, caps):
        raise ConfigError(f"illegal config {config.canonical()} for caps {caps}")
    _check_operands(shape, A, B, C)
    ops = _Operands(shape, A, B, C, out, need_c=reads_c(shape, config))
    elapsed = _launch(shape, config, caps, ops, timed=True)
    return ops.result(), max(elapsed, 1e-9)


def warm_kernels(dtype=np.float32) -> None:
    """Initialise the CUDA context and load the kernel module (kernels.py:352-361)."""
    shape = ProblemShape(4, 4, 4, alpha=1.0, beta=1.0)
    A = np.ones((4, 4), dtype)
    B = np.ones((4, 4), dtype)
    C = np.ones((4, 4), dtype)
    gemm_reference(shape, A, B, C)
    gemm_execute(shape, KernelConfig(KernelFamily.DIRECT, 8, 8, 8, 2, 2, 1), A, B, C)
    for uk in (1, 2):
        gemm_execute(shape, KernelConfig(KernelFamily.INDIRECT, 16, 16, 8, 2, 2, uk), A, B, C)


def ffma_peak_tflops() -> float:
    """Measured FP32 FFMA throughput of this GPU (CUDA-core roofline)."""
    t = _device.require_cuda()
    dev = _device.default_device()
    val = ctypes.c_double(0.0)
    rc = _native.lib().ag_ffma_peak(ctypes.c_void_p(t.cuda.current_stream(dev).cuda_stream),
                                    ctypes.byref(val))
    if rc:
        _raise_for(rc)
    return val.value
