"""Device plumbing: operand staging, per-thread workspaces, streams.

PyTorch provides CUDA memory and streams only; every GEMM runs in
libadaptgemm_b200.so.  Host (numpy) operands are staged through pinned
buffers into device tensors; device (torch.cuda) operands are used in place.
"""

import threading

import numpy as np

_torch = None


def torch():
    """Import torch lazily (the CPU-only parts of the package do not need it)."""
    global _torch
    if _torch is None:
        import torch as _t
        _torch = _t
    return _torch


class DeviceUnavailableError(RuntimeError):
    """No CUDA device: the GEMM path has no CPU fallback."""


_cuda_ok = False


def require_cuda():
    """torch, after checking (once, then cached) that a CUDA device is visible."""
    global _cuda_ok
    t = torch()
    if not _cuda_ok:
        if not t.cuda.is_available():
            raise DeviceUnavailableError(
                "no CUDA device visible: adaptgemm-b200 runs GEMMs only on the GPU (sm_100a)")
        _cuda_ok = True
    return t


def is_device_tensor(x) -> bool:
    t = _torch
    if t is None:
        # avoid importing torch just to answer "no" for numpy inputs
        return type(x).__module__.startswith("torch")
    return isinstance(x, t.Tensor)


_NP_TO_CODE = {np.dtype(np.float32): 0, np.dtype(np.float64): 1}


def dtype_code(dtype) -> int:
    """0 float32, 1 float64, -1 anything else (numpy or torch dtype)."""
    t = _torch
    if t is None and type(dtype).__module__.startswith("torch"):
        t = torch()  # a torch dtype before this module imported torch
    if t is not None and isinstance(dtype, t.dtype):
        return {t.float32: 0, t.float64: 1}.get(dtype, -1)
    try:
        return _NP_TO_CODE.get(np.dtype(dtype), -1)
    except TypeError:
        return -1


def row_major(t):
    """A 2-D tensor whose last dim is contiguous (returns it or a copy)."""
    if t.dim() == 2 and t.stride(1) == 1 and t.stride(0) >= max(1, t.shape[1]):
        return t
    return t.contiguous()


def leading_dim(t) -> int:
    return max(int(t.stride(0)), int(t.shape[1]), 1)


_tls = threading.local()


def workspace(nbytes: int, device, stream: int | None = None):
    """Per-thread, per-device, per-stream grow-only byte buffer (allocation is
    never timed).  Keyed by the stream the family path runs on: two calls
    on different streams never share pack / split-K buffers, and a buffer
    is allocated while its stream is torch's current one, so the caching
    allocator only hands a freed (outgrown) buffer back to work on that
    same stream, ordered after the kernels that used it."""
    t = torch()
    cache = getattr(_tls, "ws", None)
    if cache is None:
        cache = _tls.ws = {}
    if stream is None:
        stream = current_stream_handle(device)
    key = (device.type, device.index, int(stream))
    buf = cache.get(key)
    if buf is None or buf.numel() < nbytes:
        size = max(nbytes, 1 << 20)
        if buf is not None:
            size = max(size, buf.numel() * 2)
        buf = t.empty(size, dtype=t.uint8, device=device)
        cache[key] = buf
    return buf


class _NoGuard:
    def __enter__(self):
        return None

    def __exit__(self, *exc):
        return False


_NO_GUARD = _NoGuard()


def guard(device):
    """Make `device` the current CUDA device for a native call (kernel
    launches, events and attributes follow the current device); a no-op when
    it already is."""
    t = torch()
    idx = device.index if getattr(device, "index", None) is not None else None
    if idx is None or idx == t.cuda.current_device():
        return _NO_GUARD
    return t.cuda.device(idx)


def current_stream_handle(device) -> int:
    """Raw cudaStream_t of torch's current stream on `device` (the C++ getter
    when torch exposes it: no Stream object per call)."""
    t = torch()
    raw = getattr(t._C, "_cuda_getCurrentRawStream", None)
    if raw is not None:
        idx = device.index if getattr(device, "index", None) is not None else t.cuda.current_device()
        return int(raw(idx))
    return int(t.cuda.current_stream(device).cuda_stream)


def is_cuda_tensor(x) -> bool:
    return is_device_tensor(x) and x.is_cuda


def to_device(a, device):
    """Copy a host matrix (numpy array or torch CPU tensor) to a contiguous
    device tensor; pinned torch tensors are copied asynchronously."""
    t = torch()
    if is_device_tensor(a):
        src = a.contiguous()
        return src.to(device=device, non_blocking=bool(src.is_pinned()))
    src = t.from_numpy(np.ascontiguousarray(a))
    return src.to(device=device, non_blocking=False)


def default_device():
    t = require_cuda()
    return t.device("cuda", t.cuda.current_device())
