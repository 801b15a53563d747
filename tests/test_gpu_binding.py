"""The reference-side binding (integration/reference_kernels_b200.py) runs
the reference's `gemm_execute` convention through the C-ABI -- numpy in,
numpy out, the reference's exception order -- against the reference's own
golden outputs (tests/golden, produced by /root/reference itself)."""
import ctypes
import importlib.util

import numpy as np
import pytest

from conftest import ROOT, golden, golden_gemm, golden_shape, rel_frobenius
from paper_1806_07060_b200.kernels import ConfigError, DeviceCaps, KernelConfig, KernelFamily, ProblemShape, ShapeError

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def binding():
    spec = importlib.util.spec_from_file_location("reference_kernels_b200",
                                                  ROOT / "integration" / "reference_kernels_b200.py")
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    mod.bind(ConfigError, ShapeError)
    return mod


def test_binding_reproduces_reference_goldens(binding):
    """Every golden GEMM case: the reference's inputs and its sampled family
    configs; the output within the fp32 / fp64 bar of both the reference's
    oracle output and the reference's own family output for that config."""
    z = golden_gemm()
    n = 0
    for meta in golden()["gemm"]:
        k = meta["key"]
        s = golden_shape(meta)
        A, B, C = z[f"{k}_A"], z[f"{k}_B"], z[f"{k}_C"]
        bar = 1e-5 if A.dtype == np.float32 else 1e-12
        for j, canon in enumerate(meta["execute_configs"]):
            cfg = KernelConfig.from_canonical(canon)
            out = np.full((s.M, s.N), np.nan, dtype=A.dtype)
            got, sec = binding.gemm_execute(s, cfg, A, B, C, DeviceCaps(), out)
            assert got is out and sec > 0
            assert rel_frobenius(out, z[f"{k}_ref"]) <= bar, (meta["name"], canon)
            assert rel_frobenius(out, z[f"{k}_x{j}"]) <= bar, (meta["name"], canon)
            n += 1
    assert n > 0


def test_binding_error_order(binding):
    s = ProblemShape(8, 8, 8)
    A = np.ones((8, 8), np.float32)
    bad = np.ones((7, 8), np.float32)
    illegal = KernelConfig(KernelFamily.DIRECT, 8, 8, 8, 1, 1, 2)  # direct with unroll 2
    with pytest.raises(ConfigError):
        binding.gemm_execute(s, illegal, bad, A, A, DeviceCaps())  # legality before operands
    with pytest.raises(ShapeError, match="A has shape"):
        binding.gemm_execute(s, KernelConfig(KernelFamily.DIRECT, 8, 8, 8, 1, 1, 1), bad, A, A, DeviceCaps())
    with pytest.raises(ShapeError, match="mixed dtypes"):
        binding.gemm_execute(s, KernelConfig(KernelFamily.DIRECT, 8, 8, 8, 1, 1, 1), A, A, A.astype(np.float64),
                             DeviceCaps())


def test_binding_large_pageable_call(binding):
    """A call big enough to stage and pipeline (>= 32 MB moved): pageable
    operands through the pinned rings, the fresh result in a cached pinned
    block that returns to the cache when the array is collected."""
    import gc
    from paper_1806_07060_b200.tuner import _bench_buffers
    s = ProblemShape(2048, 3000, 1024)
    A, B, C, _ = _bench_buffers(s, np.float32, 0)
    cfg = KernelConfig.from_canonical("indirect:64-64-16-8-4-2")
    out, sec = binding.gemm_execute(s, cfg, A, B, C, DeviceCaps())
    exact = A.astype(np.float64) @ B.astype(np.float64)
    assert rel_frobenius(out, exact) <= 1e-5 and sec > 0
    L = binding.lib()
    L.ag_host_cache_bytes.restype = ctypes.c_size_t
    before = L.ag_host_cache_bytes()
    del out
    gc.collect()
    assert L.ag_host_cache_bytes() >= before + 2048 * 3000 * 4
    again, _ = binding.gemm_execute(s, cfg, A, B, C, DeviceCaps())
    assert rel_frobenius(again, exact) <= 1e-5
