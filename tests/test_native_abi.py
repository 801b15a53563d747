"""The C-ABI library loads and exports what include/adaptgemm_b200.h declares (CPU only).

No compute call is made here: the CPU container has no GPU.  The host-only
entry points (legality, registry, workspace sizing, CART, selector) are
exercised; kernels are checked to exist for every enumerated config.
"""

import ctypes
import re
import subprocess

import pytest

from conftest import ROOT
from paper_1806_07060_b200 import _native, spaces
from paper_1806_07060_b200.kernels import (TC_FAMILIES,
    DeviceCaps,
    KernelConfig,
    KernelFamily,
    ProblemShape,
    full_search_space,
    is_legal,
    native_shape,
)

HEADER = ROOT / "include" / "adaptgemm_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"\b(ag_[a-z0-9_]+)\s*\(", text)))


def test_library_loads():
    lib = _native.lib()
    assert lib.ag_version().decode().startswith("adaptgemm-b200")
    assert lib.ag_num_kernels() >= len(spaces.compiled_tuples())


def test_every_declared_symbol_is_exported():
    syms = declared_symbols()
    assert len(syms) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", str(_native.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (ag_[a-z0-9_]+)$", out, re.M))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    # and the ctypes binding covers all of them
    assert set(syms) <= set(_native.SIGNATURES)


def test_library_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(_native.LIB_PATH)],
                         capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


@pytest.mark.parametrize("caps", [DeviceCaps(), DeviceCaps.b200(), DeviceCaps(register_tile_cap_direct=16),
                                  DeviceCaps(tile_memory_cap=4096, max_threads=256)])
def test_native_legality_equals_python(caps):
    lib = _native.lib()
    ncaps = caps.native()
    grid = [(f, bm, bn, bk, tm, tn, uk)
            for f in (KernelFamily.DIRECT, KernelFamily.INDIRECT, KernelFamily.SPLITK, KernelFamily.TMA)
            for bm in (8, 16, 24, 64, 256) for bn in (8, 32, 128) for bk in (8, 16, 32)
            for tm in (1, 2, 3, 8) for tn in (1, 4, 8) for uk in (1, 2)]
    for t in grid:
        cfg = KernelConfig(*t)
        assert bool(lib.ag_is_legal(ctypes.byref(cfg.native()), ctypes.byref(ncaps))) == is_legal(cfg, caps), cfg


def test_every_enumerated_config_has_a_kernel():
    lib = _native.lib()
    for caps in (DeviceCaps(), DeviceCaps.b200()):
        for cfg in full_search_space(caps):
            assert lib.ag_has_kernel(ctypes.byref(cfg.native()), _native.AG_F32), cfg
            assert lib.ag_has_kernel(ctypes.byref(cfg.native()), _native.AG_F64), cfg


def test_workspace_sizes():
    lib = _native.lib()
    s = native_shape(ProblemShape(33, 33, 17))
    d = KernelConfig(KernelFamily.DIRECT, 16, 16, 8, 2, 2, 1)
    i = KernelConfig(KernelFamily.INDIRECT, 32, 32, 16, 4, 4, 1)
    assert lib.ag_workspace_bytes(ctypes.byref(s), ctypes.byref(d.native()), 0) == 0
    # Ap: 32 x 64 floats, Bp: 32 x 64 floats, each 256-byte rounded
    assert lib.ag_workspace_bytes(ctypes.byref(s), ctypes.byref(i.native()), 0) == 2 * 32 * 64 * 4


def test_native_tc_legality_equals_python():
    lib = _native.lib()
    ncaps = DeviceCaps.b200_tc().native()
    for fam in (KernelFamily.TF32, KernelFamily.BF16, KernelFamily.TF32X3):
        for bm in (64, 128, 256):
            for bn in (16, 32, 64, 96, 128, 192, 256, 288):
                for bk in (16, 32, 64):
                    for tm in (1, 2, 4, 6, 7, 8, 9):
                        for tn, uk in ((1, 1), (2, 1), (1, 2)):
                            cfg = KernelConfig(fam, bm, bn, bk, tm, tn, uk)
                            assert bool(lib.ag_is_legal(ctypes.byref(cfg.native()), ctypes.byref(ncaps))) == \
                                is_legal(cfg, DeviceCaps.b200_tc()), cfg


def test_tc_space_has_kernels_float32_only():
    lib = _native.lib()
    tc = [c for c in full_search_space(DeviceCaps.b200_tc()) if c.family in TC_FAMILIES]
    assert len(tc) >= 44
    assert {c.family for c in tc} == set(TC_FAMILIES)
    assert {c.block_m for c in tc} == {128, 256}  # one CTA and CTA-pair (cta_group::2) tiles
    for cfg in tc:
        assert lib.ag_has_kernel(ctypes.byref(cfg.native()), _native.AG_F32), cfg


def test_tc_workspace_sizes():
    lib = _native.lib()
    cfg = KernelConfig(KernelFamily.BF16, 128, 128, 64, 4, 1, 1)
    s = native_shape(ProblemShape(33, 70, 17))
    # bf16 staging keeps the layout with 128-byte rows: A 33 x 64 (17 -> 64), B 17 x 128 (70 -> 128),
    # each 1 KiB rounded
    want = -(-33 * 64 * 2 // 1024) * 1024 + -(-17 * 128 * 2 // 1024) * 1024
    assert lib.ag_workspace_bytes(ctypes.byref(s), ctypes.byref(cfg.native()), 0) == want
    # tf32x3 stages like tf32 (re-strided copies only for unaligned rows: fp32
    # rows rounded to 32 elements, each 1 KiB rounded); its lo parts are made
    # in shared memory
    x3 = KernelConfig(KernelFamily.TF32X3, 128, 128, 32, 2, 1, 1)
    want3 = -(-33 * 32 * 4 // 1024) * 1024 + -(-17 * 96 * 4 // 1024) * 1024
    assert lib.ag_workspace_bytes(ctypes.byref(s), ctypes.byref(x3.native()), 0) == want3


def test_tf32x3_split_is_exact():
    """hi keeps the bits a tf32 MMA reads, lo = x - hi is exact in fp32 and
    below 2^-10 |x| (the 3xTF32 error budget, tc_kernels.cuh)."""
    import numpy as np
    x = np.random.default_rng(0).uniform(-1e3, 1e3, 100000).astype(np.float32)
    hi = (x.view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)
    lo = x - hi
    assert np.array_equal(hi.astype(np.float64) + lo.astype(np.float64), x.astype(np.float64))
    assert np.all(np.abs(lo) <= np.abs(x) * 2.0 ** -10)


def test_host_scratch_bytes():
    lib = _native.lib()
    cfg = KernelConfig(KernelFamily.INDIRECT, 32, 32, 16, 4, 4, 1)
    shape = ProblemShape(1000, 300, 50)
    s = native_shape(shape)
    up = lambda n: -(-n // 256) * 256  # noqa: E731
    # beta == 0, indirect: staged A, B, out + the workspace of the largest row panel (1 panel: the whole call)
    ws = lib.ag_workspace_bytes(ctypes.byref(s), ctypes.byref(cfg.native()), 0)
    want = up(1000 * 50 * 4) + up(50 * 300 * 4) + up(1000 * 300 * 4) + up(ws)
    assert lib.ag_host_scratch_bytes(ctypes.byref(s), ctypes.byref(cfg.native()), 0, 1) == want
    # 4 row panels of 256 rows: workspace of a 256-row panel; the direct family also stages C
    p = native_shape(ProblemShape(256, 300, 50))
    ws4 = lib.ag_workspace_bytes(ctypes.byref(p), ctypes.byref(cfg.native()), 0)
    assert lib.ag_host_scratch_bytes(ctypes.byref(s), ctypes.byref(cfg.native()), 0, 4) == want - up(ws) + up(ws4)
    d = KernelConfig(KernelFamily.DIRECT, 16, 16, 8, 2, 2, 1)
    assert lib.ag_host_scratch_bytes(ctypes.byref(s), ctypes.byref(d.native()), 0, 1) == \
        up(1000 * 50 * 4) + up(50 * 300 * 4) + 2 * up(1000 * 300 * 4)


def test_null_selector_reports_an_error():
    """ag_select / ag_select_many on a null selector fail with AG_ERR_CONFIG
    and a message (no stale or empty ag_last_error)."""
    lib = _native.lib()
    cfg = _native.AgConfig()
    assert lib.ag_select(None, 64, 64, 64, ctypes.byref(cfg)) == -1
    assert b"null selector" in lib.ag_last_error()
    mnk = (ctypes.c_int64 * 3)(64, 64, 64)
    ids = (ctypes.c_int64 * 1)()
    assert lib.ag_select_many(None, mnk, 1, ids) != 0
    assert b"null selector" in lib.ag_last_error()
