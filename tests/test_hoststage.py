"""CPU checks of the pageable-staging host code (csrc/hoststage.h): the
copy-worker pool runs every item exactly once under concurrent callers, the
parallel pitched copy is byte-exact for contiguous and strided blocks, and
the slot chunking covers a block exactly with chunks that fit a 4 MB slot.
(No GPU: the header's CUDA calls are not exercised here; the staged GEMM
path itself is checked on the B200 by test_gpu_dispatch.py.)"""
import ctypes
import subprocess
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
SRC = ROOT / "tests" / "native" / "hoststage_harness.cpp"
SLOT = 4 << 20


@pytest.fixture(scope="module")
def hs(tmp_path_factory):
    out = tmp_path_factory.mktemp("hs") / "libhs.so"
    cmd = ["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-pthread", "-I/usr/local/cuda/include", str(SRC), "-o",
           str(out), "-L/usr/local/cuda/lib64", "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        pytest.skip(f"cannot build the harness: {r.stderr[-400:]}")
    L = ctypes.CDLL(str(out))
    L.hs_copy_rows.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                               ctypes.c_int64]
    L.hs_chunks.argtypes = [ctypes.c_int64] * 4 + [ctypes.c_void_p, ctypes.c_int]
    L.hs_pool_stress.argtypes = [ctypes.c_int] * 3
    return L


def test_pool_runs_every_item_once_under_concurrent_callers(hs):
    assert hs.hs_pool_threads() >= 1
    assert hs.hs_pool_stress(4, 50, 37) == 0
    assert hs.hs_pool_stress(1, 200, 1) == 0


@pytest.mark.parametrize("rows,width,spitch,dpitch", [
    (1, 64, 64, 64), (3, 1000, 1000, 1000), (1 << 10, 4096, 4096, 4096),  # contiguous (flattened)
    (700, 2800, 33828, 2800), (513, 4 * 875, 4 * 7000, 4 * 875), (2048, 64, 4096, 128),  # strided
])
def test_copy_rows_byte_exact(hs, rows, width, spitch, dpitch):
    rng = np.random.default_rng(rows + width)
    src = rng.integers(0, 255, rows * spitch, dtype=np.uint8)
    dst = np.zeros(rows * dpitch, np.uint8)
    hs.hs_copy_rows(dst.ctypes.data, dpitch, src.ctypes.data, spitch, width, rows)
    got = dst.reshape(rows, dpitch)[:, :width]
    np.testing.assert_array_equal(got, src.reshape(rows, spitch)[:, :width])
    assert not dst.reshape(rows, dpitch)[:, width:].any()  # nothing written past each row


@pytest.mark.parametrize("rows,width,hpitch,dpitch", [
    (2048, 8192, 8192, 8192),          # contiguous: flattened into byte chunks
    (35, 2800, 33828, 2800),           # strided rows
    (4096, 4 * 2048, 4 * 4096, 4 * 2048),
    (3, 3 << 20, 3 << 20, 4 << 20),    # rows just under a slot
])
def test_chunks_cover_the_block_and_fit_a_slot(hs, rows, width, hpitch, dpitch):
    buf = (ctypes.c_int64 * (4 * 4096))()
    n = hs.hs_chunks(hpitch, dpitch, width, rows, buf, 4096)
    ch = [tuple(buf[4 * i:4 * i + 4]) for i in range(n)]
    if hpitch == width and dpitch == width:
        total = rows * width
        assert sum(c[3] for c in ch) == total and all(c[0] == 0 and c[1] == 1 for c in ch)
        assert [c[2] for c in ch] == [sum(x[3] for x in ch[:i]) for i in range(n)]
        assert max(c[3] for c in ch) <= SLOT
    else:
        assert sum(c[1] for c in ch) == rows
        assert [c[0] for c in ch] == [sum(x[1] for x in ch[:i]) for i in range(n)]
        assert all(c[1] * c[3] <= SLOT and c[3] == width and c[2] == 0 for c in ch)
