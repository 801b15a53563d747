import json
import math
import sys
from functools import lru_cache
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = Path(__file__).resolve().parent / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

from paper_1806_07060_b200 import rng  # noqa: E402
from paper_1806_07060_b200.kernels import DeviceCaps, ProblemShape, full_search_space  # noqa: E402
from paper_1806_07060_b200.tuner import Measurement, TuningTable, flops_of  # noqa: E402

FAST_TIMING_KW = dict(warmup=0, repeats=1)
# the north-star parity bar for fp32 variants (BASELINE.json): relative
# Frobenius error vs the float64-accumulating reference
RF_TOL_F32 = 1e-5
RF_TOL_F64 = 1e-12


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@lru_cache(maxsize=None)
def golden() -> dict:
    with open(GOLDEN / "golden.json") as fh:
        return json.load(fh)


@lru_cache(maxsize=None)
def golden_gemm():
    return np.load(GOLDEN / "gemm_golden.npz")


def golden_shape(meta) -> ProblemShape:
    return ProblemShape(meta["M"], meta["N"], meta["K"], meta["alpha"], meta["beta"],
                        meta["transA"], meta["transB"])


@pytest.fixture(scope="session")
def default_caps():
    return DeviceCaps()


@pytest.fixture(scope="session")
def search_space(default_caps):
    return full_search_space(default_caps)


def rand_operands(shape: ProblemShape, dtype=np.float32, seed=0):
    """The reference's test operand recipe (tests/conftest.py:24-31)."""
    gen = np.random.default_rng(rng.mix(seed, shape.M, shape.N, shape.K))
    a_dims = (shape.K, shape.M) if shape.transA else (shape.M, shape.K)
    b_dims = (shape.N, shape.K) if shape.transB else (shape.K, shape.N)
    A = gen.uniform(-1.0, 1.0, a_dims).astype(dtype)
    B = gen.uniform(-1.0, 1.0, b_dims).astype(dtype)
    C = gen.uniform(-1.0, 1.0, (shape.M, shape.N)).astype(dtype)
    return A, B, C


def rel_frobenius(x, ref) -> float:
    x = np.asarray(x, np.float64)
    ref = np.asarray(ref, np.float64)
    den = np.linalg.norm(ref)
    return float(np.linalg.norm(x - ref) / (den if den > 0 else 1.0))


def assert_rf(out, ref, dtype=np.float32):
    tol = RF_TOL_F32 if np.dtype(dtype) == np.float32 else RF_TOL_F64
    err = rel_frobenius(out, ref)
    assert err <= tol, f"relative Frobenius error {err:.3e} > {tol:.0e}"


def fake_gflops(shape: ProblemShape, config) -> float:
    """The reference's deterministic synthetic performance model (conftest.py:39-55)."""
    m, n, k = shape.mnk
    gmean = (m * n * k) ** (1.0 / 3.0)
    target = 8 if gmean < 96 else (16 if gmean < 192 else (32 if gmean < 768 else 64))
    fit = (-abs(math.log2(config.block_m) - math.log2(target))
           - 0.5 * abs(math.log2(config.block_n) - math.log2(target)))
    direct = config.family.value == "direct"
    bonus = 0.6 if direct == (gmean < 192) else -0.6
    jitter = (rng.mix(m, n, k, config.block_k, config.tile_m, config.tile_n,
                      config.unroll_k, int(direct)) % 997) / 1e4
    return 10.0 + fit + bonus + jitter


@pytest.fixture(scope="session")
def fake_table_factory(search_space):
    def make(shape: ProblemShape) -> TuningTable:
        fl = flops_of(shape)
        ms = []
        for c in search_space:
            gf = fake_gflops(shape, c)
            ms.append(Measurement(c, fl / (gf * 1e9), gf))
        return TuningTable.from_measurements(shape, ms, {"mode": "fixture"})
    return make
