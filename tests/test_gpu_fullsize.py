"""Full-size parity of every kernel choice the benchmark makes.

At BASELINE.json's own sizes -- the DeepBench-style set (configs[2]), the
po2 64..4096 held-out split (configs[1]) and the tf32/bf16 random held-out
split (configs[4]) -- the decision tree's pick (through the native dispatch,
ag_dispatch_gemm), the per-shape oracle config and the default tile each run
on the bench's own operands (tuner._bench_buffers, tuner.py:128-136) and the
WHOLE output matrix is compared with the float64 product.

The float64 product is cuBLAS DGEMM via torch (test infrastructure only);
`test_fp64_blas_matches_reference_oracle` pins it against the bit-exact
gemm_reference kernel (kernels.py:294-301) on shapes from the same sets.
Bars: relative Frobenius error <= 1e-5 for the fp32
families, <= 1e-3 for tf32, <= 1e-2 for bf16.
"""
import numpy as np
import pytest

from paper_1806_07060_b200 import codegen
from paper_1806_07060_b200.kernels import (DeviceCaps, KernelConfig, KernelFamily, ProblemShape, gemm_execute,
                                           gemm_reference)
from paper_1806_07060_b200.tuner import _bench_buffers

pytestmark = pytest.mark.gpu

RF_BAR = {KernelFamily.TF32: 1e-3, KernelFamily.BF16: 1e-2}


def _bar(cfg) -> float:
    return RF_BAR.get(cfg.family, 1e-5)


@pytest.fixture(scope="module")
def shipped():
    import bench
    m = bench.build_model()
    m["tc"] = bench.build_tc_model(m["policy"])
    return m


def _device_operands(s):
    import torch
    A, B, C, _ = _bench_buffers(s, np.float32, 0)
    return tuple(torch.from_numpy(x).cuda() for x in (A, B, C))


def _rf(out, exact) -> float:
    import torch
    return float(torch.linalg.norm(out.double() - exact) / torch.linalg.norm(exact))


def _check(shapes, selector, classes_tables, policy, caps, picked_families):
    """DT pick (native dispatch), oracle and default on every shape; whole-matrix RF."""
    import torch
    worst = {}
    for s in shapes:
        dA, dB, dC = _device_operands(s)
        exact = dA.double() @ dB.double()  # alpha = 1, beta = 0
        out, picked, _fb = codegen.dispatch_native(selector, s, dA, dB, dC, caps)
        torch.cuda.synchronize()
        runs = [("dt", picked, out)]
        table = classes_tables[s.mnk]
        for label, cfg in (("oracle", table.best_config), ("default", policy.select_config(s))):
            o, _ = gemm_execute(s, cfg, dA, dB, dC, caps)
            runs.append((label, cfg, o))
        for label, cfg, o in runs:
            rf = _rf(o, exact)
            assert rf <= _bar(cfg), (s.mnk, label, cfg.canonical(), rf)
            key = cfg.family.value
            worst[key] = max(worst.get(key, 0.0), rf)
            picked_families.add((cfg.family, cfg.unroll_k if cfg.family is KernelFamily.SPLITK else 0))
        del dA, dB, dC, exact, runs
    return worst


def test_deepbench_all_picks_full_size(shipped):
    sel = codegen.CompiledSelector(shipped["tree"], shipped["classes"])
    fams = set()
    worst = _check(shipped["db_all"], sel, shipped["tables"], shipped["policy"], DeviceCaps.b200(), fams)
    print("deepbench worst RF per family:", worst)
    assert len(shipped["db_all"]) == 40


def test_po2_held_out_all_picks_full_size(shipped):
    sel = codegen.CompiledSelector(shipped["tree"], shipped["classes"])
    fams = set()
    worst = _check(shipped["po2_test"], sel, shipped["tables"], shipped["policy"], DeviceCaps.b200(), fams)
    print("po2 held-out worst RF per family:", worst)


def test_tc_held_out_all_picks_full_size(shipped):
    tc = shipped["tc"]
    if tc is None:
        pytest.skip("no tc tables shipped")
    sel = codegen.CompiledSelector(tc["tree"], tc["classes"])
    fams = set()
    worst = _check(tc["test"], sel, tc["tables"], shipped["policy"], DeviceCaps.b200_tc(), fams)
    print("tc held-out worst RF per family:", worst)
    assert any(f in (KernelFamily.TF32, KernelFamily.BF16) for f, _ in fams)


@pytest.mark.parametrize("mnk,canon", [
    ((2048, 16, 2048), "splitk:32-16-32-4-2-8"),      # in-place core, 8-slice cluster (DSMEM) reduction
    ((2048, 128, 2048), "splitk:128-128-32-8-8-16"),  # 16 slices: in-place core + slab reduction
    ((7680, 128, 2560), "splitk:64-128-16-8-8-16"),
    ((35, 8457, 2560), "splitk:64-128-32-8-8-8"),     # N % 4 != 0: packed core + splitk_reduce_kernel
    ((4096, 16, 4096), "splitk:32-16-32-4-2-16"),
])
def test_cluster_splitk_full_size(mnk, canon):
    s = ProblemShape(*mnk)
    dA, dB, dC = _device_operands(s)
    exact = dA.double() @ dB.double()
    cfg = KernelConfig.from_canonical(canon)
    out, _ = gemm_execute(s, cfg, dA, dB, dC, DeviceCaps.b200())
    again, _ = gemm_execute(s, cfg, dA, dB, dC, DeviceCaps.b200())
    assert _rf(out, exact) <= 1e-5
    import torch
    assert torch.equal(out, again)  # fixed-order reduction: bitwise repeatable at full size


@pytest.mark.parametrize("mnk", [(35, 700, 2048), (1760, 16, 1760), (256, 256, 256), (3072, 32, 1024)])
def test_fp64_blas_matches_reference_oracle(mnk):
    """The float64 product used above agrees with gemm_reference (bit-exact to
    the reference's _kernel_reference) to float64 rounding."""
    s = ProblemShape(*mnk)
    dA, dB, dC = _device_operands(s)
    blas = dA.double() @ dB.double()
    ref = gemm_reference(s, dA.double(), dB.double(), dC.double())
    assert _rf(blas, ref) <= 1e-13


def test_x3_deepbench_all_picks_full_size():
    """The fp32 space + tf32x3 (bench.py fp32_accurate_tc): the tree the
    reference pipeline trains on the merged po2 + random tables, its pick,
    the merged oracle and the default on every DeepBench shape, whole output
    vs the float64 product at the fp32 bar (1e-5) -- tf32x3 included."""
    import bench
    train, db = bench.load_x3_tables()
    pipe = bench._pipeline(train, "hybrid")
    sel = codegen.CompiledSelector(pipe["tree"], pipe["classes"])
    fams = set()
    worst = _check([t.shape for t in db], sel, {t.shape.mnk: t for t in db}, pipe["policy"], DeviceCaps.b200_tc(),
                   fams)
    print("deepbench + tf32x3 worst RF per family:", worst)
    assert (KernelFamily.TF32X3, 0) in fams
    assert worst["tf32x3"] <= 1e-5
