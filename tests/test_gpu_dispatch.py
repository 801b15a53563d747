"""Dispatch (compiled selector + GPU launch) and the full CLI pipeline on the GPU."""

import ctypes
import json

import numpy as np
import pytest

from conftest import rand_operands
from paper_1806_07060_b200 import codegen, evaluation
from paper_1806_07060_b200 import model as M
from paper_1806_07060_b200.dataset import dataset_from_tables, gen_po2
from paper_1806_07060_b200.kernels import DeviceCaps, KernelConfig, KernelFamily, ProblemShape, gemm_execute

pytestmark = pytest.mark.gpu

FIXTURE = [((64, 1, 1), 0), ((128, 1, 1), 0), ((256, 1, 1), 1), ((512, 1, 1), 1)]
SIDE = {0: KernelConfig(KernelFamily.DIRECT, 16, 16, 8, 2, 2, 1),
        1: KernelConfig(KernelFamily.INDIRECT, 32, 32, 16, 4, 4, 2)}


@pytest.fixture(scope="module")
def fixture_tree():
    return M.train(FIXTURE, M.TrainConfig(max_height=1))


def test_dispatch_bit_identical_to_direct_call(fixture_tree):
    s = ProblemShape(33, 20, 15, alpha=1.25, beta=0.5)
    A, B, C = rand_operands(s, seed=31)
    res = codegen.dispatch_and_run(fixture_tree, s, A, B, C, classes=SIDE)
    direct, _ = gemm_execute(s, res.selected, A, B, C)
    np.testing.assert_array_equal(res.output, direct)
    assert res.selected == SIDE[0] and not res.used_fallback and res.exec_seconds > 0


def test_dispatch_sources_and_selector(fixture_tree):
    s = ProblemShape(256, 8, 8)
    A, B, C = rand_operands(s, seed=37)
    for model in (codegen.emit_dispatcher(fixture_tree, SIDE, "python"),
                  codegen.CompiledSelector(fixture_tree, SIDE)):
        res = codegen.dispatch_and_run(model, s, A, B, C)
        assert res.selected == SIDE[M.predict(fixture_tree, s.mnk)]


def test_dispatch_fallback(fixture_tree):
    caps = DeviceCaps(register_tile_cap_indirect=2)
    s = ProblemShape(256, 8, 8)
    A, B, C = rand_operands(s, seed=41)
    res = codegen.dispatch_and_run(fixture_tree, s, A, B, C, caps=caps, classes=SIDE)
    assert res.used_fallback and res.selected.family is KernelFamily.DIRECT
    ref, _ = gemm_execute(s, res.selected, A, B, C, caps)
    np.testing.assert_array_equal(res.output, ref)
    sel = codegen.CompiledSelector(fixture_tree, SIDE)
    out, picked, fb = codegen.dispatch_native(sel, s, A, B, C, caps)
    assert fb and picked == codegen.FALLBACK_CONFIG
    np.testing.assert_array_equal(out, ref)


def test_dispatch_native_device_tensors(fixture_tree):
    import torch
    sel = codegen.CompiledSelector(fixture_tree, SIDE)
    s = ProblemShape(512, 300, 200, alpha=1.0, beta=0.5)
    A, B, C = rand_operands(s, seed=2)
    dA, dB, dC = (torch.from_numpy(x).cuda() for x in (A, B, C))
    out, picked, fb = codegen.dispatch_native(sel, s, dA, dB, dC)
    assert picked == SIDE[1] and not fb
    ref, _ = gemm_execute(s, picked, A, B, C)
    np.testing.assert_array_equal(out.cpu().numpy(), ref)


def test_overhead_below_one_percent(fake_table_factory):
    tables = [fake_table_factory(s) for s in gen_po2(64, 512)]
    ds = dataset_from_tables(tables, "po2")
    tree = M.train(ds.features_and_labels())
    samples = evaluation.overhead_bench(tree, [ProblemShape(1024, 1024, 1024)], 20, ds.class_index)
    s = samples[0]
    assert s.dispatch_ns < 1000 and s.overhead_fraction < 0.01


def _config(tmp, out, **over):
    shapes = tmp / "shapes.txt"
    shapes.write_text("8 8 8\n16 16 16\n24 24 24\n32 32 32\n")
    doc = {"out_dir": str(out), "timing": {"warmup": 0, "repeats": 1},
           "dataset": {"strategy": "workload", "path": str(shapes)},
           "split": {"fraction": 0.5, "seed": 7}, "grid": {"heights": [1, "max"], "min_leaf": [1]},
           "baseline": {"threshold": 16, "direct_anchor": [8, 8, 8], "indirect_anchor": [32, 32, 32]}}
    doc.update(over)
    p = tmp / "config.json"
    p.write_text(json.dumps(doc))
    return p


def test_cli_pipeline_on_gpu(tmp_path, capsys):
    from paper_1806_07060_b200.cli import main
    out = tmp_path / "run"
    cfg = _config(tmp_path, out)
    for stage in ("tune", "dataset", "train", "eval", "codegen", "bench"):
        assert main([stage, "--config", str(cfg)]) == 0, stage
    for name in ("dataset.csv", "split.json", "scores.csv", "best_model.json", "baseline.json",
                 "dispatcher.c", "dispatcher.py", "bench.csv", "bench.txt"):
        assert (out / name).exists(), name
    capsys.readouterr()
    assert main(["tune", "--config", str(cfg)]) == 0
    assert "4 already done, 0 to run" in capsys.readouterr().out
    assert main(["bench", "--config", str(cfg), "--live", "--subset", "all"]) == 0


def test_cli_tune_sharded_workers(tmp_path, capsys):
    from paper_1806_07060_b200.cli import main
    out = tmp_path / "par"
    cfg = _config(tmp_path, out, caps={"profile": "b200"})
    assert main(["tune", "--config", str(cfg), "--gpus", "2", "--share-gpus"]) == 0
    tables = sorted(p.name for p in (out / "tables").glob("*.csv"))
    assert tables == ["16x16x16.csv", "24x24x24.csv", "32x32x32.csv", "8x8x8.csv"]
    assert main(["tune", "--config", str(cfg), "--gpus", "2", "--share-gpus", "--force"]) == 0
    assert "0 already done, 4 to run" in capsys.readouterr().out


# ---------------------------------------------------------------------------
# pipelined host path (ag_gemm_host / ag_dispatch_gemm_host): host operands in,
# host result out; panels must not change a single bit


def _one_class_selector(cfg):
    tree = M.train([((64, 1, 1), 0), ((128, 1, 1), 0)])
    return codegen.CompiledSelector(tree, {0: cfg})


HOST_CASES = [
    # (M, N, K, alpha, beta, transA, transB, config)
    (700, 300, 129, 1.0, 0.0, False, False, "indirect:64-64-16-8-4-1"),    # row panels
    (300, 700, 129, 1.0, 0.0, False, False, "indirect:64-64-16-8-4-1"),    # column panels
    (517, 211, 77, 1.5, 0.5, True, False, "indirect:32-64-16-4-8-2"),     # transA, beta
    (211, 517, 77, 1.5, 0.5, False, True, "indirect:64-32-16-8-4-1"),     # transB, beta
    (333, 333, 64, 1.0, 0.0, True, True, "direct:32-32-16-2-4-1"),        # direct reads C always
    (1000, 64, 1024, 1.0, 0.0, False, False, "splitk:64-64-16-8-4-8"),    # split-K
    (600, 520, 300, 1.0, 0.25, False, False, "bf16:256-128-64-4-1-1"),    # tensor-core pair
    (260, 650, 96, 1.0, 0.0, False, True, "tf32:128-64-32-4-1-1"),
    (700, 300, 128, 1.0, 0.5, False, False, "tma:64-64-32-8-8-1"),        # TMA core, row panels
    (300, 700, 128, 1.0, 0.0, False, False, "tma:128-128-32-8-8-1"),      # TMA core, column panels
]


@pytest.mark.parametrize("case", HOST_CASES, ids=lambda c: f"{c[0]}x{c[1]}x{c[2]}-{c[7].split(':')[0]}")
@pytest.mark.parametrize("panels", [1, 3])
def test_host_path_equals_device_path(case, panels):
    import torch
    m, n, k, alpha, beta, ta, tb, name = case
    cfg = KernelConfig.from_canonical(name)
    caps = DeviceCaps.b200_tc()
    s = ProblemShape(m, n, k, alpha=alpha, beta=beta, transA=ta, transB=tb)
    A, B, C = rand_operands(s, seed=m + n + k)
    sel = _one_class_selector(cfg)
    dA, dB, dC = (torch.from_numpy(x).cuda() for x in (A, B, C))
    ref, picked, _ = codegen.dispatch_native(sel, s, dA, dB, dC, caps)
    ref = ref.cpu().numpy()
    got, picked_h, fb = codegen.dispatch_native(sel, s, A, B, C, caps, panels=panels)
    assert picked_h == picked == cfg and not fb
    assert isinstance(got, np.ndarray)
    np.testing.assert_array_equal(got, ref)
    # pinned torch tensors, result into a caller-owned pinned buffer
    pA, pB, pC = (torch.from_numpy(x).pin_memory() for x in (A, B, C))
    hout = torch.empty((m, n), dtype=torch.float32).pin_memory()
    got2, _, _ = codegen.dispatch_native(sel, s, pA, pB, pC, caps, out=hout, panels=panels)
    assert got2 is hout
    np.testing.assert_array_equal(hout.numpy(), ref)


def test_host_path_strided_operands_and_out():
    cfg = KernelConfig.from_canonical("indirect:64-64-16-8-4-1")
    s = ProblemShape(300, 200, 50, alpha=1.0, beta=1.0)
    A, B, C = rand_operands(s, seed=5)
    big = np.zeros((300, 260), np.float32)
    big[:, :50] = A  # row-major view with a leading dimension > K
    outbuf = np.zeros((200, 300), np.float32).T  # column-major out: written via a temporary
    sel = _one_class_selector(cfg)
    got, _, _ = codegen.dispatch_native(sel, s, big[:, :50], B, C, out=outbuf, panels=2)
    assert got is outbuf
    ref, _ = gemm_execute(s, cfg, A, B, C)
    np.testing.assert_array_equal(outbuf, ref)


def test_host_path_errors():
    from paper_1806_07060_b200.kernels import ShapeError
    cfg = KernelConfig.from_canonical("indirect:64-64-16-8-4-1")
    s = ProblemShape(30, 20, 10)
    A, B, C = rand_operands(s, seed=1)
    sel = _one_class_selector(cfg)
    with pytest.raises(ShapeError):
        codegen.dispatch_native(sel, s, A, B, C, out=np.zeros((20, 30), np.float32))
    with pytest.raises(ShapeError):
        codegen.dispatch_native(sel, s, A[:, :5], B, C)


def test_host_path_random_shapes_and_panels():
    """Seeded random shapes / transposes / beta / panel counts: the pipelined
    host path returns exactly the device path's bits."""
    import torch
    from paper_1806_07060_b200 import rng
    stream = rng.SplitMix64(0x405)
    names = ["indirect:64-64-16-8-4-1", "splitk:32-32-16-4-4-4", "tma:64-64-32-8-8-1", "direct:16-16-8-2-2-1",
             "indirect:128-128-32-8-8-1"]
    caps = DeviceCaps.b200_tc()
    for case in range(20):
        m, n, k = (1 + stream.below(700) for _ in range(3))
        s = ProblemShape(m, n, k, alpha=1.0, beta=(0.0, 0.5)[stream.below(2)],
                         transA=bool(stream.below(2)), transB=bool(stream.below(2)))
        cfg = KernelConfig.from_canonical(names[stream.below(len(names))])
        A, B, C = rand_operands(s, seed=case)
        sel = _one_class_selector(cfg)
        dA, dB, dC = (torch.from_numpy(x).cuda() for x in (A, B, C))
        ref, _, _ = codegen.dispatch_native(sel, s, dA, dB, dC, caps)
        got, _, _ = codegen.dispatch_native(sel, s, A, B, C, caps, panels=1 + stream.below(5))
        np.testing.assert_array_equal(got, ref.cpu().numpy(), err_msg=f"{s} {cfg.canonical()}")


def test_acceptance_c11_pipeline_on_gpu(tmp_path, capsys):
    """The reference's acceptance criterion 11 (test_acceptance.py:339-387)
    on the B200: the 27-shape po2(64, 256) pipeline from one config file,
    tune -> dataset -> train -> eval -> codegen -> bench, the model's train
    DTPR >= the baseline's, within the reference's 1800 s bound (the CPU
    reference took 862 s)."""
    import json
    import time

    from paper_1806_07060_b200 import evaluation
    from paper_1806_07060_b200.cli import main
    from paper_1806_07060_b200.dataset import load_dataset, split
    from paper_1806_07060_b200.model import load_tree
    from paper_1806_07060_b200.tuner import load_table, table_filename

    started = time.monotonic()
    out = tmp_path / "run"
    config = {
        "out_dir": str(out),
        "timing": {"warmup": 1, "repeats": 3},
        "dataset": {"strategy": "po2", "min": 64, "max": 256},
        "split": {"fraction": 0.8, "seed": 20817},
        "baseline": {"threshold": 384, "direct_anchor": [64, 64, 64], "indirect_anchor": [256, 256, 256]},
    }
    cfg_path = tmp_path / "smoke.json"
    cfg_path.write_text(json.dumps(config, indent=1))
    stage_s = {}
    for stage in ("tune", "dataset", "train", "eval", "codegen", "bench"):
        t0 = time.monotonic()
        assert main([stage, "--config", str(cfg_path)]) == 0, stage
        stage_s[stage] = round(time.monotonic() - t0, 2)
    ds = load_dataset(out / "dataset.csv", out / "dataset_classes.json")
    assert len(ds.records) == 27
    sp = split(ds, 0.8, seed=20817)
    records = ds.features_and_labels()
    train_records = [records[i] for i in sp.train]
    tables = evaluation.tables_by_shape([load_table(out / "tables" / table_filename(r.input)) for r in ds.records])
    best_name = json.loads((out / "best_model.json").read_text())["name"]
    best_tree = load_tree(out / "models" / f"{best_name}.json")
    base_doc = json.loads((out / "baseline.json").read_text())
    policy = evaluation.BaselinePolicy(
        default_indirect=KernelConfig.from_canonical(base_doc["default_indirect"]),
        default_direct=KernelConfig.from_canonical(base_doc["default_direct"]),
        threshold=base_doc["threshold"]).register(ds.class_index)
    model_dtpr = evaluation.dtpr(best_tree, train_records, tables, ds.class_index)
    base_preds = [evaluation.baseline_select(policy, ds.records[i].input) for i in sp.train]
    base_dtpr = evaluation.dtpr_from_predictions(base_preds, train_records, tables, ds.class_index)
    assert model_dtpr >= base_dtpr
    assert (out / "dispatcher.c").exists() and (out / "dispatcher.py").exists()
    elapsed = time.monotonic() - started
    with capsys.disabled():
        print(f"\n[acceptance C11 on B200] {elapsed:.1f} s (CPU reference 862 s); stages {stage_s}; "
              f"best={best_name} train-dtpr={model_dtpr:.4f} baseline-dtpr={base_dtpr:.4f}")
    assert elapsed < 1800.0


def test_numpy_fast_path_matches_and_orders_errors():
    """The compiled numpy path (csrc/fastpath.c -> ag_gemm_host_ex): same
    result as the device path, the reference's error order, out in place."""
    import torch

    from paper_1806_07060_b200.kernels import ConfigError, ShapeError, _fastpath
    assert _fastpath() is not None, "the _fastpath extension is not built"
    s = ProblemShape(300, 200, 150, alpha=1.5, beta=0.5)
    A, B, C = rand_operands(s, seed=61)
    cfg = KernelConfig.from_canonical("indirect:64-64-16-8-4-2")
    gemm_execute(s, cfg, A, B, C)  # first call: CUDA verified, fast path enabled
    out = np.empty((s.M, s.N), np.float32)
    got, sec = gemm_execute(s, cfg, A, B, C, DeviceCaps(), out)
    assert got is out and sec > 0
    dev, _ = gemm_execute(s, cfg, *(torch.from_numpy(x).cuda() for x in (A, B, C)))
    np.testing.assert_array_equal(out, dev.cpu().numpy())
    bad = np.ones((3, 3), np.float32)
    with pytest.raises(ConfigError):
        gemm_execute(s, KernelConfig(KernelFamily.DIRECT, 8, 8, 8, 1, 1, 2), bad, B, C)
    with pytest.raises(ShapeError, match="A has shape"):
        gemm_execute(s, cfg, bad, B, C)
    with pytest.raises(ShapeError, match="mixed dtypes"):
        gemm_execute(s, cfg, A, B, C.astype(np.float64))


def test_dispatch_and_run_numpy_overhead(capsys):
    """dispatch_and_run (codegen.py:285-325) with a DecisionTree and numpy
    operands: the compiled selector is built once per tree, the call is
    bit-identical to gemm_execute of the selected config, and the Python-side
    cost of the call (wall time minus the native host-path call) is small."""
    import time

    from paper_1806_07060_b200 import _native
    from paper_1806_07060_b200.kernels import native_shape
    s = ProblemShape(64, 64, 64)
    A, B, C = rand_operands(s, seed=62)
    tree = M.train([((64, 64, 64), 0), ((2048, 2048, 2048), 1)])
    classes = {0: KernelConfig(KernelFamily.DIRECT, 16, 16, 16, 1, 1, 1),
               1: KernelConfig(KernelFamily.INDIRECT, 64, 64, 16, 8, 4, 2)}
    r = codegen.dispatch_and_run(tree, s, A, B, C, DeviceCaps(), classes=classes)
    sel = tree.__dict__["_ag_selectors"][id(classes)][1]
    r2 = codegen.dispatch_and_run(tree, s, A, B, C, DeviceCaps(), classes=classes)
    assert tree.__dict__["_ag_selectors"][id(classes)][1] is sel  # cached
    ref, _ = gemm_execute(s, r.selected, A, B, C)
    np.testing.assert_array_equal(r.output, ref)
    np.testing.assert_array_equal(r2.output, ref)
    # Python-side overhead: the whole call vs the bare native host-path call
    lib = _native.lib()
    ns, nc, ncaps = native_shape(s), r.selected.native(), DeviceCaps().native()
    out = np.empty((64, 64), np.float32)
    secs = ctypes.c_double()

    def native():
        lib.ag_gemm_host_ex(ctypes.byref(ns), ctypes.byref(nc), ctypes.byref(ncaps), 0, A.ctypes.data, 64,
                            B.ctypes.data, 64, C.ctypes.data, 64, out.ctypes.data, 64, None, 0, 0, 1, None,
                            ctypes.byref(secs))

    def best(fn, n=200):
        ts = []
        for _ in range(n):
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
        ts.sort()
        return ts[n // 2]

    t_native = best(native)
    t_exec = best(lambda: gemm_execute(s, r.selected, A, B, C))
    t_disp = best(lambda: codegen.dispatch_and_run(tree, s, A, B, C, DeviceCaps(), classes=classes))
    with capsys.disabled():
        print(f"\n[numpy path 64^3] native host call {t_native * 1e6:.1f} us, gemm_execute "
              f"{t_exec * 1e6:.1f} us (+{(t_exec - t_native) * 1e6:.1f}), dispatch_and_run {t_disp * 1e6:.1f} us "
              f"(+{(t_disp - t_native) * 1e6:.1f})")
    assert t_exec - t_native < 20e-6


@pytest.mark.parametrize("mnk,name", [((3000, 700, 2048), "indirect:64-128-32-8-8-2"),   # row panels (8)
                                      ((700, 3000, 2048), "indirect:64-128-32-8-8-2"),   # column panels
                                      ((4096, 16, 4096), "skinny_n:64-16-32-2-4-4"),     # one big operand
                                      ((35, 8457, 2560), "skinny_m:40-256-32-1-2-16")])  # N % 4 != 0 rows
def test_staged_host_path_multi_panel_bit_exact(mnk, name):
    """Pageable numpy operands big enough for several output panels: the
    staged rings (AG_HOST_STAGE, 4 MB slots, the output draining on its own
    host thread) return exactly the device path's bits, through both the
    numpy fast path (gemm_execute) and dispatch_native, with a fresh output
    and with a caller-owned one."""
    import torch
    cfg = KernelConfig.from_canonical(name)
    s = ProblemShape(*mnk, alpha=1.0, beta=0.5)
    A, B, C = rand_operands(s, seed=sum(mnk))
    caps = DeviceCaps.b200()
    dA, dB, dC = (torch.from_numpy(x).cuda() for x in (A, B, C))
    ref, _ = gemm_execute(s, cfg, dA, dB, dC, caps)
    ref = ref.cpu().numpy()
    got, _ = gemm_execute(s, cfg, A, B, C, caps)
    np.testing.assert_array_equal(got, ref)
    out = np.full((s.M, s.N), np.nan, np.float32)
    got2, _ = gemm_execute(s, cfg, A, B, C, caps, out=out)
    assert got2 is out
    np.testing.assert_array_equal(out, ref)
    got3, picked, _ = codegen.dispatch_native(_one_class_selector(cfg), s, A, B, C, caps)
    assert picked == cfg
    np.testing.assert_array_equal(got3, ref)


def test_pinned_result_blocks_are_cached_and_exact():
    """A fresh result of >= 64 KB lives in a block of the library's caching
    pinned allocator (ag_host_alloc): a plain, writable numpy array with the
    device path's bits; dropping it returns the block to the cache and the
    next call of that size reuses it."""
    import gc

    import torch

    from paper_1806_07060_b200 import _native
    fp = pytest.importorskip("paper_1806_07060_b200._fastpath")
    cfg = KernelConfig.from_canonical("indirect:64-64-16-8-4-1")
    s = ProblemShape(1024, 1024, 64)
    A, B, C = rand_operands(s, seed=3)
    ref, _ = gemm_execute(s, cfg, *(torch.from_numpy(x).cuda() for x in (A, B, C)))
    out, _ = gemm_execute(s, cfg, A, B, C)
    assert isinstance(out, np.ndarray) and out.shape == (1024, 1024) and out.flags.writeable
    owner, chain = out, []
    while owner is not None:  # ndarray views -> frombuffer array -> (memoryview ->) PinnedBlock
        chain.append(type(owner).__name__)
        owner = getattr(owner, "base", None) if not isinstance(owner, memoryview) else owner.obj
    assert "PinnedBlock" in chain, chain
    np.testing.assert_array_equal(out, ref.cpu().numpy())
    out[0, 0] = 1.0  # an ordinary array for the caller
    before = fp.cache_bytes()
    del out
    gc.collect()
    assert fp.cache_bytes() >= before + 4 * 1024 * 1024
    again, _ = gemm_execute(s, cfg, A, B, C)
    assert fp.cache_bytes() == before
    np.testing.assert_array_equal(again, ref.cpu().numpy())
    assert _native.lib().ag_host_cache_bytes() == fp.cache_bytes()
    small, _ = gemm_execute(ProblemShape(64, 64, 64), cfg, *rand_operands(ProblemShape(64, 64, 64), seed=4))
    assert small.base is None  # under 64 KB: np.empty


def test_host_alloc_double_free_is_ignored():
    """ag_host_free on a block twice must not cache it twice (two later
    allocations would then share it); foreign pointers are ignored."""
    from paper_1806_07060_b200 import _native
    L = _native.lib()
    n = 3 << 20
    p = L.ag_host_alloc(n)
    assert p
    L.ag_host_free(p)
    L.ag_host_free(p)
    L.ag_host_free(12345)  # not a block of the cache
    a, b = L.ag_host_alloc(n), L.ag_host_alloc(n)
    assert a and b and a != b
    L.ag_host_free(a)
    L.ag_host_free(b)


def test_staged_host_path_concurrent_callers():
    """Two host threads in the staged numpy path at once (the fast path
    releases the GIL): per-thread pipes and rings, the shared copy pool and
    the pinned result cache; every result equals its device-path bits."""
    import threading

    import torch
    cfg = KernelConfig.from_canonical("indirect:64-64-32-8-8-1")
    shapes = [ProblemShape(1500, 900, 700), ProblemShape(900, 1500, 600, beta=0.5)]
    data = [rand_operands(s, seed=i + 7) for i, s in enumerate(shapes)]
    caps = DeviceCaps.b200()
    refs = [gemm_execute(s, cfg, *(torch.from_numpy(x).cuda() for x in d), caps)[0].cpu().numpy()
            for s, d in zip(shapes, data)]
    errors = []

    def work(i):
        try:
            for _ in range(6):
                out, _ = gemm_execute(shapes[i], cfg, *data[i], caps)
                if not np.array_equal(out, refs[i]):
                    errors.append(f"thread {i}: mismatch")
        except Exception as exc:  # noqa: BLE001
            errors.append(f"thread {i}: {exc!r}")

    ts = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors, errors
