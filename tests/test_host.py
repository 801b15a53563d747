"""Product host logic vs the reference's own outputs (CPU only).

Search space, legality, rng, shape generators, splits, sampling picks,
native CART (bit-exact trees via sha256 fingerprints), compiled selector,
emitted dispatcher sources, evaluation metrics, persistence formats and
the CLI's deterministic stages -- all compared with tests/golden/, which
tests/golden/make_golden.py produced by running the reference.
"""

import json
import math
import shutil

import numpy as np
import pytest

from conftest import GOLDEN, ROOT, golden
from oracle import cart as ocart
from paper_1806_07060_b200 import codegen, evaluation, rng, sharding
from paper_1806_07060_b200 import model as M
from paper_1806_07060_b200.dataset import (
    ClassIndex,
    Dataset,
    DatasetRecord,
    WorkloadParseError,
    dataset_from_tables,
    dedup_shapes,
    gen_go2,
    gen_po2,
    load_dataset,
    load_workload_shapes,
    save_dataset,
    split,
)
from paper_1806_07060_b200.kernels import (
    ConfigError,
    DeviceCaps,
    KernelConfig,
    KernelFamily,
    ProblemShape,
    ShapeError,
    enumerate_search_space,
    full_search_space,
    is_legal,
)
from paper_1806_07060_b200.tuner import (
    Measurement,
    TableLookupError,
    TimingPolicy,
    TuningTable,
    flops_of,
    load_table,
    random_configs,
    save_table,
    table_filename,
)

# ---------------------------------------------------------------------------
# kernels: types, legality, space


def test_shape_validation():
    with pytest.raises(ShapeError):
        ProblemShape(0, 1, 1)
    with pytest.raises(ShapeError):
        ProblemShape(4, -2, 4)
    with pytest.raises(ShapeError):
        ProblemShape(True, 1, 1)
    assert ProblemShape(1, 1, 1).mnk == (1, 1, 1)


def test_search_space_equals_reference(default_caps):
    assert [c.canonical() for c in full_search_space(default_caps)] == golden()["space"]
    assert len(enumerate_search_space(KernelFamily.DIRECT, default_caps)) == 144
    assert len(enumerate_search_space(KernelFamily.INDIRECT, default_caps)) == 432
    relaxed = DeviceCaps(register_tile_cap_direct=16)
    assert len(enumerate_search_space(KernelFamily.DIRECT, relaxed)) == golden()["space_relaxed_direct_count"] == 162
    tight = DeviceCaps(tile_memory_cap=8192)
    assert [c.canonical() for c in enumerate_search_space(KernelFamily.INDIRECT, tight)] == \
        golden()["space_tight_indirect"]


def test_is_legal_spec_cases(default_caps):
    assert not is_legal(KernelConfig(KernelFamily.DIRECT, 16, 16, 8, 4, 4, 1), default_caps)
    assert is_legal(KernelConfig(KernelFamily.DIRECT, 16, 16, 8, 2, 2, 1), default_caps)
    assert not is_legal(KernelConfig(KernelFamily.DIRECT, 16, 16, 8, 2, 2, 2), default_caps)
    assert not is_legal(KernelConfig(KernelFamily.INDIRECT, 16, 16, 8, 3, 2, 1), default_caps)
    tight = DeviceCaps(tile_memory_cap=(64 + 64) * 32 * 4 - 1)
    assert not is_legal(KernelConfig(KernelFamily.INDIRECT, 64, 64, 32, 4, 4, 2), tight)


def test_b200_profile_extends_reference_space():
    ref = full_search_space()
    b200 = full_search_space(DeviceCaps.b200())
    assert {c.canonical() for c in ref} <= {c.canonical() for c in b200}
    assert len(b200) > len(ref)
    assert all(is_legal(c, DeviceCaps.b200()) for c in b200)
    assert any(c.block_m == 128 and c.block_n == 128 for c in b200)
    # reference-profile enumeration unaffected by the B200 extras
    assert len(enumerate_search_space(KernelFamily.INDIRECT, DeviceCaps())) == 432


def test_canonical_round_trip(search_space):
    for c in search_space[::37]:
        assert KernelConfig.from_canonical(c.canonical()) == c
    with pytest.raises(ConfigError):
        KernelConfig.from_canonical("nope")
    with pytest.raises(ConfigError):
        KernelConfig.from_canonical("bogus:1-2-3-4-5-6")


def test_caps_validation():
    with pytest.raises(ConfigError):
        DeviceCaps(tile_memory_cap=0)
    with pytest.raises(ConfigError):
        DeviceCaps(profile="mystery")


# ---------------------------------------------------------------------------
# rng, shapes, splits, sampling


def test_rng_streams_match_reference():
    g = golden()
    for seed, want in g["splitmix"].items():
        st = rng.SplitMix64(int(seed))
        assert [st.next_u64() for _ in range(8)] == want["u64"]
        assert [st.below(b) for b in (1, 2, 3, 7, 96, 1000, 2**63 + 5, 8192)] == want["below"]
    assert rng.mix(0, 256, 256, 256) == g["mix"]["0,256,256,256"]
    assert rng.mix(7) == g["mix"]["7"]
    assert rng.mix(1, 2, 3, 4, 5) == g["mix"]["1,2,3,4,5"]
    assert rng.mix(-1) == g["mix"]["-1"]
    for key, want in g["shuffled"].items():
        n, s = map(int, key.split(","))
        assert rng.shuffled(n, s) == want
    for key, want in g["sample"].items():
        n, k, s = map(int, key.split(","))
        assert rng.sample_without_replacement(n, k, s) == want
    with pytest.raises(ValueError):
        rng.SplitMix64(1).below(0)
    with pytest.raises(ValueError):
        rng.sample_without_replacement(3, 4, 0)


def test_shape_generators_match_reference():
    g = golden()
    assert [s.mnk for s in gen_po2(64, 2048)] == [tuple(x) for x in g["po2_64_2048"]]
    go2 = gen_go2(256, 3840, 256)
    assert len(go2) == g["go2_count"] == 3375
    assert [s.mnk for s in go2[:40]] == [tuple(x) for x in g["go2_head"]]
    assert len(gen_po2(64, 4096)) == 343
    assert [s.mnk for s in gen_po2(64, 64)] == [(64, 64, 64)]
    assert len(gen_go2(100, 300, 100)) == 27
    for bad in ((60, 2048), (64, 96), (128, 64)):
        with pytest.raises(ValueError):
            gen_po2(*bad)
    with pytest.raises(ValueError):
        gen_go2(300, 100, 100)


def test_splits_match_reference():
    cfg = KernelConfig(KernelFamily.DIRECT, 8, 8, 8, 1, 1, 1)
    for key, (train, test) in golden()["splits"].items():
        n, seed, frac = key.split(",")
        n, seed, frac = int(n), int(seed), float(frac)
        idx = ClassIndex()
        idx.ensure(cfg)
        ds = Dataset([DatasetRecord(ProblemShape(i + 1, 1, 1), cfg, 1.0) for i in range(n)], idx, "workload")
        sp = split(ds, frac, seed)
        assert list(sp.train) == train and list(sp.test) == test
        assert len(sp.train) == int(frac * n)


def test_tune_random_picks_match_reference(default_caps):
    space_size = len(full_search_space(default_caps))
    for key, want in golden()["tune_random"].items():
        n, seed = map(int, key.split(","))
        if n >= space_size:
            continue
        assert [c.canonical() for c in random_configs(default_caps, n, seed)] == want
    picks = random_configs(default_caps, 10, 42)
    assert sum(1 for c in picks if c.family is KernelFamily.DIRECT) == 3


def test_workload_files(tmp_path):
    p = tmp_path / "w.txt"
    p.write_text("# header\n128 1000 1\n128,1000,1\n64 64 64  # trailing\n\n")
    assert [s.mnk for s in load_workload_shapes(p)] == [(128, 1000, 1), (64, 64, 64)]
    p.write_text("1 2 3\n4 5\n")
    with pytest.raises(WorkloadParseError, match=":2"):
        load_workload_shapes(p)
    p.write_text("1 0 3\n")
    with pytest.raises(WorkloadParseError):
        load_workload_shapes(p)
    p.write_text("# nothing\n")
    with pytest.warns(RuntimeWarning):
        assert load_workload_shapes(p) == []
    shapes = [ProblemShape(2, 2, 2), ProblemShape(1, 1, 1), ProblemShape(2, 2, 2)]
    assert [s.mnk for s in dedup_shapes(shapes)] == [(2, 2, 2), (1, 1, 1)]


def test_deepbench_workload_file_parses():
    from paper_1806_07060_b200 import workloads
    shapes = load_workload_shapes(workloads.DEEPBENCH_PATH)
    mnks = {s.mnk for s in shapes}
    assert (5124, 700, 2048) in mnks and (35, 8457, 2560) in mnks
    assert len(shapes) >= 20


# ---------------------------------------------------------------------------
# tables, datasets, persistence


def test_table_argmax_and_ties():
    s = ProblemShape(4, 4, 4)
    a = KernelConfig(KernelFamily.DIRECT, 8, 8, 8, 1, 1, 1)
    b = KernelConfig(KernelFamily.INDIRECT, 16, 16, 8, 2, 2, 1)
    c = KernelConfig(KernelFamily.DIRECT, 16, 16, 8, 2, 2, 1)
    t = TuningTable.from_measurements(s, [Measurement(a, 1e-3, 2.0), Measurement(b, 1e-3, 2.0),
                                          Measurement(c, 1e-3, 1.0)])
    assert t.best_overall == 0 and t.best_direct == 0 and t.best_indirect == 1
    assert t.gflops_for(c) == 1.0
    with pytest.raises(TableLookupError):
        t.gflops_for(KernelConfig(KernelFamily.DIRECT, 32, 32, 16, 4, 2, 1))
    only = TuningTable.from_measurements(s, [Measurement(a, 1e-3, 2.0)])
    with pytest.raises(TableLookupError):
        only.best_for_family(KernelFamily.INDIRECT)
    with pytest.raises(ValueError):
        Measurement(a, 0.0, 1.0)
    with pytest.raises(ValueError):
        TimingPolicy(warmup=-1)


def test_flops_of():
    assert flops_of(ProblemShape(1024, 1024, 1024)) == 2147483648
    assert flops_of(ProblemShape(2, 3, 4)) == 48


def test_table_csv_round_trip_and_reference_tables(tmp_path, fake_table_factory):
    t = fake_table_factory(ProblemShape(9, 8, 7))
    path = tmp_path / table_filename(t.shape)
    assert path.name == "9x8x7.csv"
    save_table(t, path, {"config_hash": "abc123"})
    back = load_table(path)
    assert [(m.config, m.elapsed, m.gflops) for m in back.measurements] == \
        [(m.config, m.elapsed, m.gflops) for m in t.measurements]
    assert back.meta["config_hash"] == "abc123"
    # tables written by the reference CLI load unchanged
    for p in sorted((GOLDEN / "cli" / "run" / "tables").glob("*.csv")):
        ref = load_table(p)
        assert len(ref.measurements) in (144, 432, 576)
        assert table_filename(ref.shape) == p.name
    bad = tmp_path / "bad.csv"
    bad.write_text("this,is,not\na,table,file\n")
    with pytest.raises(ValueError):
        load_table(bad)


def test_dataset_labels_and_round_trip(tmp_path, fake_table_factory):
    shapes = gen_po2(64, 256)
    tables = [fake_table_factory(s) for s in shapes]
    ds = dataset_from_tables(tables, "po2")
    for rec, table in zip(ds.records, tables):
        assert rec.label == table.best_config and rec.peak_gflops == table.peak_gflops
    save_dataset(ds, tmp_path / "d.csv", tmp_path / "c.json", {"config_hash": "deadbeef"})
    back = load_dataset(tmp_path / "d.csv", tmp_path / "c.json")
    assert back.features_and_labels() == ds.features_and_labels()
    with pytest.raises(ValueError):
        dataset_from_tables([tables[0], tables[0]], "po2")
    with pytest.raises(ValueError):
        dataset_from_tables(tables, "mystery")


def test_class_index_dense_first_appearance():
    idx = ClassIndex()
    a = KernelConfig(KernelFamily.DIRECT, 8, 8, 8, 1, 1, 1)
    b = KernelConfig(KernelFamily.INDIRECT, 16, 16, 8, 2, 2, 1)
    assert (idx.ensure(a), idx.ensure(b), idx.ensure(a)) == (0, 1, 0)
    assert idx.config_of(1) == b and idx.family_of(1) is KernelFamily.INDIRECT and len(idx) == 2


# ---------------------------------------------------------------------------
# CART (native, exact) vs the reference's trees


def _hl(name):
    h_txt, l_txt = name[1:].split("-L")
    return (None if h_txt == "Max" else int(h_txt)), (float(l_txt) if "." in l_txt else int(l_txt))


def test_gini_and_majority():
    assert M.gini(["A"] * 4) == 0.0 and M.gini(["A", "A", "B", "B"]) == 0.5
    assert M.gini(["A", "A", "A", "B"]) == 0.375
    with pytest.raises(ValueError):
        M.gini([])
    assert M.predict(M.train([((5, 5, 5), 2), ((5, 5, 5), 1)]), (5, 5, 5)) == 1


def test_best_split_matches_reference():
    g = golden()["cart"]
    fixture = [((64, 1, 1), 0), ((128, 1, 1), 0), ((256, 1, 1), 1), ((512, 1, 1), 1)]
    assert list(M.best_split(fixture, 1)) == g["best_split_fixture"]
    for case in g["best_split_cases"]:
        got = M.best_split([(tuple(f), lab) for f, lab in case["samples"]], case["min_leaf"])
        want = case["result"]
        assert (got is None) == (want is None)
        if want is not None:
            assert (got[0], got[1]) == (want[0], want[1])
            assert got[2] == want[2]


@pytest.mark.parametrize("world", ["po2_64_256", "po2_64_512", "po2_64_2048"])
def test_grid_trees_bit_exact(world):
    g = golden()["cart"]["grids"][world]
    lo, hi = 64, int(world.split("_")[-1])
    recs = list(zip([s.mnk for s in gen_po2(lo, hi)], g["labels"]))
    named = M.grid_train(recs)
    assert [n for n, _ in named] == list(g["trees"])
    for name, tree in named:
        want = g["trees"][name]
        assert codegen.tree_fingerprint(tree) == want["fingerprint"], name
        assert tree.height() == want["height"] and len(tree.leaves()) == want["leaves"]


def test_random_and_comb_trees_bit_exact():
    for case in golden()["cart"]["random_trees"]:
        recs = [(tuple(f), lab) for f, lab in case["records"]]
        t = M.train(recs, M.TrainConfig(case["max_height"], case["min_leaf"]))
        assert codegen.tree_fingerprint(t) == case["fingerprint"]


def test_go2_scale_trees_bit_exact():
    g = golden()["cart"]["go2_trees"]
    recs = list(zip([s.mnk for s in gen_go2(256, 3840, 256)], g["labels"]))
    for name, want in g["trees"].items():
        h, L = _hl(name)
        t = M.train(recs, M.TrainConfig(h, L))
        assert codegen.tree_fingerprint(t) == want["fingerprint"], name


def test_native_cart_matches_oracle_on_fresh_cases():
    # beyond the fixtures: the native trainer vs the pure-Python oracle
    import sys
    sys.setrecursionlimit(20000)
    stream = rng.SplitMix64(31337)
    for _ in range(25):
        n = 2 + stream.below(400)
        span = 1 + stream.below(1 << (1 + stream.below(20)))
        recs = [((1 + stream.below(span), 1 + stream.below(span), 1 + stream.below(span)),
                 stream.below(1 + stream.below(30))) for _ in range(n)]
        h = (1, 3, 8, None)[stream.below(4)]
        L = (1, 2, 5, 0.05, 0.25)[stream.below(5)]
        t = M.train(recs, M.TrainConfig(h, L))
        assert t.to_dict()["nodes"] == ocart.grow(recs, h, L)


def test_train_config_semantics():
    assert M.TrainConfig(min_samples_leaf=0.25).effective_min_leaf(10) == 3
    assert M.TrainConfig(min_samples_leaf=0.5).effective_min_leaf(3) == 2
    assert M.TrainConfig(min_samples_leaf=0.3).effective_min_leaf(3) == 1
    for bad in (dict(max_height=0), dict(min_samples_leaf=0), dict(min_samples_leaf=0.75)):
        with pytest.raises(ValueError):
            M.TrainConfig(**bad)
    with pytest.raises(ValueError):
        M.train([])


def test_tree_json_round_trip(tmp_path):
    fixture = [((64, 1, 1), 0), ((128, 1, 1), 0), ((256, 1, 1), 1), ((512, 1, 1), 1)]
    t = M.train(fixture, M.TrainConfig(max_height=2))
    M.save_tree(t, tmp_path / "t.json")
    assert M.load_tree(tmp_path / "t.json").to_dict() == t.to_dict()
    with pytest.raises(ValueError):
        M.DecisionTree.from_dict({"format_version": 99, "nodes": []})


# ---------------------------------------------------------------------------
# dispatch: emitted sources, probes, compiled selector


def _classes(doc):
    return ClassIndex_from(golden()["cart"]["grids"]["po2_64_512"]["classes"])


def ClassIndex_from(canon):
    idx = ClassIndex()
    for c in canon:
        idx.ensure(KernelConfig.from_canonical(c))
    return idx


@pytest.mark.parametrize("name", ["h1-L1", "h4-L1", "hMax-L1", "h8-L0.1", "hMax-L0.5"])
def test_emitted_sources_byte_identical(name):
    doc = golden()["cart"]["full_trees"][name]
    tree = M.DecisionTree.from_dict(doc["tree"])
    classes = _classes(doc)
    assert codegen.emit_dispatcher(tree, classes, "c", "golden").text == doc["c_source"]
    assert codegen.emit_dispatcher(tree, classes, "python", "golden").text == doc["py_source"]
    assert [list(p) for p in codegen.boundary_probes(tree)] == doc["probes"]
    for p, cid in doc["predictions"]:
        assert M.predict(tree, p) == cid


@pytest.mark.parametrize("kind", ["auto", "table", "walk"])
@pytest.mark.parametrize("name", ["h1-L1", "h4-L1", "hMax-L1", "h8-L0.1", "hMax-L0.5"])
def test_compiled_selector_matches_predict(name, kind):
    doc = golden()["cart"]["full_trees"][name]
    tree = M.DecisionTree.from_dict(doc["tree"])
    sel = codegen.CompiledSelector(tree, _classes(doc), kind=kind)
    assert sel.tree_fingerprint == codegen.tree_fingerprint(tree)
    assert codegen.roundtrip_check(tree, sel, [tuple(p) for p, _ in doc["predictions"]])
    pts = [tuple(p) for p, _ in doc["predictions"]]
    assert sel.select_many(pts) == [cid for _, cid in doc["predictions"]]
    stream = rng.SplitMix64(5)
    for _ in range(500):
        p = (1 + stream.below(5000), 1 + stream.below(5000), 1 + stream.below(5000))
        assert sel.select_id(*p) == M.predict(tree, p)


def test_random_feasible_trees_selector_and_sources(search_space):
    for case in golden()["cart"]["random_feasible_trees"]:
        tree = M.DecisionTree.from_dict(case["tree"])
        classes = {int(k): KernelConfig.from_canonical(v) for k, v in case["classes"].items()}
        assert [list(p) for p in codegen.boundary_probes(tree)] == case["probes"]
        import hashlib
        assert hashlib.sha256(codegen.emit_dispatcher(tree, classes, "c").text.encode()).hexdigest() == case["c_sha"]
        for kind in ("table", "walk"):
            try:
                sel = codegen.CompiledSelector(tree, classes, kind=kind)
            except codegen.CodegenError:
                assert kind == "table"  # grid too large for a table: the walk covers it
                continue
            assert codegen.roundtrip_check(tree, sel, [(1, 1, 1), (4096, 4096, 4096)])
            mutant = M.DecisionTree.from_dict(tree.to_dict())
            internal = [i for i, n in enumerate(mutant.nodes) if isinstance(n, M.SplitNode)]
            if internal:
                mutant.nodes[internal[0]].threshold += 1.0
                msel = codegen.CompiledSelector(mutant, classes, kind="walk")
                assert not codegen.roundtrip_check(tree, msel, [])


def test_c_source_compiles_and_matches():
    if shutil.which("cc") is None:
        pytest.skip("no C compiler")
    doc = golden()["cart"]["full_trees"]["hMax-L1"]
    tree = M.DecisionTree.from_dict(doc["tree"])
    src = codegen.emit_dispatcher(tree, _classes(doc), "c")
    assert codegen.roundtrip_check(tree, src, [(64, 64, 64), (512, 64, 128)])


def test_selector_dispatch_overhead_sub_microsecond():
    doc = golden()["cart"]["full_trees"]["hMax-L1"]
    tree = M.DecisionTree.from_dict(doc["tree"])
    for kind in ("table", "walk"):
        sel = codegen.CompiledSelector(tree, _classes(doc), kind=kind)
        assert sel.bench_ns(1024, 1024, 1024, 200000) < 1000.0


# ---------------------------------------------------------------------------
# evaluation


def test_evaluation_matches_reference(fake_table_factory):
    g = golden()["cart"]["evaluation"]
    shapes = gen_po2(64, 256)
    tables = [fake_table_factory(s) for s in shapes]
    ds = dataset_from_tables(tables, "po2")
    records = ds.features_and_labels()
    tbs = evaluation.tables_by_shape(tables)
    tree = M.train(records, M.TrainConfig(max_height=4, min_samples_leaf=1))
    assert codegen.tree_fingerprint(tree) == g["tree"]["fingerprint"]
    pol = evaluation.BaselinePolicy(KernelConfig(KernelFamily.INDIRECT, 32, 32, 16, 4, 4, 1),
                                    KernelConfig(KernelFamily.DIRECT, 16, 16, 8, 2, 2, 1), threshold=128)
    pol.register(ds.class_index)
    assert evaluation.accuracy(tree, records) == g["accuracy"]
    assert evaluation.dtpr(tree, records, tbs, ds.class_index) == g["dtpr"]
    assert evaluation.dttr(tree, records, tbs, ds.class_index, pol) == g["dttr"]
    assert [evaluation.baseline_select(pol, r.input) for r in ds.records] == g["baseline_select"]
    scores = evaluation.score_models(M.grid_train(records), records, tbs, ds.class_index, pol)
    assert [[s.name, s.accuracy, s.dtpr, s.dttr, s.stats.total_leaves, s.stats.height] for s in scores] == g["scores"]
    assert evaluation.select_best_model(scores).name == g["best"]
    preds = [cid for _, cid in records]
    assert evaluation.dtpr_from_predictions(preds, records, tbs, ds.class_index) == 1.0


def test_baseline_policy_cut_cases():
    d = KernelConfig(KernelFamily.DIRECT, 16, 16, 8, 2, 2, 1)
    i = KernelConfig(KernelFamily.INDIRECT, 32, 32, 16, 4, 4, 1)
    pol = evaluation.BaselinePolicy(i, d, threshold=384).register(ClassIndex())
    assert evaluation.baseline_select(pol, ProblemShape(64, 64, 64)) == pol.direct_class_id
    assert evaluation.baseline_select(pol, ProblemShape(1024, 1024, 1024)) == pol.indirect_class_id
    assert evaluation.baseline_select(pol, ProblemShape(2048, 64, 64)) == pol.direct_class_id
    assert evaluation.baseline_select(pol, ProblemShape(384, 384, 384)) == pol.indirect_class_id
    with pytest.raises(ValueError):
        evaluation.BaselinePolicy(d, d)
    assert evaluation.geomean([1.0, 4.0]) == pytest.approx(2.0)


# ---------------------------------------------------------------------------
# CLI stages vs the reference's artifacts


def test_cli_stages_reproduce_reference_artifacts(tmp_path, monkeypatch):
    from paper_1806_07060_b200.cli import PipelineConfig, main
    src = GOLDEN / "cli"
    work = tmp_path / "w"
    shutil.copytree(src, work)
    monkeypatch.chdir(work)
    ref_out = src / "run"
    run = work / "run"
    for name in ("dataset.csv", "dataset_classes.json", "split.json", "scores.csv", "best_model.json",
                 "dispatcher.c", "dispatcher.py"):
        (run / name).unlink()
    shutil.rmtree(run / "models")
    # same config -> same hash as the reference CLI
    cfg = PipelineConfig.load("config.json")
    assert f"config_hash={cfg.hash()}" in (ref_out / "dataset.csv").read_text().splitlines()[0]
    for stage in ("dataset", "train", "eval", "codegen"):
        assert main([stage, "--config", "config.json"]) == 0, stage
    for name in ("dataset.csv", "dataset_classes.json", "split.json", "scores.csv", "best_model.json",
                 "dispatcher.c", "dispatcher.py"):
        assert (run / name).read_bytes() == (ref_out / name).read_bytes(), name
    for p in (ref_out / "models").glob("*.json"):
        assert (run / "models" / p.name).read_bytes() == p.read_bytes(), p.name


def test_cli_errors(tmp_path, capsys):
    from paper_1806_07060_b200.cli import PipelineConfig, main
    assert main(["tune"]) == 1
    assert main(["frobnicate", "--config", "x.json"]) == 1
    assert main(["tune", "--config", str(tmp_path / "absent.json")]) == 2
    cfg = tmp_path / "c.json"
    cfg.write_text(json.dumps({"out_dir": str(tmp_path / "o"),
                               "dataset": {"strategy": "workload", "path": str(tmp_path / "s.txt")}}))
    (tmp_path / "s.txt").write_text("8 8 8\n")
    assert main(["dataset", "--config", str(cfg)]) == 2
    assert "missing tuning tables" in capsys.readouterr().err


def test_cli_env_caps_override(tmp_path, monkeypatch):
    from paper_1806_07060_b200.cli import PipelineConfig
    cfg = tmp_path / "c.json"
    cfg.write_text(json.dumps({"dataset": {"strategy": "po2", "min": 64, "max": 64}}))
    monkeypatch.setenv("ADAPTGEMM_REGISTER_TILE_CAP_DIRECT", "16")
    assert PipelineConfig.load(cfg).caps.register_tile_cap_direct == 16
    monkeypatch.delenv("ADAPTGEMM_REGISTER_TILE_CAP_DIRECT")
    b = tmp_path / "b.json"
    b.write_text(json.dumps({"caps": {"profile": "b200"}, "dataset": {"strategy": "po2", "min": 64, "max": 64}}))
    pc = PipelineConfig.load(b)
    assert pc.caps.profile == "b200" and pc.caps.register_tile_cap_indirect == 128
    assert pc.hash() != PipelineConfig.load(cfg).hash()


# ---------------------------------------------------------------------------
# sharding


def test_lpt_partition_properties():
    shapes = [s.mnk for s in gen_po2(64, 4096)]
    for n in (1, 2, 4, 8):
        parts = sharding.lpt_partition(shapes, n, lambda t: sharding.sweep_cost(t, 576))
        flat = [x for p in parts for x in p]
        assert sorted(flat) == sorted(shapes) and len(flat) == len(set(flat))
        loads = [sum(sharding.sweep_cost(t, 576) for t in p) for p in parts]
        biggest = max(sharding.sweep_cost(t, 576) for t in shapes)
        assert max(loads) - min(loads) <= biggest + 1e-9
    assert sharding.lpt_partition(shapes, 3, lambda t: 1.0) == sharding.lpt_partition(shapes, 3, lambda t: 1.0)


def test_gen_random_shapes_deterministic_and_in_range():
    from paper_1806_07060_b200.dataset import gen_random
    a = gen_random(64, 1, 8192, 1806)
    b = gen_random(64, 1, 8192, 1806)
    assert [s.mnk for s in a] == [s.mnk for s in b]
    assert len({s.mnk for s in a}) == 64
    assert all(1 <= d <= 8192 for s in a for d in s.mnk)
    assert [s.mnk for s in gen_random(64, 1, 8192, 7)] != [s.mnk for s in a]
    # first draws: M, N, K in order from one SplitMix64 stream
    g = rng.SplitMix64(1806)
    assert a[0].mnk == tuple(1 + g.below(8192) for _ in range(3))
    with pytest.raises(ValueError):
        gen_random(9, 1, 2, 0)


def test_gen_random_log2_octave_uniform():
    from paper_1806_07060_b200.dataset import gen_random
    a = gen_random(512, 16, 4096, 2026, "log2")
    assert [s.mnk for s in a] == [s.mnk for s in gen_random(512, 16, 4096, 2026, "log2")]
    assert len({s.mnk for s in a}) == 512
    assert all(16 <= d < 4096 for s in a for d in s.mnk)
    # first draw: an octave index, then an offset inside the octave
    g = rng.SplitMix64(2026)
    first = []
    for _ in range(3):
        base = 16 << g.below(8)
        first.append(base + g.below(base))
    assert a[0].mnk == tuple(first)
    # every octave of [16, 4096) is populated in every dimension
    for dim in range(3):
        assert {s.mnk[dim].bit_length() for s in a} == set(range(5, 13))
    with pytest.raises(ValueError):
        gen_random(8, 16, 1000, 0, "log2")
    with pytest.raises(ValueError):
        gen_random(8, 16, 1024, 0, "gauss")
    # the sweep config that produced tables_b200_lograndom.csv.gz
    from paper_1806_07060_b200 import cli
    cfg = cli.PipelineConfig.load(ROOT / "configs" / "lograndom_b200.json")
    shapes, tag = cfg.shapes()
    assert tag == "random" and [s.mnk for s in shapes] == [s.mnk for s in a]


def test_sampling_list_configs_and_tc_config_file():
    from paper_1806_07060_b200 import cli
    from paper_1806_07060_b200.kernels import KernelFamily, enumerate_search_space
    cfg = cli.PipelineConfig.load(ROOT / "configs" / "random_tc_b200.json")
    assert cfg.caps.profile == "b200tc"
    shapes, tag = cfg.shapes()
    assert tag == "random" and len(shapes) == 256
    picked = cli.sampling_configs(cfg.sampling, cfg.caps)
    tc = enumerate_search_space(KernelFamily.TF32, cfg.caps) + enumerate_search_space(KernelFamily.BF16, cfg.caps)
    assert picked[:len(tc)] == tc
    assert len(picked) == len(set(picked))
    assert all(c.family not in (KernelFamily.TF32, KernelFamily.BF16) for c in picked[len(tc):])


def test_merge_tables_keeps_base_and_order():
    from paper_1806_07060_b200.kernels import KernelConfig, ProblemShape
    from paper_1806_07060_b200.tuner import Measurement, TuningTable, merge_tables
    s = ProblemShape(64, 64, 64)
    c1, c2, c3 = (KernelConfig.from_canonical(x) for x in
                  ("direct:8-8-8-1-1-1", "bf16:128-64-64-2-1-1", "bf16:256-128-64-2-1-1"))
    meta = {"warmup": "1", "repeats": "3", "timer": "cuda-events"}
    a = TuningTable.from_measurements(s, [Measurement(c1, 1.0, 1.0), Measurement(c2, 0.5, 2.0)], meta)
    b = TuningTable.from_measurements(s, [Measurement(c3, 0.25, 4.0), Measurement(c2, 0.1, 9.0)], meta)
    m = merge_tables(a, b, order=[c2, c3, c1])
    assert [x.config for x in m.measurements] == [c2, c3, c1]
    assert m.find(c2).gflops == 2.0 and m.best_config == c3
    with pytest.raises(ValueError):
        merge_tables(a, TuningTable.from_measurements(s, [Measurement(c3, 1.0, 1.0)], dict(meta, repeats="5")))


def test_shipped_b200_models_match_reference():
    """The models bench.py trains on the shipped B200 tables equal the
    reference's own CART on the same records: split indices, all 40 grid
    fingerprints and every model's predictions on the DeepBench shapes
    (tests/golden/make_b200_golden.py ran the reference itself)."""
    import json

    import bench
    from paper_1806_07060_b200 import codegen, model
    from paper_1806_07060_b200.dataset import dataset_from_tables, split
    from paper_1806_07060_b200.tuner import load_table_bundle
    path = GOLDEN / "b200_trees.json"
    doc = json.loads(path.read_text())
    po2 = load_table_bundle(bench.PO2_BUNDLE)
    db = load_table_bundle(bench.DB_BUNDLE)
    assert doc["bundles"] == [bench.PO2_BUNDLE.name, bench.DB_BUNDLE.name, bench.LOGRANDOM_BUNDLE.name]
    hybrid = bench.dedup_tables(po2 + db)
    _, headline = bench.training_tables()
    probes = [tuple(p) for p in doc["probe_shapes"]]
    for key, tables, prov in (("po2", po2, "po2"), ("hybrid", hybrid, "hybrid"),
                              ("headline", headline, "hybrid")):
        want = doc[key]
        ds = dataset_from_tables(tables, prov)
        recs = ds.features_and_labels()
        assert [c for _, c in recs] == want["labels"]
        sp = split(ds, bench.SPLIT_FRACTION, bench.SPLIT_SEED)
        assert list(sp.train) == want["train"] and list(sp.test) == want["test"]
        named = model.grid_train([recs[i] for i in sp.train])
        assert len(named) == len(want["trees"]) == 40
        for name, tree in named:
            w = want["trees"][name]
            assert codegen.tree_fingerprint(tree) == w["fingerprint"], (key, name)
            assert [model.predict(tree, p) for p in probes] == w["predictions"], (key, name)
