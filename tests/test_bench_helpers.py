"""CPU checks of bench.py's host-side helpers: the regime floor, the launch
counts it claims per family, the merged tf32x3 tables and the headline
model's protocol (no DeepBench shape in training)."""
import sys

import pytest

from conftest import ROOT

sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_1806_07060_b200.kernels import KernelConfig, KernelFamily, ProblemShape  # noqa: E402


def test_regime_floor_is_the_slower_of_compute_and_read():
    small = ProblemShape(2048, 16, 2048)       # 17 MB, 134 MFLOP: read-bound
    big = ProblemShape(5124, 9124, 2560)       # compute-bound
    assert bench.regime_floor_s(small, 72.5) == pytest.approx(10.07e-6, rel=0.02)
    assert bench.regime_floor_s(big, 72.5) == pytest.approx(2 * 5124 * 9124 * 2560 / 72.5e12)
    tiny = ProblemShape(8, 8, 8)
    assert bench.regime_floor_s(tiny, 72.5) == pytest.approx(6.18e-6)
    sizes = [ProblemShape(1024, 16, k) for k in (256, 1024, 4096, 16384, 65536)]
    floors = [bench.regime_floor_s(s, 72.5) for s in sizes]
    assert floors == sorted(floors)  # monotone in the bytes moved


@pytest.mark.parametrize("canon,shape,n", [
    ("tf32x3:128-128-32-3-1-1", (512, 512, 512), 1),
    ("bf16:256-256-64-6-1-1", (512, 512, 512), 3),
    ("tf32:256-256-32-4-1-1", (512, 512, 512), 1),
    ("skinny_n:64-16-32-2-4-4", (2048, 16, 2048), 1),
    ("direct:16-16-8-2-2-1", (64, 64, 64), 1),
    ("splitk:64-128-32-8-8-4", (5124, 700, 2048), 1),  # in-place core, cluster reduction
    ("splitk:32-64-16-4-4-16", (35, 1500, 2560), 2),  # 16 slices: in-place core + slab reduction
    ("splitk:16-16-32-2-2-16", (64, 16, 64), 1),  # 16-slice config, 2 K tiles: 2 slices, cluster
    # N = 8457 is not a multiple of 4: pack A, pack-pad B, core, slab reduction
    # (the four launches of profiles/r02_splitk_packed_35x8457x2560.json)
    ("splitk:32-64-16-4-4-16", (35, 8457, 2560), 4),
])
def test_pack_launches_per_family(canon, shape, n):
    assert bench.pack_launches(ProblemShape(*shape), KernelConfig.from_canonical(canon)) == n


def test_x3_tables_merge_every_shape_with_fp32_rows_first():
    train, db = bench.load_x3_tables()
    assert len(train) == 729 + 512 and len(db) == 40
    assert [t.shape.mnk for t in train] == [t.shape.mnk for t in bench.training_tables()[1]]
    for t in db + train[::97]:
        fams = [m.config.family for m in t.measurements]
        first_x3 = fams.index(KernelFamily.TF32X3)
        assert all(f is not KernelFamily.TF32X3 for f in fams[:first_x3])
        assert all(f is KernelFamily.TF32X3 for f in fams[first_x3:])
        assert t.peak_gflops == max(m.gflops for m in t.measurements)


def test_headline_model_trains_on_generated_shapes_only():
    """The headline tree sees the po2 and octave-uniform random tables only
    (no DeepBench table): its training set is the CLI hybrid of the two
    sweeps, one seeded split; the DeepBench shapes that are not training
    shapes are reported separately (dt_vs.unseen)."""
    from paper_1806_07060_b200.dataset import gen_po2, gen_random
    from paper_1806_07060_b200.tuner import load_table_bundle
    po2, tables = bench.training_tables()
    gen = [s.mnk for s in gen_po2(16, 4096)] + [s.mnk for s in gen_random(512, 16, 4096, 2026, "log2")]
    assert [t.shape.mnk for t in tables] == list(dict.fromkeys(gen))
    assert [t.shape.mnk for t in po2] == [s.mnk for s in gen_po2(16, 4096)]
    pipe = bench._pipeline(tables, "hybrid")
    assert pipe["n_train"] == int(0.8 * len(tables))
    db = {t.shape.mnk for t in load_table_bundle(bench.DB_BUNDLE)}
    pow2 = lambda v: v & (v - 1) == 0  # noqa: E731
    off_grid = {mnk for mnk in db if not all(pow2(x) for x in mnk)}
    assert len(off_grid) == 32 and not off_grid & pipe["train"]

def test_headline_training_set_is_a_cli_hybrid_config():
    """configs/headline_b200.json reproduces the headline training set through
    the reference-compatible CLI (tune / dataset / train): its hybrid dataset
    lists exactly the shapes of bench.training_tables(), in order."""
    from paper_1806_07060_b200 import cli
    cfg = cli.PipelineConfig.load(bench.ROOT / "configs" / "headline_b200.json")
    shapes, tag = cfg.shapes()
    assert tag == "hybrid" and cfg.caps.profile == "b200"
    assert [s.mnk for s in shapes] == [t.shape.mnk for t in bench.training_tables()[1]]


def test_headline_cli_stages_pick_the_bench_tree(tmp_path):
    """The CLI's dataset / train / eval stages on the shipped tables of
    configs/headline_b200.json (written where `tune` would put them) choose
    the same model, with the same tree, as bench.build_model()."""
    import json

    from paper_1806_07060_b200 import cli, codegen, model
    from paper_1806_07060_b200.tuner import save_table, table_filename
    doc = json.loads((bench.ROOT / "configs" / "headline_b200.json").read_text())
    doc["out_dir"] = str(tmp_path / "out")
    path = tmp_path / "headline.json"
    path.write_text(json.dumps(doc))
    cfg = cli.PipelineConfig.load(path)
    cfg.tables_dir.mkdir(parents=True)
    for t in bench.training_tables()[1]:
        save_table(t, cfg.tables_dir / table_filename(t.shape), {"config_hash": cfg.hash()})
    for stage in ("dataset", "train", "eval"):
        assert cli.main([stage, "--config", str(path)]) == 0
    best = json.loads((cfg.out / "best_model.json").read_text())
    m = bench.build_model()
    assert best["name"] == m["name"]
    cli_tree = model.load_tree(best["path"])
    assert cli_tree.meta.pop("config_hash") == cfg.hash()  # the CLI stamps its config; otherwise equal
    assert codegen.tree_fingerprint(cli_tree) == codegen.tree_fingerprint(m["tree"])
