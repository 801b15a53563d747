"""Generate the golden fixtures by running the REFERENCE implementation.

Run in the build container (the reference is importable only there):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

It imports `adaptgemm` from /root/reference/pkg/src (read-only; the numba
cache is redirected) and the reference's own test helpers
(/root/reference/pkg/tests/conftest.py) and records, from the reference
itself:

* gemm_golden.npz -- operands and outputs of gemm_reference and of
  gemm_execute for sampled direct/indirect configs (KATs from
  test_kernels.py + the C1 shape generator of test_acceptance.py:78-111);
* golden.json -- search spaces, rng streams, shape generators, splits,
  tune_random picks, CART splits/trees/fingerprints/predictions,
  boundary probes, emitted dispatcher sources and evaluation metrics;
* cli/ -- a complete reference pipeline run (tables + every stage
  artifact) on a tiny workload, for byte-level artifact parity.

The GPU box never runs this script; tests read the committed outputs.
"""

import hashlib
import itertools
import json
import os
import shutil
import sys
import tempfile
from pathlib import Path

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
HERE = Path(__file__).resolve().parent
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, REF_SRC)
sys.path.insert(0, REF_TESTS)

import adaptgemm  # noqa: E402
from adaptgemm import codegen, evaluation, rng  # noqa: E402
from adaptgemm import model as M  # noqa: E402
from adaptgemm.cli import main as ref_main  # noqa: E402
from adaptgemm.dataset import (ClassIndex, Dataset, DatasetRecord, dataset_from_tables,  # noqa: E402
                               gen_go2, gen_po2, split)
from adaptgemm.kernels import (DeviceCaps, KernelConfig, KernelFamily, ProblemShape,  # noqa: E402
                               full_search_space, gemm_execute, gemm_reference)
from adaptgemm.tuner import TimingPolicy, tune_random  # noqa: E402

import conftest as refconf  # noqa: E402  (the reference's test helpers)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


# ---------------------------------------------------------------------------
# GEMM


def gemm_cases():
    """(name, ProblemShape, dtype, seed) in a fixed order."""
    cases = []
    ft = list(itertools.product([False, True], repeat=2))
    cases.append(("padding_33x33x17", ProblemShape(33, 33, 17), np.float32, 11))
    cases.append(("agree_41x29x37", ProblemShape(41, 29, 37, alpha=0.75, beta=1.5), np.float32, 5))
    for ta, tb in ft:
        cases.append((f"trans_{int(ta)}{int(tb)}", ProblemShape(19, 23, 31, 1.5, 0.5, ta, tb), np.float32, 13))
    for mnk in [(1, 1, 1), (1, 37, 5), (37, 1, 5), (5, 37, 1), (64, 1, 1)]:
        cases.append((f"edge_{mnk}", ProblemShape(*mnk, alpha=1.0, beta=0.5), np.float32, 17))
    cases.append(("f64_21x18x40", ProblemShape(21, 18, 40, alpha=2.0, beta=0.25), np.float64, 19))
    cases.append(("neutral_64x32x48", ProblemShape(64, 32, 48, alpha=1.0, beta=0.5), np.float32, 23))
    # C1 generator (test_acceptance.py:78-95), first 24 random shapes
    stream = rng.SplitMix64(0xC1)
    for i in range(24):
        s = ProblemShape(1 + stream.below(96), 1 + stream.below(96), 1 + stream.below(96),
                         alpha=(1.0, 1.5, 2.0)[stream.below(3)],
                         beta=(0.0, 0.0, 0.5, 1.0)[stream.below(4)],
                         transA=bool(stream.below(2)), transB=bool(stream.below(2)))
        cases.append((f"c1_{i}", s, np.float32, 1000 + i))
    return cases


def make_gemm():
    space = full_search_space()
    arrays = {}
    meta = []
    for idx, (name, s, dt, seed) in enumerate(gemm_cases()):
        A, B, C = refconf.rand_operands(s, dt, seed)
        ref = gemm_reference(s, A, B, C)
        key = f"c{idx}"
        arrays[f"{key}_A"], arrays[f"{key}_B"], arrays[f"{key}_C"] = A, B, C
        arrays[f"{key}_ref"] = ref
        picks = rng.sample_without_replacement(len(space), 6, rng.mix(idx, 77))
        execs = []
        for j, p in enumerate(picks):
            cfg = space[p]
            out, _ = gemm_execute(s, cfg, A, B, C)
            arrays[f"{key}_x{j}"] = out
            execs.append(cfg.canonical())
        meta.append({"key": key, "name": name, "M": s.M, "N": s.N, "K": s.K, "alpha": s.alpha,
                     "beta": s.beta, "transA": s.transA, "transB": s.transB,
                     "dtype": np.dtype(dt).name, "seed": seed, "ref_sha": sha(ref),
                     "A_sha": sha(A), "execute_configs": execs})
    np.savez_compressed(HERE / "gemm_golden.npz", **arrays)
    return meta


# ---------------------------------------------------------------------------
# search space, rng, shapes, splits, sampling


def make_basics():
    caps = DeviceCaps()
    g = {}
    g["space"] = [c.canonical() for c in full_search_space(caps)]
    g["space_relaxed_direct_count"] = len(adaptgemm.enumerate_search_space(
        KernelFamily.DIRECT, DeviceCaps(register_tile_cap_direct=16)))
    g["space_tight_indirect"] = [c.canonical() for c in adaptgemm.enumerate_search_space(
        KernelFamily.INDIRECT, DeviceCaps(tile_memory_cap=8192))]
    r = {}
    for seed in (0, 1, 42, 2024, 0xC1, 2**64 - 1):
        st = rng.SplitMix64(seed)
        r[str(seed)] = {"u64": [st.next_u64() for _ in range(8)],
                        "below": [st.below(b) for b in (1, 2, 3, 7, 96, 1000, 2**63 + 5, 8192)]}
    g["splitmix"] = r
    g["mix"] = {"0,256,256,256": rng.mix(0, 256, 256, 256), "7": rng.mix(7),
                "1,2,3,4,5": rng.mix(1, 2, 3, 4, 5), "-1": rng.mix(-1)}
    g["shuffled"] = {f"{n},{s}": rng.shuffled(n, s) for n, s in ((10, 1), (27, 20817), (216, 4242), (50, 0))}
    g["sample"] = {f"{n},{k},{s}": rng.sample_without_replacement(n, k, s)
                   for n, k, s in ((576, 10, 3), (144, 20, 9), (432, 20, 12345))}
    g["po2_64_2048"] = [s.mnk for s in gen_po2(64, 2048)]
    g["go2_count"] = len(gen_go2(256, 3840, 256))
    g["go2_head"] = [s.mnk for s in gen_go2(256, 3840, 256)[:40]]
    cfg = KernelConfig(KernelFamily.DIRECT, 8, 8, 8, 1, 1, 1)
    splits = {}
    for n in (2, 10, 216, 343, 3375):
        idx = ClassIndex()
        idx.ensure(cfg)
        ds = Dataset([DatasetRecord(ProblemShape(i + 1, 1, 1), cfg, 1.0) for i in range(n)], idx, "workload")
        for seed, frac in ((4242, 0.8), (2024, 0.8), (7, 0.5)):
            sp = split(ds, frac, seed)
            splits[f"{n},{seed},{frac}"] = [list(sp.train), list(sp.test)]
    g["splits"] = splits
    # tune_random picks (timing-independent): TINY shape from test_tuner.py
    tiny = ProblemShape(9, 8, 7)
    fast = TimingPolicy(warmup=0, repeats=1)
    g["tune_random"] = {f"{n},{s}": [m.config.canonical() for m in
                                     tune_random(tiny, caps, samples=n, seed=s, timing=fast).measurements]
                        for n, s in ((10, 42), (10, 43), (37, 7), (200, 1))}
    return g


# ---------------------------------------------------------------------------
# CART, dispatch, evaluation


def tree_doc(tree):
    return {"fingerprint": codegen.tree_fingerprint(tree), "height": tree.height(),
            "leaves": len(tree.leaves())}


def make_cart(search_space):
    g = {}
    fixture = [((64, 1, 1), 0), ((128, 1, 1), 0), ((256, 1, 1), 1), ((512, 1, 1), 1)]
    g["best_split_fixture"] = list(M.best_split(fixture, 1))
    # random sample sets (test_model.py:181-193 generator) with best_split results
    cases = []
    stream = rng.SplitMix64(2024)
    for _ in range(150):
        n = 2 + stream.below(30)
        samples = [((1 + stream.below(64), 1 + stream.below(64), 1 + stream.below(64)), stream.below(4))
                   for _ in range(n)]
        ml = 1 + stream.below(3)
        res = M.best_split(samples, ml)
        cases.append({"samples": samples, "min_leaf": ml, "result": list(res) if res else None})
    g["best_split_cases"] = cases
    # fixture-table datasets, full 40-model grids
    grids = {}
    def fake(shape):
        # the reference's fake_table_factory fixture (conftest.py:58-68)
        from adaptgemm.tuner import Measurement, TuningTable, flops_of
        fl = flops_of(shape)
        ms = []
        for c in search_space:
            gf = refconf.fake_gflops(shape, c)
            ms.append(Measurement(c, fl / (gf * 1e9), gf))
        return TuningTable.from_measurements(shape, ms, {"mode": "fixture"})
    worlds = {}
    for tag, shapes in (("po2_64_256", gen_po2(64, 256)), ("po2_64_512", gen_po2(64, 512)),
                        ("po2_64_2048", gen_po2(64, 2048))):
        tables = [fake(s) for s in shapes]
        ds = dataset_from_tables(tables, "po2")
        records = ds.features_and_labels()
        named = M.grid_train(records)
        grids[tag] = {"labels": [cid for _, cid in records],
                      "classes": [c.canonical() for c in ds.class_index.configs()],
                      "trees": {name: tree_doc(t) for name, t in named}}
        worlds[tag] = (ds, tables, records, named)
    g["grids"] = grids
    # full JSON + emitted sources + probes for a few trees
    ds, tables, records, named = worlds["po2_64_512"]
    by = dict(named)
    full = {}
    for name in ("h1-L1", "h4-L1", "hMax-L1", "h8-L0.1", "hMax-L0.5"):
        t = by[name]
        probes = codegen.boundary_probes(t)
        pts = sorted(set(probes) | {f for f, _ in records})
        full[name] = {"tree": t.to_dict(), "probes": probes,
                      "predictions": [[list(p), M.predict(t, p)] for p in pts],
                      "c_source": codegen.emit_dispatcher(t, ds.class_index, "c", "golden").text,
                      "py_source": codegen.emit_dispatcher(t, ds.class_index, "python", "golden").text}
    g["full_trees"] = full
    # random records with duplicates, deep combs and large n (int128 range)
    rand_trees = []
    stream = rng.SplitMix64(99)
    for case in range(30):
        n = 2 + stream.below(300)
        span = 1 + stream.below(200)
        recs = [((1 + stream.below(span), 1 + stream.below(span), 1 + stream.below(span)),
                 stream.below(1 + stream.below(12))) for _ in range(n)]
        h = (1, 2, 4, 8, None)[stream.below(5)]
        L = (1, 2, 4, 0.1, 0.2, 0.3, 0.4, 0.5)[stream.below(8)]
        t = M.train(recs, M.TrainConfig(max_height=h, min_samples_leaf=L))
        rand_trees.append({"records": recs, "max_height": h, "min_leaf": L, **tree_doc(t)})
    comb = [((i, 1, 1), i % 2) for i in range(1, 80)]
    t = M.train(comb, M.TrainConfig())
    rand_trees.append({"records": comb, "max_height": None, "min_leaf": 1, **tree_doc(t)})
    g["random_trees"] = rand_trees
    # go2-scale (3375 records): exercises the > int64 cross products path
    go2 = gen_go2(256, 3840, 256)
    recs = []
    for s in go2:
        best = max(range(0, len(search_space), 7), key=lambda i: (refconf.fake_gflops(s, search_space[i]), -i))
        recs.append((s.mnk, best))
    big = {}
    for h, L in ((None, 1), (8, 1), (4, 0.1), (None, 4)):
        t = M.train(recs, M.TrainConfig(max_height=h, min_samples_leaf=L))
        big[M.grid_name(h, L)] = tree_doc(t)
    g["go2_trees"] = {"labels": [lab for _, lab in recs], "trees": big}
    # evaluation on the 27-shape fixture world (test_evaluation.py:34-44)
    ds, tables, records, named = worlds["po2_64_256"]
    tbs = evaluation.tables_by_shape(tables)
    tree = M.train(records, M.TrainConfig(max_height=4, min_samples_leaf=1))
    pol = evaluation.BaselinePolicy(KernelConfig(KernelFamily.INDIRECT, 32, 32, 16, 4, 4, 1),
                                    KernelConfig(KernelFamily.DIRECT, 16, 16, 8, 2, 2, 1), threshold=128)
    pol.register(ds.class_index)
    scores = evaluation.score_models(named, records, tbs, ds.class_index, pol)
    g["evaluation"] = {
        "tree": tree_doc(tree),
        "accuracy": evaluation.accuracy(tree, records),
        "dtpr": evaluation.dtpr(tree, records, tbs, ds.class_index),
        "dttr": evaluation.dttr(tree, records, tbs, ds.class_index, pol),
        "baseline_select": [evaluation.baseline_select(pol, r.input) for r in ds.records],
        "scores": [[s.name, s.accuracy, s.dtpr, s.dttr, s.stats.total_leaves, s.stats.height] for s in scores],
        "best": evaluation.select_best_model(scores).name,
    }
    # random feasible trees from the reference's conftest: probes + C/py text
    rft = []
    for seed in (3, 17, 42):
        t = refconf.random_feasible_tree(seed)
        classes = refconf.cycled_class_map(len(t.leaves()), search_space)
        rft.append({"seed": seed, "tree": t.to_dict(), "probes": codegen.boundary_probes(t),
                    "classes": {str(k): v.canonical() for k, v in classes.items()},
                    "c_sha": hashlib.sha256(codegen.emit_dispatcher(t, classes, "c").text.encode()).hexdigest()})
    g["random_feasible_trees"] = rft
    return g


# ---------------------------------------------------------------------------
# a complete reference CLI run


def make_cli():
    dest = HERE / "cli"
    if dest.exists():
        shutil.rmtree(dest)
    with tempfile.TemporaryDirectory() as td:
        cwd = os.getcwd()
        os.chdir(td)
        try:
            Path("shapes.txt").write_text("8 8 8\n16 16 16\n24 24 24\n32 32 32\n40 8 24\n8 40 16\n")
            cfg = {"out_dir": "run", "timing": {"warmup": 0, "repeats": 1},
                   "dataset": {"strategy": "workload", "path": "shapes.txt"},
                   "split": {"fraction": 0.5, "seed": 7},
                   "grid": {"heights": [1, 2, "max"], "min_leaf": [1, 2]},
                   "baseline": {"threshold": 16, "direct_anchor": [8, 8, 8], "indirect_anchor": [32, 32, 32]}}
            Path("config.json").write_text(json.dumps(cfg, indent=1))
            for stage in ("tune", "dataset", "train", "eval", "codegen"):
                assert ref_main([stage, "--config", "config.json"]) == 0, stage
            shutil.copytree(td, dest)
        finally:
            os.chdir(cwd)


def main():
    search_space = full_search_space()
    golden = {"reference": "adaptgemm " + adaptgemm.__version__, "numpy": np.__version__}
    golden["gemm"] = make_gemm()
    golden.update(make_basics())
    golden["cart"] = make_cart(search_space)
    with open(HERE / "golden.json", "w") as fh:
        json.dump(golden, fh, separators=(",", ":"))
    make_cli()
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
