"""Pin the shipped B200 models against the REFERENCE's CART (run here, where
/root/reference is importable; the GPU box only reads the output):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_b200_golden.py

For the datasets bench.py trains on -- the po2 16..4096 B200 tables, the
headline training set (po2 + the octave-uniform random tables) and the
reference CLI's hybrid po2 + DeepBench dataset --
the records (features, class ids) are built from the shipped table bundles
by this package (class ids in first-appearance order, dataset.py:94-183),
then the reference's own `split` (dataset.py:224-233, via rng.shuffled) and
`grid_train` (model.py:258-301) run on them.  Written to b200_trees.json:
split indices, the 40 grid fingerprints (sha256 of the reference's tree
JSON), and every grid model's predictions on the DeepBench shapes.
tests/test_host.py::test_shipped_b200_models_match_reference compares.
"""
import json
import os
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, str(ROOT))
sys.path.insert(1, "/root/reference/pkg/src")

from adaptgemm import codegen as ref_codegen  # noqa: E402
from adaptgemm import model as ref_model  # noqa: E402
from adaptgemm import rng as ref_rng  # noqa: E402

import bench  # noqa: E402
from paper_1806_07060_b200.dataset import dataset_from_tables  # noqa: E402
from paper_1806_07060_b200.tuner import load_table_bundle  # noqa: E402


def pipeline_doc(tables, provenance, probe_shapes):
    ds = dataset_from_tables(tables, provenance)
    recs = ds.features_and_labels()
    order = ref_rng.shuffled(len(recs), bench.SPLIT_SEED)
    n_train = int(bench.SPLIT_FRACTION * len(recs))
    train_idx, test_idx = list(order[:n_train]), list(order[n_train:])
    train = [(tuple(recs[i][0]), int(recs[i][1])) for i in train_idx]
    named = ref_model.grid_train(train)
    return {
        "n_records": len(recs), "labels": [int(c) for _, c in recs],
        "train": [int(i) for i in train_idx], "test": [int(i) for i in test_idx],
        "trees": {name: {"fingerprint": ref_codegen.tree_fingerprint(t),
                         "predictions": [ref_model.predict(t, p) for p in probe_shapes]}
                  for name, t in named},
    }


def main():
    po2 = load_table_bundle(bench.PO2_BUNDLE)
    db = load_table_bundle(bench.DB_BUNDLE)
    probes = [t.shape.mnk for t in db]
    hybrid, seen = [], set()
    for t in po2 + db:
        if t.shape.mnk not in seen:
            seen.add(t.shape.mnk)
            hybrid.append(t)
    _, headline = bench.training_tables()
    doc = {"bundles": [bench.PO2_BUNDLE.name, bench.DB_BUNDLE.name, bench.LOGRANDOM_BUNDLE.name],
           "probe_shapes": [list(p) for p in probes],
           "po2": pipeline_doc(po2, "po2", probes),
           "hybrid": pipeline_doc(hybrid, "hybrid", probes),
           "headline": pipeline_doc(headline, "hybrid", probes)}
    (HERE / "b200_trees.json").write_text(json.dumps(doc, separators=(",", ":")))
    print("wrote", HERE / "b200_trees.json")


if __name__ == "__main__":
    main()
