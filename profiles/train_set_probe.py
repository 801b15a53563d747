"""Which training set transfers best to the DeepBench-style set?

Table mode only (CPU): trains the reference pipeline (seeded 80/20 split,
5 x 8 CART grid, best test DTPR) on each candidate training set and scores
the chosen tree on the DeepBench tables (DTPR, DTTR, and the geomean of the
table GFLOP/s of its picks over the table best).  No DeepBench table is
used in training or model selection.

    python profiles/train_set_probe.py [extra_bundle.csv.gz ...]
"""
import json
import math
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402
from paper_1806_07060_b200 import codegen  # noqa: E402
from paper_1806_07060_b200.tuner import load_table_bundle  # noqa: E402


def dedup(tables):
    out, seen = [], set()
    for t in tables:
        if t.shape.mnk not in seen:
            seen.add(t.shape.mnk)
            out.append(t)
    return out


def score(name, tables, db, anchors):
    pipe = bench._pipeline(tables, "hybrid", anchors)
    sel = codegen.CompiledSelector(pipe["tree"], pipe["classes"])
    ratios, dttr = [], []
    per = []
    for t in db:
        cfg = sel.select(*t.shape.mnk)
        g = t.gflops_for(cfg)
        ratios.append(g / t.peak_gflops)
        dttr.append(g / t.gflops_for(pipe["policy"].select_config(t.shape)))
        per.append([list(t.shape.mnk), round(g / t.peak_gflops, 3), cfg.canonical()])
    geo = math.exp(sum(math.log(r) for r in ratios) / len(ratios))
    return {"train_set": name, "n_train": pipe["n_train"], "model": pipe["name"], "test_score": pipe["score"],
            "db_dtpr": round(sum(ratios) / len(ratios), 4), "db_dttr": round(sum(dttr) / len(dttr), 4),
            "db_geo_over_best": round(geo, 4), "worst": sorted(per, key=lambda r: r[1])[:8]}


def main():
    po2 = load_table_bundle(bench.PO2_BUNDLE)
    db = load_table_bundle(bench.DB_BUNDLE)
    sets = {} if "--skip-po2" in sys.argv else {"po2": po2}
    for p in [a for a in sys.argv[1:] if not a.startswith("--")]:
        extra = load_table_bundle(p)
        sets[Path(p).name] = extra
        sets["po2+" + Path(p).name] = dedup(po2 + extra)
    for name, tables in sets.items():
        print(json.dumps(score(name, tables, db, {t.shape.mnk: t for t in po2})), flush=True)


if __name__ == "__main__":
    main()
