"""Re-time one kernel family over a finished sweep and merge it in.

    python configs/resweep_family.py FAMILY CONFIG.json OLD_TABLES_DIR NEW_TABLES_DIR
    python configs/resweep_family.py list:CFG1,CFG2 CONFIG.json OLD NEW   (explicit configs)

For every shape of CONFIG: time the family's configs of the config's search
space (list mode: the listed ones of that family) with the config's timing
policy on resident buffers, then write the shape's table with those rows
replaced (tuner.merge_tables, the re-timed rows win) in the full enumeration
order.  Used after a kernel change that touches one family only (the
split-K in-place core), so the other families' measurements are kept.
`--odd-n-only`: only shapes with N % 4 != 0 (the in-place core's element
copies of B, round 2) are re-timed.

    python configs/resweep_family.py --unbundle BUNDLE.csv.gz TABLES_DIR
"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))

from bundle_tables import full_order  # noqa: E402

from paper_1806_07060_b200 import cli  # noqa: E402
from paper_1806_07060_b200.kernels import KernelFamily, full_search_space  # noqa: E402
from paper_1806_07060_b200.tuner import load_table, merge_tables, save_table, table_filename, tune_configs  # noqa: E402


def main():
    if len(sys.argv) == 4 and sys.argv[1] == "--unbundle":  # a shipped bundle -> per-shape tables
        from paper_1806_07060_b200.tuner import load_table_bundle
        out = Path(sys.argv[3])
        out.mkdir(parents=True, exist_ok=True)
        for t in load_table_bundle(sys.argv[2]):
            save_table(t, out / table_filename(t.shape))
        return
    ap = argparse.ArgumentParser()
    ap.add_argument("family")
    ap.add_argument("config")
    ap.add_argument("old")
    ap.add_argument("new")
    ap.add_argument("--odd-n-only", action="store_true",
                    help="re-time only shapes whose N is not a multiple of 4 (the others are copied)")
    a = ap.parse_args()
    cfg = cli.PipelineConfig.load(a.config)
    shapes, _ = cfg.shapes()
    order = full_order(cfg) or full_search_space(cfg.caps)
    if a.family.startswith("list:"):  # explicit configs (e.g. a new default tile)
        from paper_1806_07060_b200.kernels import KernelConfig
        mine = [KernelConfig.from_canonical(x) for x in a.family[5:].split(",")]
    else:
        fam = KernelFamily(a.family)
        mine = [c for c in order if c.family is fam]
    out = Path(a.new)
    out.mkdir(parents=True, exist_ok=True)
    for i, s in enumerate(shapes):
        dst = out / table_filename(s)
        if dst.exists():
            continue
        old = load_table(Path(a.old) / table_filename(s))
        if a.odd_n_only and s.N % 4 == 0:
            save_table(old, dst)
            continue
        fresh = tune_configs(s, mine, cfg.caps, cfg.timing)
        merged = merge_tables(fresh, old, order)
        merged.meta.update({k: v for k, v in old.meta.items() if k not in ("configs",)})
        save_table(merged, dst)
        if i % 20 == 0:
            print(f"{i + 1}/{len(shapes)} {s.mnk}: best {merged.best_config.canonical()}", flush=True)
    print(f"{len(shapes)} tables -> {out}")


if __name__ == "__main__":
    main()
