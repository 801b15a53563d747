"""Bundle a sweep's per-shape tables into the gzip file bench.py ships with.

    python configs/bundle_tables.py CONFIG.json TABLES_DIR OUT.csv.gz [--extra TABLES_DIR2]

Tables are written in the config's shape order.  --extra merges a second
sweep of the same shapes and timing policy (tuner.merge_tables); rows are
ordered as the config's enumeration would list them (the tc families in
enumeration order, then the fp32 shortlist), so the bundle reads as one
sweep of the full list.
"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from paper_1806_07060_b200 import cli  # noqa: E402
from paper_1806_07060_b200.kernels import KernelConfig, KernelFamily, enumerate_search_space  # noqa: E402
from paper_1806_07060_b200.tuner import load_table, merge_tables, save_table_bundle, table_filename  # noqa: E402


def full_order(cfg) -> list:
    s = cfg.sampling
    if s.get("mode") != "list":
        return None
    out = []
    for fam in s.get("families", []):
        out += enumerate_search_space(KernelFamily(fam), cfg.caps)
    out += [KernelConfig.from_canonical(t) for t in s.get("configs", [])]
    return list(dict.fromkeys(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("tables")
    ap.add_argument("out")
    ap.add_argument("--extra", default=None)
    a = ap.parse_args()
    cfg = cli.PipelineConfig.load(a.config)
    shapes, _ = cfg.shapes()
    order = full_order(cfg)
    tables = []
    for s in shapes:
        t = load_table(Path(a.tables) / table_filename(s))
        if a.extra:
            t = merge_tables(t, load_table(Path(a.extra) / table_filename(s)), order)
        tables.append(t)
    save_table_bundle(tables, a.out)
    print(f"{len(tables)} tables, {sum(len(t.measurements) for t in tables)} rows -> {a.out}")


if __name__ == "__main__":
    main()
