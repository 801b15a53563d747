"""Split-K: DSMEM cluster reduction vs HBM slab + reduce kernel, per shape.

Times every split-K config of the B200 space on the DeepBench shapes in the
bench regime (L2 flushed before every sample, trimmed mean; the timing of
configs/deepbench_b200.json).  Run once as is and once with
AG_SPLITK_REDUCE=slab (read once per process), then compare:

    python profiles/reduce_mode_probe.py > a.jsonl
    AG_SPLITK_REDUCE=slab python profiles/reduce_mode_probe.py > b.jsonl
"""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_1806_07060_b200 import cli  # noqa: E402
from paper_1806_07060_b200.kernels import KernelFamily, full_search_space  # noqa: E402
from paper_1806_07060_b200.tuner import tune_configs  # noqa: E402


def main():
    cfg = cli.PipelineConfig.load(Path(__file__).resolve().parent.parent / "configs" / "deepbench_b200.json")
    shapes, _ = cfg.shapes()
    sk = [c for c in full_search_space(cfg.caps) if c.family is KernelFamily.SPLITK]
    mode = os.environ.get("AG_SPLITK_REDUCE", "cluster")
    for s in shapes:
        t = tune_configs(s, sk, cfg.caps, cfg.timing)
        print(json.dumps({"mode": mode, "mnk": list(s.mnk),
                          "gflops": {m.config.canonical(): round(m.gflops, 1) for m in t.measurements}}), flush=True)


if __name__ == "__main__":
    main()
