"""Device-timed probe of the tensor-core families next to the fp32 best.

    python profiles/tc_probe.py [--shapes 4096x4096x4096,...] [--ncu]

Prints one JSON line per (shape, config): median seconds (ag_tune: CUDA
events, graph-replayed samples; pack helpers included) and GFLOP/s.
--ncu: run each tc config once per shape (for an ncu launch list) instead.
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_1806_07060_b200.kernels import DeviceCaps, KernelConfig, KernelFamily, ProblemShape, enumerate_search_space  # noqa: E402
from paper_1806_07060_b200.tuner import DeviceBuffers, TimingPolicy, flops_of, time_configs  # noqa: E402

DEFAULT = "4096x4096x4096,8192x8192x8192,5124x9124x2560,2048x2048x2048,1024x1024x1024,35x8457x2560,5124x700x2048"
FP32_BEST = ["indirect:128-128-32-8-8-1", "indirect:64-64-16-8-8-1"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shapes", default=DEFAULT)
    ap.add_argument("--families", default="tf32,bf16")
    ap.add_argument("--repeats", type=int, default=5)
    a = ap.parse_args()
    caps = DeviceCaps.b200_tc()
    cfgs = []
    for f in a.families.split(","):
        cfgs += enumerate_search_space(KernelFamily(f), caps)
    cfgs += [KernelConfig.from_canonical(c) for c in FP32_BEST]
    for spec in a.shapes.split(","):
        m, n, k = (int(x) for x in spec.split("x"))
        s = ProblemShape(m, n, k)
        bufs = DeviceBuffers(s)
        secs = time_configs(s, cfgs, caps, TimingPolicy(warmup=2, repeats=a.repeats), bufs)
        fl = flops_of(s)
        for c, t in zip(cfgs, secs):
            print(json.dumps({"mnk": [m, n, k], "config": c.canonical(), "s": t, "gflops": round(fl / t / 1e9, 1)}),
                  flush=True)


if __name__ == "__main__":
    main()
