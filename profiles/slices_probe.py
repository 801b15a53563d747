"""Would more split-K slice counts help the mid-N DeepBench shapes?  Times
every split-K tile x bk at S = 2..16 slices (the shipped space has S in
{2, 4, 8, 16}) in the bench regime (L2 flushed, trimmed mean of 5) and
reports the best shipped-space config against the best with any S.
Measurement only.   python profiles/slices_probe.py   (on the GPU box)"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import numpy as np

    from paper_1806_07060_b200 import spaces
    from paper_1806_07060_b200.kernels import DeviceCaps, KernelConfig, KernelFamily, ProblemShape, is_legal
    from paper_1806_07060_b200.tuner import DeviceBuffers, TimingPolicy, time_configs
    caps = DeviceCaps.b200()
    pol = TimingPolicy(warmup=1, repeats=5, l2="flush")
    cfgs = [KernelConfig(KernelFamily.SPLITK, bm, bn, bk, tm, tn, s)
            for (bm, bn, tm, tn) in spaces.SPLITK_TILES for bk in spaces.SPLITK_BLOCK_K for s in range(2, 17)]
    cfgs = [c for c in cfgs if is_legal(c, caps)]
    shapes = [(2048, 128, 2048), (2560, 128, 2560), (1760, 128, 1760), (3072, 128, 1024), (4096, 128, 4096),
              (7680, 128, 2560), (2048, 64, 2048), (2560, 64, 2560), (1760, 64, 1760), (3072, 64, 1024),
              (4096, 64, 4096), (7680, 64, 2560), (2048, 128, 1024), (1024, 128, 2048), (4096, 64, 1024)]
    for mnk in shapes:
        s = ProblemShape(*mnk)
        bufs = DeviceBuffers(s, np.float32, 0)
        ts = time_configs(s, cfgs, caps, pol, bufs)
        fl = 2.0 * s.M * s.N * s.K
        rows = sorted(((fl / t / 1e12, c.canonical()) for c, t in zip(cfgs, ts)), reverse=True)
        shipped = [r for r in rows if int(r[1].split("-")[-1]) in spaces.SPLITK_SLICES]
        print(json.dumps({"mnk": list(mnk), "best_any_S": rows[:3], "best_shipped_S": shipped[0],
                          "gain": round(rows[0][0] / shipped[0][0], 3)}), flush=True)


if __name__ == "__main__":
    main()
