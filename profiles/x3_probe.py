"""tf32x3 (3xTF32 on tcgen05) against the fp32 CUDA-core families and the
tf32 / bf16 families on DeepBench shapes, bench.py's regime (L2 flushed
before every sample, trimmed mean of 7), plus RF vs the float64 product.
Measurement only.   python profiles/x3_probe.py   (on the GPU box)"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import numpy as np
    import torch

    from paper_1806_07060_b200.kernels import (DeviceCaps, KernelConfig, KernelFamily, ProblemShape,
                                               enumerate_search_space, gemm_execute)
    from paper_1806_07060_b200.tuner import DeviceBuffers, TimingPolicy, _bench_buffers, time_configs
    caps = DeviceCaps.b200_tc()
    pol = TimingPolicy(warmup=1, repeats=7, l2="flush")
    x3 = enumerate_search_space(KernelFamily.TF32X3, caps)
    extra = [KernelConfig.from_canonical(c) for c in (
        "indirect:64-128-32-8-8-2", "indirect:128-256-32-8-16-1", "indirect:128-128-16-16-8-1",
        "splitk:64-128-32-8-8-8", "splitk:128-64-32-8-8-8", "skinny_m:40-256-32-1-2-16",
        "tf32:256-256-32-4-1-1", "bf16:256-256-64-6-1-1")]
    shapes = [(5124, 9124, 2560), (4096, 7000, 4096), (2560, 7000, 2560), (5124, 1500, 2048), (5124, 700, 2048),
              (1760, 128, 1760), (4096, 128, 4096), (7680, 128, 2560), (35, 8457, 2560), (35, 1500, 2560),
              (2048, 64, 2048), (4096, 4096, 4096), (8192, 8192, 8192)]
    for mnk in shapes:
        s = ProblemShape(*mnk)
        cfgs = [c for c in x3 + extra]
        bufs = DeviceBuffers(s, np.float32, 0)
        ts = time_configs(s, cfgs, caps, pol, bufs)
        fl = 2.0 * s.M * s.N * s.K
        row = {"mnk": list(mnk), "tflops": {c.canonical(): round(fl / t / 1e12, 2) for c, t in zip(cfgs, ts)}}
        # accuracy of the fastest x3 config and of the fp32 reference config
        best = max(x3, key=lambda c: fl / ts[cfgs.index(c)])
        if s.M * s.N * s.K <= 2 ** 34:
            A, B, C, _ = _bench_buffers(s, np.float32, 0)
            exact = (torch.from_numpy(A).cuda().double() @ torch.from_numpy(B).cuda().double())
            for c in (best, extra[0]):
                out, _ = gemm_execute(s, c, A, B, C, caps)
                o = torch.from_numpy(out).cuda().double()
                row.setdefault("rf", {})[c.canonical()] = float(torch.linalg.norm(o - exact) / torch.linalg.norm(exact))
        row["best_x3"] = best.canonical()
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
