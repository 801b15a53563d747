"""Host-path phase times for small / mid DeepBench calls (measurement only):
numpy operands through gemm_execute (fast path, AG_HOST_STAGE), with
AG_HOST_TRACE=1 printing the per-call phase timestamps from ag_gemm_host_ex.
    AG_HOST_TRACE=1 python profiles/host_small_probe.py"""
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import numpy as np

    from paper_1806_07060_b200.kernels import DeviceCaps, KernelConfig, ProblemShape, gemm_execute
    from paper_1806_07060_b200.tuner import _bench_buffers
    cases = [((35, 700, 2560), "skinny_n:64-16-32-2-8-3"), ((1760, 128, 1760), "skinny_n:64-32-32-2-8-1"),
             ((2048, 16, 2048), "skinny_n:64-16-32-2-4-8"), ((5124, 700, 2048), "indirect:32-64-32-8-8-2")]
    for mnk, name in cases:
        s = ProblemShape(*mnk)
        A, B, C, _ = _bench_buffers(s, np.float32, 0)
        cfg = KernelConfig.from_canonical(name)
        ts = []
        for r in range(8):
            t0 = time.perf_counter()
            out, sec = gemm_execute(s, cfg, A, B, C, DeviceCaps.b200())
            ts.append(time.perf_counter() - t0)
            print(f"# {mnk} call {r}: {ts[-1] * 1e3:.3f} ms (kernel {sec * 1e3:.3f})", file=sys.stderr, flush=True)
        print(f"{mnk} median {statistics.median(ts[2:]) * 1e3:.3f} ms", flush=True)


if __name__ == "__main__":
    main()
