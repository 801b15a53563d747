"""Run one config on one shape a few times (device-resident operands), for ncu.

    ncu --set full -k regex:tc_gemm -c 1 -o gpurun_out/x python profiles/one_gemm.py 8192x8192x8192 bf16:128-256-64-4-1-1
    python profiles/one_gemm.py MxNxK CONFIG [REPS] [NN|TN|NT|TT]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_1806_07060_b200.kernels import DeviceCaps, KernelConfig, ProblemShape, gemm_execute  # noqa: E402
from paper_1806_07060_b200.tuner import DeviceBuffers  # noqa: E402


def main():
    m, n, k = (int(x) for x in sys.argv[1].split("x"))
    cfg = KernelConfig.from_canonical(sys.argv[2])
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    trans = sys.argv[4] if len(sys.argv) > 4 else "NN"  # e.g. TN = transA
    s = ProblemShape(m, n, k, transA=trans[0] == "T", transB=trans[1] == "T")
    b = DeviceBuffers(s)
    for _ in range(reps):
        _, sec = gemm_execute(s, cfg, b.A, b.B, b.C, DeviceCaps.b200_tc(), out=b.out)
        print(f"{sys.argv[1]} {cfg.canonical()} {sec * 1e6:.1f} us {2 * m * n * k / sec / 1e12:.1f} TFLOP/s")


if __name__ == "__main__":
    main()
