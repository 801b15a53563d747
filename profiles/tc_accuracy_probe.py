"""Accuracy of the tensor-core families against the fp32 CUDA-core path
(measurement only).  For each K, on U(-1,1) operands:
  tf32_trunc   tf32 family on inputs pre-truncated to tf32 (products exact in
               fp32: only the tensor core's accumulation error remains)
  fp32_trunc   the CUDA-core indirect family on the same truncated inputs
  x3           tf32x3 on the raw fp32 inputs
  fp32         the CUDA-core indirect family on the raw inputs
RF = relative Frobenius error vs the float64 product.
    python profiles/tc_accuracy_probe.py   (on the GPU box)"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import numpy as np
    import torch

    from paper_1806_07060_b200.kernels import DeviceCaps, KernelConfig, ProblemShape, gemm_execute
    caps = DeviceCaps.b200_tc()
    rng = np.random.default_rng(0)
    fp32 = KernelConfig.from_canonical("indirect:64-64-16-4-4-1")
    tf32 = KernelConfig.from_canonical("tf32:128-128-32-4-1-1")
    x3s = [KernelConfig.from_canonical(c) for c in ("tf32x3:128-128-32-3-1-1", "tf32x3:256-128-32-3-1-1")]

    def trunc(x):
        return (x.view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32)

    def rf(out, exact):
        o = torch.from_numpy(out).double()
        return float(torch.linalg.norm(o - exact) / torch.linalg.norm(exact))

    for k in (32, 256, 1024, 2560, 8192, 32768):
        s = ProblemShape(512, 512, k)
        A = rng.uniform(-1, 1, (512, k)).astype(np.float32)
        B = rng.uniform(-1, 1, (k, 512)).astype(np.float32)
        C = np.zeros((512, 512), np.float32)
        At, Bt = trunc(A), trunc(B)
        ex = torch.from_numpy(A).double() @ torch.from_numpy(B).double()
        ext = torch.from_numpy(At).double() @ torch.from_numpy(Bt).double()
        row = {"K": k,
               "tf32_trunc": rf(gemm_execute(s, tf32, At, Bt, C, caps)[0], ext),
               "fp32_trunc": rf(gemm_execute(s, fp32, At, Bt, C, caps)[0], ext),
               "fp32": rf(gemm_execute(s, fp32, A, B, C, caps)[0], ex)}
        for c in x3s:
            row[c.canonical()] = rf(gemm_execute(s, c, A, B, C, caps)[0], ex)
        print(json.dumps({kk: (f"{v:.2e}" if isinstance(v, float) else v) for kk, v in row.items()}), flush=True)


if __name__ == "__main__":
    main()
