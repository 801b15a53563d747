"""tf32x3 against cuBLAS on the same operands (reference points only, not
product code): cuBLAS SGEMM (torch fp32 matmul, TF32 off), cuBLAS TF32
(torch, TF32 on), and the library's tf32x3 and best fp32 FFMA configs;
event-timed (warm, best of 5) and RF vs the float64 product.
    python profiles/x3_vs_cublas.py   (on the GPU box)"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch

    from paper_1806_07060_b200.kernels import DeviceCaps, KernelConfig, ProblemShape, gemm_execute
    caps = DeviceCaps.b200_tc()

    def timed(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e-3)
        return best

    for mnk in [(5124, 9124, 2560), (4096, 7000, 4096), (8192, 8192, 8192), (5124, 700, 2048)]:
        s = ProblemShape(*mnk)
        g = torch.Generator(device="cuda").manual_seed(0)
        a = torch.rand(s.M, s.K, device="cuda", generator=g) * 2 - 1
        b = torch.rand(s.K, s.N, device="cuda", generator=g) * 2 - 1
        c = torch.zeros(s.M, s.N, device="cuda")
        exact = a.double() @ b.double()
        rf = lambda o: float(torch.linalg.norm(o.double() - exact) / torch.linalg.norm(exact))  # noqa: E731
        fl = 2.0 * s.M * s.N * s.K
        row = {"mnk": list(mnk)}
        for name, tf32 in (("cublas_sgemm", False), ("cublas_tf32", True)):
            torch.backends.cuda.matmul.allow_tf32 = tf32
            out = torch.empty_like(c)
            t = timed(lambda: torch.matmul(a, b, out=out))
            row[name] = {"tflops": round(fl / t / 1e12, 1), "rf": f"{rf(out):.1e}"}
        torch.backends.cuda.matmul.allow_tf32 = False
        for name, cfg in (("ours_tf32x3", "tf32x3:128-128-32-3-1-1"), ("ours_fp32_ffma", "indirect:64-128-32-8-8-2")):
            k = KernelConfig.from_canonical(cfg)
            out = torch.empty_like(c)
            t = timed(lambda: gemm_execute(s, k, a, b, c, caps, out=out))
            row[name] = {"config": cfg, "tflops": round(fl / t / 1e12, 1), "rf": f"{rf(out):.1e}"}
        del exact
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
