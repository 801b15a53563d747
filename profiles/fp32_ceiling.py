"""FP32 ceilings next to the indirect core (measurement only; prints JSON lines).

* ffma_peak: the roofline denominator bench.py uses (FFMA with a uniform
  register and a reused source: the cheapest FFMA form).
* smem_outer TMxTN @ c CTA/SM: the indirect core's LDS.128 + register-tile
  inner loop with shared-memory-resident tiles and no global traffic
  (profiles/ceiling.cu) -- the ceiling of that register tiling.
* cublas_sgemm: torch.matmul fp32 with TF32 disabled (cuBLAS SGEMM), a
  library reference point only (the product path never calls cuBLAS).
* ours: the shipped tables' best indirect config, device time from ag_tune
  (median of 5, warm buffers, pack helpers included).

    python profiles/fp32_ceiling.py            (on the GPU box)
"""
import ctypes
import json
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))

SHAPES = [(4096, 4096, 4096), (8192, 8192, 8192), (5124, 9124, 2560), (4096, 7000, 4096), (2048, 7000, 2048)]


def ceiling_lib():
    so = HERE / "_ceiling.so"
    if not so.exists():
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared",
                               "-Xcompiler", "-fPIC", "-o", str(so), str(HERE / "ceiling.cu")])
    lib = ctypes.CDLL(str(so))
    lib.smem_outer_tflops.argtypes = [ctypes.c_int] * 5 + [ctypes.POINTER(ctypes.c_double)]
    return lib


def main():
    import torch

    from paper_1806_07060_b200.kernels import DeviceCaps, KernelConfig, ProblemShape, ffma_peak_tflops
    from paper_1806_07060_b200.tuner import DeviceBuffers, TimingPolicy, time_configs

    torch.cuda.init()
    print(json.dumps({"probe": "ffma_peak", "tflops": round(ffma_peak_tflops(), 2)}), flush=True)
    lib = ceiling_lib()
    for paired in (0, 1):
        for tm, tn, c in ((8, 8, 1), (8, 8, 2), (8, 4, 1), (4, 4, 1)):
            v = ctypes.c_double()
            lib.smem_outer_tflops(tm, tn, c, 2000, paired, ctypes.byref(v))
            print(json.dumps({"probe": f"smem_outer {tm}x{tn} @ {c} CTA/SM" + (" FFMA2" if paired else " FFMA"),
                              "tflops": round(v.value, 2)}), flush=True)

    torch.backends.cuda.matmul.allow_tf32 = False
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    caps = DeviceCaps.b200()
    cands = ["indirect:128-128-32-8-8-1", "indirect:128-128-16-8-8-1", "indirect:128-128-32-8-8-2",
             "indirect:64-128-32-8-8-1", "indirect:128-64-32-8-8-1", "indirect:64-64-16-8-8-1"]
    for m, n, k in SHAPES:
        a = torch.rand(m, k, device="cuda") - 0.5
        b = torch.rand(k, n, device="cuda") - 0.5
        best = float("inf")
        for _ in range(7):
            flush.fill_(1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.matmul(a, b)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e-3)
        line = {"probe": "cublas_sgemm", "mnk": [m, n, k], "tflops": round(2 * m * n * k / best / 1e12, 2)}
        s = ProblemShape(m, n, k)
        bufs = DeviceBuffers(s)
        cfgs = [KernelConfig.from_canonical(x) for x in cands]
        secs = time_configs(s, cfgs, caps, TimingPolicy(warmup=1, repeats=5), bufs)
        line["ours"] = {c: round(2 * m * n * k / t / 1e12, 2) for c, t in zip(cands, secs)}
        print(json.dumps(line), flush=True)
        del a, b, bufs
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
