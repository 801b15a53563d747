"""Time the skinny_n / skinny_m candidates (profiles/skinny_probe.cu, kernels
from csrc/skinny.cuh) against the round-1 DT picks on the DeepBench skinny
shapes, L2 flushed before every sample; RF vs the float64 product.
Measurement only.   python profiles/skinny_probe.py  (on the GPU box)"""
import ctypes
import json
import os
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
SO = Path(os.environ.get("SKINNY_SO", str(HERE / "_skinny_probe.so")))

BASE = {  # round-1 DT picks (profiles/r01_bench.json per_shape)
    (1760, 16, 1760): "splitk:64-16-32-4-2-8", (2048, 16, 2048): "splitk:32-16-32-4-2-8",
    (4096, 16, 4096): "splitk:32-16-32-4-2-8", (7680, 16, 2560): "splitk:32-16-32-4-2-8",
    (3072, 16, 1024): "splitk:32-16-32-4-2-8", (2048, 32, 2048): "splitk:32-32-32-4-4-8",
    (4096, 32, 4096): "splitk:64-32-32-4-4-8", (2048, 64, 2048): "splitk:64-64-32-8-4-8",
    (4096, 64, 4096): "splitk:128-64-32-8-8-8", (2560, 64, 2560): "splitk:32-64-32-4-4-8",
    (35, 700, 2048): "splitk:16-32-32-2-4-8", (35, 1500, 2560): "splitk:16-32-32-2-4-4",
    (35, 8457, 2048): "splitk:64-128-32-8-8-4", (35, 8457, 2560): "splitk:64-128-32-8-8-8",
    (2048, 128, 2048): "splitk:128-128-32-8-8-16",
}


def main():
    import torch
    if not SO.exists():
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-shared",
                               "-Xcompiler", "-fPIC", f"-I{HERE.parent / 'include'}", "-o", str(SO),
                               str(HERE / "skinny_probe.cu"), "-lcuda"])
    L = ctypes.CDLL(str(SO))
    L.exp_time.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                           ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t,
                           ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
    L.do_flush_ext.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
    L.empty_launch.restype = ctypes.c_double
    L.empty_launch.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
    from paper_1806_07060_b200 import _native
    from paper_1806_07060_b200.kernels import DeviceCaps, KernelConfig, ProblemShape, native_shape
    lib = _native.lib()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    fb = flush.numel()
    mode = int(os.environ.get("FLUSH_MODE", "0"))
    L.set_flush_mode(mode)
    print(json.dumps({"flush_mode": mode, "empty_launch_us_best": round(L.empty_launch(flush.data_ptr(), fb, 50) * 1e6, 2)}),
          flush=True)
    n = L.exp_count()
    infos = []
    for i in range(n):
        t = (ctypes.c_int * 4)()
        L.exp_info(i, t)
        infos.append(tuple(t))
    ws = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream()
    only = os.environ.get("SHAPES")
    base_items = dict(BASE)
    if only == "midn":  # N = 64 / 128 shapes (the skinny_n DT picks), round-2 picks as the base
        base_items = {(1760, 64, 1760): "skinny_n:64-16-32-2-8-1", (2048, 64, 2048): "skinny_n:64-16-32-2-8-1",
                      (2560, 64, 2560): "skinny_n:64-16-32-2-8-1", (1760, 128, 1760): "skinny_n:64-32-32-2-8-1",
                      (2048, 128, 2048): "skinny_n:64-32-32-2-8-1", (4096, 64, 4096): "skinny_n:64-32-32-2-8-1",
                      (3072, 64, 1024): "skinny_n:64-16-32-2-8-1", (7680, 64, 2560): "skinny_n:64-32-32-2-8-1"}
    for (m, nn, k), base in base_items.items():
        if only == "m35" and m != 35:
            continue
        a = torch.rand(m, k, device="cuda") - 0.5
        b = torch.rand(k, nn, device="cuda") - 0.5
        out = torch.empty(m, nn, device="cuda")
        exact = a.double() @ b.double()
        flops = 2.0 * m * nn * k
        res = {}
        cfg = KernelConfig.from_canonical(base).native()
        ns = native_shape(ProblemShape(m, nn, k))
        caps = DeviceCaps.b200().native()
        ts = []
        for r in range(21):
            L.do_flush_ext(flush.data_ptr(), fb, r)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            lib.ag_gemm(ctypes.byref(ns), ctypes.byref(cfg), ctypes.byref(caps), 0, ctypes.c_void_p(a.data_ptr()),
                        k, ctypes.c_void_p(b.data_ptr()), nn, ctypes.c_void_p(out.data_ptr()), nn,
                        ctypes.c_void_p(out.data_ptr()), nn, ctypes.c_void_p(ws.data_ptr()), ws.numel(),
                        ctypes.c_void_p(st.cuda_stream))
            e1.record(st)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e-3)
        ts.sort()
        res["base " + base] = [round(ts[10] * 1e6, 2), round(flops / ts[10] / 1e12, 2)]
        best = None
        for i, (kind, p1, p2, p3) in enumerate(infos):
            if (kind == 0 and nn > 128) or (kind in (1, 2) and m > 64):
                continue
            if kind == 2 and m != 35:
                continue
            for s in (1, 2, 3, 4, 6, 8, 12, 16):
                sec = ctypes.c_double()
                out.zero_()
                rc = L.exp_time(i, m, nn, k, a.data_ptr(), b.data_ptr(), out.data_ptr(), s, flush.data_ptr(), fb, 21,
                                ctypes.byref(sec))
                name = (("skinny_n", "skinny_m", "skinny_m40x2[qk,nbuf,nw]")[kind]) + f"<{p1},{p2},{p3}>/s{s}"
                if rc:
                    res[name] = f"rc={rc}"
                    continue
                rf = float(torch.linalg.norm(out.double() - exact) / torch.linalg.norm(exact))
                res[name] = [round(sec.value * 1e6, 2), round(flops / sec.value / 1e12, 2), f"{rf:.1e}"]
                if rf < 1e-5 and (best is None or sec.value < best[0]):
                    best = (sec.value, name)
        print(json.dumps({"mnk": [m, nn, k], "base_us": res["base " + base][0],
                          "best": [best[1], round(best[0] * 1e6, 2)] if best else None, "results": res}), flush=True)


if __name__ == "__main__":
    main()
