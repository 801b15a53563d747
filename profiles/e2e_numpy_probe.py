"""Host-buffer call cost per DeepBench shape for the three ways a numpy
caller's bytes can cross PCIe (measurement only):
  pageable   -- ag_gemm_host_ex, flags 0 (the driver stages each copy)
  register   -- ag_gemm_host_ex, AG_HOST_REGISTER (page-locked for the call)
  stage      -- ag_gemm_host_ex, AG_HOST_STAGE (pinned rings + host copy workers)
  stage_fresh -- AG_HOST_STAGE into a freshly allocated output each call (numpy's out=None)
  pinned     -- the operands already in pinned memory (torch pin_memory)
    python profiles/e2e_numpy_probe.py     (on the GPU box)"""
import ctypes
import json
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import numpy as np
    import torch

    import bench
    from paper_1806_07060_b200 import _native, codegen
    from paper_1806_07060_b200.kernels import DeviceCaps, ProblemShape, native_shape
    from paper_1806_07060_b200.tuner import _bench_buffers
    lib = _native.lib()
    m = bench.build_model()
    sel = codegen.CompiledSelector(m["tree"], m["classes"])
    caps = DeviceCaps.b200()
    nc = caps.native()
    for s in [ProblemShape(64, 64, 64), ProblemShape(256, 256, 256)] + m["db_all"][::4]:
        A, B, C, out = _bench_buffers(s, np.float32, 0)
        cfg = sel.select(*s.mnk).native()
        ns = native_shape(s)
        row = {"mnk": list(s.mnk), "mb": round((A.nbytes + B.nbytes + out.nbytes) / 1e6, 1)}
        secs = ctypes.c_double()
        for name, flags in (("pageable", 0), ("register", 1), ("stage", 2), ("stage_fresh", 2)):
            ts = []
            for _ in range(4):
                if name == "stage_fresh":
                    out = np.empty_like(out)
                t0 = time.perf_counter()
                rc = lib.ag_gemm_host_ex(ctypes.byref(ns), ctypes.byref(cfg), ctypes.byref(nc), 0, A.ctypes.data,
                                         A.shape[1], B.ctypes.data, B.shape[1], C.ctypes.data, C.shape[1],
                                         out.ctypes.data, out.shape[1], None, 0, 0, flags, None, ctypes.byref(secs))
                ts.append(time.perf_counter() - t0)
                assert rc == 0, _native.last_error()
            row[name + "_ms"] = round(statistics.median(ts[1:]) * 1e3, 3)
        row["kernel_ms"] = round(secs.value * 1e3, 3)
        pA, pB, pC = (torch.from_numpy(x).pin_memory() for x in (A, B, C))
        po = torch.empty(out.shape, dtype=torch.float32).pin_memory()
        ts = []
        for _ in range(4):
            t0 = time.perf_counter()
            codegen.dispatch_native(sel, s, pA, pB, pC, caps, out=po)
            ts.append(time.perf_counter() - t0)
        row["pinned_ms"] = round(statistics.median(ts[1:]) * 1e3, 3)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
