"""Per-shape end-to-end (host buffers) timings of the dispatch path with
1 / auto / 8 output panels, next to the PCIe copy rates (measurement only).

    python profiles/e2e_probe.py            (on the GPU box)
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch

    import bench
    from paper_1806_07060_b200 import codegen
    from paper_1806_07060_b200.kernels import DeviceCaps

    x = torch.empty(256 << 20, dtype=torch.uint8).pin_memory()
    d = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for name, fn in (("h2d", lambda: d.copy_(x, non_blocking=True)), ("d2h", lambda: x.copy_(d, non_blocking=True))):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        print(json.dumps({"copy": name, "GB/s": round(5 * x.numel() / (time.perf_counter() - t0) / 1e9, 1)}))
    m = bench.build_model()
    sel = codegen.CompiledSelector(m["tree"], m["classes"])
    caps = DeviceCaps.b200()
    from paper_1806_07060_b200.kernels import ProblemShape
    for s in [ProblemShape(8, 8, 8)] + m["db_all"][::3]:
        c = bench.ShapeCase(s, torch.device("cuda", 0))
        A, B, C = (torch.from_numpy(v).pin_memory() for v in c.host)
        hout = torch.empty((s.M, s.N), dtype=torch.float32).pin_memory()
        row = {"mnk": list(s.mnk), "cfg": sel.select(*s.mnk).canonical()}
        for panels in (1, 0, 8):
            best = 1e9
            for _ in range(4):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                codegen.dispatch_native(sel, s, A, B, C, caps, out=hout, panels=panels)
                best = min(best, time.perf_counter() - t0)
            row[f"ms_p{panels}"] = round(best * 1e3, 3)
        dt = 1e9
        for _ in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            codegen.dispatch_native(sel, s, c.dA, c.dB, c.dC, caps, out=c.dout)
            e1.record()
            torch.cuda.synchronize()
            dt = min(dt, e0.elapsed_time(e1))
        row["device_ms"] = round(dt, 3)
        row["bytes_mb"] = round((A.numel() + B.numel() + hout.numel()) * 4 / 1e6, 1)
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
