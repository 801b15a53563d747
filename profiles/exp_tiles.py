"""Time candidate indirect-core tiles (profiles/exp_tiles.cu) on tile-multiple
shapes, plus an RF check against a float64 product (measurement only).

    python profiles/exp_tiles.py          (on the GPU box)
"""
import ctypes
import json
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
SHAPES = [(4096, 4096, 4096), (8192, 8192, 8192), (5124, 9124, 2560), (4096, 7000, 4096), (2048, 7000, 2048),
          (1024, 1024, 1024), (1760, 7000, 1760)]


def lib():
    import os
    so = Path(os.environ.get("EXP_SO", str(HERE / "_exp_tiles.so")))
    if not so.exists():
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                               "-shared", "-Xcompiler", "-fPIC", f"-I{HERE.parent / 'include'}", "-o", str(so),
                               str(HERE / "exp_tiles.cu")])
    L = ctypes.CDLL(str(so))
    L.exp_ws.restype = ctypes.c_size_t
    L.exp_ws.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int]
    L.exp_time.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                           ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int,
                           ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
    return L


def main():
    import os
    import torch
    if os.environ.get("EXP_SKINNY"):
        return skinny(torch)
    L = lib()
    n = L.exp_count()
    tiles = []
    for i in range(n):
        t = (ctypes.c_int * 6)()
        L.exp_tile(i, t)
        tiles.append("-".join(map(str, t)))
    only_stage = os.environ.get("EXP_STAGES")  # only the ring-depth variants (uk field >= 100)
    shapes = [(5124, 9124, 2560), (4096, 7000, 4096), (2560, 7000, 2560), (8192, 8192, 8192)] if only_stage else SHAPES
    for (m, nn, k) in shapes:
        a = torch.rand(m, k, device="cuda") - 0.5
        b = torch.rand(k, nn, device="cuda") - 0.5
        out = torch.empty(m, nn, device="cuda")
        ref = None
        res = {}
        for i in range(n):
            if only_stage and int(tiles[i].split("-")[-1]) < 100:
                continue
            ws_n = L.exp_ws(i, m, nn, k, 1)
            ws = torch.empty(ws_n, dtype=torch.uint8, device="cuda")
            sec = ctypes.c_double()
            rc = L.exp_time(i, m, nn, k, a.data_ptr(), b.data_ptr(), out.data_ptr(), ws.data_ptr(), ws_n, 5,
                            1, ctypes.byref(sec))
            if rc:
                res[tiles[i]] = f"rc={rc}"
                continue
            entry = round(2 * m * nn * k / sec.value / 1e12, 2)
            if m <= 4096 and k <= 4096:
                if ref is None:
                    ref = (a.double() @ b.double())
                rf = float(torch.linalg.norm(out.double() - ref) / torch.linalg.norm(ref))
                entry = [entry, f"rf={rf:.1e}"]
            res[tiles[i]] = entry
        print(json.dumps({"mnk": [m, nn, k], "tflops": res}), flush=True)
        del a, b, out, ref
        torch.cuda.empty_cache()


SKINNY = [(4096, 16, 4096), (2048, 16, 2048), (7680, 16, 2560), (1760, 16, 1760), (3072, 16, 1024),
          (4096, 32, 4096), (1760, 32, 1760), (7680, 32, 2560)]


def skinny(torch):
    """In-place split-K candidates (uk = 0 rows) on N <= 32 shapes, slices 2..32."""
    L = lib()
    n = L.exp_count()
    tiles = []
    for i in range(n):
        t = (ctypes.c_int * 6)()
        L.exp_tile(i, t)
        tiles.append(tuple(t))
    for (m, nn, k) in SKINNY:
        a = torch.rand(m, k, device="cuda") - 0.5
        b = torch.rand(k, nn, device="cuda") - 0.5
        out = torch.empty(m, nn, device="cuda")
        res = {}
        for i, t in enumerate(tiles):
            if t[5] != 0 or t[1] > nn:
                continue
            best = None
            for splits in (2, 4, 8, 16):
                ws_n = L.exp_ws(i, m, nn, k, splits)
                ws = torch.empty(ws_n, dtype=torch.uint8, device="cuda")
                sec = ctypes.c_double()
                rc = L.exp_time(i, m, nn, k, a.data_ptr(), b.data_ptr(), out.data_ptr(), ws.data_ptr(), ws_n, 7,
                                splits, ctypes.byref(sec))
                if rc == 0 and (best is None or sec.value < best[0]):
                    best = (sec.value, splits)
            if best:
                res["-".join(map(str, t[:5]))] = [round(2 * m * nn * k / best[0] / 1e12, 2), best[1]]
        print(json.dumps({"mnk": [m, nn, k], "tflops_slices": res}), flush=True)


if __name__ == "__main__":
    main()
