"""Streaming-read floor in bench.py's regime (256 MB write flush, event,
one kernel, event): microseconds to read N bytes with a plain chunked read
kernel, for the operand sizes of the DeepBench skinny shapes.  Measurement
only.   python profiles/read_floor.py   (on the GPU box)"""
import ctypes
import json
import os
import subprocess
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
SO = Path(os.environ.get("SKINNY_SO", str(HERE / "_skinny_probe.so")))


def main():
    import torch
    if not SO.exists():
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17", "-shared",
                               "-Xcompiler", "-fPIC", f"-I{HERE.parent / 'include'}", "-o", str(SO),
                               str(HERE / "skinny_probe.cu"), "-lcuda"])
    L = ctypes.CDLL(str(SO))
    L.read_floor.restype = ctypes.c_double
    L.read_floor.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                             ctypes.c_size_t, ctypes.c_int]
    L.empty_launch.restype = ctypes.c_double
    L.empty_launch.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    src = torch.empty(128 << 20, dtype=torch.uint8, device="cuda").fill_(1)
    for mode in (0, 2):
        L.set_flush_mode(mode)
        print(json.dumps({"flush_mode": mode,
                          "empty_us": round(L.empty_launch(flush.data_ptr(), flush.numel(), 41) * 1e6, 2)}), flush=True)
        for mb in (0.25, 1, 4, 8, 17, 34, 52, 70, 87, 120):
            nbytes = int(mb * (1 << 20)) // 4096 * 4096
            res = {}
            for ctas in (148, 296, 592, 1184):
                for un in (4, 8, 16):
                    t = L.read_floor(src.data_ptr(), nbytes, ctas, un, flush.data_ptr(), flush.numel(), 21)
                    res[f"{ctas}x{un}"] = round(t * 1e6, 2)
            best = min(res.items(), key=lambda kv: kv[1])
            print(json.dumps({"flush_mode": mode, "MB": mb, "best": best, "GBps": round(nbytes / best[1] / 1e3, 1),
                              "all": res}), flush=True)


if __name__ == "__main__":
    main()
