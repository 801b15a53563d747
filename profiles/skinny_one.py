"""Run one skinny probe config a few times (for ncu).
    python profiles/skinny_one.py KIND P1 P2 P3 SLICES M N K [REPS]   (KIND 0 skinny_n, 1 skinny_m)"""
import ctypes
import sys
from pathlib import Path

import torch

HERE = Path(__file__).resolve().parent
L = ctypes.CDLL(str(HERE / "_skinny_probe.so"))
L.exp_time.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                       ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int,
                       ctypes.POINTER(ctypes.c_double)]
kind, p1, p2, p3, s, m, n, k = (int(x) for x in sys.argv[1:9])
reps = int(sys.argv[9]) if len(sys.argv) > 9 else 3
idx = None
for i in range(L.exp_count()):
    t = (ctypes.c_int * 4)()
    L.exp_info(i, t)
    if tuple(t) == (kind, p1, p2, p3):
        idx = i
assert idx is not None
L.set_flush_mode(2)
a = torch.rand(m, k, device="cuda") - 0.5
b = torch.rand(k, n, device="cuda") - 0.5
out = torch.empty(m, n, device="cuda")
sec = ctypes.c_double()
rc = L.exp_time(idx, m, n, k, a.data_ptr(), b.data_ptr(), out.data_ptr(), s, out.data_ptr(), 0, reps, ctypes.byref(sec))
print(rc, sec.value)
