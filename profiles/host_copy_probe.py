"""Host memory copy rates on the GPU box (measurement only): numpy copyto
from a touched pageable source into (a) a pinned buffer, (b) a touched
pageable buffer, (c) a freshly allocated pageable buffer (first-touch page
faults), with 1..16 threads (numpy releases the GIL in copyto).
    python profiles/host_copy_probe.py"""
import json
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np


def rate(dst_fn, src, threads, reps=5):
    n = src.size
    best = 1e9
    with ThreadPoolExecutor(threads) as ex:
        for _ in range(reps):
            dst = dst_fn()
            t0 = time.perf_counter()
            parts = [(n * i // threads, n * (i + 1) // threads) for i in range(threads)]
            list(ex.map(lambda p: np.copyto(dst[p[0]:p[1]], src[p[0]:p[1]]), parts))
            best = min(best, time.perf_counter() - t0)
    return src.nbytes / best / 1e9


def main():
    import torch
    for mb in (16, 256):
        n = mb * (1 << 20) // 4
        src = np.random.default_rng(0).random(n, dtype=np.float32)
        pinned = torch.empty(n, dtype=torch.float32).pin_memory().numpy()
        touched = np.ones(n, np.float32)
        for th in (1, 2, 4, 8, 16):
            print(json.dumps({"MB": mb, "threads": th,
                              "to_pinned_GBps": round(rate(lambda: pinned, src, th), 1),
                              "to_touched_GBps": round(rate(lambda: touched, src, th), 1),
                              "to_fresh_GBps": round(rate(lambda: np.empty(n, np.float32), src, th), 1)}),
                  flush=True)
    # pinned <-> device DMA for reference
    x = torch.empty(256 << 18, dtype=torch.float32).pin_memory()
    d = torch.empty_like(x, device="cuda")
    for name, f in (("h2d", lambda: d.copy_(x, non_blocking=True)), ("d2h", lambda: x.copy_(d, non_blocking=True))):
        f(); torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5):
            f()
        torch.cuda.synchronize()
        print(json.dumps({"dma": name, "GBps": round(5 * x.numel() * 4 / (time.perf_counter() - t0) / 1e9, 1)}))


if __name__ == "__main__":
    main()
