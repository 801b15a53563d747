"""Small calls through every kernel family for compute-sanitizer
(memcheck / racecheck / synccheck); measurement only.

    compute-sanitizer --tool memcheck python profiles/sanitize_probe.py
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_1806_07060_b200 import codegen, model  # noqa: E402
from paper_1806_07060_b200.kernels import DeviceCaps, KernelConfig, ProblemShape, gemm_execute  # noqa: E402

CASES = [
    ((67, 45, 36), "direct:16-16-8-2-2-1"),
    ((67, 45, 36), "indirect:64-32-16-8-4-2"),
    ((67, 45, 36), "indirect:128-128-32-8-8-1"),
    ((100, 68, 512), "splitk:32-32-16-4-4-4"),     # in-place core + cluster reduction
    ((100, 68, 510), "splitk:32-32-16-4-4-4"),     # packed core + slab reduction (K % 4 != 0)
    ((100, 68, 1024), "splitk:32-32-16-4-4-32"),   # in-place core, slab path (> 16 slices)
    ((130, 70, 100), "tma:64-64-32-8-8-1"),        # TMA core
    ((130, 70, 100), "tma:128-128-32-8-8-1"),
    ((300, 260, 200), "bf16:256-128-64-4-1-1"),    # tcgen05 CTA pair
    ((300, 260, 200), "tf32:128-64-32-4-1-1"),
    ((300, 260, 600), "tf32x3:128-128-32-3-1-1"),  # 3xTF32, 3 TMEM chunks, running sum
    ((300, 260, 600), "tf32x3:256-64-32-3-1-1"),   # 3xTF32 CTA pair
    ((1000, 16, 1024), "skinny_n:64-16-32-2-4-4"),  # skinny_n, 4-CTA cluster reduction
    ((35, 1001, 512), "skinny_m:40-256-32-1-2-4"),  # skinny_m, N % 4 != 0
]


def main():
    caps = DeviceCaps.b200_tc()
    rng = np.random.default_rng(0)
    for (m, n, k), name in CASES:
        s = ProblemShape(m, n, k, alpha=1.0, beta=0.5)
        A, B, C = (rng.uniform(-1, 1, d).astype(np.float32) for d in ((m, k), (k, n), (m, n)))
        out, _ = gemm_execute(s, KernelConfig.from_canonical(name), A, B, C, caps)
        ref = A.astype(np.float64) @ B.astype(np.float64) + 0.5 * C
        rf = np.linalg.norm(out - ref) / np.linalg.norm(ref)
        print(f"{name} {m}x{n}x{k} rf={rf:.1e}", flush=True)
    tree = model.train([((64, 1, 1), 0), ((128, 1, 1), 0)])
    sel = codegen.CompiledSelector(tree, {0: KernelConfig.from_canonical("tma:64-64-32-8-8-1")})
    s = ProblemShape(700, 300, 128)
    A, B, C = (rng.uniform(-1, 1, d).astype(np.float32) for d in ((700, 128), (128, 300), (700, 300)))
    codegen.dispatch_native(sel, s, A, B, C, caps, panels=3)
    print("host path ok", flush=True)
    # staged host path: pageable numpy through the pinned rings, 4 panels, the
    # output draining on its own host thread, the result in a pinned block
    s = ProblemShape(2048, 2048, 1024)
    A, B, C = (rng.uniform(-1, 1, d).astype(np.float32) for d in ((2048, 1024), (1024, 2048), (2048, 2048)))
    out, _ = gemm_execute(s, KernelConfig.from_canonical("indirect:64-64-32-8-8-1"), A, B, C, caps)
    ref = A[:64].astype(np.float64) @ B.astype(np.float64)
    print(f"staged host path rf={np.linalg.norm(out[:64] - ref) / np.linalg.norm(ref):.1e}", flush=True)


if __name__ == "__main__":
    main()
