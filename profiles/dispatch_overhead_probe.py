import cProfile, pstats, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_1806_07060_b200 import codegen, model
from paper_1806_07060_b200.kernels import KernelConfig, ProblemShape, DeviceCaps
tree = model.train([((64, 1, 1), 0), ((128, 1, 1), 0)])
sel = codegen.CompiledSelector(tree, {0: KernelConfig.from_canonical("indirect:64-64-16-8-4-1")})
s = ProblemShape(64, 64, 64)
A, B, C = (np.random.rand(64, 64).astype(np.float32) for _ in range(3))
out = np.empty((64, 64), np.float32)
caps = DeviceCaps.b200()
for _ in range(20): codegen.dispatch_native(sel, s, A, B, C, caps, out=out)
t0 = time.perf_counter()
for _ in range(200): codegen.dispatch_native(sel, s, A, B, C, caps, out=out)
print("host-path call us", (time.perf_counter() - t0) / 200 * 1e6)
dA, dB, dC, dO = (torch.from_numpy(x).cuda() for x in (A, B, C, out))
for _ in range(20): codegen.dispatch_native(sel, s, dA, dB, dC, caps, out=dO)
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(200): codegen.dispatch_native(sel, s, dA, dB, dC, caps, out=dO)
torch.cuda.synchronize(); print("device-path call us", (time.perf_counter() - t0) / 200 * 1e6)
pr = cProfile.Profile(); pr.enable()
for _ in range(200): codegen.dispatch_native(sel, s, dA, dB, dC, caps, out=dO)
pr.disable(); pstats.Stats(pr).sort_stats("tottime").print_stats(22)
