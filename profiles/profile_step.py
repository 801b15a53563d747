"""One bench step under ncu: warm passes, then exactly one DT pass between
cudaProfilerStart/Stop (run ncu with --profile-from-start off).

    ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none \
        --csv --log-file gpurun_out/launches.csv python profiles/profile_step.py
    ncu --profile-from-start off --set full --clock-control none --import-source on \
        -k regex:tiled_gemm -c 1 -o gpurun_out/prof python profiles/profile_step.py --only 5124x9124x2560
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1806_07060_b200 import codegen  # noqa: E402
from paper_1806_07060_b200.kernels import DeviceCaps  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=None, help="MxNxK: profile just this shape")
    ap.add_argument("--warm", type=int, default=2)
    args = ap.parse_args()
    device = torch.device("cuda", 0)
    m = bench.build_model()
    sel = codegen.CompiledSelector(m["tree"], m["classes"])
    fb = codegen.FALLBACK_CONFIG.native()
    shapes = m["db_all"]
    if args.only:
        want = tuple(int(x) for x in args.only.split("x"))
        shapes = [s for s in shapes if s.mnk == want]
    cases = [bench.ShapeCase(s, device) for s in shapes]
    runner = bench.Runner(device, DeviceCaps.b200())
    for _ in range(args.warm):
        runner.pass_(cases, lambda i, c: runner.launch(c, selector=sel, fallback=fb))
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    runner.pass_(cases, lambda i, c: runner.launch(c, selector=sel, fallback=fb))
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    for s in shapes:
        print(s.mnk, sel.select(*s.mnk).canonical())


if __name__ == "__main__":
    main()
