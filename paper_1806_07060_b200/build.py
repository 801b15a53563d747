"""Build libadaptgemm_b200.so in-tree (sm_100a, no GPU needed).

Generates one launcher table per translation unit from `spaces.py`,
compiles the units in parallel with nvcc (-gencode arch=compute_100a,
code=sm_100a -lineinfo) and links them with the C-ABI (abi.cu) and the
host decision-tree code (dtree.cpp) into
`paper_1806_07060_b200/_lib/libadaptgemm_b200.so`.  Incremental: a unit is
recompiled only when its source or a header is newer than its object.

    python -m paper_1806_07060_b200.build [--jobs N] [--force]
"""

import argparse
import concurrent.futures
import os
import re
import subprocess
import sys
import time
from pathlib import Path

if __package__ in (None, ""):
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    from paper_1806_07060_b200 import spaces  # type: ignore
else:
    from . import spaces

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
GEN = CSRC / "gen"
BUILD = PKG / "_build"
LIBDIR = PKG / "_lib"
LIB = LIBDIR / "libadaptgemm_b200.so"
INCLUDE = PKG.parent / "include"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
                     "-Xcompiler", "-fPIC", "-Xptxas", "-v", f"-I{INCLUDE}"]
CXX = os.environ.get("CXX", "g++")
CXX_FLAGS = ["-O2", "-fPIC", "-std=c++17", "-Wall", f"-I{INCLUDE}"]

N_UNITS = 48
FAMILY_CODE = {"direct": 0, "indirect": 1, "splitk": 2, "tf32": 3, "bf16": 4, "tma": 5, "skinny_n": 6, "skinny_m": 7, "tf32x3": 8}


def _cost(t):
    """Rough ptxas cost of one instantiation (bigger tiles unroll more)."""
    fam, bm, bn, bk, tm, tn, uk = t
    return 1.0 + tm * tn * bk / 64.0


def kernel_entries():
    """(family, dtype, bm, bn, bk, tm, tn, uk, launcher) for every instantiation."""
    out = []
    for t in spaces.compiled_tuples():
        fam, bm, bn, bk, tm, tn, uk = t
        if fam == "direct":
            fn = f"&ag::launch_direct<float, {bm}, {bn}, {bk}, {tm}, {tn}>"
        else:
            fn = f"&ag::launch_indirect<float, {bm}, {bn}, {bk}, {tm}, {tn}, {uk}>"
        out.append((FAMILY_CODE[fam], 0, bm, bn, bk, tm, tn, uk, fn, _cost(t)))
    # split-K family: the indirect core with the in-place row-major-A loader
    # (key uk = 0: the slice count is a run-time argument)
    for bm, bn, tm, tn in spaces.SPLITK_TILES:
        for bk in spaces.SPLITK_BLOCK_K:
            out.append((2, 0, bm, bn, bk, tm, tn, 0,
                        f"&ag::launch_indirect<float, {bm}, {bn}, {bk}, {tm}, {tn}, 1, true>",
                        _cost(("splitk", bm, bn, bk, tm, tn, 1))))
    # TMA family: the TMA-fed core per tile (falls back to the packed core
    # with the same tile for transposed / unaligned operands)
    for bm, bn, tm, tn in spaces.TMA_TILES:
        out.append((5, 0, bm, bn, spaces.TMA_BLOCK_K, tm, tn, 1,
                    f"&ag::f32tma::launch_tma_family<{bm}, {bn}, {tm}, {tn}>", 2.0 + tm * tn * 32 / 64.0))
    # skinny families (csrc/skinny.cuh): one kernel per tile; the K slice
    # count is a run-time argument (key uk = 0)
    for tm, bn in spaces.SKINNY_N_TILES:
        for w in spaces.SKINNY_N_WARPS:
            if spaces.is_legal_tuple("skinny_n", 32 * tm, bn, spaces.SKINNY_BLOCK_K, tm, w, 1, spaces.B200_CAPS):
                out.append((6, 0, 32 * tm, bn, spaces.SKINNY_BLOCK_K, tm, w, 0,
                            f"&ag::skinny::launch_n<{tm}, {bn}, {w}>", 3.0 + tm * bn / 16.0))
    for bm, tn in spaces.SKINNY_M_TILES:
        for w in spaces.SKINNY_M_WARPS:
            out.append((7, 0, bm, 32 * w * tn, spaces.SKINNY_BLOCK_K, 1, tn, 0,
                        f"&ag::skinny::launch_m<{bm}, {tn}, {w}>", 3.0 + bm * tn / 16.0))
    # tensor-core families: one persistent tcgen05 kernel per (kind, bn, stages)
    for fam in spaces.TC_FAMILIES:
        for t in spaces.enumerate_tuples(fam, spaces.B200_CAPS, spaces.PROFILE_B200_TC):
            _, bm, bn, bk, tm, tn, uk = t
            kind = {"tf32": "ag::tc::KIND_TF32", "bf16": "ag::tc::KIND_BF16", "tf32x3": "ag::tc::KIND_TF32X3"}[fam]
            out.append((FAMILY_CODE[fam], 0, bm, bn, bk, tm, tn, uk,
                        f"&ag::tc::launch_tc<{kind}, {bn}, {tm}, {bm // 128}>", 3.0))
    for dcode, ctype in ((0, "float"), (1, "double")):
        for tm in spaces.RUNTIME_TILES:
            for tn in spaces.RUNTIME_TILES:
                out.append((0, dcode, 0, 0, 0, tm, tn, 0,
                            f"&ag::launch_direct<{ctype}, 0, 0, 0, {tm}, {tn}>", 2.0))
                out.append((1, dcode, 0, 0, 0, tm, tn, 0,
                            f"&ag::launch_indirect<{ctype}, 0, 0, 0, {tm}, {tn}, 1>", 2.0))
    # float64 run-time kernels for the B200 wide register tiles (their float32
    # configs all have fixed instantiations)
    for tm, tn in spaces.RUNTIME_WIDE_TILES:
        out.append((1, 1, 0, 0, 0, tm, tn, 0, f"&ag::launch_indirect<double, 0, 0, 0, {tm}, {tn}, 1>", 4.0))
    return out


def _write_if_changed(path: Path, text: str):
    if path.exists() and path.read_text() == text:
        return
    path.write_text(text)


def generate():
    GEN.mkdir(parents=True, exist_ok=True)
    entries = kernel_entries()
    # greedy cost balancing into N_UNITS translation units
    units = [[] for _ in range(N_UNITS)]
    loads = [0.0] * N_UNITS
    for e in sorted(entries, key=lambda e: -e[-1]):
        i = loads.index(min(loads))
        units[i].append(e)
        loads[i] += e[-1]
    names = []
    for u, ents in enumerate(units):
        ents.sort(key=lambda e: e[:8])
        lines = ["// generated by paper_1806_07060_b200/build.py -- do not edit",
                 '#include "../launch.cuh"', '#include "../tc_kernels.cuh"', '#include "../fp32_tma.cuh"',
                 '#include "../skinny.cuh"', "", "namespace {",
                 "const ag::KernelEntry kEntries[] = {"]
        for fam, dt, bm, bn, bk, tm, tn, uk, fn, _ in ents:
            lines.append(f"    {{{fam}, {dt}, {bm}, {bn}, {bk}, {tm}, {tn}, {uk}, {fn}}},")
        lines += ["};", "}  // namespace", "",
                  f"const ag::KernelEntry* ag_gen_table_{u:02d}(int* n) {{",
                  "    *n = (int)(sizeof(kEntries) / sizeof(kEntries[0]));",
                  "    return kEntries;", "}", ""]
        _write_if_changed(GEN / f"inst_{u:02d}.cu", "\n".join(lines))
        names.append(f"ag_gen_table_{u:02d}")
    lines = ["// generated by paper_1806_07060_b200/build.py -- do not edit",
             '#include "../registry.h"', ""]
    lines += [f"const ag::KernelEntry* {n}(int* n);" for n in names]
    lines += ["", "extern const ag::EntryTableFn g_entry_tables[] = {"]
    lines += [f"    &{n}," for n in names]
    lines += ["};", f"extern const int g_num_entry_tables = {len(names)};", ""]
    _write_if_changed(GEN / "tables.cu", "\n".join(lines))
    # drop stale units from an earlier, larger N_UNITS
    for p in GEN.glob("inst_*.cu"):
        if int(p.stem.split("_")[1]) >= N_UNITS:
            p.unlink()
    return len(entries)


def _headers_mtime():
    hs = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + list(INCLUDE.glob("*.h"))
    return max(p.stat().st_mtime for p in hs)


def _compile(src: Path, obj: Path, force: bool, hdr_mtime: float):
    if (not force and obj.exists() and obj.stat().st_mtime > src.stat().st_mtime
            and obj.stat().st_mtime > hdr_mtime):
        return src.name, 0.0, ""
    t0 = time.time()
    if src.suffix == ".cpp":
        cmd = [CXX] + CXX_FLAGS + ["-c", str(src), "-o", str(obj)]
    else:
        cmd = [NVCC] + NVCC_FLAGS + ["-c", str(src), "-o", str(obj)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    (BUILD / (obj.stem + ".ptxas.log")).write_text(res.stderr)
    return src.name, time.time() - t0, res.stderr


def spill_report():
    """Kernels whose ptxas report shows spill stores/loads (empty = none)."""
    bad = []
    for log in BUILD.glob("*.ptxas.log"):
        func = None
        for line in log.read_text().splitlines():
            m = re.search(r"Compiling entry function '([^']+)'", line)
            if m:
                func = m.group(1)
            m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
            if m and (int(m.group(1)) or int(m.group(2))):
                bad.append((func, int(m.group(1)), int(m.group(2))))
    return bad


def build(jobs: int | None = None, force: bool = False, verbose: bool = True) -> Path:
    t0 = time.time()
    n = generate()
    BUILD.mkdir(parents=True, exist_ok=True)
    LIBDIR.mkdir(parents=True, exist_ok=True)
    srcs = sorted(GEN.glob("*.cu")) + [CSRC / "abi.cu", CSRC / "dtree.cpp"]
    objs = [BUILD / (s.stem + ".o") for s in srcs]
    hdr = _headers_mtime()
    jobs = jobs or os.cpu_count() or 4
    compiled = 0
    with concurrent.futures.ThreadPoolExecutor(max_workers=jobs) as ex:
        futs = [ex.submit(_compile, s, o, force, hdr) for s, o in zip(srcs, objs)]
        for f in concurrent.futures.as_completed(futs):
            name, dt, _ = f.result()
            if dt:
                compiled += 1
                if verbose:
                    print(f"  built {name} in {dt:.1f}s", flush=True)
    newest = max(o.stat().st_mtime for o in objs)
    if force or compiled or not LIB.exists() or LIB.stat().st_mtime < newest:
        tmp = LIB.with_suffix(".so.tmp")
        cmd = [NVCC] + ARCH + ["-shared", "-o", str(tmp)] + [str(o) for o in objs] + \
              ["-lpthread", "-ldl", "-lrt"]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
        os.replace(tmp, LIB)
    build_fastpath(force)
    if verbose:
        print(f"libadaptgemm_b200.so: {n} kernel instantiations, {compiled} units rebuilt, "
              f"{time.time() - t0:.1f}s", flush=True)
    return LIB


FASTPATH_SRC = CSRC / "fastpath.c"


def fastpath_path() -> Path:
    import sysconfig
    return PKG / ("_fastpath" + sysconfig.get_config_var("EXT_SUFFIX"))


def build_fastpath(force: bool = False) -> Path:
    """The CPython extension for the numpy call path (csrc/fastpath.c),
    linked against libadaptgemm_b200.so through rpath $ORIGIN/_lib."""
    import sysconfig
    out = fastpath_path()
    deps = [FASTPATH_SRC, INCLUDE / "adaptgemm_b200.h", LIB]
    if not force and out.exists() and out.stat().st_mtime > max(d.stat().st_mtime for d in deps):
        return out
    cmd = ["gcc", "-O2", "-fPIC", "-shared", "-Wall", f"-I{sysconfig.get_paths()['include']}", f"-I{INCLUDE}",
           str(FASTPATH_SRC), "-o", str(out), f"-L{LIBDIR}", "-ladaptgemm_b200", "-Wl,-rpath,$ORIGIN/_lib"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"fastpath build failed: {' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
    return out


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--jobs", type=int, default=None)
    ap.add_argument("--force", action="store_true")
    args = ap.parse_args(argv)
    build(args.jobs, args.force)
    spills = spill_report()
    if spills:
        print(f"WARNING: {len(spills)} kernels spill registers, e.g. {spills[:3]}")


if __name__ == "__main__":
    main()
