#!/usr/bin/env python
"""bench.py -- DT-selected vs oracle vs default-tile GEMM throughput on B200.

Metric (BASELINE.json): geomean GFLOP/s over a GEMM shape set for the
decision-tree-selected kernels, next to the per-shape exhaustive best
("oracle") and the fixed default tile.  Workload: the DeepBench-style
rectangular set (configs[2]; paper_1806_07060_b200/data/deepbench_fp32.txt),
fp32, alpha=1, beta=0, no transposes, operands from the reference's
_bench_buffers recipe.  The po2 64..4096 held-out split (configs[1]) is
reported beside it.

The tree is the reference pipeline's (dataset -> seeded 80/20 split ->
5x8 CART grid -> best test DTPR) trained on the exhaustive B200 tuning
tables of generated shape sets shipped in paper_1806_07060_b200/data/ (po2
16..4096 + 512 octave-uniform random shapes, configs/headline_b200.json;
produced on a B200 by `python -m paper_1806_07060_b200.cli tune`).  No
DeepBench table is used in training or model selection.  The DeepBench
tables give the oracle per shape; the default tile is the BaselinePolicy
anchored on the 256^3 / 1024^3 po2 tables; all three are re-measured live.

One step = one pass over the shape set: per shape, L2 flushed (256 MB
write), then the DT path -- native branch-free select + launch through the
C-ABI (ag_dispatch_gemm) on operands resident in HBM -- bracketed by CUDA
events on the launching stream.  value = geomean over shapes of
2MNK / trimmed-mean event time.  e2e = the same metric through the public Python
API with host (numpy) buffers, host<->device copies inside the timed call.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

DATA = ROOT / "paper_1806_07060_b200" / "data"
PO2_BUNDLE = DATA / "tables_b200_po2.csv.gz"
DB_BUNDLE = DATA / "tables_b200_deepbench.csv.gz"
TC_BUNDLE = DATA / "tables_b200tc_random.csv.gz"
GO2_BUNDLE = DATA / "tables_b200_go2.csv.gz"
# 512 octave-uniform random shapes in [16, 4096) (configs/lograndom_b200.json),
# swept over the full B200 space in the bench's regime; joins po2 in the
# headline model's training set
LOGRANDOM_BUNDLE = DATA / "tables_b200_lograndom.csv.gz"
# the tf32x3 rows of the same shapes and timing regime (configs/*_x3.json),
# merged per shape into the fp32 tables by x3_section
X3_PO2_BUNDLE = DATA / "tables_x3_po2.csv.gz"
X3_DB_BUNDLE = DATA / "tables_x3_deepbench.csv.gz"
X3_LOGRANDOM_BUNDLE = DATA / "tables_x3_lograndom.csv.gz"
TRAFFIC_FILE = ROOT / "profiles" / "roofline_traffic.json"
NOMINAL_FP32_TFLOPS = 148 * 128 * 2 * 1.965e9 / 1e12  # 74.4
FLUSH_BYTES = 256 << 20  # > 126 MB L2
SPLIT_SEED, SPLIT_FRACTION = 2024, 0.8
METRIC = "geomean GFLOP/s over GEMM shape set: DT-selected vs oracle vs default tile"
# the reference's CPU default tiles (BaselinePolicy tuned at 256^3 / 1024^3 on
# the reference's CPU kernels)
CPU_DEFAULT_DIRECT = "direct:32-32-16-2-4-1"
CPU_DEFAULT_INDIRECT = "indirect:64-32-16-4-8-2"
CPU_SAMPLE_FLOPS = 1.0e8  # per shape per reference step: output rows sized to ~20-50 ms


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def geomean(xs):
    xs = list(xs)
    return math.exp(sum(math.log(x) for x in xs) / len(xs))


def trimmed_mean(xs):
    """Mean after dropping the lowest and highest quarter.  One GEMM per
    sample, and B200 CUDA-event timestamps tick in 2.048 us steps
    (profiles/r02_skinny_probe_*.jsonl), so a median of a microsecond-scale
    GEMM is stuck on a tick; the mean of the middle samples is not."""
    xs = sorted(xs)
    d = len(xs) // 4 if len(xs) >= 4 else 0
    mid = xs[d:len(xs) - d]
    return sum(mid) / len(mid)


# ---------------------------------------------------------------------------
# model: the reference pipeline on the shipped B200 tables


def _pipeline(tables, provenance, anchors=None):
    """The reference pipeline on a list of tables (cli.py:281-373): dataset,
    seeded 80/20 split, the 5 x 8 CART grid on the train split, the model
    with the best test DTPR.  `anchors` (tables by shape) supplies the
    default-tile anchors 256^3 / 1024^3 when `tables` lacks them."""
    from paper_1806_07060_b200 import evaluation, model
    from paper_1806_07060_b200.dataset import dataset_from_tables, split

    ds = dataset_from_tables(tables, provenance)
    sp = split(ds, SPLIT_FRACTION, SPLIT_SEED)
    recs = ds.features_and_labels()
    train_recs = [recs[i] for i in sp.train]
    test_recs = [recs[i] for i in sp.test]
    named = model.grid_train(train_recs)
    by_shape = dict(anchors or {})
    by_shape.update(evaluation.tables_by_shape(tables))
    policy = evaluation.build_baseline_policy(by_shape[(256, 256, 256)], by_shape[(1024, 1024, 1024)],
                                              384).register(ds.class_index)
    scores = evaluation.score_models(named, test_recs, by_shape, ds.class_index, policy)
    best = evaluation.select_best_model(scores)
    return {"tree": dict(named)[best.name], "name": best.name, "classes": ds.class_index, "policy": policy,
            "train": {mnk for mnk, _ in train_recs}, "test": {mnk for mnk, _ in test_recs},
            "score": {"accuracy": best.accuracy, "dtpr": best.dtpr, "dttr": best.dttr,
                      "leaves": best.stats.total_leaves, "height": best.stats.height},
            "n_train": len(train_recs), "n_test": len(test_recs)}


def dedup_tables(tables):
    """Tables deduplicated by (M, N, K) in order (the CLI's hybrid strategy,
    cli.py:166-179)."""
    out, seen = [], set()
    for t in tables:
        if t.shape.mnk not in seen:
            seen.add(t.shape.mnk)
            out.append(t)
    return out


def training_tables():
    """The headline model's training set: the po2 16..4096 tables followed by
    the octave-uniform random tables (the CLI hybrid of the two sweeps), one
    seeded 80/20 split.  No DeepBench table."""
    from paper_1806_07060_b200.tuner import load_table_bundle

    for b in (PO2_BUNDLE, LOGRANDOM_BUNDLE):
        if not b.exists():
            raise SystemExit(f"missing shipped tuning tables {b.name}")
    po2 = load_table_bundle(PO2_BUNDLE)
    return po2, dedup_tables(po2 + load_table_bundle(LOGRANDOM_BUNDLE))


def build_model():
    """The headline model: the reference pipeline on the po2 + octave-uniform
    random tables (train on generated shape sets,
    evaluate on the DeepBench-style set); no DeepBench table is seen in
    training or model selection.  The DeepBench tables provide the oracle
    per shape.  profiles/r02_train_set_probe.jsonl compares training sets
    in table mode (po2 only: DeepBench DTPR 0.919; po2 + random: 0.921)."""
    from paper_1806_07060_b200.kernels import KernelFamily
    from paper_1806_07060_b200.tuner import load_table_bundle

    if not DB_BUNDLE.exists():
        raise SystemExit(f"missing shipped tuning tables {DB_BUNDLE.name}")
    po2, train_tables = training_tables()
    db = load_table_bundle(DB_BUNDLE)
    by_shape = {t.shape.mnk: t for t in train_tables}
    by_shape.update({t.shape.mnk: t for t in db})
    pipe = _pipeline(train_tables, "hybrid")
    return {
        "tree": pipe["tree"], "name": pipe["name"], "classes": pipe["classes"], "policy": pipe["policy"],
        "tables": by_shape, "po2_test": [t.shape for t in po2 if t.shape.mnk in pipe["test"]],
        "db_all": [t.shape for t in db],
        # DeepBench shapes that are not po2 training shapes (a po2 grid point such
        # as 2048 x 16 x 2048 can coincide with a DeepBench shape)
        "db_unseen": [t.shape for t in db if t.shape.mnk not in pipe["train"]],
        "score": pipe["score"], "n_train": pipe["n_train"], "n_test": pipe["n_test"],
        "train_set": "po2 16..4096 + 512 octave-uniform random shapes in [16, 4096) (seed 2026); "
                     "train split (seed 2024, 80 %)", "family_direct": KernelFamily.DIRECT,
    }


def build_hybrid_model():
    """Secondary model: the reference CLI's "hybrid" dataset (cli.py:166-179),
    po2 + DeepBench deduplicated in order, one seeded 80/20 split; reported
    with its train and test subsets separately (cli.py:413-420)."""
    from paper_1806_07060_b200.tuner import load_table_bundle

    po2 = load_table_bundle(PO2_BUNDLE)
    db = load_table_bundle(DB_BUNDLE)
    pipe = _pipeline(dedup_tables(po2 + db), "hybrid")
    db_set = {t.shape.mnk for t in db}
    pipe["db_train"] = [ProblemShapeOf(mnk) for mnk in sorted(pipe["train"] & db_set)]
    pipe["db_test"] = [ProblemShapeOf(mnk) for mnk in sorted(pipe["test"] & db_set)]
    return pipe


def build_tc_model(policy):
    """configs[4]: the reference pipeline on the b200tc tables (random
    (M, N, K) in 1..8192, tf32/bf16/tf32x3 families + the fp32 winner
    shortlist, bench regime; configs/random_tc_r02.json).  Default tile = the fp32 BaselinePolicy of
    the main model (the reference's definition); `fixed_tc` = the single tc
    config with the best geomean over the training shapes."""
    from paper_1806_07060_b200 import evaluation, model
    from paper_1806_07060_b200.dataset import dataset_from_tables, split
    from paper_1806_07060_b200.kernels import TC_FAMILIES
    from paper_1806_07060_b200.tuner import load_table_bundle

    if not TC_BUNDLE.exists():
        return None
    tables = load_table_bundle(TC_BUNDLE)
    ds = dataset_from_tables(tables, "random")
    sp = split(ds, SPLIT_FRACTION, SPLIT_SEED)
    recs = ds.features_and_labels()
    train_recs = [recs[i] for i in sp.train]
    test_recs = [recs[i] for i in sp.test]
    named = model.grid_train(train_recs)
    policy.register(ds.class_index)
    by_shape = evaluation.tables_by_shape(tables)
    scores = evaluation.score_models(named, test_recs, by_shape, ds.class_index, policy)
    best = evaluation.select_best_model(scores)
    train_shapes = [recs[i][0] for i in sp.train]
    tc_cfgs = [m.config for m in tables[0].measurements if m.config.family in TC_FAMILIES]

    def train_geo(cfg):
        return geomean(by_shape[mnk].gflops_for(cfg) for mnk in train_shapes)

    fixed = max(tc_cfgs, key=train_geo)
    return {"tree": dict(named)[best.name], "name": best.name, "classes": ds.class_index, "tables": by_shape,
            "test": [ProblemShapeOf(recs[i][0]) for i in sp.test], "fixed_tc": fixed, "n_train": len(train_recs),
            "score": {"accuracy": best.accuracy, "dtpr": best.dtpr, "dttr": best.dttr,
                      "leaves": best.stats.total_leaves, "height": best.stats.height}}


def go2_section():
    """The paper's dense dataset (go2: 256..3840 step 256, 3375 shapes) on
    B200 tables swept with the reference's seeded tune_random sampler
    (configs/go2r_b200.json: 96 of the 1114 B200 configs, tuner.py:188-221,
    bench regime), run through the reference pipeline in table mode: seeded
    80/20 split, the 5 x 8 CART grid, selection by test DTPR; reports the
    reference's metrics (accuracy, DTPR, DTTR) and the table-mode geomeans
    (no GPU time)."""
    from paper_1806_07060_b200 import evaluation, model
    from paper_1806_07060_b200.dataset import dataset_from_tables, split
    from paper_1806_07060_b200.tuner import load_table_bundle

    if not GO2_BUNDLE.exists():
        return {"unavailable": f"no {GO2_BUNDLE.name}"}
    tables = load_table_bundle(GO2_BUNDLE)
    ds = dataset_from_tables(tables, "go2")
    sp = split(ds, SPLIT_FRACTION, SPLIT_SEED)
    recs = ds.features_and_labels()
    train_recs = [recs[i] for i in sp.train]
    test_recs = [recs[i] for i in sp.test]
    t0 = time.perf_counter()
    named = model.grid_train(train_recs)
    train_s = time.perf_counter() - t0
    by_shape = dict(anchors or {})
    by_shape.update(evaluation.tables_by_shape(tables))
    policy = evaluation.build_baseline_policy(by_shape[(256, 256, 256)], by_shape[(1024, 1024, 1024)],
                                              384).register(ds.class_index)
    scores = evaluation.score_models(named, test_recs, by_shape, ds.class_index, policy)
    best = evaluation.select_best_model(scores)
    tree = dict(named)[best.name]
    dt, orc, de = [], [], []
    for mnk, _ in test_recs:
        t = by_shape[mnk]
        cid = model.predict(tree, mnk)
        cfg = ds.class_index.config_of(cid)
        dt.append(t.gflops_for(cfg))
        orc.append(t.peak_gflops)
        de.append(t.gflops_for(policy.select_config(ProblemShapeOf(mnk))))
    meta = tables[0].meta
    return {"shapes": len(tables), "configs_per_shape": len(tables[0].measurements),
            "sampling": {k: meta.get(k) for k in ("mode", "samples", "seed", "l2") if k in meta},
            "n_train": len(train_recs),
            "n_test": len(test_recs), "model": best.name,
            "accuracy": round(best.accuracy, 4), "dtpr": round(best.dtpr, 4), "dttr": round(best.dttr, 4),
            "leaves": best.stats.total_leaves, "height": best.stats.height,
            "grid_train_s": round(train_s, 2),
            "dt_geomean_table": round(geomean(dt), 1), "oracle_geomean_table": round(geomean(orc), 1),
            "default_geomean_table": round(geomean(de), 1),
            "paper_p100_go2_hmax_l1": {"accuracy": 0.60, "dtpr": 0.852, "dttr": 1.424}}


def deepbench_table_mode(m, selector):
    """The reference's DTPR / DTTR (arithmetic means of per-shape ratios,
    evaluation.py:169-183) of the headline model on the DeepBench tables:
    DT pick vs the table's best (DTPR) and vs the default tile (DTTR)."""
    dtpr, dttr = [], []
    for s in m["db_all"]:
        t = m["tables"][s.mnk]
        g = t.gflops_for(selector.select(*s.mnk))
        dtpr.append(g / t.peak_gflops)
        dttr.append(g / t.gflops_for(m["policy"].select_config(s)))
    return {"shapes": len(dtpr), "dtpr": round(math.fsum(dtpr) / len(dtpr), 4),
            "dttr": round(math.fsum(dttr) / len(dttr), 4)}


def ProblemShapeOf(mnk):
    from paper_1806_07060_b200.kernels import ProblemShape
    return ProblemShape(*mnk)


# ---------------------------------------------------------------------------
# device-side measurement


class ShapeCase:
    """Resident operands + prepared native arguments for one shape."""

    def __init__(self, shape, device, seed=0, keep_host=True):
        import ctypes

        import torch

        from paper_1806_07060_b200 import _device, _native
        from paper_1806_07060_b200.kernels import native_shape
        from paper_1806_07060_b200.tuner import _bench_buffers

        self.shape = shape
        self.flops = 2.0 * shape.M * shape.N * shape.K
        A, B, C, _ = _bench_buffers(shape, np.float32, seed)
        self.host = (A, B, C) if keep_host else None
        self.dA, self.dB, self.dC = (torch.from_numpy(x).to(device) for x in (A, B, C))
        self.dout = torch.empty((shape.M, shape.N), device=device)
        self.nshape = native_shape(shape)
        ld = _device.leading_dim
        self.ptrs = (ctypes.c_void_p(self.dA.data_ptr()), ld(self.dA), ctypes.c_void_p(self.dB.data_ptr()),
                     ld(self.dB), ctypes.c_void_p(self.dC.data_ptr()), ld(self.dC),
                     ctypes.c_void_p(self.dout.data_ptr()), ld(self.dout))
        self._native = _native


def pack_launches(shape, cfg) -> int:
    """Kernels one family path launches (mirrors launch.cuh's pack decisions)."""
    from paper_1806_07060_b200.kernels import TC_FAMILIES, KernelFamily
    if cfg.family is KernelFamily.DIRECT:
        return 1
    if cfg.family in (KernelFamily.SKINNY_N, KernelFamily.SKINNY_M) and not shape.transA and not shape.transB \
            and shape.K % 4 == 0 and (cfg.family is KernelFamily.SKINNY_M or shape.N % 4 == 0):
        return 1  # one clustered launch (skinny.cuh)
    if cfg.family in TC_FAMILIES:  # bf16: one convert pass per operand; tf32 reads fp32 in place
        if cfg.family is KernelFamily.TF32X3:
            return 1  # the lo parts are made in shared memory
        return 3 if cfg.family is KernelFamily.BF16 else 1
    if cfg.family is KernelFamily.TMA and not shape.transA and not shape.transB and shape.K % 4 == 0 \
            and shape.N % 4 == 0:
        return 1  # TMA-fed core on the caller's operands, no packs
    arow_fit = not shape.transA and shape.M % cfg.block_m == 0 and shape.K % cfg.block_k == 0
    if (cfg.family is KernelFamily.SPLITK and not shape.transA and not shape.transB and shape.K % 4 == 0
            and shape.N % 4 == 0 and (shape.N <= 64 or not arow_fit)):
        ktiles = -(-shape.K // cfg.block_k)
        kps = -(-ktiles // cfg.unroll_k)
        # in-place core; up to 8 slices reduce inside the cluster, more take
        # the slab + reduce launch (launch.cuh launch_inplace)
        return 1 if -(-ktiles // kps) <= 8 else 2
    n = 1
    a_in_place = (shape.transA and shape.M % cfg.block_m == 0 and shape.K % cfg.block_k == 0) or \
        (cfg.family is KernelFamily.SPLITK and arow_fit)
    if not a_in_place:
        n += 1
    if not (not shape.transB and shape.N % cfg.block_n == 0 and shape.K % cfg.block_k == 0 and shape.N % 4 == 0):
        n += 1
    if cfg.family is KernelFamily.SPLITK:
        ktiles = -(-shape.K // cfg.block_k)
        kps = -(-ktiles // cfg.unroll_k)
        if -(-ktiles // kps) > 1:
            n += 1  # fixed-order split-K reduction
    return n


class Runner:
    """Times native dispatches (selector or fixed config) per shape."""

    def __init__(self, device, caps):
        import ctypes

        import torch

        from paper_1806_07060_b200 import _device, _native
        self.torch = torch
        self.ctypes = ctypes
        self.lib = _native.lib()
        self.native = _native
        self.caps = caps
        self.ncaps = caps.native()
        self.device = device
        self.stream = torch.cuda.current_stream(device)
        self.hstream = ctypes.c_void_p(self.stream.cuda_stream)
        self.flush = torch.empty(FLUSH_BYTES // 4, dtype=torch.float32, device=device)
        self.ws = _device.workspace(1 << 30, device)  # >= every pack buffer in the sets
        self.ws_ptr = ctypes.c_void_p(self.ws.data_ptr())
        self.ws_n = self.ws.numel()

    def launch(self, case, selector=None, config=None, fallback=None):
        ct = self.ctypes
        a, lda, b, ldb, c, ldc, o, ldo = case.ptrs
        if selector is not None:
            sel = self.native.AgConfig()
            fb = ct.c_int(0)
            rc = self.lib.ag_dispatch_gemm(selector.handle, ct.byref(fallback), ct.byref(case.nshape),
                                           ct.byref(self.ncaps), 0, a, lda, b, ldb, c, ldc, o, ldo,
                                           self.ws_ptr, self.ws_n, self.hstream, ct.byref(sel), ct.byref(fb))
        else:
            rc = self.lib.ag_gemm(ct.byref(case.nshape), ct.byref(config), ct.byref(self.ncaps), 0,
                                  a, lda, b, ldb, c, ldc, o, ldo, self.ws_ptr, self.ws_n, self.hstream)
        if rc:
            raise RuntimeError(f"native GEMM failed ({rc}): {self.native.last_error()}")

    def pass_(self, cases, how):
        """One pass: per shape flush L2, then events around the path. Returns event pairs."""
        torch = self.torch
        evs = []
        for i, case in enumerate(cases):
            self.flush.fill_(float(i))
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(self.stream)
            how(i, case)
            e1.record(self.stream)
            evs.append((e0, e1))
        return evs


def clocks_sampler():
    """nvidia-smi sampling of SM clocks / throttle reasons during the timed region."""
    fields = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    import torch
    local = int(os.environ.get("LOCAL_RANK", "0"))
    ndev = max(1, torch.cuda.device_count())
    local = local if local < ndev else 0  # ranks sharing one GPU (AG_DIST_BACKEND=gloo)
    visible = [v for v in os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",") if v.strip()]
    idx = visible[local] if local < len(visible) else str(local)
    out = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
    try:
        proc = subprocess.Popen(["nvidia-smi", f"--id={idx}", f"--query-gpu={fields}", "--format=csv,noheader,nounits",
                                 "-lms", "100"], stdout=out, stderr=subprocess.DEVNULL)
    except (FileNotFoundError, OSError):
        return None, out.name
    return proc, out.name


def clocks_summary(proc, path):
    if proc is None:
        return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
    proc.terminate()
    try:
        proc.wait(timeout=5)
    except subprocess.TimeoutExpired:
        proc.kill()
    sm, smax, reasons = [], [], set()
    names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
    with open(path) as fh:
        for line in fh:
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                smax.append(float(f[1]))
            except ValueError:
                continue
            for name, val in zip(names, f[4:8]):
                if val.lower() == "active":
                    reasons.add(name)
    os.unlink(path)
    return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
            "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU (reference) arm


def cpu_rates(shapes, budget_flops=CPU_SAMPLE_FLOPS):
    """Reference CPU path (oracle port of the numba kernels, all host threads)
    on each shape's first m' output rows, m' sized to ~budget_flops."""
    from oracle import gemm as ogemm
    from paper_1806_07060_b200.tuner import _bench_buffers
    ogemm.build()
    ogemm.set_threads(len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count())
    rates = []
    for s in shapes:
        canon = CPU_DEFAULT_DIRECT if s.M * s.N * s.K < 384 ** 3 else CPU_DEFAULT_INDIRECT
        fam, params = canon.split(":")
        bm, bn, bk, tm, tn, uk = map(int, params.split("-"))
        # whole row blocks only, so the sample never pays padding the full
        # shape would not
        rows = int(budget_flops // (2.0 * s.N * s.K)) // bm * bm
        rows = min(s.M, max(bm, rows))
        A, B, C, _ = _bench_buffers(s, np.float32, 0)
        A = np.ascontiguousarray(A[:rows])
        C = np.ascontiguousarray(C[:rows])
        _, sec = ogemm.execute(rows, s.N, s.K, 1.0, 0.0, False, False, A, B, C, fam, bm, bn, bk, tm, tn, uk)
        rates.append(2.0 * rows * s.N * s.K / sec / 1e9)
    return rates, ogemm.num_threads()


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from paper_1806_07060_b200.dataset import load_workload_shapes
    from paper_1806_07060_b200.workloads import DEEPBENCH_PATH
    shapes = load_workload_shapes(DEEPBENCH_PATH)
    per_step = []
    t_all = time.perf_counter()
    for step in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        rates, cores = cpu_rates(shapes)
        dt = time.perf_counter() - t0
        if step >= args.warmup:
            per_step.append((rates, dt))
    per_shape = [statistics.median(r[i] for r, _ in per_step) for i in range(len(shapes))]
    value = geomean(per_shape)
    ms = 1e3 * statistics.median(dt for _, dt in per_step)
    sample = (f"all {len(shapes)} DeepBench-style shapes, each on its first m' output rows (whole "
              f"row blocks) with 2*m'*N*K ~ {CPU_SAMPLE_FLOPS:.0e} flops; reference CPU default tiles "
              f"({CPU_DEFAULT_DIRECT} below 384^3, {CPU_DEFAULT_INDIRECT} above)")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32 (f64 accumulate)",
        "data": "synthetic (reference _bench_buffers recipe)",
        "config": {"workload": "deepbench_fp32 (DeepBench-style rectangular set, configs[2])",
                   "shapes": len(shapes), "alpha": 1.0, "beta": 0.0, "l2": "n/a (CPU)"},
        "cpu_baseline": {"value": round(value, 4), "unit": "GFLOP/s", "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": round(value, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": round(time.perf_counter() - t_all, 2),
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm


def run_ours(args):
    import torch

    from paper_1806_07060_b200 import codegen, distributed
    from paper_1806_07060_b200.kernels import DeviceCaps, ffma_peak_tflops, gemm_execute

    rank, world, local = distributed.init()
    device = torch.device("cuda", local if torch.cuda.device_count() > local else 0)
    torch.cuda.set_device(device)
    caps = DeviceCaps.b200()
    m = build_model()
    tree, classes, policy, tables = m["tree"], m["classes"], m["policy"], m["tables"]
    selector = codegen.CompiledSelector(tree, classes)
    fallback = codegen.FALLBACK_CONFIG.native()
    workload = m["db_all"]
    po2_test = m["po2_test"]
    t_build = time.perf_counter()
    cases = [ShapeCase(s, device) for s in workload]
    po2_cases = [ShapeCase(s, device) for s in po2_test]
    log(f"rank {rank}: model {m['name']} ({m['score']}), {len(cases)} + {len(po2_cases)} shapes, "
        f"operands staged in {time.perf_counter() - t_build:.1f}s")
    runner = Runner(device, caps)

    def dt_pass(cs):
        return runner.pass_(cs, lambda i, c: runner.launch(c, selector=selector, fallback=fallback))

    def fixed_pass(cs, cfgs):
        nat = [c.native() for c in cfgs]
        return runner.pass_(cs, lambda i, c: runner.launch(c, config=nat[i]))

    def times(evs):
        evs[-1][1].synchronize()
        return [e0.elapsed_time(e1) * 1e-3 for e0, e1 in evs]

    # warmup (also JITs nothing: the kernels are precompiled sm_100a)
    for _ in range(args.warmup):
        dt_pass(cases)
    torch.cuda.synchronize()

    # ---- timed region: exactly K DT passes over the workload
    proc, clk_path = clocks_sampler()
    time.sleep(0.3)
    distributed.barrier()
    torch.cuda.synchronize()
    r0 = torch.cuda.Event(enable_timing=True)
    r1 = torch.cuda.Event(enable_timing=True)
    r0.record(runner.stream)
    step_evs = [dt_pass(cases) for _ in range(args.steps)]
    r1.record(runner.stream)
    torch.cuda.synchronize()
    distributed.barrier()
    clocks = clocks_summary(proc, clk_path)
    region_s = r0.elapsed_time(r1) * 1e-3
    per_step = [times(evs) for evs in step_evs]
    dt_t = [trimmed_mean([p[i] for p in per_step]) for i in range(len(cases))]
    dt_t = distributed.reduce_max(dt_t, device)
    region_s = distributed.reduce_max([region_s], device)[0]

    # ---- oracle and default tiles, same method, outside the timed region
    oracle_cfgs = [tables[c.shape.mnk].best_config for c in cases]
    default_cfgs = [policy.select_config(c.shape) for c in cases]
    dt_cfgs = [selector.select(*c.shape.mnk) for c in cases]

    def measured(cs, cfgs, reps=None):
        runs = [times(fixed_pass(cs, cfgs)) for _ in range(reps or max(4, args.steps))]
        torch.cuda.synchronize()
        return distributed.reduce_max([trimmed_mean([r[i] for r in runs]) for i in range(len(cs))], device)

    fixed_pass(cases, oracle_cfgs)
    oracle_t = measured(cases, oracle_cfgs)
    default_t = measured(cases, default_cfgs)
    # the default's indirect tile is the anchor (1024^3) argmax; configs within
    # 1 % of it are a coin flip of the sweep, so report the DT ratio vs each
    anchor = tables[(1024, 1024, 1024)]
    best_i = anchor.gflops_for(policy.default_indirect)
    near = [m.config for m in anchor.measurements
            if m.config.family is policy.default_indirect.family and m.gflops >= 0.99 * best_i]
    sensitivity = []
    for cfg in near[:4]:
        alt = [cfg if d is policy.default_indirect else d for d in default_cfgs]
        alt_t = measured(cases, alt)
        g = geomean(c.flops / t / 1e9 for c, t in zip(cases, alt_t))
        sensitivity.append({"default_indirect": cfg.canonical(), "anchor_gflops": round(anchor.gflops_for(cfg), 1),
                            "default_geomean": round(g, 2)})
    rate = lambda cs, ts: [c.flops / t / 1e9 for c, t in zip(cs, ts)]  # noqa: E731
    dt_r, or_r, de_r = rate(cases, dt_t), rate(cases, oracle_t), rate(cases, default_t)
    value_1 = geomean(dt_r)
    unseen_set = {s.mnk for s in m["db_unseen"]}
    unseen = [i for i, c in enumerate(cases) if c.shape.mnk in unseen_set]

    # po2 held-out split (configs[1])
    po2_steps = max(4, args.steps // 3)
    po2_runs = [times(dt_pass(po2_cases)) for _ in range(po2_steps)]
    torch.cuda.synchronize()
    po2_dt = [trimmed_mean([r[i] for r in po2_runs]) for i in range(len(po2_cases))]
    po2_or = measured(po2_cases, [tables[c.shape.mnk].best_config for c in po2_cases], po2_steps)
    po2_de = measured(po2_cases, [policy.select_config(c.shape) for c in po2_cases], po2_steps)
    # configs[1] is po2 64..4096: its held-out shapes are the test-split shapes with every dim >= 64
    in_c1 = [i for i, c in enumerate(po2_cases) if min(c.shape.mnk) >= 64]

    # ---- secondary model: the reference CLI's hybrid dataset (po2 + DeepBench,
    # one 80/20 split), DT on DeepBench reported per subset (cli.py:413-420)
    hy = build_hybrid_model()
    hy_sel = codegen.CompiledSelector(hy["tree"], hy["classes"])
    hy_runs = [times(runner.pass_(cases, lambda i, c: runner.launch(c, selector=hy_sel, fallback=fallback)))
               for _ in range(max(4, args.steps // 2))]
    torch.cuda.synchronize()
    hy_t = distributed.reduce_max([trimmed_mean([r[i] for r in hy_runs]) for i in range(len(cases))], device)
    case_idx = {c.shape.mnk: i for i, c in enumerate(cases)}

    def hy_sub(shapes):
        idx = [case_idx[s.mnk] for s in shapes]
        if not idx:
            return {"shapes": 0}
        d = geomean(cases[i].flops / hy_t[i] / 1e9 for i in idx)
        o = geomean(cases[i].flops / oracle_t[i] / 1e9 for i in idx)
        q = geomean(cases[i].flops / default_t[i] / 1e9 for i in idx)
        return {"shapes": len(idx), "dt_geomean": round(d, 2), "oracle_geomean": round(o, 2),
                "default_geomean": round(q, 2), "dt_over_oracle": round(d / o, 4), "dt_over_default": round(d / q, 4)}

    # ---- configs[4]: the tensor-core search space on random (M, N, K)
    # sub-measurements never take the headline line down with them
    try:
        tc_doc = tc_section(m, policy, device, distributed, times, fallback, args)
    except Exception as exc:  # noqa: BLE001
        tc_doc = {"error": f"{type(exc).__name__}: {exc}"}
    try:
        x3_doc = x3_section(cases, default_t, device, distributed, times, fallback, args)
    except Exception as exc:  # noqa: BLE001
        x3_doc = {"error": f"{type(exc).__name__}: {exc}"}
    try:
        go2_doc = go2_section() if rank == 0 else None
    except Exception as exc:  # noqa: BLE001
        go2_doc = {"error": f"{type(exc).__name__}: {exc}"}
    # ---- configs[3]: sharded exhaustive sweep throughput
    sweep_doc = sweep_section(device, distributed, rank, world,
                              with_cpu=(rank == 0 and world == 1 and not args.no_cpu_baseline)) \
        if not args.no_sweep else None

    # ---- e2e: the reference-facing call with the reference's own data
    # convention -- codegen.dispatch_and_run(tree, shape, A, B, C, caps) on
    # plain (pageable) numpy arrays (codegen.py:285-325) -- copies inside.
    from paper_1806_07060_b200.kernels import reads_c
    e2e_t, pinned_t = [], []
    h2d = d2h = 0
    for c, cfg in zip(cases, dt_cfgs):
        A, B, C = c.host
        codegen.dispatch_and_run(tree, c.shape, A, B, C, caps, classes=classes)  # warm (selector, page-lock path)
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            res = codegen.dispatch_and_run(tree, c.shape, A, B, C, caps, classes=classes)
            ts.append(time.perf_counter() - t0)
        e2e_t.append(statistics.median(ts))
        picked = res.selected
        h2d += A.nbytes + B.nbytes + (C.nbytes if reads_c(c.shape, picked) else 0)
        d2h += res.output.nbytes
        # the same call from pinned torch buffers (dispatch_native), for comparison
        pA, pB, pC = (torch.from_numpy(x).pin_memory() for x in c.host)
        hout = torch.empty((c.shape.M, c.shape.N), dtype=torch.float32).pin_memory()
        codegen.dispatch_native(selector, c.shape, pA, pB, pC, caps, out=hout)
        ts = []
        for _ in range(3):
            t0 = time.perf_counter()
            codegen.dispatch_native(selector, c.shape, pA, pB, pC, caps, out=hout)
            ts.append(time.perf_counter() - t0)
        pinned_t.append(statistics.median(ts))
    e2e_t = distributed.reduce_max(e2e_t, device)
    pinned_t = distributed.reduce_max(pinned_t, device)
    e2e_value = geomean(rate(cases, e2e_t))
    e2e_pinned = geomean(rate(cases, pinned_t))
    # spot-check the DT output against the float64 product (first rows)
    c0 = max(cases, key=lambda c: c.flops)
    rows = slice(0, 8)
    exact = c0.host[0][rows].astype(np.float64) @ c0.host[1].astype(np.float64)
    got = c0.dout[rows].double().cpu().numpy()
    rf = float(np.linalg.norm(got - exact) / np.linalg.norm(exact))

    # ---- roofline of the dominant kernel (largest share of the DT pass)
    dom = max(range(len(cases)), key=lambda i: dt_t[i])
    peak_meas = ffma_peak_tflops()
    achieved = cases[dom].flops / dt_t[dom] / 1e12
    traffic = None
    key = f"{cases[dom].shape.M}x{cases[dom].shape.N}x{cases[dom].shape.K}:{dt_cfgs[dom].canonical()}"
    if TRAFFIC_FILE.exists():
        traffic = json.loads(TRAFFIC_FILE.read_text()).get(key)

    # ---- CPU baseline (oracle port) on rank 0, bounded sample
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:  # rank 0 at N = 1 only
        t0 = time.perf_counter()
        cpu_r, cores = cpu_rates(workload)
        cpu = {"value": round(geomean(cpu_r), 4), "unit": "GFLOP/s", "cores": cores, "kind": "port",
               "sample": (f"all {len(workload)} workload shapes, each on its first m' output rows "
                          f"(2*m'*N*K ~ {CPU_SAMPLE_FLOPS:.0e} flops), reference CPU default tiles "
                          f"{CPU_DEFAULT_DIRECT}/{CPU_DEFAULT_INDIRECT}; {time.perf_counter() - t0:.1f}s"),
               }

    launches = sum(pack_launches(c.shape, cfg) for c, cfg in zip(cases, dt_cfgs)) * args.steps
    # the compiled decision tree's host cost per dispatch (ag_select_bench_ns)
    select_ns = statistics.median(selector.bench_ns(*c.shape.mnk, reps=20000) for c in cases)
    value = value_1 * world  # replicas: whole-job aggregate over N GPUs
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(region_s / args.steps * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (reference _bench_buffers recipe: PCG64(mix(0,M,N,K)) U(-1,1))",
        "config": {"workload": "deepbench_fp32: DeepBench-style rectangular set (BASELINE configs[2])",
                   "shapes": len(cases), "alpha": 1.0, "beta": 0.0, "trans": "NN",
                   "l2": "flushed (256 MB write) before every timed GEMM; per-shape time = trimmed mean "
                         "(middle half) of the steps' event times",
                   "parallelism": f"replicas x{world} (shapes independent; no collective on the data path)",
                   "model": f"{m['name']} trained on {m['n_train']} shapes ({m['train_set']}); no DeepBench "
                            f"table in training or model selection ({len(cases) - len(unseen)} of the 40 shapes "
                            f"are po2 training shapes; dt_vs.unseen covers the other {len(unseen)})",
                   "caps_profile": "b200"},
        "dt_vs": {"dt_geomean": round(value_1, 2), "oracle_geomean": round(geomean(or_r), 2),
                  "default_geomean": round(geomean(de_r), 2),
                  "dt_over_oracle": round(value_1 / geomean(or_r), 4),
                  "dt_over_default": round(value_1 / geomean(de_r), 4),
                  "default_config": [policy.default_direct.canonical(), policy.default_indirect.canonical()],
                  "default_sensitivity": [dict(s, dt_over_default=round(value_1 / s["default_geomean"], 4))
                                          for s in sensitivity],
                  "unseen": {"shapes": len(unseen), "note": "DeepBench shapes that are not training shapes",
                             "dt_geomean": round(geomean(dt_r[i] for i in unseen), 2),
                             "oracle_geomean": round(geomean(or_r[i] for i in unseen), 2),
                             "default_geomean": round(geomean(de_r[i] for i in unseen), 2)}},
        "hybrid_model": {"model": hy["name"], "n_train": hy["n_train"], "n_test": hy["n_test"],
                         "note": "reference CLI hybrid dataset (po2 + DeepBench, one 80/20 split); DT measured "
                                 "live on the DeepBench shapes of each subset",
                         "deepbench_train": hy_sub(hy["db_train"]), "deepbench_test": hy_sub(hy["db_test"]),
                         "deepbench_all": dict(hy_sub([c.shape for c in cases]),
                                               note="round 1's headline protocol (tree trained on po2 + 80 % "
                                                    "of DeepBench), for comparison only")},
        "po2_test_split": {"shapes": len(po2_cases), "dataset": "po2 16..4096 shapes in the training set's held-out 20 %",
                           "dt_geomean": round(geomean(rate(po2_cases, po2_dt)), 2),
                           "oracle_geomean": round(geomean(rate(po2_cases, po2_or)), 2),
                           "default_geomean": round(geomean(rate(po2_cases, po2_de)), 2),
                           "configs1_po2_64_4096": {
                               "shapes": len(in_c1),
                               "dt_geomean": round(geomean(rate(po2_cases, po2_dt)[i] for i in in_c1), 2),
                               "oracle_geomean": round(geomean(rate(po2_cases, po2_or)[i] for i in in_c1), 2),
                               "default_geomean": round(geomean(rate(po2_cases, po2_de)[i] for i in in_c1), 2)}},
        "model_scores_table_mode": m["score"],
        "deepbench_table_mode": deepbench_table_mode(m, selector),
        "per_shape": [[list(c.shape.mnk), round(d, 1), round(o, 1), round(q, 1), dc.canonical(),
                       oc.canonical(), qc.canonical()]
                      for c, d, o, q, dc, oc, qc in zip(cases, dt_r, or_r, de_r, dt_cfgs, oracle_cfgs, default_cfgs)],
        "per_shape_columns": ["mnk", "dt_gflops", "oracle_gflops", "default_gflops", "dt_config",
                              "oracle_config", "default_config"],
        "e2e": {"value": round(e2e_value * world, 2), "unit": "GFLOP/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h,
                "how": "codegen.dispatch_and_run(tree, shape, A, B, C, caps, classes) on plain pageable numpy "
                       "arrays (the reference's call, codegen.py:285-325): cached compiled selector, then the "
                       "compiled numpy path (csrc/fastpath.c) -> ag_gemm_host_ex(AG_HOST_STAGE): the pageable "
                       "operands and the fresh output cross through pinned staging rings filled / drained by "
                       "parallel host copies, H2D / family path / D2H pipelined over output panels on three "
                       "streams; median of 5 wall-clock calls per shape",
                "pinned_dispatch_native": round(e2e_pinned * world, 2),
                "per_shape_ms": [[list(c.shape.mnk), round(t * 1e3, 3), round(u * 1e3, 3)]
                                 for c, t, u in zip(cases, e2e_t, pinned_t)],
                "per_shape_columns": ["mnk", "numpy_dispatch_and_run_ms", "pinned_dispatch_native_ms"]},
        "regime_floor": {
            "note": "per shape, max(2MNK at the measured FFMA peak, the bench regime's streaming-read floor for "
                    "its operand + result bytes, profiles/r02_read_floor.jsonl); geomean of floor / measured time",
            "dt_frac": round(geomean(regime_floor_s(c.shape, peak_meas) / t for c, t in zip(cases, dt_t)), 4),
            "oracle_frac": round(geomean(regime_floor_s(c.shape, peak_meas) / t for c, t in zip(cases, oracle_t)), 4),
            "per_shape_dt_frac": [[list(c.shape.mnk), round(regime_floor_s(c.shape, peak_meas) / t, 3)]
                                  for c, t in zip(cases, dt_t)]},
        "roofline": {"bound": "fp32-cuda-core (compute)", "achieved": round(achieved, 3),
                     "peak": round(peak_meas, 3), "unit": "TFLOP/s", "frac": round(achieved / peak_meas, 4),
                     "traffic": traffic, "kernel": key,
                     "peak_source": "measured FFMA microbenchmark (ag_ffma_peak) in this run; "
                                    f"nominal 148x128x2x1.965GHz = {NOMINAL_FP32_TFLOPS:.1f}",
                     "frac_of_nominal": round(achieved / NOMINAL_FP32_TFLOPS, 4),
                     "note": "event time covers the whole family path (pack helpers + tiled core)"},
        "cpu_baseline": cpu,
        "tc_random": tc_doc,
        "fp32_accurate_tc": x3_doc,
        "go2_table_mode": go2_doc,
        "sweep": sweep_doc,
        "clocks": clocks,
        "gpu_launches": launches,
        "dispatch_select_ns": round(select_ns, 1),
        "parity_spot_check_rf": rf,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    distributed.finalize()
    return 0


def tc_section(m, policy, device, distributed, times, fallback, args):
    """configs[4] live: DT (compiled selector over the b200tc classes) vs
    oracle vs the fp32 default tile vs the best single tc tile, on the
    held-out random shapes; roofline of the dominant tensor-core kernel."""
    from paper_1806_07060_b200 import codegen
    from paper_1806_07060_b200.kernels import TC_FAMILIES, DeviceCaps, KernelFamily

    tcm = build_tc_model(policy)
    if tcm is None:
        return {"unavailable": f"no {TC_BUNDLE.name}"}
    runner = Runner(device, DeviceCaps.b200_tc())
    sel = codegen.CompiledSelector(tcm["tree"], tcm["classes"])
    cases = [ShapeCase(s, device, keep_host=False) for s in tcm["test"]]
    reps = max(3, args.steps // 4)

    def timed(how):
        runs = [times(runner.pass_(cases, how)) for _ in range(reps)]
        return distributed.reduce_max([statistics.median(r[i] for r in runs) for i in range(len(cases))], device)

    def fixed(cfgs):
        nat = [c.native() for c in cfgs]
        return timed(lambda i, c: runner.launch(c, config=nat[i]))

    def dt(i, c):
        runner.launch(c, selector=sel, fallback=fallback)

    runner.pass_(cases, dt)
    dt_t = timed(dt)
    dt_cfgs = [sel.select(*c.shape.mnk) for c in cases]
    or_cfgs = [tcm["tables"][c.shape.mnk].best_config for c in cases]
    de_cfgs = [policy.select_config(c.shape) for c in cases]
    or_t, de_t = fixed(or_cfgs), fixed(de_cfgs)
    fx_t = fixed([tcm["fixed_tc"]] * len(cases))
    rate = lambda ts: [c.flops / t / 1e9 for c, t in zip(cases, ts)]  # noqa: E731
    g_dt, g_or, g_de, g_fx = (geomean(rate(ts)) for ts in (dt_t, or_t, de_t, fx_t))
    # dominant tensor-core kernel of the DT pass vs the measured bf16 peak
    tc_idx = [i for i, c in enumerate(dt_cfgs) if c.family in TC_FAMILIES]
    roof = None
    if tc_idx:
        dom = max(tc_idx, key=lambda i: dt_t[i])
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
        bf16_peak = float(peaks.get("bf16_tflops", 2250.0))
        peak = bf16_peak if dt_cfgs[dom].family is KernelFamily.BF16 else bf16_peak / 2
        ach = cases[dom].flops / dt_t[dom] / 1e12
        key = f"{'x'.join(map(str, cases[dom].shape.mnk))}:{dt_cfgs[dom].canonical()}"
        traffic = json.loads(TRAFFIC_FILE.read_text()).get(key) if TRAFFIC_FILE.exists() else None
        roof = {"bound": "tensor", "achieved": round(ach, 2), "peak": round(peak, 1), "unit": "TFLOP/s",
                "frac": round(ach / peak, 4), "traffic": traffic,
                "traffic_note": "DRAM bytes of the tc_gemm launch alone (ncu --set full); the bf16 convert "
                                "passes add 6 B per operand element",
                "kernel": key,
                "peak_source": ("MEASURED_PEAKS.json bf16_tflops (burst)" if "bf16_tflops" in peaks
                                else "nominal dense bf16 2250") + ("; tf32 = half of it" if peak != bf16_peak else ""),
                "note": "event time covers the whole family path (bf16 convert passes included)"}
    fams = {}
    for c in dt_cfgs:
        fams[c.family.value] = fams.get(c.family.value, 0) + 1
    return {"workload": "random (M,N,K) in 1..8192, 256 shapes seed 1806; held-out 20% (split seed 2024)",
            "shapes": len(cases), "model": tcm["name"], "n_train": tcm["n_train"], "score_table_mode": tcm["score"],
            "dt_geomean": round(g_dt, 1), "oracle_geomean": round(g_or, 1), "default_geomean": round(g_de, 1),
            "fixed_tc_geomean": round(g_fx, 1), "fixed_tc_config": tcm["fixed_tc"].canonical(),
            "dt_over_oracle": round(g_dt / g_or, 4), "dt_over_default": round(g_dt / g_de, 4),
            "dt_over_fixed_tc": round(g_dt / g_fx, 4), "dt_families": fams, "roofline": roof,
            "per_shape": [[list(c.shape.mnk), round(a, 1), round(b, 1), d.canonical(), o.canonical()]
                          for c, a, b, d, o in zip(cases, rate(dt_t), rate(or_t), dt_cfgs, or_cfgs)]}


def load_x3_tables():
    """(training, DeepBench) tables of the fp32 space with the tf32x3 rows of
    the same shapes merged in (tuner.merge_tables: fp32 rows first).  The
    training tables are the headline's training set (po2 + the octave-uniform
    random shapes, deduplicated in order)."""
    from paper_1806_07060_b200.tuner import load_table_bundle, merge_tables

    def merged(base, extra):
        by = {t.shape.mnk: t for t in load_table_bundle(extra)}
        return [merge_tables(t, by[t.shape.mnk]) for t in load_table_bundle(base)]

    train = dedup_tables(merged(PO2_BUNDLE, X3_PO2_BUNDLE) + merged(LOGRANDOM_BUNDLE, X3_LOGRANDOM_BUNDLE))
    return train, merged(DB_BUNDLE, X3_DB_BUNDLE)


# The bench regime's streaming-read floor (profiles/r02_read_floor.jsonl,
# profiles/read_floor.py): event time of a plain chunked read kernel of N MB
# after the 256 MB write flush, best over grid sizes and unroll depths.
READ_FLOOR_US = ((0.25, 6.18), (1, 6.18), (4, 8.19), (8, 8.19), (17, 10.24), (34, 14.34), (52, 18.43),
                 (70, 22.53), (87, 24.61), (120, 31.74))


def regime_floor_s(shape, ffma_tflops):
    """The fastest any kernel could be in the bench regime: the FFMA time of
    2MNK at the measured peak, or the time to merely read the operands and
    write the result (interpolated read floor), whichever is longer."""
    mb = 4.0 * (shape.M * shape.K + shape.K * shape.N + shape.M * shape.N) / (1 << 20)
    pts = READ_FLOOR_US
    if mb <= pts[0][0]:
        us = pts[0][1]
    elif mb >= pts[-1][0]:
        us = pts[-1][1] + (mb - pts[-1][0]) * (pts[-1][1] - pts[-2][1]) / (pts[-1][0] - pts[-2][0])
    else:
        for (m0, t0), (m1, t1) in zip(pts, pts[1:]):
            if m0 <= mb <= m1:
                us = t0 + (mb - m0) * (t1 - t0) / (m1 - m0)
                break
    return max(2.0 * shape.M * shape.N * shape.K / (ffma_tflops * 1e12), us * 1e-6)


def x3_section(cases, default_t, device, distributed, times, fallback, args):
    """The fp32 space plus tf32x3 (fp32-accurate 3xTF32 on tcgen05, RF <=
    1e-5 like the fp32 families): the reference pipeline on the merged
    po2 + random tables (no DeepBench table in training), the DT measured live on the
    DeepBench set against the merged oracle and the fp32 default tile; the
    whole output of the largest tf32x3 pick checked against the float64
    product; roofline of the dominant tf32x3 kernel against tf32 peak / 3."""
    import torch

    from paper_1806_07060_b200 import codegen
    from paper_1806_07060_b200.kernels import DeviceCaps, KernelFamily
    missing = [b.name for b in (X3_PO2_BUNDLE, X3_DB_BUNDLE, X3_LOGRANDOM_BUNDLE) if not b.exists()]
    if missing:
        return {"unavailable": f"no {' / '.join(missing)}"}
    train, db_list = load_x3_tables()
    db = {t.shape.mnk: t for t in db_list}
    pipe = _pipeline(train, "hybrid")
    sel = codegen.CompiledSelector(pipe["tree"], pipe["classes"])
    runner = Runner(device, DeviceCaps.b200_tc())
    reps = max(4, args.steps // 2)

    def timed(how):
        runner.pass_(cases, how)
        runs = [times(runner.pass_(cases, how)) for _ in range(reps)]
        return distributed.reduce_max([trimmed_mean([r[i] for r in runs]) for i in range(len(cases))], device)

    dt_t = timed(lambda i, c: runner.launch(c, selector=sel, fallback=fallback))
    dt_cfgs = [sel.select(*c.shape.mnk) for c in cases]
    or_cfgs = [db[c.shape.mnk].best_config for c in cases]
    nat = [c.native() for c in or_cfgs]
    or_t = timed(lambda i, c: runner.launch(c, config=nat[i]))
    rate = lambda ts: [c.flops / t / 1e9 for c, t in zip(cases, ts)]  # noqa: E731
    g_dt, g_or, g_de = geomean(rate(dt_t)), geomean(rate(or_t)), geomean(rate(default_t))
    x3_idx = [i for i, c in enumerate(dt_cfgs) if c.family is KernelFamily.TF32X3]
    roof, parity = None, None
    if x3_idx:
        dom = max(x3_idx, key=lambda i: dt_t[i])
        c = cases[dom]
        runner.launch(c, config=dt_cfgs[dom].native())
        torch.cuda.synchronize()
        exact = c.dA.double() @ c.dB.double()
        parity = {"shape": list(c.shape.mnk), "config": dt_cfgs[dom].canonical(),
                  "rf_whole_matrix": float(torch.linalg.norm(c.dout.double() - exact) / torch.linalg.norm(exact)),
                  "bar": 1e-5}
        del exact
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) if (ROOT / "MEASURED_PEAKS.json").exists() else {}
        tf32_peak = float(peaks.get("bf16_tflops", 2250.0)) / 2
        ach = c.flops / dt_t[dom] / 1e12
        key = f"{'x'.join(map(str, c.shape.mnk))}:{dt_cfgs[dom].canonical()}"
        traffic = json.loads(TRAFFIC_FILE.read_text()).get(key) if TRAFFIC_FILE.exists() else None
        roof = {"bound": "tensor", "achieved": round(ach, 2), "peak": round(tf32_peak / 3, 1), "unit": "TFLOP/s",
                "frac": round(ach / (tf32_peak / 3), 4), "kernel": key, "traffic": traffic,
                "traffic_note": "DRAM bytes of the tc_gemm launch (ncu --set full); the lo parts are made in "
                                "shared memory, no other launch",
                "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst) / 2 = tf32, / 3 products per K step",
                "note": "event time covers the family path (one launch)"}
    fams = {}
    for c in dt_cfgs:
        fams[c.family.value] = fams.get(c.family.value, 0) + 1
    return {"workload": "deepbench_fp32 (same 40 shapes, same regime as the headline)",
            "space": "b200 fp32 families + tf32x3 (fp32-accurate, RF <= 1e-5)",
            "model": pipe["name"], "n_train": pipe["n_train"], "score_table_mode": pipe["score"],
            "dt_geomean": round(g_dt, 1), "oracle_geomean": round(g_or, 1), "default_geomean": round(g_de, 1),
            "dt_over_oracle": round(g_dt / g_or, 4), "dt_over_default": round(g_dt / g_de, 4),
            "dt_families": fams, "roofline": roof, "parity": parity,
            "per_shape": [[list(c.shape.mnk), round(a, 1), round(b, 1), d.canonical(), o.canonical()]
                          for c, a, b, d, o in zip(cases, rate(dt_t), rate(or_t), dt_cfgs, or_cfgs)]}


def _cpu_sweep_worker(job):
    """One single-threaded reference-CPU process of `tune --jobs nproc`
    (cli.py:198-228): times its shapes' sampled configs with the oracle port
    of the reference's numba kernels, warmup + repeats runs each."""
    shapes, cfgs, warmup, repeats = job
    from oracle import gemm as ogemm
    from paper_1806_07060_b200.kernels import KernelConfig
    from paper_1806_07060_b200.tuner import _bench_buffers
    ogemm.set_threads(1)
    n = 0
    flops = 0.0
    for mnk in shapes:
        from paper_1806_07060_b200.kernels import ProblemShape
        sh = ProblemShape(*mnk)
        A, B, C, _ = _bench_buffers(sh, np.float32, 0)
        for canon in cfgs:
            c = KernelConfig.from_canonical(canon)
            for _ in range(warmup + repeats):
                ogemm.execute(sh.M, sh.N, sh.K, 1.0, 0.0, False, False, A, B, C, c.family.value, *c.param_tuple())
            n += 1
            flops += 2.0 * sh.M * sh.N * sh.K * (warmup + repeats)
    return n, flops


def cpu_sweep(shapes, stride=8, warmup=1, repeats=3):
    """The reference's CPU sweep of the same shapes on all host cores (one
    single-threaded process per core, as `tune --jobs $(nproc)`), on every
    `stride`-th config of the reference space: configs/s measured, the full
    sweep's wall time extrapolated (labelled an estimate)."""
    import concurrent.futures
    import multiprocessing

    from oracle import gemm as ogemm
    from paper_1806_07060_b200.kernels import DeviceCaps, full_search_space
    from paper_1806_07060_b200.sharding import lpt_partition
    ogemm.build()
    space = [c.canonical() for c in full_search_space(DeviceCaps())]
    sample = space[::stride]
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    parts = [p for p in lpt_partition([s.mnk for s in shapes], cores, lambda m: m[0] * m[1] * m[2]) if p]
    t0 = time.perf_counter()
    with concurrent.futures.ProcessPoolExecutor(max_workers=len(parts),
                                                mp_context=multiprocessing.get_context("spawn")) as ex:
        res = list(ex.map(_cpu_sweep_worker, [(p, sample, warmup, repeats) for p in parts]))
    wall = time.perf_counter() - t0
    n = sum(r[0] for r in res)
    flops = sum(r[1] for r in res)
    full = len(space) * len(shapes)
    return {"configs_timed": n, "configs_per_shape_sampled": len(sample), "configs_per_shape_full": len(space),
            "wall_s": round(wall, 2), "configs_per_s": round(n / wall, 2),
            "swept_gflops_per_s": round(flops / wall / 1e9, 2), "processes": len(parts), "cores": cores,
            "full_sweep_wall_s_estimate": round(full / (n / wall), 1),
            "shapes_per_h_estimate": round(len(shapes) / (full / (n / wall)) * 3600, 1),
            "kind": "port", "how": f"oracle port of the reference's numba kernels, one single-threaded process "
                                   f"per core (tune --jobs nproc), every {stride}th config of the 576-config "
                                   f"reference space, warmup {warmup} + repeats {repeats}"}


def sweep_section(device, distributed, rank, world, with_cpu):
    """configs[3]: the exhaustive tuning sweep of acceptance C11's dataset,
    po2(64, 256) = 27 shapes, timing warmup 1 + repeats 3 (the reference's
    smoke config, test_acceptance.py:339-387), LPT-sharded shape-wise over the
    ranks with no collective (cli tune --gpus); wall time = max over ranks.
    Both the reference space (576 configs, what the CPU sweep times) and the
    B200 profile, the latter also in the shipped labels' regime (L2 flushed
    before every sample, 1 + 5); the reference's CPU sweep of the same
    shapes beside it."""
    import torch

    from paper_1806_07060_b200 import distributed as dist_mod
    from paper_1806_07060_b200.dataset import gen_po2
    from paper_1806_07060_b200.kernels import DeviceCaps, ProblemShape, full_search_space
    from paper_1806_07060_b200.sharding import sweep_cost
    from paper_1806_07060_b200.tuner import TimingPolicy, tune_exhaustive

    timing = TimingPolicy(warmup=1, repeats=3)
    shapes = [s if isinstance(s, ProblemShape) else ProblemShape(*s) for s in gen_po2(64, 256)]
    out = {"shapes": len(shapes), "dataset": "po2(64, 256) (acceptance C11)", "ranks": world, "scaling": "strong",
           "timing": "warmup 1 + repeats 3 (warm)"}
    tune_exhaustive(ProblemShape(64, 64, 64), DeviceCaps.b200(), timing)  # warm every kernel once
    flush = TimingPolicy(warmup=1, repeats=5, l2="flush")  # the shipped tables' label regime
    for name, caps, timing in (("reference_space", DeviceCaps(), timing), ("b200_space", DeviceCaps.b200(), timing),
                               ("b200_space_label_regime", DeviceCaps.b200(), flush)):
        n_cfg = len(full_search_space(caps))
        mine = dist_mod.shard(shapes, rank, world, lambda s: sweep_cost(s.mnk, n_cfg, 8))
        distributed.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for s in mine:
            tune_exhaustive(s, caps, timing)
        torch.cuda.synchronize()
        wall = distributed.reduce_max([time.perf_counter() - t0], device)[0]
        flops = sum(2.0 * s.M * s.N * s.K for s in shapes) * n_cfg * (timing.warmup + timing.repeats)
        out[name] = {"timing": f"warmup {timing.warmup} + repeats {timing.repeats} ({timing.l2})",
                     "configs_per_shape": n_cfg, "configs_timed": n_cfg * len(shapes), "wall_s": round(wall, 3),
                     "configs_per_s": round(n_cfg * len(shapes) / wall, 1),
                     "shapes_per_h": round(len(shapes) / wall * 3600, 1),
                     "swept_gflops_per_s": round(flops / wall / 1e9, 1)}
    if with_cpu:
        cpu = cpu_sweep(shapes)
        out["cpu_reference"] = cpu
        out["gpu_over_cpu_configs_per_s"] = round(out["reference_space"]["configs_per_s"] / cpu["configs_per_s"], 1)
    out["how"] = ("tune_exhaustive per shape on this rank's LPT shard; wall clock around the shard, max over "
                  "ranks (device-timed samples inside, CUDA events)")
    return out


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="skip the sharded-sweep sub-measurement")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        log("note: warmup raised to 3 (timing rules)")
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
