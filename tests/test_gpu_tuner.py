"""Device-timed tuning sweeps on the GPU (tuner.py semantics)."""

import warnings

import numpy as np
import pytest

from conftest import golden
from paper_1806_07060_b200.kernels import DeviceCaps, KernelConfig, KernelFamily, ProblemShape, is_legal
from paper_1806_07060_b200.tuner import (
    DeviceBuffers,
    TimingPolicy,
    flops_of,
    load_table,
    save_table,
    table_filename,
    time_configs,
    tune_exhaustive,
    tune_random,
)

pytestmark = pytest.mark.gpu
FAST = TimingPolicy(warmup=0, repeats=1)
TINY = ProblemShape(9, 8, 7)


@pytest.fixture(scope="module")
def tiny_table():
    return tune_exhaustive(TINY, DeviceCaps(), FAST)


def test_exhaustive_covers_both_families(tiny_table):
    assert len(tiny_table.measurements) == 576
    assert {m.config.family for m in tiny_table.measurements} == {KernelFamily.DIRECT, KernelFamily.INDIRECT}


def test_exhaustive_argmax_invariants(tiny_table, default_caps):
    best = tiny_table.measurements[tiny_table.best_overall]
    assert all(best.gflops >= m.gflops for m in tiny_table.measurements)
    for fam, idx in ((KernelFamily.DIRECT, tiny_table.best_direct), (KernelFamily.INDIRECT, tiny_table.best_indirect)):
        fb = tiny_table.measurements[idx]
        assert fb.config.family is fam
        assert all(fb.gflops >= m.gflops for m in tiny_table.measurements if m.config.family is fam)
    for m in tiny_table.measurements:
        assert m.elapsed > 0 and is_legal(m.config, default_caps)
        assert m.gflops == pytest.approx(flops_of(TINY) / m.elapsed / 1e9)
        assert m.elapsed < 1e-3  # device time of a 9x8x7 GEMM, not launch + sync overhead


def test_family_restricted_and_random(default_caps):
    t = tune_exhaustive(TINY, default_caps, FAST, families=(KernelFamily.DIRECT,))
    assert len(t.measurements) == 144 and t.best_indirect is None
    r = tune_random(TINY, default_caps, samples=10, seed=42, timing=FAST)
    assert [m.config.canonical() for m in r.measurements] == golden()["tune_random"]["10,42"]
    with pytest.warns(RuntimeWarning, match="clamping"):
        c = tune_random(TINY, default_caps, samples=10_000, seed=1, timing=FAST)
    assert len(c.measurements) == 576
    with pytest.raises(ValueError):
        tune_random(TINY, default_caps, samples=0, seed=1, timing=FAST)


def test_table_round_trip(tmp_path, tiny_table):
    p = tmp_path / table_filename(TINY)
    save_table(tiny_table, p, {"config_hash": "abc"})
    back = load_table(p)
    assert [(m.config, m.elapsed, m.gflops) for m in back.measurements] == \
        [(m.config, m.elapsed, m.gflops) for m in tiny_table.measurements]
    assert back.best_overall == tiny_table.best_overall
    assert back.meta["timer"] == "cuda-events" and back.meta["aggregate"] == "median"


def test_b200_profile_sweep_and_perf_floor():
    caps = DeviceCaps.b200()
    s = ProblemShape(2048, 2048, 2048)
    t = tune_exhaustive(s, caps, TimingPolicy(1, 3))
    assert len(t.measurements) == 144 + 626 + 120 + 8 + 88 + 128  # direct + indirect + split-K + tma + skinny_n + skinny_m
    # a big square must reach a large fraction of the FP32 FFMA peak
    assert t.peak_gflops > 35000, t.best_config.canonical()
    assert t.best_config.family is KernelFamily.INDIRECT


def test_timing_repeatability():
    s = ProblemShape(1024, 1024, 1024)
    bufs = DeviceBuffers(s)
    cfg = [KernelConfig(KernelFamily.INDIRECT, 64, 64, 16, 8, 4, 1), KernelConfig(KernelFamily.DIRECT, 32, 32, 16, 2, 4, 1)]
    a = time_configs(s, cfg, DeviceCaps(), TimingPolicy(2, 7), bufs)
    b = time_configs(s, cfg, DeviceCaps(), TimingPolicy(2, 7), bufs)
    for x, y in zip(a, b):
        assert abs(x - y) / min(x, y) < 0.25


@pytest.mark.parametrize("profile", ["b200", "b200_tc"])
def test_tune_random_b200_profiles(profile):
    """tune_random (tuner.py:188-221) over the enlarged B200 spaces: the
    seeded sample is the host-side sampler's, allocated per family by
    largest remainder, every pick legal and timed on the device."""
    from paper_1806_07060_b200.kernels import enumerate_search_space, full_search_space
    from paper_1806_07060_b200.tuner import random_configs

    caps = getattr(DeviceCaps, profile)()
    s = ProblemShape(300, 200, 500)
    samples, seed = 64, 1806
    t = tune_random(s, caps, samples=samples, seed=seed, timing=FAST)
    picked = [m.config for m in t.measurements]
    assert picked == random_configs(caps, samples, seed)
    assert len(set(picked)) == samples and all(is_legal(c, caps) for c in picked)
    assert all(m.gflops > 0 for m in t.measurements) and t.best_config in picked
    total = len(full_search_space(caps))
    for fam in KernelFamily:
        size = len(enumerate_search_space(fam, caps))
        got = sum(1 for c in picked if c.family is fam)
        exact = samples * size / total
        assert int(exact) <= got <= int(exact) + 1, (fam, got, exact)
    again = tune_random(s, caps, samples=samples, seed=seed, timing=FAST)
    assert [m.config for m in again.measurements] == picked
