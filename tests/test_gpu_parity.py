"""GPU parity: the sm_100a kernels vs the reference (golden) and the CPU oracle.

Bars (written in the asserts):
* gemm_reference (fp64-accumulating parity kernel): bit-identical to the
  reference's _kernel_reference;
* fp32 families: relative Frobenius error <= 1e-5 vs the float64 reference
  (BASELINE.json north star); float64 inputs: <= 1e-12;
* pack helper: bit-identical.
Full-size shapes (4096^3, DeepBench) are checked through size-independent
properties: a checksum identity (column sums) and exact rows.
"""

import itertools

import numpy as np
import pytest

from conftest import assert_rf, golden, golden_gemm, golden_shape, rand_operands, rel_frobenius
from oracle import gemm as ogemm
from paper_1806_07060_b200 import rng
from paper_1806_07060_b200.kernels import (
    ConfigError,
    DeviceCaps,
    KernelConfig,
    KernelFamily,
    ProblemShape,
    ShapeError,
    full_search_space,
    gemm_execute,
    gemm_reference,
    pack_padded,
)

pytestmark = pytest.mark.gpu

DIRECT_CFG = KernelConfig(KernelFamily.DIRECT, 16, 16, 8, 2, 2, 1)
INDIRECT_CFG = KernelConfig(KernelFamily.INDIRECT, 32, 32, 16, 4, 4, 2)
B200 = DeviceCaps.b200()


def _oracle_ref(s, A, B, C):
    return ogemm.reference(s.M, s.N, s.K, s.alpha, s.beta, s.transA, s.transB, A, B, C)


@pytest.mark.parametrize("meta", golden()["gemm"], ids=lambda m: m["name"])
def test_gemm_reference_bit_exact_vs_reference(meta):
    z = golden_gemm()
    k = meta["key"]
    s = golden_shape(meta)
    out = gemm_reference(s, z[f"{k}_A"], z[f"{k}_B"], z[f"{k}_C"])
    np.testing.assert_array_equal(out, z[f"{k}_ref"])


@pytest.mark.parametrize("meta", golden()["gemm"], ids=lambda m: m["name"])
def test_families_vs_reference_golden(meta):
    z = golden_gemm()
    k = meta["key"]
    s = golden_shape(meta)
    A, B, C = z[f"{k}_A"], z[f"{k}_B"], z[f"{k}_C"]
    for j, canon in enumerate(meta["execute_configs"]):
        cfg = KernelConfig.from_canonical(canon)
        out, sec = gemm_execute(s, cfg, A, B, C)
        assert sec > 0
        assert_rf(out, z[f"{k}_ref"], A.dtype)
        assert_rf(out, z[f"{k}_x{j}"], A.dtype)  # vs the reference's own family output


def test_identity_and_hand_example():
    s = ProblemShape(24, 24, 24)
    A = np.eye(24, dtype=np.float32)
    B = np.arange(576, dtype=np.float32).reshape(24, 24) / 100.0
    C = np.zeros((24, 24), np.float32)
    for cfg in (DIRECT_CFG, INDIRECT_CFG):
        out, _ = gemm_execute(s, cfg, A, B, C)
        np.testing.assert_array_equal(out, B)
    s1 = ProblemShape(1, 1, 1, alpha=2.0, beta=1.0)
    one = lambda v: np.array([[v]])  # noqa: E731
    assert gemm_reference(s1, one(2.0), one(3.0), one(5.0)).tolist() == [[17.0]]
    for cfg in (DIRECT_CFG, INDIRECT_CFG):
        assert gemm_execute(s1, cfg, one(2.0), one(3.0), one(5.0))[0].tolist() == [[17.0]]


@pytest.mark.parametrize("ta,tb", list(itertools.product([False, True], repeat=2)))
def test_transposes_all_families(ta, tb, search_space):
    s = ProblemShape(67, 45, 39, alpha=1.5, beta=0.5, transA=ta, transB=tb)
    A, B, C = rand_operands(s, seed=13)
    ref = _oracle_ref(s, A, B, C)
    for cfg in search_space[:: 7]:
        out, _ = gemm_execute(s, cfg, A, B, C)
        assert_rf(out, ref)


def test_every_config_of_both_profiles():
    """All 576 reference configs and every B200-profile config on a ragged shape."""
    s = ProblemShape(131, 77, 53, alpha=0.75, beta=1.25, transA=True)
    A, B, C = rand_operands(s, seed=3)
    ref = _oracle_ref(s, A, B, C)
    seen = set()
    for caps in (DeviceCaps(), B200):
        for cfg in full_search_space(caps):
            if cfg in seen:
                continue
            seen.add(cfg)
            out, _ = gemm_execute(s, cfg, A, B, C, caps)
            assert rel_frobenius(out, ref) <= 1e-5, cfg.canonical()
    assert len(seen) > 576


@pytest.mark.parametrize("mnk", [(1, 1, 1), (1, 37, 5), (37, 1, 5), (5, 37, 1), (64, 1, 1), (1, 1, 96),
                                 (96, 96, 1), (1, 96, 96), (300, 1, 700), (3, 1000, 2)])
def test_edge_dimensions(mnk, search_space):
    s = ProblemShape(*mnk, alpha=1.0, beta=0.5)
    A, B, C = rand_operands(s, seed=17)
    ref = _oracle_ref(s, A, B, C)
    for idx in rng.sample_without_replacement(len(search_space), 24, rng.mix(*mnk)):
        out, _ = gemm_execute(s, search_space[idx], A, B, C)
        assert_rf(out, ref)


def test_randomized_c1_generator(search_space):
    """The reference acceptance C1 generator (test_acceptance.py:78-111): 200
    shapes x 20 configs per family, vs the bit-exact CPU oracle."""
    stream = rng.SplitMix64(0xC1)
    fams = {f: [c for c in search_space if c.family is f] for f in (KernelFamily.DIRECT, KernelFamily.INDIRECT)}
    for case in range(200):
        s = ProblemShape(1 + stream.below(96), 1 + stream.below(96), 1 + stream.below(96),
                         alpha=(1.0, 1.5, 2.0)[stream.below(3)], beta=(0.0, 0.0, 0.5, 1.0)[stream.below(4)],
                         transA=bool(stream.below(2)), transB=bool(stream.below(2)))
        A, B, C = rand_operands(s, np.float32, seed=case)
        ref = _oracle_ref(s, A, B, C)
        for space in fams.values():
            for idx in rng.sample_without_replacement(len(space), 20, rng.mix(case, len(space))):
                out, _ = gemm_execute(s, space[idx], A, B, C)
                assert rel_frobenius(out, ref) <= 1e-5, (s, space[idx].canonical())


def test_float64_path(search_space):
    s = ProblemShape(53, 38, 70, alpha=2.0, beta=0.25, transB=True)
    A, B, C = rand_operands(s, np.float64, seed=19)
    ref = _oracle_ref(s, A, B, C)
    np.testing.assert_array_equal(gemm_reference(s, A, B, C), ref)
    for cfg in search_space[::11]:
        out, _ = gemm_execute(s, cfg, A, B, C)
        assert out.dtype == np.float64
        assert_rf(out, ref, np.float64)


def test_beta_zero_nan_semantics():
    """beta == 0: the direct family (like _kernel_direct) still reads C, so a
    NaN in C propagates; the indirect family skips C (kernels.py:318-321)."""
    s = ProblemShape(40, 40, 16, beta=0.0)
    A, B, C = rand_operands(s, seed=2)
    C[3, 5] = np.nan
    d, _ = gemm_execute(s, DIRECT_CFG, A, B, C)
    i, _ = gemm_execute(s, INDIRECT_CFG, A, B, C)
    od, _ = ogemm.execute(40, 40, 16, 1.0, 0.0, False, False, A, B, C, "direct", 16, 16, 8, 2, 2, 1)
    oi, _ = ogemm.execute(40, 40, 16, 1.0, 0.0, False, False, A, B, C, "indirect", 32, 32, 16, 4, 4, 2)
    assert np.isnan(d[3, 5]) and np.isnan(od[3, 5]) and np.isnan(d).sum() == 1
    assert np.isfinite(i).all() and np.isfinite(oi).all()


def test_padding_neutrality_bit_identical():
    """Aligned operands skip the pack; the packed path must give the same bits."""
    cfg = KernelConfig(KernelFamily.INDIRECT, 32, 32, 16, 4, 4, 2)
    s = ProblemShape(64, 32, 48, alpha=1.0, beta=0.5)
    A, B, C = rand_operands(s, seed=23)
    out, _ = gemm_execute(s, cfg, A, B, C)
    st = ProblemShape(64, 32, 48, alpha=1.0, beta=0.5, transA=True, transB=True)
    out_t, _ = gemm_execute(st, cfg, np.ascontiguousarray(A.T), np.ascontiguousarray(B.T), C)
    np.testing.assert_array_equal(out, out_t)


def test_pack_padded_matches_oracle():
    X = rand_operands(ProblemShape(37, 1, 21), seed=4)[0]
    for transpose in (False, True):
        rows, cols = (21, 37) if transpose else (37, 21)
        got = pack_padded(X, rows, cols, transpose, 64, 48)
        np.testing.assert_array_equal(got, ogemm.pack_padded(X, rows, cols, transpose, 64, 48))


def test_error_order_and_operands():
    s = ProblemShape(8, 8, 8)
    A, B, C = rand_operands(s)
    bad_cfg = KernelConfig(KernelFamily.DIRECT, 16, 16, 8, 4, 4, 1)
    with pytest.raises(ConfigError):
        gemm_execute(s, bad_cfg, A[:4], B, C)  # legality is checked before operands
    with pytest.raises(ShapeError):
        gemm_execute(s, DIRECT_CFG, A[:4], B, C)
    with pytest.raises(ShapeError):
        gemm_execute(s, DIRECT_CFG, A, B.astype(np.float64), C)
    with pytest.raises(ShapeError):
        gemm_execute(s, DIRECT_CFG, A.astype(np.int32), B.astype(np.int32), C.astype(np.int32))
    with pytest.raises(ShapeError):
        gemm_execute(s, DIRECT_CFG, A, B, C, out=np.empty((8, 7), np.float32))


def test_out_buffer_and_device_tensors():
    import torch
    s = ProblemShape(100, 70, 33, alpha=1.0, beta=1.0)
    A, B, C = rand_operands(s, seed=9)
    ref = _oracle_ref(s, A, B, C)
    out = np.empty((100, 70), np.float32)
    res, _ = gemm_execute(s, INDIRECT_CFG, A, B, C, out=out)
    assert res is out
    assert_rf(out, ref)
    dA, dB, dC = (torch.from_numpy(x).cuda() for x in (A, B, C))
    dout = torch.empty((100, 70), device="cuda")
    for cfg in (DIRECT_CFG, INDIRECT_CFG):
        r, _ = gemm_execute(s, cfg, dA, dB, dC, out=dout)
        assert r is dout
        assert_rf(dout.cpu().numpy(), ref)
    # non-contiguous device views are handled (copied to row-major)
    st = ProblemShape(100, 70, 33, alpha=1.0, beta=1.0, transA=True)
    dAt = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()
    r, _ = gemm_execute(st, INDIRECT_CFG, dAt, dB, dC)
    assert_rf(r.cpu().numpy(), ref)


def _checksum_ok(s, A, B, C, out, tol=1e-5):
    """Column-sum identity: 1^T (alpha op(A) op(B) + beta C) = alpha (1^T op(A)) op(B) + beta 1^T C."""
    opA = (A.T if s.transA else A).astype(np.float64)
    opB = (B.T if s.transB else B).astype(np.float64)
    want = s.alpha * (opA.sum(axis=0) @ opB) + s.beta * C.astype(np.float64).sum(axis=0)
    got = out.astype(np.float64).sum(axis=0)
    return rel_frobenius(got, want) <= tol


def test_wide_register_tiles_float32_and_float64():
    """B200 wide tiles (8x16 / 16x8 per thread): their own FFMA2 kernels in
    float32; float64 runs the 8-wide run-time-tile kernel (same elements)."""
    from paper_1806_07060_b200.spaces import B200_INDIRECT_WIDE
    for dt, bar in ((np.float32, 1e-5), (np.float64, 1e-12)):
        s = ProblemShape(301, 277, 97, alpha=1.5, beta=0.5, transB=True)
        A, B, C = rand_operands(s, dt, seed=23)
        ref = _oracle_ref(s, A, B, C)
        for w in B200_INDIRECT_WIDE:
            cfg = KernelConfig(KernelFamily.INDIRECT, *w)
            out, _ = gemm_execute(s, cfg, A, B, C, B200)
            assert out.dtype == dt
            assert rel_frobenius(out, ref) <= bar, (cfg.canonical(), dt)


@pytest.mark.parametrize("mnk,cfg", [
    ((5124, 9124, 2560), "indirect:128-256-32-8-16-1"),
    ((4096, 4096, 4096), "indirect:128-128-32-8-8-1"),
    ((5124, 700, 2048), "indirect:128-64-16-8-8-2"),
    ((35, 8457, 2560), "direct:8-32-16-2-4-1"),
    ((35, 8457, 2560), "indirect:16-64-32-2-8-1"),
    ((2048, 7000, 2048), "indirect:256-64-16-8-8-2"),
])
def test_full_size_properties(mnk, cfg):
    import torch
    s = ProblemShape(*mnk)
    A, B, C = rand_operands(s, seed=1)
    config = KernelConfig.from_canonical(cfg)
    out, _ = gemm_execute(s, config, A, B, C, B200)
    assert _checksum_ok(s, A, B, C, out)
    # 32 exact rows from the float64 product
    rows = np.array(rng.sample_without_replacement(s.M, min(32, s.M), 5))
    exact = A[rows].astype(np.float64) @ B.astype(np.float64)
    assert rel_frobenius(out[rows], exact) <= 1e-5
    # linearity in B on the device path: G(A, 2B) == 2 G(A, B) exactly (power-of-two scaling)
    dA, dB, dC = (torch.from_numpy(x).cuda() for x in (A, B, C))
    o1, _ = gemm_execute(s, config, dA, dB, dC, B200)
    o2, _ = gemm_execute(s, config, dA, dB * 2, dC, B200)
    assert torch.equal(o2, o1 * 2)


# ---------------------------------------------------------------------------
# split-K family (B200 profile)


@pytest.mark.parametrize("ta,tb", list(itertools.product([False, True], repeat=2)))
def test_splitk_parity_and_determinism(ta, tb):
    s = ProblemShape(70, 33, 1000, alpha=1.25, beta=0.75, transA=ta, transB=tb)
    A, B, C = rand_operands(s, seed=29)
    ref = _oracle_ref(s, A, B, C)
    for canon in ("splitk:16-16-16-2-2-2", "splitk:32-32-32-4-4-8", "splitk:64-64-32-8-4-16",
                  "splitk:128-64-16-8-8-4"):
        cfg = KernelConfig.from_canonical(canon)
        out1, _ = gemm_execute(s, cfg, A, B, C, B200)
        out2, _ = gemm_execute(s, cfg, A, B, C, B200)
        assert_rf(out1, ref)
        np.testing.assert_array_equal(out1, out2)  # fixed-order reduction: bitwise repeatable


def test_splitk_more_slices_than_k_tiles():
    s = ProblemShape(40, 40, 20, beta=0.5)  # 2 K tiles of 16, 16 slices requested
    A, B, C = rand_operands(s, seed=30)
    out, _ = gemm_execute(s, KernelConfig.from_canonical("splitk:16-16-16-2-2-16"), A, B, C, B200)
    assert_rf(out, _oracle_ref(s, A, B, C))


def test_splitk_illegal_under_reference_caps():
    s = ProblemShape(8, 8, 8)
    A, B, C = rand_operands(s)
    with pytest.raises(ConfigError):
        gemm_execute(s, KernelConfig.from_canonical("splitk:16-16-16-2-2-1"), A, B, C, B200)  # 1 slice


@pytest.mark.parametrize("mnk", [(4096, 16, 4096), (2048, 32, 2048), (35, 700, 2560)])
def test_splitk_full_size_skinny(mnk):
    s = ProblemShape(*mnk)
    A, B, C = rand_operands(s, seed=3)
    out, _ = gemm_execute(s, KernelConfig.from_canonical("splitk:32-16-32-4-2-16"), A, B, C, B200)
    assert _checksum_ok(s, A, B, C, out)
    rows = np.array(rng.sample_without_replacement(s.M, min(16, s.M), 9))
    exact = A[rows].astype(np.float64) @ B.astype(np.float64)
    assert rel_frobenius(out[rows], exact) <= 1e-5


@pytest.mark.parametrize("canon", ["splitk:32-16-32-4-2-16", "splitk:64-64-16-8-4-8", "splitk:128-128-32-8-8-2"])
def test_splitk_row_major_a_path(canon):
    """Aligned M, K with row-major A: split-K reads A in place (no pack)."""
    cfg = KernelConfig.from_canonical(canon)
    s = ProblemShape(4 * cfg.block_m, 48, 8 * cfg.block_k, alpha=0.5, beta=1.5, transB=True)
    A, B, C = rand_operands(s, seed=41)
    ref = _oracle_ref(s, A, B, C)
    out1, _ = gemm_execute(s, cfg, A, B, C, B200)
    out2, _ = gemm_execute(s, cfg, A, B, C, B200)
    assert_rf(out1, ref)
    np.testing.assert_array_equal(out1, out2)


SPLITK_ALL = [c for c in full_search_space(B200) if c.family is KernelFamily.SPLITK]


@pytest.mark.parametrize("mnk", [(70, 36, 1000), (257, 100, 644), (35, 708, 2560), (1000, 16, 64)])
def test_splitk_inplace_path_bit_identical_to_packed(mnk):
    """Row-major A and B with K, N multiples of 4: the split-K family runs the
    pack-free in-place core.  Storing A transposed (transA) forces the packed
    core on the same products in the same order: the bits must agree."""
    s = ProblemShape(*mnk, alpha=1.25, beta=0.5)
    A, B, C = rand_operands(s, seed=mnk[0])
    st = ProblemShape(*mnk, alpha=1.25, beta=0.5, transA=True)
    At = np.ascontiguousarray(A.T)
    ref = _oracle_ref(s, A, B, C)
    for cfg in SPLITK_ALL[::3]:
        out_inplace, _ = gemm_execute(s, cfg, A, B, C, B200)
        out_packed, _ = gemm_execute(st, cfg, At, B, C, B200)
        np.testing.assert_array_equal(out_inplace, out_packed, err_msg=cfg.canonical())
        assert rel_frobenius(out_inplace, ref) <= 1e-5, cfg.canonical()


def test_splitk_inplace_device_offsets_and_fallbacks():
    """Sub-matrix views (leading dimension > K) stay in place; K % 4 != 0 or
    an unaligned base falls back to the packed path with the same result."""
    import torch
    cfg = KernelConfig.from_canonical("splitk:64-64-16-8-4-8")
    for (m, n, k), off in (((300, 64, 512), 0), ((300, 64, 510), 0), ((300, 64, 512), 1)):
        s = ProblemShape(m, n, k)
        A, B, C = rand_operands(s, seed=k + off)
        big = torch.zeros((m, k + 8 + off), dtype=torch.float32, device="cuda")
        big[:, off:off + k] = torch.from_numpy(A).cuda()
        dA = big[:, off:off + k]
        dB, dC = torch.from_numpy(B).cuda(), torch.from_numpy(C).cuda()
        out, _ = gemm_execute(s, cfg, dA, dB, dC, B200)
        want, _ = gemm_execute(ProblemShape(m, n, k, transA=True), cfg, np.ascontiguousarray(A.T), B, C, B200)
        np.testing.assert_array_equal(out.cpu().numpy(), want)


@pytest.mark.parametrize("slices", [3, 8, 16, 32, 64])
def test_splitk_inplace_cluster_and_slab_reductions(slices):
    """Up to 8 slices reduce inside a thread-block cluster over DSMEM; more
    (legal up to 64) take the partial-slab + reduction-kernel path.  Both sum
    the slices in order, so the packed (transA) path gives the same bits."""
    cfg = KernelConfig(KernelFamily.SPLITK, 32, 32, 16, 4, 4, slices)
    s = ProblemShape(100, 68, 2048, alpha=1.5, beta=0.25)
    A, B, C = rand_operands(s, seed=slices)
    out, _ = gemm_execute(s, cfg, A, B, C, B200)
    st = ProblemShape(100, 68, 2048, alpha=1.5, beta=0.25, transA=True)
    want, _ = gemm_execute(st, cfg, np.ascontiguousarray(A.T), B, C, B200)
    np.testing.assert_array_equal(out, want)
    assert_rf(out, _oracle_ref(s, A, B, C))


TMA_ALL = [c for c in full_search_space(B200) if c.family is KernelFamily.TMA]


@pytest.mark.parametrize("mnk,beta", [((300, 260, 516), 0.0), ((129, 68, 36), 0.5), ((1000, 1000, 1000), 0.0),
                                      ((77, 1024, 4), 1.0)])
def test_tma_family_bit_identical_to_packed_core(mnk, beta):
    """The TMA-fed core (row-major operands, zero fill by the TMA unit) and the
    packed indirect core with the same tile compute the same FMA sequence."""
    s = ProblemShape(*mnk, alpha=1.25, beta=beta)
    A, B, C = rand_operands(s, seed=sum(mnk))
    ref = _oracle_ref(s, A, B, C)
    assert len(TMA_ALL) == 8
    for cfg in TMA_ALL:
        packed = KernelConfig(KernelFamily.INDIRECT, cfg.block_m, cfg.block_n, 32, cfg.tile_m, cfg.tile_n, 1)
        out_tma, _ = gemm_execute(s, cfg, A, B, C, B200)
        out_packed, _ = gemm_execute(s, packed, A, B, C, B200)
        np.testing.assert_array_equal(out_tma, out_packed, err_msg=cfg.canonical())
        assert rel_frobenius(out_tma, ref) <= 1e-5


def test_tma_family_fallbacks():
    """Transposed operands, K % 4 != 0 and float64 run the packed path."""
    cfg = KernelConfig.from_canonical("tma:64-64-32-8-8-1")
    for s in (ProblemShape(90, 70, 50, transA=True, beta=0.5), ProblemShape(90, 70, 50, transB=True),
              ProblemShape(90, 70, 51)):
        A, B, C = rand_operands(s, seed=5)
        out, _ = gemm_execute(s, cfg, A, B, C, B200)
        assert_rf(out, _oracle_ref(s, A, B, C))
    s = ProblemShape(90, 70, 52, beta=0.5)
    A, B, C = rand_operands(s, np.float64, seed=6)
    out, _ = gemm_execute(s, cfg, A, B, C, B200)
    assert out.dtype == np.float64 and rel_frobenius(out, _oracle_ref(s, A, B, C)) <= 1e-12


def test_every_b200_fp32_family_config_runs_float64():
    """Legality is dtype-independent (kernels.py:145-158): every config of the
    B200 profile's CUDA-core families runs float64 operands (run-time-tile
    kernels; a larger register tile when the float64 CTA would exceed the
    kernel's thread bound) at the float64 bar."""
    from paper_1806_07060_b200.kernels import full_search_space
    s = ProblemShape(67, 45, 33, alpha=1.5, beta=0.5)
    A, B, C = rand_operands(s, np.float64, seed=41)
    ref = _oracle_ref(s, A, B, C)
    bad = []
    for cfg in full_search_space(B200):
        out, _ = gemm_execute(s, cfg, A, B, C, B200)
        if rel_frobenius(out, ref) > 1e-12:
            bad.append(cfg.canonical())
    assert not bad, bad[:10]


def test_tc_config_on_float64_falls_back_in_dispatch():
    """The tf32/bf16 families have no float64 kernels: gemm_execute raises
    ConfigError, and the native dispatch takes the fallback config."""
    from paper_1806_07060_b200 import codegen, model
    s = ProblemShape(40, 30, 20)
    A, B, C = rand_operands(s, np.float64, seed=42)
    tc = KernelConfig.from_canonical("bf16:128-128-64-4-1-1")
    with pytest.raises(ConfigError):
        gemm_execute(s, tc, A, B, C, DeviceCaps.b200_tc())
    tree = model.train([((40, 30, 20), 0)])
    sel = codegen.CompiledSelector(tree, {0: tc})
    out, picked, fb = codegen.dispatch_native(sel, s, A, B, C, DeviceCaps.b200_tc())
    assert fb and picked == codegen.FALLBACK_CONFIG
    assert rel_frobenius(out, _oracle_ref(s, A, B, C)) <= 1e-12


# ---------------------------------------------------------------------------
# skinny families (csrc/skinny.cuh, B200 profile)


@pytest.mark.parametrize("family,mnk", [
    ("skinny_n", (300, 16, 517)), ("skinny_n", (97, 40, 96)), ("skinny_n", (1000, 64, 1000)),
    ("skinny_m", (35, 700, 517)), ("skinny_m", (9, 333, 96)), ("skinny_m", (64, 1001, 300)),
])
def test_skinny_every_config(family, mnk):
    """Every config of the family on ragged shapes (M, N not tile multiples,
    K not a multiple of 32, N odd for skinny_m), alpha / beta with C read:
    RF <= 1e-5 vs the fp64 reference, and bitwise repeatable (fixed-order
    cluster reduction)."""
    from paper_1806_07060_b200.kernels import enumerate_search_space
    s = ProblemShape(*mnk, alpha=1.25, beta=0.5)
    A, B, C = rand_operands(s, seed=51)
    ref = _oracle_ref(s, A, B, C)
    fam = KernelFamily(family)
    cfgs = enumerate_search_space(fam, B200)
    assert cfgs
    for cfg in cfgs:
        out1, _ = gemm_execute(s, cfg, A, B, C, B200)
        assert rel_frobenius(out1, ref) <= 1e-5, cfg.canonical()
    for cfg in cfgs[::7]:
        out1, _ = gemm_execute(s, cfg, A, B, C, B200)
        out2, _ = gemm_execute(s, cfg, A, B, C, B200)
        np.testing.assert_array_equal(out1, out2)


@pytest.mark.parametrize("ta,tb", list(itertools.product([False, True], repeat=2)))
def test_skinny_fallback_paths(ta, tb):
    """Transposed operands, unaligned rows and float64 run the families'
    split-K fallback at the same bars."""
    for canon in ("skinny_n:64-16-32-2-4-4", "skinny_m:40-256-32-1-2-8"):
        cfg = KernelConfig.from_canonical(canon)
        for dt, bar in ((np.float32, 1e-5), (np.float64, 1e-12)):
            s = ProblemShape(45, 37, 203, alpha=0.75, beta=0.25, transA=ta, transB=tb)  # K % 4 != 0
            A, B, C = rand_operands(s, dt, seed=52)
            out, _ = gemm_execute(s, cfg, A, B, C, B200)
            assert rel_frobenius(out, _oracle_ref(s, A, B, C)) <= bar, (canon, dt)


def test_skinny_full_size_deepbench():
    import torch
    for mnk, canon in (((4096, 16, 4096), "skinny_n:64-16-32-2-4-4"), ((7680, 16, 2560), "skinny_n:64-16-32-2-4-2"),
                       ((35, 8457, 2560), "skinny_m:40-256-32-1-2-16"), ((35, 700, 2048), "skinny_m:16-256-32-1-2-16")):
        s = ProblemShape(*mnk)
        A, B, C = rand_operands(s, seed=53)
        dA, dB, dC = (torch.from_numpy(x).cuda() for x in (A, B, C))
        exact = dA.double() @ dB.double()
        out, _ = gemm_execute(s, KernelConfig.from_canonical(canon), dA, dB, dC, B200)
        rf = float(torch.linalg.norm(out.double() - exact) / torch.linalg.norm(exact))
        assert rf <= 1e-5, (mnk, canon, rf)
