"""GPU parity of the tensor-core families (tf32, bf16, tf32x3; csrc/tc_kernels.cuh).

No reference analogue (BASELINE.json configs[4] adds them to the search
space).  Bars, as SURVEY.md section 8(c) states them:
* vs the float64 reference on the float32 inputs: relative Frobenius error
  <= 1e-3 (tf32) / <= 1e-2 (bf16) -- the input-rounding floor is ~2.6e-4 /
  ~2.1e-3 independent of K;
* vs the float64 reference on inputs pre-rounded the way the family sees
  them (tf32: the tensor core reads the fp32 bits and drops the low 13
  mantissa bits; bf16: the convert pass rounds to nearest even): <= 1e-5,
  i.e. only fp32 accumulation error remains.
* tf32x3 (3xTF32: hi/lo operand split, three tf32 MMAs per K step) is held
  to the fp32 families' bar: <= 1e-5 vs the float64 reference on the
  float32 inputs themselves, at every K.
beta == 0 never reads C (the indirect family's semantics, kernels.py:318-321).
"""

import numpy as np
import pytest

from conftest import rand_operands, rel_frobenius
from oracle import gemm as ogemm
from paper_1806_07060_b200.kernels import (DeviceCaps, KernelConfig, KernelFamily, ProblemShape,
                                           enumerate_search_space, gemm_execute)

pytestmark = pytest.mark.gpu

TC = DeviceCaps.b200_tc()
RF_TOL = {KernelFamily.TF32: 1e-3, KernelFamily.BF16: 1e-2, KernelFamily.TF32X3: 1e-5}
FAMS = [KernelFamily.TF32, KernelFamily.BF16, KernelFamily.TF32X3]
RF_TOL_ROUNDED = 1e-5


def round_tf32(x):
    """The tensor core's reading of an fp32 operand as tf32: 10 mantissa
    bits kept, the low 13 dropped (truncation toward zero)."""
    b = np.ascontiguousarray(x, np.float32).view(np.uint32)
    return (b & np.uint32(0xFFFFE000)).view(np.float32)


def round_tf32_rna(x):
    b = np.ascontiguousarray(x, np.float32).view(np.uint32)
    return ((b + np.uint32(0x1000)) & np.uint32(0xFFFFE000)).view(np.float32)


def round_bf16(x):
    """__float2bfloat16_rn: keep 7 mantissa bits, round half to even."""
    b = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    r = (b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000
    return r.astype(np.uint32).view(np.float32)


ROUND = {KernelFamily.TF32: round_tf32, KernelFamily.BF16: round_bf16, KernelFamily.TF32X3: lambda x: x}


def _ref(s, A, B, C):
    return ogemm.reference(s.M, s.N, s.K, s.alpha, s.beta, s.transA, s.transB, A, B, C)


def _check(s, cfg, seed=0):
    A, B, C = rand_operands(s, np.float32, seed)
    out, sec = gemm_execute(s, cfg, A, B, C, TC)
    assert sec > 0
    err = rel_frobenius(out, _ref(s, A, B, C))
    assert err <= RF_TOL[cfg.family], (cfg.canonical(), s, err)
    rnd = ROUND[cfg.family]
    err_r = rel_frobenius(out, _ref(s, rnd(A), rnd(B), C))
    if err_r > RF_TOL_ROUNDED and cfg.family is KernelFamily.TF32:
        alt = rel_frobenius(out, _ref(s, round_tf32_rna(A), round_tf32_rna(B), C))
        raise AssertionError(f"{cfg.canonical()} {s}: rf vs truncated {err_r:.3e}, vs rna {alt:.3e}")
    assert err_r <= RF_TOL_ROUNDED, (cfg.canonical(), s, err_r)
    return err, err_r


def _configs(fam):
    return enumerate_search_space(fam, TC)


def test_tc_space_enumerates_only_in_tc_profile():
    for fam in FAMS:
        assert enumerate_search_space(fam, DeviceCaps.b200()) == []
        assert len(_configs(fam)) >= 6


@pytest.mark.parametrize("fam", FAMS, ids=lambda f: f.value)
@pytest.mark.parametrize("mnk", [(1, 1, 1), (7, 13, 5), (128, 128, 32), (129, 257, 33), (35, 1000, 2560),
                                 (300, 64, 1), (64, 300, 4097)])
@pytest.mark.parametrize("trans", [(False, False), (True, False), (False, True), (True, True)],
                         ids=["NN", "TN", "NT", "TT"])
def test_tc_shapes_and_transposes(fam, mnk, trans):
    s = ProblemShape(*mnk, alpha=1.0, beta=0.0, transA=trans[0], transB=trans[1])
    _check(s, _configs(fam)[0])


@pytest.mark.parametrize("fam", FAMS, ids=lambda f: f.value)
def test_tc_every_config(fam):
    # 333 x 517 x 260: ragged in every dimension; the persistent grid wraps
    # when tiles exceed the SM count (checked at 2048^2 below)
    s = ProblemShape(333, 517, 260, alpha=1.25, beta=-0.5)
    for cfg in _configs(fam):
        _check(s, cfg)


@pytest.mark.parametrize("fam", FAMS, ids=lambda f: f.value)
def test_tc_persistent_wrap_rows(fam):
    """2048 x 2048 x 1024: up to 512 tiles over 148 persistent CTAs.  Checked
    on 64 exact rows spread over the matrix (pre-rounded float64)."""
    s = ProblemShape(2048, 2048, 1024)
    A, B, C = rand_operands(s, np.float32, 3)
    rnd = ROUND[fam]
    rows = np.arange(0, 2048, 32)
    exact = rnd(A)[rows].astype(np.float64) @ rnd(B).astype(np.float64)
    for cfg in _configs(fam):
        out, _ = gemm_execute(s, cfg, A, B, C, TC)
        assert rel_frobenius(out[rows], exact) <= RF_TOL_ROUNDED, cfg.canonical()


@pytest.mark.parametrize("fam", FAMS, ids=lambda f: f.value)
def test_tc_beta_zero_never_reads_c(fam):
    s = ProblemShape(70, 90, 40, alpha=2.0, beta=0.0)
    A, B, C = rand_operands(s, np.float32, 5)
    C[:] = np.nan
    out, _ = gemm_execute(s, _configs(fam)[0], A, B, C, TC)
    assert np.isfinite(out).all()
    s1 = ProblemShape(70, 90, 40, alpha=2.0, beta=1.0)
    out1, _ = gemm_execute(s1, _configs(fam)[0], A, B, C, TC)
    assert np.isnan(out1).all()


def test_tc_rejects_float64():
    from paper_1806_07060_b200.kernels import ConfigError
    s = ProblemShape(16, 16, 16)
    A, B, C = rand_operands(s, np.float64)
    with pytest.raises(ConfigError):
        gemm_execute(s, _configs(KernelFamily.TF32)[0], A, B, C, TC)


@pytest.mark.parametrize("mnk", [(256, 256, 8192), (1000, 700, 4096), (35, 2000, 2560)])
def test_tf32x3_accuracy_matches_fp32_families(mnk):
    """3xTF32 against the CUDA-core fp32 path on the same inputs: both within
    the fp32 bar of the float64 product, and the tensor-pipe error no more
    than 4x the FFMA error (long K included)."""
    s = ProblemShape(*mnk)
    A, B, C = rand_operands(s, np.float32, 11)
    ref = _ref(s, A, B, C)
    x3, _ = gemm_execute(s, _configs(KernelFamily.TF32X3)[-1], A, B, C, TC)
    f32, _ = gemm_execute(s, KernelConfig(KernelFamily.INDIRECT, 64, 64, 16, 4, 4, 1), A, B, C, TC)
    e3, e32 = rel_frobenius(x3, ref), rel_frobenius(f32, ref)
    assert e3 <= 1e-5 and e32 <= 1e-5, (e3, e32)
    assert e3 <= 4 * e32 + 1e-7, (e3, e32)
