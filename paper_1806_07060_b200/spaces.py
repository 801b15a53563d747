"""Tuning-parameter domains and legality rules (dependency-free).

Restates the reference's parameter space (/root/reference/pkg/src/adaptgemm/
kernels.py:122-177) and adds the explicit B200 profile.  The build script
imports this module to decide which sm_100a kernel instantiations to
compile, so it must stay importable without numpy/torch.

Config tuples are ``(family, bm, bn, bk, tm, tn, uk)`` with family
``"direct"`` or ``"indirect"``.
"""

import itertools

# kernels.py:123-138 -- the reference domains, canonical order
DIRECT_DOMAINS = {
    "block_m": (8, 16, 32),
    "block_n": (8, 16, 32),
    "block_k": (8, 16),
    "tile_m": (1, 2, 4),
    "tile_n": (1, 2, 4),
    "unroll_k": (1,),
}
INDIRECT_DOMAINS = {
    "block_m": (16, 32, 64),
    "block_n": (16, 32, 64),
    "block_k": (8, 16, 32),
    "tile_m": (2, 4, 8),
    "tile_n": (2, 4, 8),
    "unroll_k": (1, 2),
}

# B200 profile: the reference space plus large CTA tiles that only pay off
# on a 148-SM part with 227 KB of shared memory per CTA.  Enumerated after
# the reference configs so that reference-profile class ids keep their
# meaning.  Kept small on purpose: every entry is a compiled instantiation.
B200_INDIRECT_EXTRA_DOMAINS = {
    "block_m": (64, 128, 256),
    "block_n": (64, 128, 256),
    "block_k": (8, 16, 32),
    "tile_m": (4, 8),
    "tile_n": (4, 8),
    "unroll_k": (1, 2),
}

# B200 profile, wide register tiles: 8 x 16 / 16 x 8 accumulators per
# thread (128 fp32 = 64 FFMA2 pairs), half the shared-memory fragment loads
# per FMA of an 8 x 8 tile; +3-5 % over 8 x 8 on >= 4096-class shapes
# (profiles/r01_exp_tiles.jsonl).  An explicit list: each is a compiled
# kernel, enumerated after the extra domains.
B200_INDIRECT_WIDE = ((128, 128, 16, 8, 16, 1), (128, 128, 32, 8, 16, 1), (128, 128, 16, 16, 8, 1),
                      (128, 128, 32, 16, 8, 1), (128, 256, 16, 8, 16, 1), (128, 256, 32, 8, 16, 1),
                      (256, 128, 16, 16, 8, 1), (256, 128, 32, 16, 8, 1))

# B200 profile, split-K family ("splitk"): the indirect core over `uk` equal
# K slices plus a fixed-order reduction.  For skinny / small-N shapes whose
# tile grid cannot fill 148 SMs.  Tiles are ones the indirect family already
# compiles (unroll 1), so the family adds no instantiations.
SPLITK_TILES = ((16, 16, 2, 2), (32, 16, 4, 2), (16, 32, 2, 4), (32, 32, 4, 4), (64, 16, 4, 2),
                (16, 64, 2, 4), (64, 32, 4, 4), (32, 64, 4, 4), (64, 64, 8, 4), (64, 64, 4, 8),
                (128, 64, 8, 4), (64, 128, 4, 8), (128, 64, 8, 8), (64, 128, 8, 8), (128, 128, 8, 8))
SPLITK_BLOCK_K = (16, 32)
SPLITK_SLICES = (2, 4, 8, 16)

# B200 tensor-core profile ("b200tc"), families "tf32" and "bf16": tcgen05.mma
# with TMEM accumulators fed by TMA (csrc/tc_kernels.cuh).  bm is the UMMA M
# (128: one CTA per tile; 256: a CTA pair on one TPC, tcgen05 cta_group::2),
# bn the UMMA N, bk one 128-byte K block (32 tf32 / 64 bf16 elements), tm
# the shared-memory pipeline depth; tn = uk = 1.  They enter
# only the b200tc search space: their numerics (tf32 / bf16 inputs, fp32
# accumulation) differ from the fp32 families, so fp32 tables and trees
# keep their meaning.
# "tf32x3" (3xTF32, fp32-accurate): the tf32 kernel with [hi | lo] parts of
# both operands in every stage and three MMAs per K step (twice the stage
# bytes of tf32); TMEM accumulates 256-k chunks that the epilogue sums in
# IEEE fp32, so bn <= 128.
TC_FAMILIES = ("tf32", "bf16", "tf32x3")
TC_BLOCK_M = (128, 256)
TC_BLOCK_N = (64, 128, 256)
TC_BLOCK_K = {"tf32": 32, "bf16": 64, "tf32x3": 32}
TC_PARTS = {"tf32": 1, "bf16": 1, "tf32x3": 2}
TC_STAGES = (2, 3, 4, 6)
TC_SMEM_LIMIT = 227 * 1024
# B200 profiles, TMA family ("tma"): the indirect core's tiles fed by TMA
# straight from the caller's row-major A and B (csrc/fp32_tma.cuh): no pack
# passes, mbarrier ring instead of cp.async + __syncthreads.  bk is one
# 128-byte swizzle row (32 fp32); uk = 1.  Transposed or unaligned operands
# run the same tile through the packed core (same bits).
TMA_TILES = ((128, 128, 8, 8), (128, 64, 8, 8), (64, 128, 8, 8), (64, 64, 8, 8), (64, 64, 8, 4),
             (64, 64, 4, 8), (64, 32, 8, 4), (32, 64, 4, 8))
TMA_BLOCK_K = 32
# B200 profiles, skinny families (csrc/skinny.cuh), K over `uk` cluster slices.
# skinny_n (N small): (tm, bn) register tiles (tm rows x all bn columns per
# thread); bm = 32 tm rows per CTA; tn = warps splitting the CTA's K range.
SKINNY_N_TILES = ((1, 16), (2, 16), (4, 16), (1, 32), (2, 32), (1, 64))
SKINNY_N_WARPS = (4, 8)
# skinny_m (M small): bm = M tile, tn = columns per thread (pairs for FFMA2),
# warps per CTA; bn = 32 * warps * tn; accumulators bm * tn <= 96.
SKINNY_M_TILES = ((8, 2), (8, 4), (16, 2), (16, 4), (24, 2), (32, 2), (40, 2), (48, 2))
SKINNY_M_WARPS = (4, 8)
SKINNY_SLICES = (1, 2, 3, 4, 6, 8, 12, 16)  # cluster sizes > 8 are non-portable
SKINNY_BLOCK_K = 32
SKINNY_FAMILIES = ("skinny_n", "skinny_m")
FAMILIES = ("direct", "indirect", "splitk") + TC_FAMILIES + ("tma",) + SKINNY_FAMILIES

PROFILE_REFERENCE = "reference"
PROFILE_B200 = "b200"
PROFILE_B200_TC = "b200tc"
PROFILES = (PROFILE_REFERENCE, PROFILE_B200, PROFILE_B200_TC)


def is_b200_profile(profile) -> bool:
    """The B200 profiles share the fp32 space; b200tc adds the tc families."""
    return profile in (PROFILE_B200, PROFILE_B200_TC)


TC_EPILOGUE_BYTES = 4 * 32 * 36 * 4  # per-warp 32 x 32 fp32 staging blocks (tc_kernels.cuh EPI_BYTES)


def tc_smem_bytes(bm, bn, stages, parts=1) -> int:
    """Dynamic shared memory of one tc CTA: the stage ring (128 rows of A and
    bn / (bm / 128) rows of B per stage and operand part) + slack + epilogue
    staging + barriers."""
    ctas = bm // 128
    return stages * parts * (128 + bn // ctas) * 128 + 1024 + TC_EPILOGUE_BYTES + 256

# DeviceCaps defaults (kernels.py:64-71) and the B200 profile caps
REFERENCE_CAPS = dict(tile_memory_cap=32768, register_tile_cap_direct=8,
                      register_tile_cap_indirect=32, element_size=4, max_threads=1024)
B200_CAPS = dict(tile_memory_cap=65536, register_tile_cap_direct=8,
                 register_tile_cap_indirect=128, element_size=4, max_threads=1024)

REGISTER_FILE = 65536  # 32-bit registers per SM (and per CTA) on sm_100

_FIELDS = ("block_m", "block_n", "block_k", "tile_m", "tile_n", "unroll_k")


def is_legal_tuple(family, bm, bn, bk, tm, tn, uk, caps) -> bool:
    """kernels.is_legal (kernels.py:145-158) + two sm_100 launch limits.

    The CTA thread limit (bm/tm)*(bn/tn) <= max_threads and the register
    file limit threads * (tm*tn + tm + tn + 24) <= 65536 (accumulators,
    fragments and ~24 addressing registers per thread) never bind on the
    reference domains under the reference caps (their maxima are 1024
    threads and 32768 registers), so the 144/432 legal counts are unchanged.
    """
    if min(bm, bn, bk, tm, tn, uk) < 1:
        return False
    if family not in FAMILIES:
        return False
    if family in TC_FAMILIES:
        # tensor-core resources are TMEM and the stage ring, not the
        # CUDA-core register/tile caps
        if bm not in TC_BLOCK_M or bk != TC_BLOCK_K[family] or tn != 1 or uk != 1:
            return False
        if bn % 32 or not 32 <= bn <= 256 or not 2 <= tm <= 8:
            return False
        # a pair splits B into whole 128-byte chunks per CTA (64 bf16 / 32 tf32)
        if bm == 256 and (bn // 2) % (128 // (2 if family == "bf16" else 4)):
            return False
        # tf32x3 keeps a bn-wide fp32 running sum per epilogue thread (tc_kernels.cuh)
        if family == "tf32x3" and bn > 128:
            return False
        return tc_smem_bytes(bm, bn, tm, TC_PARTS[family]) <= TC_SMEM_LIMIT
    if family == "direct" and uk != 1:
        return False
    if family == "skinny_n":
        if (tm, bn) not in SKINNY_N_TILES or bm != 32 * tm or bk != SKINNY_BLOCK_K:
            return False
        # a 2-deep TMA ring per warp fits one CTA's shared memory
        return tn in SKINNY_N_WARPS and uk in SKINNY_SLICES and tn * (4096 * tm + 128 * bn) <= 110 * 1024
    if family == "skinny_m":
        if (bm, tn) not in SKINNY_M_TILES or tm != 1 or bk != SKINNY_BLOCK_K or bn % (32 * tn):
            return False
        return bn // (32 * tn) in SKINNY_M_WARPS and uk in SKINNY_SLICES
    if family == "tma":
        # one 128-byte A row per k block, boxes of at most 256 rows, whole warps
        if bk != TMA_BLOCK_K or uk != 1 or bm > 256 or bn > 256 or bn % 4:
            return False
        if bm % tm or bn % tn or ((bm // tm) * (bn // tn)) % 32:
            return False
    if family == "splitk":
        if not 2 <= uk <= 64:  # uk carries the number of K slices
            return False
        if bm % tm or bn % tn:
            return False
    elif family != "tma" and (bm % tm or bn % tn or bk % uk):
        return False
    cap = caps["register_tile_cap_direct"] if family == "direct" else caps["register_tile_cap_indirect"]
    if tm * tn > cap:
        return False
    if (bm + bn) * bk * caps["element_size"] > caps["tile_memory_cap"]:
        return False
    threads = (bm // tm) * (bn // tn)
    if threads > caps.get("max_threads", 1024):
        return False
    if threads * (tm * tn + tm + tn + 24) > REGISTER_FILE:
        return False
    return True


def _product(family, domains):
    for vals in itertools.product(*(domains[f] for f in _FIELDS)):
        yield (family,) + vals


def enumerate_tuples(family, caps, profile=PROFILE_REFERENCE):
    """Legal configs of one family in deterministic canonical order."""
    if family in TC_FAMILIES:
        if profile != PROFILE_B200_TC:
            return []
        return [t for bm in TC_BLOCK_M for bn in TC_BLOCK_N for st in TC_STAGES
                for t in [(family, bm, bn, TC_BLOCK_K[family], st, 1, 1)] if is_legal_tuple(*t, caps)]
    if family == "tma":
        if not is_b200_profile(profile):
            return []
        return [t for (bm, bn, tm, tn) in TMA_TILES
                for t in [("tma", bm, bn, TMA_BLOCK_K, tm, tn, 1)] if is_legal_tuple(*t, caps)]
    if family == "skinny_n":
        if not is_b200_profile(profile):
            return []
        return [t for (tm, bn) in SKINNY_N_TILES for w in SKINNY_N_WARPS for s in SKINNY_SLICES
                for t in [("skinny_n", 32 * tm, bn, SKINNY_BLOCK_K, tm, w, s)] if is_legal_tuple(*t, caps)]
    if family == "skinny_m":
        if not is_b200_profile(profile):
            return []
        return [t for (bm, tn) in SKINNY_M_TILES for w in SKINNY_M_WARPS for s in SKINNY_SLICES
                for t in [("skinny_m", bm, 32 * w * tn, SKINNY_BLOCK_K, 1, tn, s)] if is_legal_tuple(*t, caps)]
    if family == "splitk":
        if not is_b200_profile(profile):
            return []
        return [t for (bm, bn, tm, tn) in SPLITK_TILES for bk in SPLITK_BLOCK_K for s in SPLITK_SLICES
                for t in [("splitk", bm, bn, bk, tm, tn, s)] if is_legal_tuple(*t, caps)]
    base = DIRECT_DOMAINS if family == "direct" else INDIRECT_DOMAINS
    out = [t for t in _product(family, base) if is_legal_tuple(*t, caps)]
    if is_b200_profile(profile) and family == "indirect":
        seen = set(out)
        for t in _product(family, B200_INDIRECT_EXTRA_DOMAINS):
            bm, bn = t[1], t[2]
            if max(bm, bn) < 128 or t in seen:
                continue
            # big tiles only with >= 64 threads: a 148-SM part needs warps
            if (bm // t[4]) * (bn // t[5]) < 64:
                continue
            if is_legal_tuple(*t, caps):
                out.append(t)
                seen.add(t)
        for w in B200_INDIRECT_WIDE:
            t = ("indirect",) + w
            if t not in seen and is_legal_tuple(*t, caps):
                out.append(t)
                seen.add(t)
    return out


def compiled_tuples():
    """Every (family, bm, bn, bk, tm, tn, uk) with a fully templated fp32
    kernel: both profiles' enumerations under their own caps."""
    out = []
    seen = set()
    for profile, caps in ((PROFILE_REFERENCE, REFERENCE_CAPS), (PROFILE_B200, B200_CAPS)):
        for fam in ("direct", "indirect"):
            for t in enumerate_tuples(fam, caps, profile):
                if t not in seen:
                    seen.add(t)
                    out.append(t)
    return out


# register-tile shapes with a run-time-tile-size kernel (any bm/bn/bk):
# float64 runs these, as do legal float32 configs outside the domains
RUNTIME_TILES = (1, 2, 4, 8)
RUNTIME_WIDE_TILES = ((8, 16), (16, 8))  # float64 only (build.py)
