"""Pin the CPU oracle against outputs of the reference itself (CPU only).

The oracle (oracle/) is the checker of every GPU parity test and the CPU
baseline of bench.py, so it is pinned first: its GEMM loop nests must be
bit-identical to the reference's numba kernels, and its CART must grow the
reference's trees, on the golden fixtures made by tests/golden/make_golden.py.
"""

import hashlib
import json

import numpy as np
import pytest

from conftest import golden, golden_gemm, golden_shape
from oracle import cart as ocart
from oracle import gemm as ogemm


@pytest.fixture(scope="module", autouse=True)
def _built():
    ogemm.build()


def _case_ids():
    return [m["key"] for m in golden()["gemm"]]


@pytest.mark.parametrize("key", _case_ids())
def test_oracle_reference_bit_exact(key):
    meta = next(m for m in golden()["gemm"] if m["key"] == key)
    z = golden_gemm()
    s = golden_shape(meta)
    A, B, C = z[f"{key}_A"], z[f"{key}_B"], z[f"{key}_C"]
    out = ogemm.reference(s.M, s.N, s.K, s.alpha, s.beta, s.transA, s.transB, A, B, C)
    np.testing.assert_array_equal(out, z[f"{key}_ref"])


@pytest.mark.parametrize("key", _case_ids())
def test_oracle_families_bit_exact(key):
    meta = next(m for m in golden()["gemm"] if m["key"] == key)
    z = golden_gemm()
    s = golden_shape(meta)
    A, B, C = z[f"{key}_A"], z[f"{key}_B"], z[f"{key}_C"]
    for j, canon in enumerate(meta["execute_configs"]):
        fam, params = canon.split(":")
        bm, bn, bk, tm, tn, uk = map(int, params.split("-"))
        out, sec = ogemm.execute(s.M, s.N, s.K, s.alpha, s.beta, s.transA, s.transB, A, B, C,
                                 fam, bm, bn, bk, tm, tn, uk)
        np.testing.assert_array_equal(out, z[f"{key}_x{j}"], err_msg=canon)
        assert sec > 0


def test_oracle_pack_padded():
    X = np.arange(12, dtype=np.float32).reshape(3, 4)
    P = ogemm.pack_padded(X, 3, 4, False, 4, 8)
    assert P.shape == (4, 8) and P[:3, :4].tolist() == X.tolist() and not P[3:].any() and not P[:, 4:].any()
    T = ogemm.pack_padded(X, 4, 3, True, 8, 4)
    np.testing.assert_array_equal(T[:4, :3], X.T)


def test_oracle_hand_example():
    # test_kernels.py:44-49: 2 * (2 * 3) + 1 * 5 = 17
    out = ogemm.reference(1, 1, 1, 2.0, 1.0, False, False, np.array([[2.0]]), np.array([[3.0]]),
                          np.array([[5.0]]))
    assert out.tolist() == [[17.0]]


# ---------------------------------------------------------------------------
# CART


def _fingerprint(nodes, meta):
    doc = {"format_version": 1, "feature_names": ["M", "N", "K"], "root": 0, "nodes": nodes, "meta": meta}
    return hashlib.sha256(json.dumps(doc, sort_keys=True, separators=(",", ":")).encode()).hexdigest()


def _meta(records, h, L):
    return {"max_height": h, "min_samples_leaf": L,
            "effective_min_samples_leaf": ocart.effective_leaf(L, len(records)), "train_size": len(records)}


def test_oracle_best_split_cases():
    g = golden()["cart"]
    fixture = [((64, 1, 1), 0), ((128, 1, 1), 0), ((256, 1, 1), 1), ((512, 1, 1), 1)]
    f, t, _ = ocart.split_search(fixture, 1)
    assert [f, t] == g["best_split_fixture"][:2]
    for case in g["best_split_cases"]:
        samples = [(tuple(f), lab) for f, lab in case["samples"]]
        got = ocart.split_search(samples, case["min_leaf"])
        want = case["result"]
        if want is None:
            assert got is None
        else:
            assert (got[0], got[1]) == (want[0], want[1])
            num, den = got[2]
            assert 1.0 - (num / den) / len(samples) == pytest.approx(want[2], abs=1e-15)


def test_oracle_random_trees_match_reference():
    import sys
    sys.setrecursionlimit(10000)
    for case in golden()["cart"]["random_trees"]:
        recs = [(tuple(f), lab) for f, lab in case["records"]]
        nodes = ocart.grow(recs, case["max_height"], case["min_leaf"])
        assert _fingerprint(nodes, _meta(recs, case["max_height"], case["min_leaf"])) == case["fingerprint"]


def test_oracle_grid_trees_match_reference():
    g = golden()["cart"]["grids"]["po2_64_512"]
    from paper_1806_07060_b200.dataset import gen_po2
    feats = [s.mnk for s in gen_po2(64, 512)]
    recs = list(zip(feats, g["labels"]))
    for name, doc in g["trees"].items():
        h_txt, l_txt = name[1:].split("-L")
        h = None if h_txt == "Max" else int(h_txt)
        L = float(l_txt) if "." in l_txt else int(l_txt)
        nodes = ocart.grow(recs, h, L)
        assert _fingerprint(nodes, _meta(recs, h, L)) == doc["fingerprint"], name


def test_oracle_route_matches_reference_predictions():
    for name, doc in golden()["cart"]["full_trees"].items():
        nodes = doc["tree"]["nodes"]
        for p, cid in doc["predictions"]:
            assert ocart.route(nodes, p) == cid
