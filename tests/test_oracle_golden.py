"""Pin the C oracle (oracle/rs_oracle.c) to the reference's own outputs.

The fixtures were produced by running the reference package itself
(tests/golden/make_golden.py).  If these pass, the oracle is a faithful
restatement and can judge the CUDA path in the -m gpu tests.
"""

import numpy as np
import pytest

from golden_io import (MODES, OVERFLOWS, SCENES, SOUPS, TREE_FIELDS, TREE_SIZES,
                       assert_result_fields, expected, load)
from oracle import oracle as O


def test_morton_known_answers():
    fx = load("morton")
    assert np.array_equal(O.morton_codes(fx["q"]), fx["codes"])
    lo, hi = O.support(fx["pts"])
    assert np.array_equal(lo, fx["lo"]) and np.array_equal(hi, fx["hi"])
    assert np.array_equal(O.quantize(fx["pts"], lo, hi), fx["pts_q"])
    # test_morton.py:55-66
    top = O.GRID_MAX
    q = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [top, top, top]], np.uint32)
    assert O.morton_codes(q).tolist() == [0, 1, 2, 4, 2**63 - 1]
    # test_morton.py:38-41 midpoint
    assert O.quantize(np.array([[0.5, 0, 0]]), np.zeros(3), np.array([1.0, 2, 4]))[0, 0] == 1048575


@pytest.mark.parametrize("n", TREE_SIZES)
def test_tree_bit_identical(n):
    fx = load(f"tree_{n}")
    V, T = fx["vertices"], fx["triangles"]
    codes, ids = O.sorted_keys(V, T)
    assert np.array_equal(codes, fx["sorted_codes"])
    assert np.array_equal(ids, fx["sorted_ids"])
    tree = O.build_tree(V, T, codes, ids)
    for f in TREE_FIELDS:
        assert np.array_equal(tree[f], fx[f"tree_{f}"]), f


def test_duplicate_code_scene_tree():
    """scene_dup: every triangle repeated, so runs of equal Morton codes --
    the sort's (code, id) order and the climb's id-XOR / position tie-breaks
    (_core.pyx:52-64)."""
    fx = load("scene_dup")
    V, T = fx["vertices"], fx["triangles"]
    codes, ids = O.sorted_keys(V, T)
    assert len(np.unique(codes)) < len(codes)
    assert np.array_equal(codes, fx["sorted_codes"]) and np.array_equal(ids, fx["sorted_ids"])
    tree = O.build_tree(V, T, codes, ids)
    for f in TREE_FIELDS:
        assert np.array_equal(tree[f], fx[f"tree_{f}"]), f
    args = (V, T, fx["starts"], fx["ends"])
    for mode in MODES:
        for cap in (4, 8):
            got = O.run_batch(*args, mode=mode, max_coll=cap)
            assert_result_fields(got, expected(fx, f"cap{cap}", mode), f"dup cap{cap} {mode}")


@pytest.mark.parametrize("name", SCENES)
@pytest.mark.parametrize("mode", MODES)
def test_scene_results(name, mode):
    fx = load(f"scene_{name}")
    args = (fx["vertices"], fx["triangles"], fx["starts"], fx["ends"])
    got = O.run_batch(*args, mode=mode)
    assert_result_fields(got, expected(fx, "batch", mode), f"{name} batch {mode}")
    base = O.run_baseline(*args, mode=mode)
    assert_result_fields(base, expected(fx, "base", mode), f"{name} baseline {mode}")


@pytest.mark.parametrize("name", SOUPS)
@pytest.mark.parametrize("mode", MODES)
def test_soup_results(name, mode):
    fx = load(f"soup_{name}")
    args = (fx["vertices"], fx["triangles"], fx["starts"], fx["ends"])
    assert_result_fields(O.run_batch(*args, mode=mode), expected(fx, "batch", mode), name)
    assert_result_fields(O.run_baseline(*args, mode=mode), expected(fx, "base", mode), name)
    for cap in (4, 8):
        got = O.run_batch(*args, mode=mode, max_coll=cap)
        assert_result_fields(got, expected(fx, f"cap{cap}", mode), f"{name} cap{cap}")


@pytest.mark.parametrize("name", OVERFLOWS)
def test_overflow_index(name):
    fx = load(f"soup_{name}")
    args = (fx["vertices"], fx["triangles"], fx["starts"], fx["ends"])
    for mode_i, cap, st, idx in fx["overflow"].tolist():
        try:
            O.run_batch(*args, mode=MODES[mode_i], max_coll=cap, max_stack=st, nthreads=3)
            got = -1
        except O.OracleOverflow as exc:
            got = exc.segment_index
        assert got == idx, (MODES[mode_i], cap, st)


@pytest.mark.parametrize("cap", (32, 8))
@pytest.mark.parametrize("mode", MODES)
def test_layered(cap, mode):
    fx = load("layered")
    args = (fx["vertices"], fx["triangles"], fx["starts"], fx["ends"])
    got = O.run_batch(*args, mode=mode, max_coll=cap)
    assert_result_fields(got, expected(fx, f"cap{cap}", mode), f"layered cap{cap}")


@pytest.mark.parametrize("mode", MODES)
def test_reference_arm_matches_golden(mode):
    """oracle/ref_engine.py (the reference's compiled kernel, or the C port
    when it is absent) reproduces the reference results."""
    from oracle import ref_engine

    fx = load("scene_s19")
    res, _ = ref_engine.run_batch(fx["vertices"], fx["triangles"], fx["starts"], fx["ends"],
                                  mode=mode, workers=3)
    assert_result_fields(res, expected(fx, "batch", mode), f"ref arm {mode}")


SORT_BATCHES = ("scene_c1", "scene_s19", "soup_17", "layered")


@pytest.mark.parametrize("name", SORT_BATCHES)
def test_segment_morton_order_matches_reference(name):
    """The oracle's restatement of sort_segments_by_morton (f64 midpoints,
    support, per-axis quantisation, 63-bit codes, stable sort; engine.py:
    125-147) reproduces the reference's permutation."""
    fx = load("sortperm")
    s, e = fx[f"{name}_starts"], fx[f"{name}_ends"]
    mid = (s.astype(np.float64) + e.astype(np.float64)) / 2.0
    lo, hi = O.support(mid)
    _, ids = O.sort_by_code(O.morton_codes(O.quantize(mid, lo, hi)))
    assert np.array_equal(ids.astype(np.int64), fx[f"{name}_perm"])
    assert np.array_equal(s[ids], fx[f"{name}_sorted_starts"])
