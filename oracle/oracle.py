"""ctypes front-end of the C restatement in rs_oracle.c.

TEST INFRASTRUCTURE ONLY -- imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline leg as the parity checker.  The product package never
imports this module.

The orchestration below restates the reference's engine.run_batch
(engine.py:222-290) and _assemble (engine.py:183-215) around the C kernels.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "liboracle.so"

MODE_TAGS = {"boolean": 0, "barycentric": 1, "count": 2}  # _compiled.py:17-21
MODES = ("boolean", "barycentric", "count")               # lbvh.py:33-36
GRID_MAX = (1 << 21) - 1                                   # morton.py:15-16
TREE_FIELDS = (                                            # test_backends.py:17-30
    "internal_bounds", "internal_child_left", "internal_child_right",
    "internal_range_left", "internal_range_right", "internal_triangle_id",
    "internal_visit", "leaf_bounds", "leaf_triangle_id", "leaf_range_left",
    "leaf_range_right", "sorted_triangle_ids",
)


class _RoTree(C.Structure):
    _fields_ = [("int_bounds", C.c_void_p)] + [
        (n, C.c_void_p)
        for n in ("child_l", "child_r", "range_l", "range_r", "int_tri", "visit",
                  "leaf_bounds", "leaf_tri", "leaf_range_l", "leaf_range_r", "sorted_ids")
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            subprocess.run(["make", "-s", "-f", str(HERE / "Makefile"), str(LIB_PATH)], check=True)
        _lib = C.CDLL(str(LIB_PATH))
        _lib.ro_query.restype = C.c_int
        _lib.ro_mt_hit.restype = C.c_int
    return _lib


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return C.c_void_p(a.ctypes.data)


def _i64(v):
    return C.c_int64(int(v))


# ------------------------------------------------------------------ morton --

def tri_boxes(V, T):
    """mesh.py:69-79."""
    out = np.empty((T.shape[0], 6), np.float32)
    lib().ro_tri_boxes(_p(V), _p(T), _i64(T.shape[0]), _p(out))
    return out


def centroids(V, T):
    """morton.py:34-37."""
    out = np.empty((T.shape[0], 3), np.float64)
    lib().ro_centroids(_p(V), _p(T), _i64(T.shape[0]), _p(out))
    return out


def support(points):
    """morton.py:40-45."""
    points = np.ascontiguousarray(points, np.float64)
    lo = np.empty(3, np.float64)
    hi = np.empty(3, np.float64)
    lib().ro_support(_p(points), _i64(points.shape[0]), _p(lo), _p(hi))
    return lo, hi


def quantize(points, lo, hi, iso_bits: int | None = None):
    """morton.py:48-63 (iso_bits=None) or the fast tree's isotropic grid."""
    points = np.ascontiguousarray(points, np.float64)
    q = np.empty(points.shape, np.uint32)
    lo = np.ascontiguousarray(lo, np.float64)
    hi = np.ascontiguousarray(hi, np.float64)
    if iso_bits is None:
        lib().ro_quantize(_p(points), _i64(points.shape[0]), _p(lo), _p(hi), _p(q))
    else:
        lib().ro_quantize_iso(_p(points), _i64(points.shape[0]), _p(lo), _p(hi),
                              C.c_int(iso_bits), _p(q))
    return q


def morton_codes(q):
    """morton.py:117-128."""
    q = np.ascontiguousarray(q, np.uint32)
    out = np.empty(q.shape[0], np.uint64)
    lib().ro_morton_codes(_p(q), _i64(q.shape[0]), _p(out))
    return out


def sort_by_code(codes, ids=None):
    """morton.py:131-146 (ascending by (code, id))."""
    codes = np.array(codes, np.uint64, copy=True)
    ids = np.arange(codes.shape[0], dtype=np.int32) if ids is None else np.array(ids, np.int32)
    lib().ro_sort(_p(codes), _p(ids), _i64(codes.shape[0]))
    return codes, ids


def sorted_keys(V, T, kind: str = "reference", iso_bits: int = 10):
    """engine.py:250-262 (kind='reference'); kind='fast' swaps in the isotropic grid."""
    c = centroids(V, T)
    lo, hi = support(c)
    q = quantize(c, lo, hi, None if kind == "reference" else iso_bits)
    return sort_by_code(morton_codes(q))


# -------------------------------------------------------------------- tree --

def build_tree(V, T, codes, ids) -> dict:
    """lbvh._reset_tree + climb (lbvh.py:148-233) -> the 12 BvhTree fields."""
    n = T.shape[0]
    tr = {
        "internal_bounds": np.empty((n, 6), np.float32),
        "leaf_bounds": np.empty((n, 6), np.float32),
    }
    for f in TREE_FIELDS:
        if f not in tr:
            tr[f] = np.empty(n, np.int32)
    s = _RoTree(*[C.c_void_p(tr[f].ctypes.data) for f in (
        "internal_bounds", "internal_child_left", "internal_child_right",
        "internal_range_left", "internal_range_right", "internal_triangle_id",
        "internal_visit", "leaf_bounds", "leaf_triangle_id", "leaf_range_left",
        "leaf_range_right", "sorted_triangle_ids")])
    codes = np.ascontiguousarray(codes, np.uint64)
    ids = np.ascontiguousarray(ids, np.int32)
    boxes = tri_boxes(V, T)
    lib().ro_build(_i64(n), _p(codes), _p(ids), _p(boxes), C.byref(s))
    tr["_struct"] = s
    tr["root"] = int(tr["internal_child_left"][n - 1])
    return tr


def empty_outputs(n):
    """engine.py:150-157."""
    return {
        "detected": np.zeros(n, np.int32),
        "counts": np.zeros(n, np.int32),
        "tri": np.full(n, -1, np.int32),
        "dist": np.zeros(n, np.float32),
        "points": np.zeros((n, 3), np.float32),
    }


class OracleOverflow(Exception):
    def __init__(self, segment_index):
        super().__init__(f"traversal stack overflow at segment {segment_index}")
        self.segment_index = segment_index


def query(V, T, starts, ends, tree, mode, max_coll=32, max_stack=64, nthreads=0,
          out=None, stats=None):
    """_core.pyx:195-352 over all segments; raises OracleOverflow(min index)."""
    n = starts.shape[0]
    out = empty_outputs(n) if out is None else out
    bad = C.c_int64(-1)
    st = np.zeros(2, np.int64)
    status = lib().ro_query(
        _p(V), _p(T), _p(starts), _p(ends), C.byref(tree["_struct"]), C.c_int32(tree["root"]),
        _i64(T.shape[0]), C.c_int(MODE_TAGS[mode]), C.c_int(max_coll), C.c_int(max_stack),
        _i64(0), _i64(n), _p(out["detected"]), _p(out["counts"]), _p(out["tri"]),
        _p(out["dist"]), _p(out["points"]), C.byref(bad), C.c_int(nthreads), _p(st))
    if stats is not None:
        stats["internal_visits"] = int(st[0])
        stats["mt_tests"] = int(st[1])
    if status == 1:
        raise OracleOverflow(int(bad.value))
    return out


def baseline(V, T, starts, ends, mode, nthreads=0):
    """_core.pyx:355-433 over all segments."""
    n = starts.shape[0]
    out = empty_outputs(n)
    boxes = tri_boxes(V, T)
    lib().ro_baseline(_p(V), _p(T), _i64(T.shape[0]), _p(boxes), _p(starts), _p(ends),
                      C.c_int(MODE_TAGS[mode]), _i64(0), _i64(n), _p(out["detected"]),
                      _p(out["counts"]), _p(out["tri"]), _p(out["dist"]), _p(out["points"]),
                      C.c_int(nthreads))
    return out


def assemble(mode, out) -> dict:
    """engine.py:183-215 without the permutation (results as plain arrays)."""
    if mode == "boolean":
        return {"mode": mode, "crossing": out["detected"]}
    if mode == "count":
        return {"mode": mode, "counts": out["counts"]}
    idx = np.nonzero(out["detected"])[0].astype(np.int32)
    return {"mode": mode, "ray_index": idx, "distance": out["dist"][idx],
            "triangle_id": out["tri"][idx], "point": out["points"][idx]}


def _canon(V, T, starts, ends):
    return (np.ascontiguousarray(V, np.float32).reshape(-1, 3),
            np.ascontiguousarray(T, np.int32).reshape(-1, 3),
            np.ascontiguousarray(starts, np.float32).reshape(-1, 3),
            np.ascontiguousarray(ends, np.float32).reshape(-1, 3))


def run_batch(V, T, starts, ends, mode="boolean", max_coll=32, max_stack=64,
              tree_kind="reference", nthreads=0, stats=None) -> dict:
    """engine.py:222-290: keys -> tree -> query -> assemble."""
    V, T, starts, ends = _canon(V, T, starts, ends)
    if starts.shape[0] == 0 or T.shape[0] == 0:
        return assemble(mode, empty_outputs(starts.shape[0]))
    codes, ids = sorted_keys(V, T, tree_kind)
    tree = build_tree(V, T, codes, ids)
    out = query(V, T, starts, ends, tree, mode, max_coll, max_stack, nthreads, stats=stats)
    return assemble(mode, out)


def run_baseline(V, T, starts, ends, mode="boolean", nthreads=0) -> dict:
    """engine.py:293-335."""
    V, T, starts, ends = _canon(V, T, starts, ends)
    if starts.shape[0] == 0 or T.shape[0] == 0:
        return assemble(mode, empty_outputs(starts.shape[0]))
    return assemble(mode, baseline(V, T, starts, ends, mode, nthreads))


def threads() -> int:
    return int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
