"""The reference arm: the reference's own compiled CPU kernels, driven the way
the reference engine drives them.

TEST/BENCH INFRASTRUCTURE ONLY (bench.py --impl reference and the
cpu_baseline leg).  `_ref/_core*.so` is the reference's `_core.pyx` compiled
from /root/reference by oracle/Makefile (flags of setup.py:17-35); this module
restates the Python orchestration around it:
  engine.py:222-290  run_batch phases and timings
  engine.py:115-122  segment boxes
  morton.py:34-146   centroids, support, quantise, encode, lexsort
  lbvh.py:175-195    _reset_tree
  _compiled.py:27-112 threaded construct_range / batch_query
  engine.py:160-183  _run_chunked (min(4w, n/256) chunks, chunk-order errors)
When _ref is absent the C port (rs_oracle.c, OpenMP) stands in (kind "port").
"""

from __future__ import annotations

import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
MODE_TAGS = {"boolean": 0, "barycentric": 1, "count": 2}
_MIN_PER_WORKER = 256
_PAR_BUILD = 2048
_MASKS = (0x1F00000000FFFF, 0x1F0000FF0000FF, 0x100F00F00F00F00F, 0x10C30C30C30C30C3,
          0x1249249249249249)


def load_ref_core():
    """The reference's compiled kernel module, or None."""
    d = HERE / "_ref"
    if not any(d.glob("_core*.so")):
        return None
    if str(d) not in sys.path:
        sys.path.insert(0, str(d))
    import _core  # noqa: E402

    return _core


def kind() -> str:
    return "reference" if load_ref_core() is not None else "port"


def _keys(V, T):
    v = V.astype(np.float64)
    c = (v[T[:, 0]] + v[T[:, 1]] + v[T[:, 2]]) / 3.0
    lo, hi = c.min(axis=0), c.max(axis=0)
    q = np.zeros(c.shape, np.uint32)
    for k in range(3):
        ext = hi[k] - lo[k]
        if ext > 0.0:
            s = np.floor((c[:, k] - lo[k]) / ext * float((1 << 21) - 1))
            q[:, k] = np.clip(s, 0.0, float((1 << 21) - 1)).astype(np.uint32)
    codes = np.zeros(c.shape[0], np.uint64)
    for k in range(3):
        x = q[:, k].astype(np.uint64)
        for sh, m in zip((32, 16, 8, 4, 2), _MASKS):
            x = (x | x << np.uint64(sh)) & np.uint64(m)
        codes |= x << np.uint64(k)
    ids = np.arange(codes.shape[0], dtype=np.int32)
    order = np.lexsort((ids, codes))
    return codes[order], ids[order]


def _chunks(n, workers):
    workers = min(workers, max(1, n // _MIN_PER_WORKER))
    if workers <= 1:
        return 1, [(0, n)]
    chunks = min(workers * 4, max(1, n // _MIN_PER_WORKER))
    b = np.linspace(0, n, chunks + 1).astype(int)
    return workers, [(int(b[c]), int(b[c + 1])) for c in range(chunks)]


def run_batch(V, T, starts, ends, mode="boolean", workers=None, max_coll=32, max_stack=64):
    """engine.py:222-290 with the compiled backend; returns (outputs, timings)."""
    core = load_ref_core()
    workers = workers or os.cpu_count() or 1
    if core is None:
        from . import oracle as O

        t0 = time.perf_counter()
        res = O.run_batch(V, T, starts, ends, mode=mode, max_coll=max_coll, max_stack=max_stack,
                          nthreads=workers)
        return res, {"total": time.perf_counter() - t0}
    timings = {}
    t_all = time.perf_counter()
    n, nt = starts.shape[0], T.shape[0]
    t0 = time.perf_counter()
    boxes = np.empty((n, 6), np.float32)
    boxes[:, 0::2] = np.minimum(starts, ends)
    boxes[:, 1::2] = np.maximum(starts, ends)
    timings["ray boxes"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    codes, ids = _keys(V, T)
    timings["keys"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    va, vb, vc = V[T[:, 0]], V[T[:, 1]], V[T[:, 2]]
    tb = np.empty((nt, 6), np.float32)
    tb[:, 0::2] = np.minimum(np.minimum(va, vb), vc)
    tb[:, 1::2] = np.maximum(np.maximum(va, vb), vc)
    child_l = np.full(nt, -1, np.int32)
    child_r = np.full(nt, -1, np.int32)
    range_l = np.full(nt, -1, np.int32)
    range_r = np.full(nt, -1, np.int32)
    int_tri = np.full(nt, -1, np.int32)
    visit = np.zeros(nt, np.int32)
    int_bounds = np.zeros((nt, 6), np.float32)
    leaf_bounds = np.ascontiguousarray(tb[ids])
    leaf_tri = ids.copy()
    timings["reset"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    if nt == 1:
        child_l[0] = 0
    else:
        def construct(lo, hi):
            core.construct_range(codes, ids, child_l, child_r, range_l, range_r, visit, int_tri,
                                 int_bounds, leaf_bounds, nt, lo, hi)

        if workers <= 1 or nt < _PAR_BUILD:
            construct(0, nt)
        else:
            b = np.linspace(0, nt, workers + 1).astype(int)
            with ThreadPoolExecutor(max_workers=workers) as pool:
                for f in [pool.submit(construct, int(b[w]), int(b[w + 1])) for w in range(workers)]:
                    f.result()
    timings["construct"] = time.perf_counter() - t0
    out = {"detected": np.zeros(n, np.int32), "counts": np.zeros(n, np.int32),
           "tri": np.full(n, -1, np.int32), "dist": np.zeros(n, np.float32),
           "points": np.zeros((n, 3), np.float32)}
    root = int(child_l[nt - 1])
    t0 = time.perf_counter()

    def query(lo, hi):
        st, bad = core.batch_query(V, T, starts, ends, boxes, int_bounds, child_l, child_r,
                                   leaf_tri, leaf_bounds, root, nt, MODE_TAGS[mode], max_coll,
                                   max_stack, lo, hi, out["detected"], out["counts"], out["tri"],
                                   out["dist"], out["points"])
        if st == 1:
            raise OverflowError(bad)

    nw, parts = _chunks(n, workers)
    if nw <= 1:
        query(0, n)
    else:
        with ThreadPoolExecutor(max_workers=nw) as pool:
            for f in [pool.submit(query, lo, hi) for lo, hi in parts]:
                f.result()
    timings["query"] = time.perf_counter() - t0
    if mode == "boolean":
        res = {"crossing": out["detected"]}
    elif mode == "count":
        res = {"counts": out["counts"]}
    else:
        idx = np.nonzero(out["detected"])[0].astype(np.int32)
        res = {"ray_index": idx, "distance": out["dist"][idx], "triangle_id": out["tri"][idx],
               "point": out["points"][idx]}
    timings["total"] = time.perf_counter() - t_all
    return res, timings
