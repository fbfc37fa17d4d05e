"""Generate the golden fixtures in tests/golden/ by running the REFERENCE itself.

Run in the build container (the reference is mounted at /root/reference):

    python tests/golden/make_golden.py

It imports the reference package `raysurf` from /root/reference/pkg/src.  The
reference's compiled kernel (`_core.pyx`) is built by oracle/Makefile into
oracle/_ref/ and injected as `raysurf._backend._core`, so both of the
reference's own backends (pure and compiled) run; every fixture is produced by
the compiled backend and cross-checked against the pure backend where the
reference's own tests do (test_backends.py).

Nothing on the GPU box runs this script; the .npz files it writes are
committed.  Fixture contents (all arrays exactly as the reference returned
them):
  scene_*.npz   generate_scene inputs + ground truth, reference sorted keys,
                the 12 BvhTree fields, run_batch / run_baseline_allpairs
                results in all three modes
  soup_*.npz    random-soup inputs (tests/helpers.py random_mesh/segments)
                with results and max_stack overflow indices
  tree_*.npz    trees for random meshes (test_backends.py:46-84 sizes)
  sortperm.npz  sort_segments_by_morton permutations (engine.py:125-147)
  tree_dup5.npz, scene_dup.npz   equal Morton codes (test_backends.py:70-84
                and a terrain with repeated triangles): trees + results
"""

from __future__ import annotations

import subprocess
import sys
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parents[2]
REF_SRC = Path("/root/reference/pkg/src")
REF_TESTS = Path("/root/reference/pkg/tests")
OUT = Path(__file__).resolve().parent


def _import_reference():
    subprocess.run(["make", "-s", "-f", str(REPO / "oracle/Makefile"), "ref"], check=True)
    sys.path.insert(0, str(REPO / "oracle/_ref"))
    import _core  # the reference's own Cython kernels, compiled by oracle/Makefile

    sys.modules["raysurf._backend._core"] = _core
    sys.path.insert(0, str(REF_SRC))
    sys.path.insert(0, str(REF_TESTS))
    import raysurf

    assert raysurf.available_backends() == ("compiled", "pure"), raysurf.available_backends()
    return raysurf


TREE_FIELDS = (
    "internal_bounds", "internal_child_left", "internal_child_right",
    "internal_range_left", "internal_range_right", "internal_triangle_id",
    "internal_visit", "leaf_bounds", "leaf_triangle_id", "leaf_range_left",
    "leaf_range_right", "sorted_triangle_ids",
)
MODES = ("boolean", "barycentric", "count")


def _result_arrays(prefix, rs):
    d = {}
    for f in ("crossing", "counts", "ray_index", "distance", "triangle_id", "point"):
        v = getattr(rs, f)
        if v is not None:
            d[f"{prefix}_{f}"] = v
    return d


def _tree_arrays(rs_mod, mesh, prefix="tree"):
    from raysurf import morton
    from raysurf._backend import get_backend

    c = morton.triangle_centroids(mesh.vertices, mesh.triangles)
    sup = morton.centroid_support(c)
    codes = morton.morton_encode_points(morton.quantize_points(c, sup))
    sc, si = morton.sort_by_morton(codes)
    tree, _, _ = get_backend("compiled").build_tree(mesh, sc, si)
    pure, _, _ = get_backend("pure").build_tree(mesh, sc, si)
    for f in TREE_FIELDS:
        assert np.array_equal(getattr(tree, f), getattr(pure, f)), f
    d = {f"{prefix}_{f}": getattr(tree, f) for f in TREE_FIELDS}
    d["codes_unsorted"] = codes
    d["sorted_codes"] = sc
    d["sorted_ids"] = si
    d["support_lo"] = np.array(sup.min)
    d["support_hi"] = np.array(sup.max)
    return d


def scene_case(rs, name, n_tri, n_ray, frac, seed, modes=MODES, baseline=True):
    from raysurf import EngineConfig, run_baseline_allpairs, run_batch
    from raysurf.oracle import generate_scene

    sc = generate_scene(n_tri, n_ray, frac, seed=seed)
    d = {
        "vertices": sc.mesh.vertices, "triangles": sc.mesh.triangles,
        "starts": sc.segments.starts, "ends": sc.segments.ends,
        "expected": sc.expected_crossings,
        "params": np.array([n_tri, n_ray, seed]), "frac": np.array(frac),
    }
    d.update(_tree_arrays(rs, sc.mesh))
    for m in modes:
        d.update(_result_arrays(f"batch_{m}", run_batch(sc.mesh, sc.segments, EngineConfig(mode=m))))
        if baseline:
            d.update(_result_arrays(
                f"base_{m}", run_baseline_allpairs(sc.mesh, sc.segments, EngineConfig(mode=m))))
    np.savez_compressed(OUT / f"scene_{name}.npz", **d)
    print("wrote", name, {k: v.shape for k, v in d.items() if k.startswith("batch_boolean")})


def soup_case(rs, name, seed, n_tri, n_seg, span=12.0, overflow_stack=None):
    from helpers import random_mesh, random_segments
    from raysurf import EngineConfig, run_baseline_allpairs, run_batch
    from raysurf.exceptions import TraversalStackOverflow

    rng = np.random.default_rng(seed)
    mesh = random_mesh(rng, n_tri)
    if span > 0:
        batch = random_segments(rng, n_seg, span=span)
    else:  # short segments: overflow only on some, so the index is informative
        from raysurf import SegmentBatch

        st = rng.uniform(-10.0, 10.0, size=(n_seg, 3)).astype(np.float32)
        en = (st + rng.normal(scale=-span, size=(n_seg, 3))).astype(np.float32)
        batch = SegmentBatch.from_arrays(st, en)
    d = {"vertices": mesh.vertices, "triangles": mesh.triangles,
         "starts": batch.starts, "ends": batch.ends}
    d.update(_tree_arrays(rs, mesh))
    if overflow_stack is None:
        for m in MODES:
            d.update(_result_arrays(f"batch_{m}", run_batch(mesh, batch, EngineConfig(mode=m))))
            d.update(_result_arrays(f"base_{m}", run_baseline_allpairs(mesh, batch, EngineConfig(mode=m))))
            for cap in (4, 8):
                rs_cap = run_batch(mesh, batch, EngineConfig(mode=m, max_collisions=cap))
                d.update(_result_arrays(f"cap{cap}_{m}", rs_cap))
    else:
        # overflow index for every (mode, max_collisions, max_stack) combination
        rows = []
        for m in MODES:
            for cap in (2, 4, 32):
                for st in overflow_stack:
                    idx = -1
                    try:
                        run_batch(mesh, batch, EngineConfig(
                            mode=m, max_collisions=cap, max_stack=st, workers=1, backend="compiled"))
                    except TraversalStackOverflow as exc:
                        idx = exc.segment_index
                    try:
                        run_batch(mesh, batch, EngineConfig(
                            mode=m, max_collisions=cap, max_stack=st, workers=1, backend="pure"))
                        idx_p = -1
                    except TraversalStackOverflow as exc:
                        idx_p = exc.segment_index
                    assert idx == idx_p, (m, cap, st, idx, idx_p)
                    rows.append((MODES.index(m), cap, st, idx))
        d["overflow"] = np.array(rows, np.int64)
    np.savez_compressed(OUT / f"soup_{name}.npz", **d)
    print("wrote soup", name)


def tree_case(rs, n_tri, seed):
    from helpers import random_mesh

    mesh = random_mesh(np.random.default_rng(seed), n_tri)
    d = {"vertices": mesh.vertices, "triangles": mesh.triangles}
    d.update(_tree_arrays(rs, mesh))
    np.savez_compressed(OUT / f"tree_{n_tri}.npz", **d)


def dup_cases(rs):
    """Equal Morton codes: the all-duplicate mesh of test_backends.py:70-84
    (one tree) and a terrain whose triangles are each repeated (every code
    appears 2-3 times): trees (the Apetrei climb's id-XOR / position
    tie-breaks, _core.pyx:52-64, and the sort's stability, morton.py:131-146)
    and results in every mode."""
    from raysurf import EngineConfig, Mesh, SegmentBatch, run_baseline_allpairs, run_batch
    from raysurf.oracle import generate_scene

    rng = np.random.default_rng(56)
    verts = rng.uniform(-1, 1, size=(6, 3)).astype(np.float32)
    tris = np.array([[0, 1, 2], [1, 2, 3], [2, 3, 4], [0, 2, 4], [1, 3, 5]], dtype=np.int32)
    mesh = Mesh.from_arrays(np.tile(verts[:1], (6, 1)) * 0 + verts[:1], tris)
    d = {"vertices": mesh.vertices, "triangles": mesh.triangles}
    d.update(_tree_arrays(rs, mesh))
    assert len(set(d["sorted_codes"].tolist())) == 1
    np.savez_compressed(OUT / "tree_dup5.npz", **d)

    sc = generate_scene(1500, 8000, 0.5, seed=2023)
    T = sc.mesh.triangles
    pick = np.random.default_rng(3).permutation(T.shape[0])
    # every triangle twice, a third of them three times; shuffled ids
    T2 = np.concatenate([T, T[pick], T[pick[: T.shape[0] // 3]]])
    T2 = T2[np.random.default_rng(4).permutation(T2.shape[0])]
    mesh = Mesh.from_arrays(sc.mesh.vertices, T2)
    batch = SegmentBatch.from_arrays(sc.segments.starts, sc.segments.ends)
    d = {"vertices": mesh.vertices, "triangles": mesh.triangles, "starts": batch.starts,
         "ends": batch.ends, "expected": sc.expected_crossings}
    d.update(_tree_arrays(rs, mesh))
    assert len(np.unique(d["sorted_codes"])) < mesh.num_triangles
    for m in MODES:
        d.update(_result_arrays(f"batch_{m}", run_batch(mesh, batch, EngineConfig(mode=m))))
        d.update(_result_arrays(f"base_{m}", run_baseline_allpairs(mesh, batch, EngineConfig(mode=m))))
        for cap in (4, 8):
            d.update(_result_arrays(f"cap{cap}_{m}", run_batch(mesh, batch, EngineConfig(mode=m, max_collisions=cap))))
    np.savez_compressed(OUT / "scene_dup.npz", **d)
    print("wrote dup cases")


def layered_case(rs):
    """Small C4 analogue: 3 z-offset copies of a scene, stretched crossers, count mode."""
    from raysurf import EngineConfig, Mesh, SegmentBatch, run_batch
    from raysurf.oracle import generate_scene

    sc = generate_scene(500, 3000, 0.5, seed=2022)
    layers, dz = 3, 8.0
    V = np.concatenate([sc.mesh.vertices + np.float32([0, 0, dz * k]) for k in range(layers)])
    T = np.concatenate([sc.mesh.triangles + k * sc.mesh.num_vertices for k in range(layers)])
    s = sc.segments.starts.copy()
    e = sc.segments.ends.copy()
    cross = sc.expected_crossings.astype(bool)
    zlo = float(sc.mesh.vertices[:, 2].min()) - 3.0
    zhi = float(sc.mesh.vertices[:, 2].max()) + dz * (layers - 1) + 3.0
    up = e[:, 2] > s[:, 2]
    s[cross, 2] = np.where(up[cross], zlo, zhi)
    e[cross, 2] = np.where(up[cross], zhi, zlo)
    mesh = Mesh.from_arrays(V, T)
    batch = SegmentBatch.from_arrays(s, e)
    d = {"vertices": mesh.vertices, "triangles": mesh.triangles, "starts": batch.starts,
         "ends": batch.ends}
    for cap in (32, 8):
        for m in MODES:
            d.update(_result_arrays(f"cap{cap}_{m}", run_batch(mesh, batch, EngineConfig(mode=m, max_collisions=cap))))
    assert set(np.unique(d["cap32_count_counts"]).tolist()) <= {0, layers}
    np.savez_compressed(OUT / "layered.npz", **d)
    print("wrote layered")


def sortperm_case(rs):
    """engine.sort_segments_by_morton (engine.py:125-147) on three batches:
    the permutation and the permuted endpoints."""
    from raysurf.engine import sort_segments_by_morton

    d = {}
    for name in ("scene_c1", "scene_s19", "soup_17", "layered"):
        with np.load(OUT / f"{name}.npz") as z:
            batch = rs.SegmentBatch.from_arrays(z["starts"], z["ends"])
        sb, perm = sort_segments_by_morton(batch)
        d[f"{name}_starts"] = batch.starts
        d[f"{name}_ends"] = batch.ends
        d[f"{name}_perm"] = perm
        d[f"{name}_sorted_starts"] = sb.starts
        d[f"{name}_sorted_ends"] = sb.ends
    np.savez_compressed(OUT / "sortperm.npz", **d)
    print("wrote sortperm")


def main():
    rs = _import_reference()
    if sys.argv[1:] == ["sortperm"]:
        sortperm_case(rs)
        return
    if sys.argv[1:] == ["dup"]:
        dup_cases(rs)
        return
    from raysurf import morton

    # morton known answers straight from the reference (test_morton.py:33-74)
    q = np.random.default_rng(11).integers(0, morton.GRID_MAX + 1, size=(4096, 3)).astype(np.uint32)
    pts = np.random.default_rng(12).normal(size=(2048, 3)) * np.array([100.0, 3.0, 0.01])
    sup = morton.centroid_support(pts)
    np.savez_compressed(
        OUT / "morton.npz", q=q, codes=morton.morton_encode_points(q), pts=pts,
        pts_q=morton.quantize_points(pts, sup), lo=np.array(sup.min), hi=np.array(sup.max))

    scene_case(rs, "c1", 2000, 10_000, 0.5, 2022)              # BASELINE configs[0]
    scene_case(rs, "s19", 300, 2500, 0.5, 19)                  # test_backends.py:87-94
    scene_case(rs, "s77", 250, 2000, 0.25, 77)                 # test_engine.py:206-211
    scene_case(rs, "full", 100, 500, 1.0, 1001)                # acceptance fraction 1.0
    scene_case(rs, "none", 20, 100, 0.0, 1000)                 # acceptance fraction 0.0
    soup_case(rs, "17", 17, 150, 600)                          # test_engine.py:130-140
    soup_case(rs, "20", 20, 120, 500)                          # test_backends.py:96-104
    soup_case(rs, "ovf21", 21, 256, 6, span=15.0, overflow_stack=(3, 4, 6))   # test_backends.py:108-119
    soup_case(rs, "ovf31", 31, 256, 8, span=15.0, overflow_stack=(3, 5))      # test_engine.py:188-195
    soup_case(rs, "ovfshort", 41, 400, 300, span=-2.5, overflow_stack=(4, 5, 6, 7, 8))
    for n in (1, 2, 3, 7, 8, 100, 5000):                        # test_backends.py:46-56
        tree_case(rs, n, n)
    layered_case(rs)
    sortperm_case(rs)
    dup_cases(rs)


if __name__ == "__main__":
    main()
