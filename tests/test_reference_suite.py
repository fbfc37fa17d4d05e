"""The reference's own test suite against the B200 backend, through the
reference's plugin registry exactly as INTEGRATION.md section 1 shows.

oracle/Makefile copies /root/reference/pkg (src + tests) into
oracle/_ref/refpkg (a git-ignored build output that travels to the GPU box)
and appends the three-line `_BACKENDS["b200"] = b200` registration to its
_backend/__init__.py.  Then, on the GPU:

- test_backends.py runs with the registry's "compiled" entry pointing at the
  b200 module, so the reference's pure-vs-compiled bitwise suite (all 12
  tree fields at N_t 1..5000, parallel-build determinism, the all-duplicate-
  code mesh, scene and soup results, baseline, the overflow segment index)
  becomes pure-vs-b200 (test_backends.py:46-119);
- test_engine.py, test_acceptance.py (every criterion but the three timing
  ones, test_acceptance.py:289-401) and test_io_cli.py run with
  RAYSURF_BACKEND=b200: the reference engine drives the plugin, its thread
  pool calling b200.batch_query concurrently on disjoint ranges
  (engine.py:160-180);
- in-process: the structural suite (test_acceptance.py:113-127) on trees
  the GPU built and downloaded, the 50-scene equivalence set
  (test_acceptance.py:52-85) through this engine's own fast path against
  the reference's compiled engine run right here, and concurrent callers.
"""

from __future__ import annotations

import os
import subprocess
import sys
import threading
from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

REPO = Path(__file__).resolve().parents[1]
REFPKG = REPO / "oracle" / "_ref" / "refpkg"
TIMING = "not performance_lbvh_vs_baseline and not performance_multiworker and not sorted_segment_variant"


def _env(**extra):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(REFPKG / "src"), str(REPO), str(REPO / "tests")])
    env.update(extra)
    return env


def _pytest(files, k=None, **env):
    assert (REFPKG / "src" / "raysurf").is_dir(), "oracle/_ref/refpkg missing: run make -f oracle/Makefile"
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", "-p", "refsuite_alias"]
    cmd += [str(REFPKG / "tests" / f) for f in files]
    if k:
        cmd += ["-k", k]
    r = subprocess.run(cmd, cwd=str(REFPKG / "tests"), env=_env(**env), capture_output=True, text=True,
                       timeout=1800)
    tail = (r.stdout + r.stderr)[-3000:]
    assert r.returncode == 0, tail
    assert " passed" in tail and " skipped" not in tail.split("\n")[-2], tail
    return tail


def test_reference_backend_suite_pure_vs_b200():
    """test_backends.py with "compiled" := b200 (tests/refsuite_alias.py)."""
    tail = _pytest(["test_backends.py"], RS_REFSUITE_ALIAS="compiled")
    assert "18 passed" in tail, tail


def test_reference_engine_suites_on_b200():
    tail = _pytest(["test_engine.py", "test_acceptance.py", "test_io_cli.py"], k=TIMING,
                   RAYSURF_BACKEND="b200")
    assert "passed" in tail


# ------------------------------------------------------------- in-process --

@pytest.fixture(scope="module")
def ref():
    """The vendored reference package (its compiled backend is the CPU
    reference; b200 is registered beside it)."""
    sys.path.insert(0, str(REFPKG / "src"))
    sys.path.insert(0, str(REFPKG / "tests"))
    import raysurf

    assert set(raysurf.available_backends()) >= {"b200", "compiled", "pure"}, raysurf.available_backends()
    return raysurf


def test_structural_suite_on_gpu_trees(ref):
    """test_acceptance.py:113-127's 1000 random meshes, built on the GPU:
    the plugin's tree (from the reference's sorted keys) equals the
    reference's compiled tree in all 12 fields and passes the reference's
    validate_structure; the device-keyed reference and fast trees pass
    validate_structure too."""
    from helpers import random_mesh
    from raysurf import morton
    from raysurf._backend import get_backend
    from raysurf.lbvh import validate_structure

    import paper_2209_02878_b200 as rs
    from paper_2209_02878_b200._backend import b200
    from golden_io import TREE_FIELDS

    plan = [(1, 200), (2, 200), (3, 200), (7, 150), (8, 150), (100, 80), (5000, 20)]
    comp = get_backend("compiled")
    for n_tri, repeats in plan:
        for r in range(repeats):
            mesh = random_mesh(np.random.default_rng(7_000_000 + 1000 * n_tri + r), n_tri)
            c = morton.triangle_centroids(mesh.vertices, mesh.triangles)
            codes = morton.morton_encode_points(morton.quantize_points(c, morton.centroid_support(c)))
            sc, si = morton.sort_by_morton(codes)
            want, _, _ = comp.build_tree(mesh, sc, si)
            got, _, _ = b200.build_tree(mesh, sc, si)
            for f in TREE_FIELDS:
                assert np.array_equal(getattr(got, f), getattr(want, f)), (n_tri, r, f)
            validate_structure(got)
            if r % 10 == 0:
                m = rs.Mesh.from_arrays(mesh.vertices, mesh.triangles)
                for kind in ("reference", "fast"):
                    validate_structure(b200.DeviceTree(m, kind=kind).download())


def test_fifty_scene_equivalence_fast_path(ref):
    """test_acceptance.py:52-85's 50 seeded scenes through this engine's own
    run_batch (device keys, fast tree, tile traversal), host and device
    inputs: bitwise equal to the reference's compiled run_batch computed
    here, and to the reference's independent oracle (floats to 1e-4, as
    the reference test)."""
    from helpers import assert_results_equal
    from raysurf import EngineConfig as RefConfig
    from raysurf import run_batch as ref_run_batch
    from raysurf.oracle import generate_scene, oracle_intersect_all_modes

    import paper_2209_02878_b200 as rs

    sizes = [(20, 100), (100, 500), (500, 2000), (1000, 5000), (2000, 10000)]
    fractions = [0.0, 0.25, 0.5, 1.0]
    for i in range(50):
        n_tri, n_ray = sizes[i % len(sizes)]
        scene = generate_scene(n_tri, n_ray, fractions[i % len(fractions)], seed=1000 + i)
        oracle = oracle_intersect_all_modes(scene.mesh, scene.segments)
        mesh = rs.Mesh.from_arrays(scene.mesh.vertices, scene.mesh.triangles)
        segs = rs.SegmentBatch.from_arrays(scene.segments.starts, scene.segments.ends)
        dm = rs.Mesh.from_arrays(torch.from_numpy(scene.mesh.vertices).cuda(),
                                 torch.from_numpy(scene.mesh.triangles).cuda())
        ds = rs.SegmentBatch.from_arrays(torch.from_numpy(scene.segments.starts).cuda(),
                                         torch.from_numpy(scene.segments.ends).cuda())
        for mode in ("boolean", "barycentric", "count"):
            want = ref_run_batch(scene.mesh, scene.segments, RefConfig(mode=mode, backend="compiled"))
            for got in (rs.run_batch(mesh, segs, rs.EngineConfig(mode=mode)),
                        rs.run_batch(dm, ds, rs.EngineConfig(mode=mode))):
                got = _as_ref(ref, got)
                assert_results_equal(got, want, context=f"scene {i} {mode}")
                assert_results_equal(got, oracle[mode], float_tol=1e-4, context=f"scene {i} {mode} oracle")


def _as_ref(ref, r):
    """This engine's ResultSet as the reference's (numpy fields)."""
    from raysurf.engine import ResultSet

    f = {k: (v.cpu().numpy() if hasattr(v, "cpu") else v) for k, v in
         ((k, getattr(r, k)) for k in ("crossing", "counts", "ray_index", "distance", "triangle_id", "point"))}
    return ResultSet(mode=r.mode, num_rays=r.num_rays, **f)


def test_concurrent_callers(ref):
    """SURVEY 8(b) threading: run_batch on device tensors from 4 threads at
    once (each capturing and replaying its own graph) and 4 threads sharing
    one plugin tree through batch_query on disjoint ranges; every result
    equals the single-threaded one."""
    from raysurf._backend import get_backend

    import paper_2209_02878_b200 as rs
    from paper_2209_02878_b200._backend import b200

    scenes = [rs.generate_scene(400 + 300 * k, 40_000 + 7_000 * k, 0.5, seed=90 + k) for k in range(4)]
    errors = []

    def device_worker(sc):
        try:
            dm = rs.Mesh.from_arrays(torch.from_numpy(sc.mesh.vertices).cuda(),
                                     torch.from_numpy(sc.mesh.triangles).cuda())
            ds = rs.SegmentBatch.from_arrays(torch.from_numpy(sc.segments.starts).cuda(),
                                             torch.from_numpy(sc.segments.ends).cuda())
            truth = sc.expected_crossings.astype(np.int32)
            with torch.cuda.stream(torch.cuda.Stream()):
                for _ in range(5):
                    for mode in ("boolean", "count", "barycentric"):
                        r = rs.run_batch(dm, ds, rs.EngineConfig(mode=mode))
                        got = r.crossing if mode == "boolean" else r.counts if mode == "count" else r.ray_index
                        want = truth if mode != "barycentric" else np.nonzero(truth)[0]
                        assert np.array_equal(got.cpu().numpy(), want), mode
        except Exception as exc:  # pragma: no cover - reported below
            errors.append(repr(exc))

    threads = [threading.Thread(target=device_worker, args=(sc,)) for sc in scenes]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors

    # one tree, four threads, disjoint ranges of one output dict
    from raysurf import morton
    from raysurf.engine import _empty_outputs

    sc = scenes[3]
    c = morton.triangle_centroids(sc.mesh.vertices, sc.mesh.triangles)
    codes = morton.morton_encode_points(morton.quantize_points(c, morton.centroid_support(c)))
    scodes, sids = morton.sort_by_morton(codes)
    mesh = rs.Mesh.from_arrays(sc.mesh.vertices, sc.mesh.triangles)
    segs = rs.SegmentBatch.from_arrays(sc.segments.starts, sc.segments.ends)
    tree, _, _ = b200.build_tree(mesh, scodes, sids)
    n = segs.count
    for mode in ("boolean", "count", "barycentric"):
        out = _empty_outputs(n)
        want = _empty_outputs(n)
        bounds = np.linspace(0, n, 9).astype(int)
        jobs = [threading.Thread(target=b200.batch_query,
                                 args=(mesh, tree, segs, None, mode, 32, 64, int(lo), int(hi), out))
                for lo, hi in zip(bounds[:-1], bounds[1:])]
        for j in jobs:
            j.start()
        for j in jobs:
            j.join()
        ref_tree = get_backend("compiled").build_tree(sc.mesh, scodes, sids)[0]
        from raysurf.engine import compute_segment_boxes

        get_backend("compiled").batch_query(sc.mesh, ref_tree, sc.segments, compute_segment_boxes(sc.segments),
                                            mode, 32, 64, 0, n, want)
        for k in want:
            assert np.array_equal(out[k], want[k]), (mode, k)
