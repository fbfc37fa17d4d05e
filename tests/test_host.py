"""CPU-only checks of the host side: the C-ABI library loads and exports
what the header declares, the scene generator reproduces the reference,
config validation and the sort_rays permutation logic."""

import ctypes as C

import numpy as np
import pytest

import paper_2209_02878_b200 as rs
from paper_2209_02878_b200 import _lib
from golden_io import SCENES, load
from oracle import oracle as O


def test_library_exports_every_header_symbol():
    names = _lib.header_symbols()
    assert len(names) >= 13
    dll = C.CDLL(str(_lib.LIB_PATH))
    for n in names:
        assert hasattr(dll, n), n
    assert set(names) == set(_lib._SIGS), "ctypes signatures out of sync with the header"
    assert _lib.lib().rs_abi_version() == 1


def test_library_is_sm100a():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


@pytest.mark.parametrize("name", [s for s in SCENES if s != "dup"])  # dup: not a generate_scene output
def test_generate_scene_reproduces_reference(name):
    fx = load(f"scene_{name}")
    n_tri, n_ray, seed = fx["params"].tolist()
    sc = rs.generate_scene(n_tri, n_ray, float(fx["frac"]), seed)
    assert np.array_equal(sc.mesh.vertices, fx["vertices"])
    assert np.array_equal(sc.mesh.triangles, fx["triangles"])
    assert np.array_equal(sc.segments.starts, fx["starts"])
    assert np.array_equal(sc.segments.ends, fx["ends"])
    assert np.array_equal(sc.expected_crossings, fx["expected"])


def test_layered_scene_counts_by_construction():
    base = rs.generate_scene(300, 2000, 0.5, seed=3)
    lay = rs.layered_scene(base, layers=4)
    assert lay.mesh.num_triangles == 4 * 300
    want = O.run_batch(lay.mesh.vertices, lay.mesh.triangles, lay.segments.starts,
                       lay.segments.ends, mode="count")
    assert np.array_equal(want["counts"], lay.expected_crossings)


def test_config_validation():
    with pytest.raises(rs.ValidationError):
        rs.EngineConfig(mode="nope").validate()
    with pytest.raises(rs.ValidationError):
        rs.EngineConfig(workers=0).validate()
    with pytest.raises(rs.ValidationError):
        rs.EngineConfig(max_collisions=1).validate()  # reference compiled path would overrun
    with pytest.raises(rs.ValidationError):
        rs.EngineConfig(max_stack=0).validate()
    with pytest.raises(rs.ValidationError):
        rs.EngineConfig(backend="compiled").validate()
    with pytest.raises(rs.ValidationError):
        rs.EngineConfig(tree="bvh8").validate()
    assert rs.EngineConfig().resolved_tree() == "fast"
    assert rs.EngineConfig(max_stack=3).resolved_tree() == "reference"
    assert rs.EngineConfig(tree="reference").resolved_tree() == "reference"


def test_segment_and_mesh_validation():
    with pytest.raises(rs.ValidationError):
        rs.SegmentBatch.from_arrays(np.zeros((2, 3)), np.zeros((3, 3)))
    with pytest.raises(rs.ValidationError):
        rs.SegmentBatch.from_arrays([[0, 0, np.nan]], [[1, 1, 1]])
    with pytest.raises(rs.ValidationError):
        rs.Mesh.from_arrays(np.zeros((3, 3)), [[0, 1, 3]])
    with pytest.raises(rs.ValidationError):
        rs.Mesh.from_arrays(np.zeros((3, 3)), [[0, 1, 1]])
    with pytest.raises(rs.ValidationError):
        rs.Mesh.from_arrays([[0, 0, np.inf]] * 3, [[0, 1, 2]])


@pytest.mark.gpu
def test_sort_rays_permutation_matches_reference_rule():
    rng = np.random.default_rng(2)
    s = rng.uniform(-12, 12, size=(5000, 3)).astype(np.float32)
    e = rng.uniform(-12, 12, size=(5000, 3)).astype(np.float32)
    batch = rs.SegmentBatch.from_arrays(s, e)
    sorted_batch, perm = rs.sort_segments_by_morton(batch)
    mid = (s.astype(np.float64) + e.astype(np.float64)) / 2.0
    lo, hi = O.support(mid)
    codes = O.morton_codes(O.quantize(mid, lo, hi))
    _, want = O.sort_by_code(codes)
    assert np.array_equal(perm, want)
    restored = np.empty_like(sorted_batch.starts)
    restored[perm] = sorted_batch.starts
    assert np.array_equal(restored, s)
    again, perm2 = rs.sort_segments_by_morton(sorted_batch)  # fixed point (test_engine.py:65-71)
    assert np.array_equal(perm2, np.arange(5000))


def test_morton_encode_known_answers():
    """The checker's Morton restatement on the reference's known answers
    (test_morton.py:33-74); the engine's own keys are checked on the GPU."""
    top = (1 << 21) - 1
    q = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [top, top, top]], np.uint32)
    assert O.morton_codes(q).tolist() == [0, 1, 2, 4, 2**63 - 1]
    fx = load("morton")
    assert np.array_equal(O.morton_codes(fx["q"]), fx["codes"])
    lo, hi = O.support(fx["pts"])
    assert np.array_equal(O.quantize(fx["pts"], lo, hi), fx["pts_q"])


@pytest.mark.gpu
def test_unpermute_barycentric_rows():
    """rs_unpermute_rows / rs_unpermute_dense (sort_rays un-permutation)."""
    import torch

    from paper_2209_02878_b200.engine import ResultSet, _unpermute

    cuda = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
    perm = cuda(np.array([3, 0, 2, 1], np.int64))
    r = ResultSet("barycentric", 4, ray_index=cuda(np.array([0, 2, 3], np.int32)),
                  distance=cuda(np.array([1, 2, 3], np.float32)),
                  triangle_id=cuda(np.array([7, 8, 9], np.int32)),
                  point=cuda(np.arange(9, dtype=np.float32).reshape(3, 3)))
    r = _unpermute(r, perm)
    assert r.ray_index.tolist() == [1, 2, 3]
    assert r.triangle_id.tolist() == [9, 8, 7]
    assert r.distance.tolist() == [3, 2, 1]
    assert r.point.tolist() == [[6, 7, 8], [3, 4, 5], [0, 1, 2]]
    b = _unpermute(ResultSet("boolean", 4, crossing=cuda(np.array([1, 0, 0, 1], np.int32))), perm)
    assert b.crossing.tolist() == [0, 1, 0, 1]
    # a large random permutation against numpy
    rng = np.random.default_rng(5)
    n = 300_000
    pm = rng.permutation(n).astype(np.int64)
    rows = np.sort(rng.choice(n, 100_000, replace=False)).astype(np.int32)
    dist = rng.random(rows.size).astype(np.float32)
    tri = rng.integers(0, 1000, rows.size).astype(np.int32)
    pt = rng.random((rows.size, 3)).astype(np.float32)
    r = _unpermute(ResultSet("barycentric", n, ray_index=cuda(rows), distance=cuda(dist),
                             triangle_id=cuda(tri), point=cuda(pt)), cuda(pm))
    orig = pm[rows]
    order = np.argsort(orig, kind="stable")
    assert np.array_equal(r.ray_index.cpu().numpy(), orig[order])
    assert np.array_equal(r.distance.cpu().numpy(), dist[order])
    assert np.array_equal(r.triangle_id.cpu().numpy(), tri[order])
    assert np.array_equal(r.point.cpu().numpy(), pt[order])


def test_bench_reference_arm_line():
    """bench.py --impl reference (the driver's reference arm) runs the
    reference package's own run_batch on the host cores and prints one JSON
    line with the contract's keys (small --rays so it takes seconds)."""
    import json
    import subprocess
    import sys
    from pathlib import Path

    repo = Path(__file__).resolve().parents[1]
    r = subprocess.run([sys.executable, str(repo / "bench.py"), "--impl", "reference", "--rays", "20000",
                        "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=600,
                       cwd=str(repo))
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["same_config"] is True  # every step ran the whole (small) batch
    assert line["e2e"]["h2d_bytes_per_step"] == 0
