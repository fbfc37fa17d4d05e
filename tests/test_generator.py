"""On-device terrain segment generator (rs_generate_segments, BASELINE
configs[4]'s 1B segments): the numpy restatement (oracle/gen_oracle.py) is
checked on CPU against the C oracle's intersection results (its ground-truth
flags are real: a generated crosser crosses exactly once, a miss never) and
for shard invariance; on the GPU the kernel must reproduce the restatement
bit for bit and the engine must reproduce the flags."""

import numpy as np
import pytest

import paper_2209_02878_b200 as rs
from oracle import gen_oracle as G
from oracle import oracle as O


@pytest.fixture(scope="module")
def terrain():
    return rs.generate_scene(2000, 0, 0.5, seed=2022).mesh


def test_generator_flags_are_ground_truth(terrain):
    s, e, f = G.generate_segments(terrain.vertices, terrain.triangles, 30_000, seed=7, first=123_456)
    got = O.run_batch(terrain.vertices, terrain.triangles, s, e, mode="count")
    assert np.array_equal(got["counts"], f.astype(np.int32))
    assert abs(f.mean() - 0.5) < 0.02
    # crossers are vertical; misses' three kinds all occur
    assert np.array_equal(s[f == 1, :2], e[f == 1, :2])
    assert (s[f == 0, 0] < -1.0).any() and (s[f == 0, 2] > terrain.vertices[:, 2].max()).any()


def test_generator_shard_invariance(terrain):
    s, e, f = G.generate_segments(terrain.vertices, terrain.triangles, 1000, seed=3)
    s2, e2, f2 = G.generate_segments(terrain.vertices, terrain.triangles, 400, seed=3, first=600)
    assert np.array_equal(s[600:], s2) and np.array_equal(e[600:], e2) and np.array_equal(f[600:], f2)
    s3, _, _ = G.generate_segments(terrain.vertices, terrain.triangles, 1000, seed=4)
    assert not np.array_equal(s, s3)


def test_generator_crossing_fraction_edges(terrain):
    for frac in (0.0, 1.0):
        s, e, f = G.generate_segments(terrain.vertices, terrain.triangles, 2000, seed=1,
                                      crossing_fraction=frac)
        assert f.mean() == frac
        got = O.run_batch(terrain.vertices, terrain.triangles, s, e, mode="boolean")
        assert np.array_equal(got["crossing"], f.astype(np.int32))


@pytest.mark.gpu
@pytest.mark.parametrize("first,n", [(0, 200_000), (2**32 - 7, 50), (999_999_000, 1000), (5, 0)])
def test_device_generator_matches_restatement(terrain, first, n):
    import torch

    segs, flags = rs.scene.generate_segments_device(terrain, n, 0.5, seed=2022, first=first)
    torch.cuda.synchronize()
    s, e, f = G.generate_segments(terrain.vertices, terrain.triangles, n, seed=2022, first=first)
    assert np.array_equal(segs.starts.cpu().numpy(), s)
    assert np.array_equal(segs.ends.cpu().numpy(), e)
    assert np.array_equal(flags.cpu().numpy(), f)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["boolean", "count"])
def test_engine_on_generated_segments(mode):
    """2M-triangle terrain (BASELINE configs[4]'s mesh) x 4M generated
    segments: every flag reproduced, and a sample matches the C oracle."""
    import torch

    mesh = rs.generate_scene(2_000_000, 0, 0.5, seed=2022).mesh
    segs, flags = rs.scene.generate_segments_device(mesh, 4_000_000, 0.5, seed=2022, first=10**8)
    dmesh = rs.Mesh.from_arrays(torch.from_numpy(mesh.vertices).cuda(),
                                torch.from_numpy(mesh.triangles).cuda())
    got = rs.run_batch(dmesh, segs, rs.EngineConfig(mode=mode))
    out = (got.crossing if mode == "boolean" else got.counts).cpu().numpy()
    truth = flags.cpu().numpy().astype(np.int32)
    assert np.array_equal(out, truth)
    idx = np.random.default_rng(0).choice(out.size, 5000, replace=False)
    want = O.run_batch(mesh.vertices, mesh.triangles, segs.starts.cpu().numpy()[idx],
                       segs.ends.cpu().numpy()[idx], mode=mode)
    assert np.array_equal(out[idx], want["crossing" if mode == "boolean" else "counts"])
