"""inside_closed_surface: odd parity on count mode.

Cube and icosphere (convex, watertight) against a convex-containment
oracle: inside iff on the inner side of every face plane.  Points closer
than 1e-3 to the surface are excluded (the parity answer there hinges on
f32 rounding of the points themselves, not on the engine).  On CPU the
per-segment counts come from the C oracle (the parity logic and the target
construction); the GPU tests run the engine's count mode."""

import numpy as np
import pytest

import paper_2209_02878_b200 as rs
from oracle import oracle as O


def cube():
    v = np.array([[x, y, z] for x in (-0.5, 0.5) for y in (-0.5, 0.5) for z in (-0.5, 0.5)], np.float32)
    quads = [(0, 1, 3, 2), (4, 6, 7, 5), (0, 4, 5, 1), (2, 3, 7, 6), (0, 2, 6, 4), (1, 5, 7, 3)]
    t = []
    for a, b, c, d in quads:
        t += [(a, b, c), (a, c, d)]
    return rs.Mesh.from_arrays(v, np.array(t, np.int32))


def icosphere(subdiv=2):
    p = (1 + 5 ** 0.5) / 2
    v = [(-1, p, 0), (1, p, 0), (-1, -p, 0), (1, -p, 0), (0, -1, p), (0, 1, p), (0, -1, -p), (0, 1, -p),
         (p, 0, -1), (p, 0, 1), (-p, 0, -1), (-p, 0, 1)]
    v = [np.array(x, float) / np.linalg.norm(x) for x in v]
    f = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11), (1, 5, 9), (5, 11, 4), (11, 10, 2),
         (10, 7, 6), (7, 1, 8), (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9), (4, 9, 5),
         (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    for _ in range(subdiv):
        cache, nf = {}, []

        def mid(a, b):
            k = (min(a, b), max(a, b))
            if k not in cache:
                m = v[a] + v[b]
                v.append(m / np.linalg.norm(m))
                cache[k] = len(v) - 1
            return cache[k]

        for a, b, c in f:
            ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
            nf += [(a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca)]
        f = nf
    return rs.Mesh.from_arrays(np.array(v, np.float32), np.array(f, np.int32))


def containment(mesh, pts):
    """(inside, distance to the nearest face plane) for a convex mesh."""
    V = mesh.vertices.astype(np.float64)
    T = mesh.triangles
    a, b, c = V[T[:, 0]], V[T[:, 1]], V[T[:, 2]]
    n = np.cross(b - a, c - a)
    n /= np.linalg.norm(n, axis=1, keepdims=True)
    cen = V.mean(axis=0)
    flip = np.einsum("ij,ij->i", n, a - cen) < 0
    n[flip] *= -1
    d = (pts.astype(np.float64)[:, None, :] - a[None]) @ np.eye(3)
    s = np.einsum("kfj,fj->kf", d, n)  # signed distance per face (outward +)
    return (s < 0).all(axis=1), np.abs(s).min(axis=1)


def oracle_run(mesh, segs, cfg):
    d = O.run_batch(mesh.vertices, mesh.triangles, segs.starts, segs.ends, mode=cfg.mode)
    return rs.ResultSet(cfg.mode, segs.count, counts=d["counts"])


def sample_points(mesh, n, seed):
    rng = np.random.default_rng(seed)
    lo, hi = mesh.vertices.min(axis=0), mesh.vertices.max(axis=0)
    pts = (lo - 0.3 + rng.random((n, 3)) * (hi - lo + 0.6)).astype(np.float32)
    inside, dist = containment(mesh, pts)
    keep = dist > 1e-3
    return pts[keep], inside[keep]


@pytest.mark.parametrize("make", [cube, icosphere], ids=["cube", "icosphere"])
def test_parity_matches_convex_containment_oracle(make):
    mesh = make()
    pts, want = sample_points(mesh, 1000, 7)
    got = rs.inside_closed_surface(pts, mesh, run=oracle_run)
    assert np.array_equal(got, want)
    assert want.any() and (~want).any()


def test_parity_trivial_cases():
    mesh = cube()
    got = rs.inside_closed_surface(np.array([[0, 0, 0], [2, 0, 0], [0.49, -0.49, 0.3]], np.float32),
                                   mesh, run=oracle_run)
    assert got.tolist() == [True, False, True]
    assert rs.inside_closed_surface(np.zeros((0, 3), np.float32), mesh, run=oracle_run).shape == (0,)


def test_parity_targets_outside_and_deterministic():
    mesh = icosphere(1)
    t1, t2 = rs.parity_targets(mesh, 100, seed=3), rs.parity_targets(mesh, 100, seed=3)
    assert np.array_equal(t1, t2)
    assert (t1 > mesh.vertices.max(axis=0)).all()
    assert not np.array_equal(t1, rs.parity_targets(mesh, 100, seed=4))


@pytest.mark.gpu
@pytest.mark.parametrize("device", [False, True], ids=["host", "device"])
@pytest.mark.parametrize("make", [cube, icosphere], ids=["cube", "icosphere"])
def test_parity_engine(make, device):
    import torch

    mesh = make()
    pts, want = sample_points(mesh, 20000, 11)
    if device:
        dmesh = rs.Mesh.from_arrays(torch.from_numpy(mesh.vertices).cuda(),
                                    torch.from_numpy(mesh.triangles).cuda())
        got = rs.inside_closed_surface(torch.from_numpy(pts).cuda(), dmesh).cpu().numpy()
    else:
        got = rs.inside_closed_surface(pts, mesh)
    assert np.array_equal(got, want)
    ref = rs.inside_closed_surface(pts[:2000], mesh, run=oracle_run)
    assert np.array_equal(got[:2000], ref)
