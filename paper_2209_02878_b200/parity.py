"""Point-in-closed-surface by odd parity on count mode.

The reference paper's wrapper notes that "the odd parity test may be used to
find ray starting points that lie inside a closed surface" (PAPER.md:84,
SPEC.md:486-500); the reference package itself ships no code for it.  This
is that operation on top of the engine's count mode: one segment per point,
from the point to a target outside the mesh bounds, and the point is inside
iff the segment crosses the surface an odd number of times.

Targets follow SPEC.md:500: the mesh bounds' max corner plus 10% of the
bounds' diagonal on every axis, jittered per point by a fixed seeded offset
(up to another 10% of the diagonal per axis) so that neighbouring points'
segments do not all graze the same edges -- count mode counts a segment
through a shared edge once per triangle, which would flip the
parity.  The mesh must be watertight (caller-asserted).
"""

from __future__ import annotations

import numpy as np

from .engine import MODE_COUNT, EngineConfig, ResultSet, SegmentBatch, run_batch
from .exceptions import ValidationError
from .mesh import Mesh, is_device_array


def parity_targets(mesh: Mesh, n: int, seed: int = 2022, device=None):
    """(n,3) f32 exterior targets: bounds max + 10% diagonal + seeded jitter
    in [0, 10%) of the diagonal per axis."""
    if is_device_array(mesh.vertices):
        import torch

        v = mesh.vertices
        lo, hi = v.amin(dim=0).double().cpu().numpy(), v.amax(dim=0).double().cpu().numpy()
    else:
        v = np.asarray(mesh.vertices, dtype=np.float64)
        lo, hi = v.min(axis=0), v.max(axis=0)
    diag = float(np.linalg.norm(hi - lo)) or 1.0
    base = hi + 0.1 * diag
    jitter = np.random.default_rng(seed).random((n, 3)) * (0.1 * diag)
    tgt = (base[None, :] + jitter).astype(np.float32)
    if device is not None:
        import torch

        return torch.from_numpy(tgt).to(device)
    return tgt


def inside_closed_surface(points, mesh: Mesh, seed: int = 2022, config: EngineConfig | None = None,
                          run=None):
    """Boolean array: points[i] lies inside the closed surface `mesh`.

    `points` (N,3) f32: numpy (numpy result) or a CUDA tensor (CUDA tensor
    result).  `config` may set the tree/limits; its mode is forced to count.
    `run(mesh, segments, config) -> ResultSet` defaults to run_batch (the
    CPU tests substitute the C oracle)."""
    dev = is_device_array(points)
    if dev:
        import torch

        pts = points.to(torch.float32).reshape(-1, 3).contiguous()
        n = pts.shape[0]
        ends = parity_targets(mesh, n, seed, device=pts.device)
    else:
        pts = np.ascontiguousarray(points, dtype=np.float32).reshape(-1, 3)
        n = pts.shape[0]
        ends = parity_targets(mesh, n, seed)
    if n == 0:
        return pts[:0, 0] != 0
    cfg = EngineConfig(mode=MODE_COUNT) if config is None else EngineConfig(
        mode=MODE_COUNT, max_collisions=config.max_collisions, max_stack=config.max_stack,
        tree=config.tree, workers=config.workers, backend=config.backend)
    segs = SegmentBatch.from_arrays(pts, ends)
    res: ResultSet = (run or run_batch)(mesh, segs, cfg)
    counts = res.counts
    if counts is None:
        raise ValidationError("count mode returned no counts")
    return (counts % 2) == 1
