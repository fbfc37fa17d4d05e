"""Synthetic terrain scenes with known answers.

`generate_scene` reproduces the reference generator
(raysurf/oracle.py:167-274) draw for draw, so the same seed yields the same
mesh and segments bit for bit (checked against tests/golden/scene_*.npz):
a single-valued height field over an integer grid, half of the segments
vertical through a strictly interior point of a random triangle (ground truth
= exactly one crossing) and the rest entirely above, below or beside the
surface.  `layered_scene` stacks z-shifted copies for the count-mode config
(BASELINE.json configs[3]).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .engine import SegmentBatch
from .exceptions import ValidationError
from .mesh import Mesh

MARGIN = 0.05  # barycentric clearance of constructed crossing points (oracle.py:27)


@dataclass
class SyntheticScene:
    mesh: Mesh
    segments: SegmentBatch
    expected_crossings: np.ndarray  # (N_r,) uint8


def _height_field(nx: int, ny: int, phase: np.ndarray):
    gx, gy = np.meshgrid(np.arange(nx + 1, dtype=np.float64),
                         np.arange(ny + 1, dtype=np.float64), indexing="ij")
    height = (1.5 * np.sin(0.37 * gx + phase[0]) * np.cos(0.23 * gy + phase[1])
              + 0.8 * np.sin(0.11 * gx + 0.19 * gy + phase[2])
              + 0.1 * np.sin(1.7 * gx + phase[3]))
    return np.column_stack([gx.ravel(), gy.ravel(), height.ravel()]).astype(np.float32)


def _grid_triangles(nx: int, ny: int) -> np.ndarray:
    ix, iy = np.meshgrid(np.arange(nx), np.arange(ny), indexing="ij")
    ix, iy = ix.ravel(), iy.ravel()
    stride = ny + 1
    c00 = ix * stride + iy
    c10 = (ix + 1) * stride + iy
    c01 = ix * stride + iy + 1
    c11 = (ix + 1) * stride + iy + 1
    tris = np.empty((2 * nx * ny, 3), dtype=np.int32)
    tris[0::2] = np.column_stack([c00, c10, c11])
    tris[1::2] = np.column_stack([c00, c11, c01])
    return tris


def generate_scene(num_triangles: int, num_rays: int, crossing_fraction: float,
                   seed: int) -> SyntheticScene:
    if not 0.0 <= crossing_fraction <= 1.0:
        raise ValidationError("crossing fraction must be within [0, 1]")
    if num_triangles < 1:
        raise ValidationError("need at least one triangle")
    rng = np.random.default_rng(seed)

    nx = max(1, int(math.ceil(math.sqrt(num_triangles / 2.0))))
    ny = max(1, int(math.ceil(num_triangles / (2.0 * nx))))
    phase = rng.uniform(0.0, 2.0 * np.pi, size=4)
    verts = _height_field(nx, ny, phase)
    mesh = Mesh.from_arrays(verts, _grid_triangles(nx, ny)[:num_triangles])

    z_lo = float(verts[:, 2].min())
    z_hi = float(verts[:, 2].max())
    pad = 0.5 + 0.1 * (z_hi - z_lo)

    flags = np.zeros(num_rays, dtype=np.uint8)
    flags[: int(round(crossing_fraction * num_rays))] = 1
    rng.shuffle(flags)
    p0 = np.zeros((num_rays, 3))
    p1 = np.zeros((num_rays, 3))

    hit_rows = np.nonzero(flags)[0]
    if hit_rows.size:
        m = hit_rows.size
        pick = rng.integers(0, mesh.num_triangles, size=m)
        w = rng.random((m, 2))
        flip = w.sum(axis=1) > 1.0
        w[flip] = 1.0 - w[flip]
        bary = np.column_stack([1.0 - w.sum(axis=1), w[:, 0], w[:, 1]])
        bary = MARGIN + (1.0 - 3.0 * MARGIN) * bary
        corners = mesh.vertices[mesh.triangles[pick]].astype(np.float64)
        xy = np.einsum("kc,kcj->kj", bary, corners)
        low = z_lo - pad * (1.0 + rng.random(m))
        high = z_hi + pad * (1.0 + rng.random(m))
        going_up = rng.random(m) < 0.5
        p0[hit_rows, 0] = p1[hit_rows, 0] = xy[:, 0]
        p0[hit_rows, 1] = p1[hit_rows, 1] = xy[:, 1]
        p0[hit_rows, 2] = np.where(going_up, low, high)
        p1[hit_rows, 2] = np.where(going_up, high, low)

    miss_rows = np.nonzero(flags == 0)[0]
    if miss_rows.size:
        m = miss_rows.size
        where = rng.integers(0, 3, size=m)  # 0 above, 1 below, 2 beside
        x = rng.uniform(-1.0, nx + 1.0, size=(m, 2))
        y = rng.uniform(-1.0, ny + 1.0, size=(m, 2))
        z = np.empty((m, 2))
        up, down, side = where == 0, where == 1, where == 2
        z[up] = z_hi + pad + rng.uniform(0.0, 2.0 * pad, size=(up.sum(), 2))
        z[down] = z_lo - pad - rng.uniform(0.0, 2.0 * pad, size=(down.sum(), 2))
        z[side] = rng.uniform(z_lo - pad, z_hi + pad, size=(side.sum(), 2))
        x[side] = rng.uniform(-6.0, -1.0, size=(side.sum(), 2))
        p0[miss_rows] = np.column_stack([x[:, 0], y[:, 0], z[:, 0]])
        p1[miss_rows] = np.column_stack([x[:, 1], y[:, 1], z[:, 1]])

    return SyntheticScene(mesh=mesh, segments=SegmentBatch.from_arrays(p0, p1),
                          expected_crossings=flags)


def layered_scene(scene: SyntheticScene, layers: int = 7, dz: float = 8.0) -> SyntheticScene:
    """`layers` copies of the surface shifted by dz in z; every crossing
    segment is stretched (direction kept) to span all of them, so its count
    is `layers`; misses stay misses."""
    v = scene.mesh.vertices
    t = scene.mesh.triangles
    verts = np.concatenate([v + np.float32([0.0, 0.0, dz * k]) for k in range(layers)])
    tris = np.concatenate([t + k * v.shape[0] for k in range(layers)])
    s = scene.segments.starts.copy()
    e = scene.segments.ends.copy()
    cross = scene.expected_crossings.astype(bool)
    z_bottom = float(v[:, 2].min()) - 3.0
    z_top = float(v[:, 2].max()) + dz * (layers - 1) + 3.0
    up = e[:, 2] > s[:, 2]
    s[cross, 2] = np.where(up[cross], z_bottom, z_top)
    e[cross, 2] = np.where(up[cross], z_top, z_bottom)
    # misses keep their z: with dz = 8 the highest "above" miss
    # (z_hi + 3 pad) stays below the second layer's lowest vertex
    exp = scene.expected_crossings.astype(np.int32) * layers
    return SyntheticScene(mesh=Mesh.from_arrays(verts, tris),
                          segments=SegmentBatch.from_arrays(s, e), expected_crossings=exp)


def _terrain_extent(vertices) -> tuple[float, float, float, float]:
    """(z_lo, z_hi, x_hi, y_hi) of a generate_scene height field: the f32
    vertex z range (oracle.py:213-214) and the grid extent + 1 that bounds
    the misses' xy draws (oracle.py:256-257)."""
    import torch

    v = vertices if isinstance(vertices, torch.Tensor) else torch.from_numpy(np.asarray(vertices))
    lo = v.amin(dim=0).cpu().numpy()
    hi = v.amax(dim=0).cpu().numpy()
    return float(lo[2]), float(hi[2]), float(hi[0]) + 1.0, float(hi[1]) + 1.0


def generate_segments_device(mesh: Mesh, num_rays: int, crossing_fraction: float = 0.5,
                             seed: int = 2022, first: int = 0, device=None,
                             out: tuple | None = None):
    """Rows [first, first + num_rays) of a synthetic segment batch over a
    generate_scene terrain, generated on the GPU (rs_generate_segments): the
    reference generator's distribution (oracle.py:228-271) from a Philox
    stream keyed by (seed, global row), so every sharding of a batch sees the
    same rows.  Returns (SegmentBatch of CUDA tensors, ground-truth flags u8
    CUDA tensor).  This is how BASELINE configs[4]'s 1B segments are made:
    24 GB that would otherwise cross PCIe from a numpy generator.
    `out` = (starts, ends, flags) preallocated CUDA tensors (flags may be None)."""
    import torch

    from . import _lib

    if not 0.0 <= crossing_fraction <= 1.0:
        raise ValidationError("crossing fraction must be within [0, 1]")
    if num_rays < 0 or first < 0:
        raise ValidationError("num_rays and first must be non-negative")
    device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    dev_v = torch.as_tensor(np.asarray(mesh.vertices) if not isinstance(mesh.vertices, torch.Tensor)
                            else mesh.vertices).to(device).contiguous()
    dev_t = torch.as_tensor(np.asarray(mesh.triangles) if not isinstance(mesh.triangles, torch.Tensor)
                            else mesh.triangles).to(device).contiguous()
    z_lo, z_hi, x_hi, y_hi = _terrain_extent(dev_v)
    if out is None:
        starts = torch.empty((num_rays, 3), dtype=torch.float32, device=device)
        ends = torch.empty((num_rays, 3), dtype=torch.float32, device=device)
        flags = torch.empty(num_rays, dtype=torch.uint8, device=device)
    else:
        starts, ends, flags = out
    stream = torch.cuda.current_stream(device).cuda_stream
    _lib.check(_lib.lib().rs_generate_segments(
        dev_v.data_ptr(), dev_t.data_ptr(), dev_t.shape[0], z_lo, z_hi, x_hi, y_hi,
        float(crossing_fraction), int(seed), int(first), int(num_rays), starts.data_ptr(),
        ends.data_ptr(), flags.data_ptr() if flags is not None else None, stream))
    return SegmentBatch(starts, ends), flags
