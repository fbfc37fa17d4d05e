"""Two more of the reference's public names, on the device.

- `build_bvh(mesh, sorted_codes, sorted_ids)` (lbvh.py:148-241): the radix
  tree over caller-sorted Morton keys, built on the GPU (rs_build_from_sorted)
  and returned as the reference's `BvhTree` arrays -- bit-identical in all 12
  fields (tests/test_gpu_parity.py tree goldens).
- `oracle_intersect(mesh, segments, mode)` (oracle.py:88-158): the reference's
  independent verification oracle, every (segment, triangle) pair with a
  plane intersection and three edge sign tests in f64 (rs_oracle_intersect),
  a formulation algebraically independent of the engine's Moller-Trumbore.
  It agrees with run_batch except for grazing pairs (the reference's own
  tests compare the two at 1e-4 on distance/point).

The scalar CPU helpers (`traverse`, `find_collisions`, `CollisionBuffer`,
`TraversalStack`, `buffer_insert`) are the reference's per-segment
semantics objects; here that role belongs to the C oracle under oracle/
(test infrastructure), and the product has no CPU traversal.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .engine import (MODE_BARYCENTRIC, MODES, ResultSet, SegmentBatch, _empty_result, _ptr, _stream,
                     _to_device, _to_host)
from .exceptions import ValidationError
from .mesh import MAX_TRIANGLES, Mesh
from .tree import BvhTree


def build_bvh(mesh: Mesh, sorted_codes, sorted_ids) -> BvhTree:
    n = mesh.num_triangles
    if n < 1:
        raise ValidationError("cannot build a BVH over an empty mesh")
    if n > MAX_TRIANGLES:
        raise ValidationError(f"triangle count {n} exceeds capacity {MAX_TRIANGLES}")
    from ._backend import b200

    return b200.DeviceTree(mesh, sorted_codes=sorted_codes, sorted_ids=sorted_ids).download()


def oracle_intersect(mesh: Mesh, segments: SegmentBatch, mode: str = "boolean") -> ResultSet:
    if mode not in MODES:
        raise ValidationError(f"unknown mode {mode!r}")
    n = segments.count
    dev = segments.on_device
    if n == 0 or mesh.num_triangles == 0:
        return _empty_result(mode, n, segments.starts.device if dev else None)
    if not dev:
        return _to_host(oracle_intersect(*_to_device(mesh, segments), mode))
    import torch

    d = segments.starts.device
    k = C.c_int64(0)
    if mode == MODE_BARYCENTRIC:
        ray = torch.empty(n, dtype=torch.int32, device=d)
        dist = torch.empty(n, dtype=torch.float32, device=d)
        tri = torch.empty(n, dtype=torch.int32, device=d)
        pt = torch.empty((n, 3), dtype=torch.float32, device=d)
        flags = None
    else:
        flags = torch.empty(n, dtype=torch.int32, device=d)
        ray = dist = tri = pt = None
    _lib.check(_lib.lib().rs_oracle_intersect(
        _ptr(mesh.vertices), mesh.num_vertices, _ptr(mesh.triangles), mesh.num_triangles,
        _ptr(segments.starts), _ptr(segments.ends), n, _lib.MODE_TAGS[mode], _ptr(flags), _ptr(ray),
        _ptr(dist), _ptr(tri), _ptr(pt), C.byref(k), _stream(d.index)))
    if mode == "boolean":
        return ResultSet(mode, n, crossing=flags)
    if mode == "count":
        return ResultSet(mode, n, counts=flags)
    m = k.value
    return ResultSet(mode, n, ray_index=ray[:m], distance=dist[:m], triangle_id=tri[:m], point=pt[:m])
