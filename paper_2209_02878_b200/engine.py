"""Batch orchestration: the reference's public engine API on the B200 path.

`run_batch` / `run_baseline_allpairs` keep the reference signatures and
ResultSet semantics (raysurf/engine.py:35-335).  Where the reference fans
segment chunks out to CPU threads (engine.py:160-180), this engine makes one
native call: for host (numpy) inputs `rs_run_batch_host` streams the rays
through the GPU (H2D / build / query / D2H overlapped in C++), for torch CUDA
inputs `rs_run_batch_device` runs build + query + compaction on device.
Nothing here computes intersections on the CPU.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .exceptions import ValidationError
from .mesh import Mesh, is_device_array

MAX_COLLISIONS = 32  # lbvh.py:30-31
MAX_STACK = 64
MODE_BOOLEAN = "boolean"
MODE_BARYCENTRIC = "barycentric"
MODE_COUNT = "count"
MODES = (MODE_BOOLEAN, MODE_BARYCENTRIC, MODE_COUNT)
TREES = ("auto", "fast", "reference")
BACKEND_NAME = "b200"


@dataclass
class SegmentBatch:
    """Paired segment endpoints, (N_r,3) f32 each (engine.py:35-61); numpy
    arrays or torch CUDA tensors."""

    starts: object
    ends: object

    @classmethod
    def from_arrays(cls, starts, ends) -> "SegmentBatch":
        if is_device_array(starts):
            import torch

            s = starts.to(torch.float32).reshape(-1, 3).contiguous()
            e = ends.to(device=s.device, dtype=torch.float32).reshape(-1, 3).contiguous()
        else:
            s = np.ascontiguousarray(starts, dtype=np.float32).reshape(-1, 3)
            e = np.ascontiguousarray(ends, dtype=np.float32).reshape(-1, 3)
        batch = cls(starts=s, ends=e)
        batch.validate()
        return batch

    @property
    def count(self) -> int:
        return int(self.starts.shape[0])

    @property
    def on_device(self) -> bool:
        return is_device_array(self.starts)

    def validate(self) -> None:
        if tuple(self.starts.shape) != tuple(self.ends.shape):
            raise ValidationError(
                f"segment start/end arrays differ in shape: "
                f"{tuple(self.starts.shape)} vs {tuple(self.ends.shape)}")
        if self.on_device:
            import torch

            ok = bool(torch.isfinite(self.starts).all()) and bool(torch.isfinite(self.ends).all())
        else:
            ok = bool(np.isfinite(self.starts).all() and np.isfinite(self.ends).all())
        if not ok:
            raise ValidationError("segment endpoints contain non-finite values")


@dataclass(eq=False)
class ResultSet:
    """Per-mode output (engine.py:64-90).  boolean: `crossing` (N_r,) i32;
    count: `counts` (N_r,) i32; barycentric: `ray_index` ascending with
    `distance`, `triangle_id`, `point` rows.  Arrays are numpy for host
    inputs and torch CUDA tensors for device inputs."""

    mode: str
    num_rays: int
    crossing: object = None
    counts: object = None
    ray_index: object = None
    distance: object = None
    triangle_id: object = None
    point: object = None
    timings: dict = field(default_factory=dict)

    def num_crossing(self) -> int:
        if self.mode == MODE_BOOLEAN:
            return int((self.crossing != 0).sum())
        if self.mode == MODE_COUNT:
            return int((self.counts != 0).sum())
        return int(self.ray_index.shape[0])


@dataclass
class EngineConfig:
    """engine.py:93-112 plus the tree choice.

    tree="auto" builds the isotropic 30-bit "fast" tree (identical results,
    ~3.7x fewer node visits on terrain) unless max_stack is lowered below the
    default, in which case the reference tree is built so the
    TraversalStackOverflow segment index matches the reference exactly.
    `workers` is validated for compatibility; the GPU path ignores it.
    """

    mode: str = MODE_BOOLEAN
    sort_rays: bool = False
    workers: int | None = None
    max_collisions: int = MAX_COLLISIONS
    max_stack: int = MAX_STACK
    backend: str | None = None
    tree: str = "auto"
    chunk_rays: int = 0

    def resolved_workers(self) -> int:
        if self.workers is None:
            return max(1, os.cpu_count() or 1)
        if self.workers < 1:
            raise ValidationError("workerCount must be >= 1")
        return self.workers

    def resolved_tree(self) -> str:
        if self.tree != "auto":
            return self.tree
        return "reference" if self.max_stack < MAX_STACK else "fast"

    def validate(self) -> None:
        if self.mode not in MODES:
            raise ValidationError(f"unknown mode {self.mode!r}")
        self.resolved_workers()
        if self.backend not in (None, BACKEND_NAME):
            raise ValidationError(f"unknown backend {self.backend!r} (have: {BACKEND_NAME})")
        if self.tree not in TREES:
            raise ValidationError(f"unknown tree {self.tree!r} (have: {', '.join(TREES)})")
        if self.max_collisions < 2:  # lbvh.py:92-93
            raise ValidationError("collision buffer needs capacity >= 2")
        if self.max_stack < 1:
            raise ValidationError("traversal stack needs capacity >= 1")


def compute_segment_boxes(segments: SegmentBatch):
    """(N_r,6) f32 segment AABBs [xmin,xmax,ymin,ymax,zmin,zmax]
    (engine.py:115-122), on the device (rs_segment_boxes); kept for API
    parity (the query kernels form the same boxes in registers).  numpy in,
    numpy out; CUDA tensors in, CUDA tensor out."""
    import torch

    host = not segments.on_device
    s = torch.from_numpy(np.ascontiguousarray(segments.starts)).cuda() if host else segments.starts
    e = torch.from_numpy(np.ascontiguousarray(segments.ends)).cuda() if host else segments.ends
    boxes = torch.empty((s.shape[0], 6), dtype=torch.float32, device=s.device)
    _lib.check(_lib.lib().rs_segment_boxes(_ptr(s), _ptr(e), int(s.shape[0]), _ptr(boxes),
                                           _stream(s.device.index)))
    return boxes.cpu().numpy() if host else boxes


def sort_segments_by_morton(segments: SegmentBatch):
    """Z-order of segment midpoints (engine.py:125-147), computed on the GPU
    (rs_sort_segments): returns the permuted batch and perm (perm[k] =
    original index of sorted slot k; int64 numpy for host batches, an int64
    CUDA tensor for device batches)."""
    import torch

    n = segments.count
    if n == 0:
        return segments, np.empty(0, dtype=np.int64)
    host = not segments.on_device
    if host:
        s = torch.from_numpy(np.ascontiguousarray(segments.starts)).cuda()
        e = torch.from_numpy(np.ascontiguousarray(segments.ends)).cuda()
    else:
        s, e = segments.starts, segments.ends
    so, eo = torch.empty_like(s), torch.empty_like(e)
    perm = torch.empty(n, dtype=torch.int64, device=s.device)
    _lib.check(_lib.lib().rs_sort_segments(_ptr(s), _ptr(e), n, _ptr(so), _ptr(eo), _ptr(perm),
                                           _stream()))
    if host:
        return SegmentBatch(so.cpu().numpy(), eo.cpu().numpy()), perm.cpu().numpy()
    return SegmentBatch(so, eo), perm


# --------------------------------------------------------------- internals --

def _ptr(a) -> C.c_void_p:
    if a is None:
        return C.c_void_p(0)
    if isinstance(a, np.ndarray):
        return C.c_void_p(a.ctypes.data)
    return C.c_void_p(a.data_ptr())


def _stream(device_index: int | None = None):
    """The caller's current CUDA stream (raw handle).  The raw getter skips
    building a torch Stream object on every call (~2 us per run_batch)."""
    import torch

    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if raw is not None:
        return raw(torch.cuda.current_device() if device_index is None else device_index)
    return torch.cuda.current_stream().cuda_stream


def _host_empty(shape, dtype):
    """Pinned host array (so D2H runs at full PCIe rate); torch caches the
    pinned blocks across calls."""
    import torch

    tdt = {np.int32: torch.int32, np.float32: torch.float32}[dtype]
    return torch.empty(shape, dtype=tdt, pin_memory=True).numpy()


def _empty_result(mode: str, n: int, like_device=None) -> ResultSet:
    if like_device is not None:
        import torch

        dev = like_device
        z = lambda *s, dt=torch.int32: torch.zeros(*s, dtype=dt, device=dev)  # noqa: E731
        if mode == MODE_BOOLEAN:
            return ResultSet(mode, n, crossing=z(n))
        if mode == MODE_COUNT:
            return ResultSet(mode, n, counts=z(n))
        return ResultSet(mode, n, ray_index=z(0), distance=z(0, dt=torch.float32),
                         triangle_id=z(0), point=z(0, 3, dt=torch.float32))
    if mode == MODE_BOOLEAN:
        return ResultSet(mode, n, crossing=np.zeros(n, np.int32))
    if mode == MODE_COUNT:
        return ResultSet(mode, n, counts=np.zeros(n, np.int32))
    return ResultSet(mode, n, ray_index=np.zeros(0, np.int32), distance=np.zeros(0, np.float32),
                     triangle_id=np.zeros(0, np.int32), point=np.zeros((0, 3), np.float32))


def _unpermute(rs: ResultSet, perm) -> ResultSet:
    """engine.py:191-198: results of Morton-sorted segments back in the
    caller's order, on the device (rs_unpermute_dense / rs_unpermute_rows:
    a scatter for the dense rows, an ordered gather-compaction for the
    barycentric rows).  sort_rays always runs on the device (run_batch moves
    host batches there), so `perm` is an int64 CUDA tensor."""
    if perm is None:
        return rs
    import torch

    n = int(perm.shape[0])
    lib = _lib.lib()
    if rs.mode in (MODE_BOOLEAN, MODE_COUNT):
        key = "crossing" if rs.mode == MODE_BOOLEAN else "counts"
        vals = getattr(rs, key)
        out = torch.empty_like(vals)
        _lib.check(lib.rs_unpermute_dense(_ptr(perm), n, _ptr(vals), _ptr(out), _stream(vals.device.index)))
        setattr(rs, key, out)
        return rs
    k = int(rs.ray_index.shape[0])
    dev = rs.ray_index.device
    o_ray = torch.empty(k, dtype=torch.int32, device=dev)
    o_dist = torch.empty(k, dtype=torch.float32, device=dev)
    o_tri = torch.empty(k, dtype=torch.int32, device=dev)
    o_pt = torch.empty((k, 3), dtype=torch.float32, device=dev)
    _lib.check(lib.rs_unpermute_rows(
        _ptr(perm), n, _ptr(rs.ray_index.contiguous()), _ptr(rs.distance.contiguous()),
        _ptr(rs.triangle_id.contiguous()), _ptr(rs.point.contiguous()), k, _ptr(o_ray), _ptr(o_dist),
        _ptr(o_tri), _ptr(o_pt), _stream(dev.index)))
    rs.ray_index, rs.distance, rs.triangle_id, rs.point = o_ray, o_dist, o_tri, o_pt
    return rs


def _run_host(mesh: Mesh, seg: SegmentBatch, config: EngineConfig, kind: str) -> ResultSet:
    n = seg.count
    mode = config.mode
    flags = ray = dist = tri = pt = None
    if mode == MODE_BARYCENTRIC:
        ray, dist = _host_empty(n, np.int32), _host_empty(n, np.float32)
        tri, pt = _host_empty(n, np.int32), _host_empty((n, 3), np.float32)
    else:
        flags = _host_empty(n, np.int32)
    n_hits, bad = C.c_int64(0), C.c_int64(-1)
    st = _lib.lib().rs_run_batch_host(
        _ptr(mesh.vertices), mesh.num_vertices, _ptr(mesh.triangles), mesh.num_triangles,
        _ptr(seg.starts), _ptr(seg.ends), n, _lib.MODE_TAGS[mode], _lib.TREE_KINDS[kind],
        config.max_collisions, config.max_stack, int(config.chunk_rays),
        _ptr(flags), _ptr(ray), _ptr(dist), _ptr(tri), _ptr(pt), C.byref(n_hits), C.byref(bad),
        _stream())
    _lib.check(st, bad.value, config.max_stack)
    timings = _lib.last_phases()
    if mode == MODE_BOOLEAN:
        return ResultSet(mode, n, crossing=flags, timings=timings)
    if mode == MODE_COUNT:
        return ResultSet(mode, n, counts=flags, timings=timings)
    k = n_hits.value
    return ResultSet(mode, n, ray_index=ray[:k], distance=dist[:k], triangle_id=tri[:k],
                     point=pt[:k], timings=timings)


def run_device(mesh: Mesh, seg: SegmentBatch, config: EngineConfig, kind: str,
               out: dict | None = None) -> ResultSet:
    """Device-resident run_batch: torch CUDA tensors in, torch CUDA tensors
    out, one native call (build + query + compaction).  `out` may supply
    preallocated output tensors (bench.py reuses them across steps)."""
    import torch

    n = seg.count
    mode = config.mode
    dev = seg.starts.device
    out = out or {}
    if mode == MODE_BARYCENTRIC:
        ray = out.get("ray") if out.get("ray") is not None else torch.empty(n, dtype=torch.int32, device=dev)
        dist = out.get("dist") if out.get("dist") is not None else torch.empty(n, dtype=torch.float32, device=dev)
        tri = out.get("tri") if out.get("tri") is not None else torch.empty(n, dtype=torch.int32, device=dev)
        pt = out.get("pt") if out.get("pt") is not None else torch.empty((n, 3), dtype=torch.float32, device=dev)
        flags = None
    else:
        flags = out.get("flags") if out.get("flags") is not None else torch.empty(n, dtype=torch.int32, device=dev)
        ray = dist = tri = pt = None
    n_hits, bad = C.c_int64(0), C.c_int64(-1)
    st = _lib.lib().rs_run_batch_device(
        _ptr(mesh.vertices), mesh.num_vertices, _ptr(mesh.triangles), mesh.num_triangles,
        _ptr(seg.starts), _ptr(seg.ends), n, _lib.MODE_TAGS[mode], _lib.TREE_KINDS[kind],
        config.max_collisions, config.max_stack, _ptr(flags), _ptr(ray), _ptr(dist), _ptr(tri),
        _ptr(pt), C.byref(n_hits), C.byref(bad), _stream(dev.index))
    _lib.check(st, bad.value, config.max_stack)
    timings = _lib.last_phases()
    if mode == MODE_BOOLEAN:
        return ResultSet(mode, n, crossing=flags, timings=timings)
    if mode == MODE_COUNT:
        return ResultSet(mode, n, counts=flags, timings=timings)
    k = n_hits.value
    return ResultSet(mode, n, ray_index=ray[:k], distance=dist[:k], triangle_id=tri[:k], point=pt[:k],
                     timings=timings)


def _to_device(mesh: Mesh, segments: SegmentBatch):
    import torch

    t = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    return (Mesh.from_arrays(t(mesh.vertices), t(mesh.triangles)),
            SegmentBatch(t(segments.starts), t(segments.ends)))


def _to_host(rs: ResultSet) -> ResultSet:
    for f in ("crossing", "counts", "ray_index", "distance", "triangle_id", "point"):
        v = getattr(rs, f)
        if v is not None and is_device_array(v):
            setattr(rs, f, v.cpu().numpy())
    return rs


def run_batch(mesh: Mesh, segments: SegmentBatch, config: EngineConfig | None = None) -> ResultSet:
    """Index the mesh on the GPU and test every segment (engine.py:222-290).

    Results equal the reference's for the same inputs in every mode.  With
    sort_rays, host inputs are moved to the device once: the Morton order,
    the query and the un-permutation all run there."""
    config = config or EngineConfig()
    config.validate()
    n = segments.count
    dev = segments.on_device
    if dev != mesh.on_device and mesh.num_triangles and n:
        raise ValidationError("mesh and segments must both be host arrays or both CUDA tensors")
    if n == 0 or mesh.num_triangles == 0:
        return _empty_result(config.mode, n, segments.starts.device if dev else None)
    if config.sort_rays and not dev:
        return _to_host(run_batch(*_to_device(mesh, segments), config))
    timings = {}
    perm = None
    if config.sort_rays:
        segments, perm, timings["ray sort"] = _timed_sort(segments)
    kind = config.resolved_tree()
    rs = run_device(mesh, segments, config, kind) if dev else _run_host(mesh, segments, config, kind)
    rs.timings.update(timings)
    return _unpermute(rs, perm)


def _timed_sort(segments: SegmentBatch):
    """sort_segments_by_morton with its device time ("ray sort")."""
    import torch

    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    segments, perm = sort_segments_by_morton(segments)
    ev[1].record()
    ev[1].synchronize()
    return segments, perm, ev[0].elapsed_time(ev[1]) / 1e3


def run_baseline_allpairs(mesh: Mesh, segments: SegmentBatch,
                          config: EngineConfig | None = None) -> ResultSet:
    """Every (segment, triangle) pair on the GPU (engine.py:293-335); results
    identical to run_batch."""
    from ._backend import b200

    config = config or EngineConfig()
    config.validate()
    n = segments.count
    dev = segments.on_device
    if n == 0 or mesh.num_triangles == 0:
        return _empty_result(config.mode, n, segments.starts.device if dev else None)
    if not dev:  # compaction and un-permutation run on the device too
        return _to_host(run_baseline_allpairs(*_to_device(mesh, segments), config))
    perm = None
    timings = {}
    if config.sort_rays:
        segments, perm, timings["ray sort"] = _timed_sort(segments)
    if config.mode == MODE_BARYCENTRIC:  # ordered compaction on device (rs_baseline_compact)
        rs = b200.baseline_compact(mesh, segments)
    else:
        rs = _assemble_dense(config.mode, b200.baseline_dense(mesh, segments, config.mode), n, dev)
    timings.update(_lib.last_phases())
    rs.timings = timings
    return _unpermute(rs, perm)


def _assemble_dense(mode: str, out: dict, n: int, dev: bool) -> ResultSet:
    """engine.py:200-215 over dense per-segment rows (boolean / count; the
    barycentric rows come compacted from rs_baseline_compact)."""
    if mode == MODE_BOOLEAN:
        return ResultSet(mode, n, crossing=out["detected"])
    return ResultSet(mode, n, counts=out["counts"])
