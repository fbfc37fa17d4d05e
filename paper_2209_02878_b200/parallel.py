"""Segment sharding across GPUs (one process per GPU, torch.distributed).

Every segment is independent, so a batch is split
into contiguous ranges [r*N/W, (r+1)*N/W).  Each rank runs the ordinary
single-GPU run_batch on its range against its own replica of the mesh (a
build takes ~0.15 ms on B200 at 30k triangles, cheaper than shipping a
BVH).  There is no collective on the data path.  Afterwards:

1. one tiny all_gather of (status, global bad-segment index) so that every
   rank agrees on failure: if any shard raised, every rank raises the same
   exception -- TraversalStackOverflow with the batch-global lowest index
   (reference engine.py:179-180 takes the minimum over chunks the same way)
   -- instead of the healthy ranks blocking in the gather;
2. one gather of the result rows to `dst` (default rank 0), or an
   all_gather when gather="all".  Barycentric rows are concatenated in rank
   order, which keeps ray_index ascending (engine.py:206-215).  Over NCCL the
   rows move GPU to GPU (NVLink); over gloo they move as CPU tensors.

Inputs may be numpy arrays (each rank uploads only its own range) or CUDA
tensors (each rank's range is a view, no copy).  Ranks other than the
gather destination return their own shard's ResultSet (ray indices global).
"""

from __future__ import annotations

import numpy as np

from .engine import (MODE_BARYCENTRIC, MODE_BOOLEAN, EngineConfig, ResultSet, SegmentBatch,
                     run_batch)
from .exceptions import TraversalStackOverflow, ValidationError

_FIELDS_BARY = ("ray_index", "distance", "triangle_id", "point")
_ERR_NONE, _ERR_OVERFLOW, _ERR_VALIDATION, _ERR_OTHER = 0, 1, 2, 3


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    return n * rank // world, n * (rank + 1) // world


def _comm_device(dist, group):
    import torch

    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def _as_tensor(x, device):
    import torch

    t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x))
    return t.to(device).contiguous()


def _agree_on_errors(dist, group, device, err: BaseException | None, lo: int) -> None:
    """Every rank learns every rank's outcome; all raise together."""
    import torch

    code, bad = _ERR_NONE, -1
    if isinstance(err, TraversalStackOverflow):
        code = _ERR_OVERFLOW
        bad = lo + int(err.segment_index) if err.segment_index is not None and err.segment_index >= 0 else -1
    elif isinstance(err, ValidationError):
        code = _ERR_VALIDATION
    elif err is not None:
        code = _ERR_OTHER
    mine = torch.tensor([code, bad], dtype=torch.int64, device=device)
    world = dist.get_world_size(group)
    every = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(every, mine, group=group)
    rows = [tuple(int(v) for v in t.cpu().tolist()) for t in every]
    if err is not None:
        if code == _ERR_OVERFLOW:
            overflow = [b for c, b in rows if c == _ERR_OVERFLOW and b >= 0]
            raise TraversalStackOverflow(str(err), segment_index=min(overflow) if overflow else bad) from err
        raise err
    failed = [(r, c, b) for r, (c, b) in enumerate(rows) if c != _ERR_NONE]
    if not failed:
        return
    overflow = [b for _, c, b in failed if c == _ERR_OVERFLOW and b >= 0]
    if overflow and all(c == _ERR_OVERFLOW for _, c, _ in failed):
        raise TraversalStackOverflow("traversal stack overflow on another rank",
                                     segment_index=min(overflow))
    r, c, _ = failed[0]
    if c == _ERR_VALIDATION:
        raise ValidationError(f"rank {r} rejected its shard")
    raise RuntimeError(f"rank {r} failed its shard of run_batch_sharded")


def _gather_rows(dist, group, rows, device, dst: int | None):
    """Gather variable-length row blocks to `dst` (None: to every rank).
    Returns the concatenation on the receiving rank(s), else None."""
    import torch

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    t = _as_tensor(rows, device)
    n = torch.tensor([t.shape[0]], dtype=torch.int64, device=device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    m = max(sizes) if sizes else 0
    if t.shape[0] < m:  # collectives need equal shapes: pad to the longest shard
        pad = torch.zeros((m - t.shape[0],) + tuple(t.shape[1:]), dtype=t.dtype, device=device)
        t = torch.cat([t, pad])
    if dst is None:
        bufs = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(bufs, t, group=group)
    else:
        bufs = [torch.empty_like(t) for _ in range(world)] if rank == dst else None
        dist.gather(t, gather_list=bufs, dst=dst, group=group)
        if rank != dst:
            return None
    return torch.cat([b[:k] for b, k in zip(bufs, sizes)])


def run_batch_sharded(mesh, segments: SegmentBatch, config: EngineConfig | None = None,
                      group=None, local_run=None, gather: str = "rank0", dst: int = 0) -> ResultSet:
    """run_batch over all ranks of `group`, segments sharded by contiguous
    ranges, mesh replicated.

    gather="rank0" (default): rank `dst` returns the whole batch's result,
    the other ranks their own shard's; gather="all": every rank returns the
    whole result.  Results are numpy for numpy inputs, torch tensors (on the
    communication device) for CUDA-tensor inputs.  `local_run(mesh,
    segments, config) -> ResultSet` defaults to the GPU run_batch (the CPU
    tests substitute the C oracle to exercise the sharding, error and gather
    logic without a device)."""
    import torch
    import torch.distributed as dist

    config = config or EngineConfig()
    config.validate()
    if gather not in ("rank0", "all"):
        raise ValidationError(f"unknown gather {gather!r}")
    local_run = local_run or run_batch
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    n = segments.count
    lo, hi = shard_range(n, rank, world)
    on_device = segments.on_device
    if on_device:
        part = SegmentBatch(segments.starts[lo:hi], segments.ends[lo:hi])
    else:
        part = SegmentBatch(np.ascontiguousarray(segments.starts[lo:hi]),
                            np.ascontiguousarray(segments.ends[lo:hi]))
    device = _comm_device(dist, group)
    err, res = None, None
    try:
        res = local_run(mesh, part, config)
    except Exception as e:  # noqa: BLE001 -- re-raised on every rank below
        err = e
    _agree_on_errors(dist, group, device, err, lo)
    to = None if gather == "all" else dst

    def out(t):
        if t is None:
            return None
        return t if on_device else t.cpu().numpy()

    if config.mode == MODE_BARYCENTRIC:
        ri = _as_tensor(res.ray_index, device).to(torch.int64) + lo
        local = ResultSet(config.mode, hi - lo, ray_index=out(ri.to(torch.int32)),
                          distance=res.distance, triangle_id=res.triangle_id, point=res.point,
                          timings=res.timings)
        got = {"ray_index": _gather_rows(dist, group, ri, device, to)}
        for f in _FIELDS_BARY[1:]:
            got[f] = _gather_rows(dist, group, getattr(res, f), device, to)
        if got["ray_index"] is None:
            return local
        got["ray_index"] = got["ray_index"].to(torch.int32)
        got["point"] = got["point"].reshape(-1, 3)
        return ResultSet(config.mode, n, timings=res.timings, **{k: out(v) for k, v in got.items()})
    key = "crossing" if config.mode == MODE_BOOLEAN else "counts"
    flat = _gather_rows(dist, group, getattr(res, key), device, to)
    if flat is None:
        return ResultSet(config.mode, hi - lo, timings=res.timings, **{key: getattr(res, key)})
    return ResultSet(config.mode, n, timings=res.timings, **{key: out(flat.to(torch.int32))})
