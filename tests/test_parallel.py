"""Multi-process sharding logic (world_size 2, gloo, CPU).

The per-rank compute is the C oracle here (no GPU in the build container),
so this exercises exactly the host-side parts of the multi-GPU path: the
contiguous shard split, the variable-length all_gather and the barycentric
ray-index rebasing/concatenation."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2209_02878_b200 as rs
from paper_2209_02878_b200.parallel import run_batch_sharded, shard_range
from golden_io import MODES, assert_result_fields, expected, load


def _oracle_local(mesh, segs, cfg):
    from oracle import oracle as O

    d = O.run_batch(mesh.vertices, mesh.triangles, segs.starts, segs.ends, mode=cfg.mode)
    return rs.ResultSet(cfg.mode, segs.count, **{k: v for k, v in d.items() if k != "mode"})


def _worker(rank, world, port, name, q, gpu=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fx = load(name)
        mesh = rs.Mesh.from_arrays(fx["vertices"], fx["triangles"])
        segs = rs.SegmentBatch.from_arrays(fx["starts"], fx["ends"])
        out = {}
        for mode in MODES:
            r = run_batch_sharded(mesh, segs, rs.EngineConfig(mode=mode),
                                  local_run=None if gpu else _oracle_local)
            out[mode] = {f: np.asarray(getattr(r, f)) for f in
                         ("crossing", "counts", "ray_index", "distance", "triangle_id", "point")
                         if getattr(r, f) is not None}
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_ranges_partition():
    for n in (0, 1, 7, 10_000_001):
        for w in (1, 2, 3, 8):
            r = [shard_range(n, k, w) for k in range(w)]
            assert r[0][0] == 0 and r[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(r, r[1:]))


def _run_two_ranks(name, gpu):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, q, gpu)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("name", ["scene_s19", "soup_17"])
def test_two_rank_gloo_matches_reference(name):
    res = _run_two_ranks(name, gpu=False)
    fx = load(name)
    for rank in (0, 1):
        for mode in MODES:
            assert_result_fields(res[rank][mode], expected(fx, "batch", mode), f"rank {rank} {mode}")


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["scene_c1", "soup_20"])
def test_two_rank_sharded_gpu_matches_reference(name):
    """Both ranks run the real CUDA run_batch on their shard (sharing one
    GPU here), gather over gloo, and every rank holds the reference result."""
    res = _run_two_ranks(name, gpu=True)
    fx = load(name)
    for rank in (0, 1):
        for mode in MODES:
            assert_result_fields(res[rank][mode], expected(fx, "batch", mode), f"gpu rank {rank} {mode}")
