"""Multi-process sharding logic (world_size 2, gloo).

On CPU the per-rank compute is the C oracle (no GPU in the build container),
so this exercises exactly the host-side parts of the multi-GPU path: the
contiguous shard split, the gather to rank 0 (or to every rank), the
barycentric ray-index rebasing/concatenation, and the error agreement (one
rank's TraversalStackOverflow / ValidationError raised on every rank with
the batch-global segment index, instead of a hang in the gather).  The GPU
variants run the real CUDA run_batch on each rank (both ranks share one
device here), on numpy inputs and on CUDA-tensor inputs."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2209_02878_b200 as rs
from paper_2209_02878_b200.parallel import run_batch_sharded, shard_range
from golden_io import MODES, assert_result_fields, expected, load

FIELDS = ("crossing", "counts", "ray_index", "distance", "triangle_id", "point")


def _oracle_local(mesh, segs, cfg):
    from oracle import oracle as O

    d = O.run_batch(mesh.vertices, mesh.triangles, segs.starts, segs.ends, mode=cfg.mode)
    return rs.ResultSet(cfg.mode, segs.count, **{k: v for k, v in d.items() if k != "mode"})


def _np(x):
    return x.cpu().numpy() if hasattr(x, "cpu") else np.asarray(x)


def _worker(rank, world, port, name, q, kind, gather):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fx = load(name)
        V, T, s, e = fx["vertices"], fx["triangles"], fx["starts"], fx["ends"]
        if kind == "gpu_device":
            import torch

            V, T, s, e = (torch.from_numpy(a).cuda() for a in (V, T, s, e))
        mesh = rs.Mesh.from_arrays(V, T)
        segs = rs.SegmentBatch.from_arrays(s, e)
        out = {}
        for mode in MODES:
            r = run_batch_sharded(mesh, segs, rs.EngineConfig(mode=mode), gather=gather,
                                  local_run=_oracle_local if kind == "cpu" else None)
            out[mode] = {f: _np(getattr(r, f)) for f in FIELDS if getattr(r, f) is not None}
            out[mode]["num_rays"] = r.num_rays
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def _failing_worker(rank, world, port, q, failing_rank, exc):
    """`failing_rank`'s local run raises `exc`; every rank must raise."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fx = load("scene_s19")
        mesh = rs.Mesh.from_arrays(fx["vertices"], fx["triangles"])
        segs = rs.SegmentBatch.from_arrays(fx["starts"], fx["ends"])

        def local(m, part, cfg):
            if rank == failing_rank or failing_rank < 0:
                if exc == "overflow":
                    raise rs.TraversalStackOverflow("overflow", segment_index=3 + rank)
                raise rs.ValidationError("bad shard")
            return _oracle_local(m, part, cfg)

        try:
            run_batch_sharded(mesh, segs, rs.EngineConfig(), local_run=local)
            q.put((rank, ("ok", None)))
        except rs.TraversalStackOverflow as e:
            q.put((rank, ("overflow", e.segment_index)))
        except rs.ValidationError:
            q.put((rank, ("validation", None)))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _spawn(target, args_of_rank, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port) + args_of_rank(q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_shard_ranges_partition():
    for n in (0, 1, 7, 10_000_001):
        for w in (1, 2, 3, 8):
            r = [shard_range(n, k, w) for k in range(w)]
            assert r[0][0] == 0 and r[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(r, r[1:]))


def _check(res, fx, gather):
    n = fx["starts"].shape[0]
    for rank in (0, 1):
        for mode in MODES:
            got = res[rank][mode]
            if gather == "all" or rank == 0:
                assert got["num_rays"] == n
                assert_result_fields(got, expected(fx, "batch", mode), f"rank {rank} {mode}")
            else:  # rank 1 keeps its own shard (global ray indices)
                lo, hi = shard_range(n, 1, 2)
                want = expected(fx, "batch", mode)
                assert got["num_rays"] == hi - lo
                if mode == "barycentric":
                    keep = (want["ray_index"] >= lo) & (want["ray_index"] < hi)
                    assert np.array_equal(got["ray_index"], want["ray_index"][keep])
                    assert np.array_equal(got["point"], want["point"][keep])
                else:
                    key = "crossing" if mode == "boolean" else "counts"
                    assert np.array_equal(got[key], want[key][lo:hi])


@pytest.mark.parametrize("gather", ["rank0", "all"])
@pytest.mark.parametrize("name", ["scene_s19", "soup_17"])
def test_two_rank_gloo_matches_reference(name, gather):
    res = _spawn(_worker, lambda q: (name, q, "cpu", gather))
    _check(res, load(name), gather)


@pytest.mark.parametrize("failing_rank,exc,want", [
    (1, "overflow", ("overflow", None)),     # rank 1's local index 4 -> global lo + 4
    (-1, "overflow", ("overflow", 3)),       # both ranks: the batch-global minimum (rank 0's 3)
    (0, "validation", ("validation", None)),
])
def test_error_agreement(failing_rank, exc, want):
    res = _spawn(_failing_worker, lambda q: (q, failing_rank, exc))
    n = load("scene_s19")["starts"].shape[0]
    lo1 = shard_range(n, 1, 2)[0]
    for rank in (0, 1):
        kind, idx = res[rank]
        assert kind == want[0], (rank, res)
        if kind == "overflow":
            assert idx == (want[1] if want[1] is not None else lo1 + 4), (rank, res)


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["gpu", "gpu_device"])
@pytest.mark.parametrize("name", ["scene_c1", "soup_20"])
def test_two_rank_sharded_gpu_matches_reference(name, kind):
    """Both ranks run the real CUDA run_batch on their shard (sharing one
    GPU here) on numpy or CUDA-tensor inputs, gather to rank 0 over gloo."""
    res = _spawn(_worker, lambda q: (name, q, kind, "rank0"))
    _check(res, load(name), "rank0")


def _generated_worker(rank, world, port, q):
    """BASELINE configs[4]'s sharding: each rank generates its own contiguous
    shard of one batch on its GPU (rs_generate_segments, keyed by the global
    row), runs it, and the flags are gathered to rank 0."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch

        mesh = rs.generate_scene(20_000, 0, 0.5, seed=2022).mesh
        dmesh = rs.Mesh.from_arrays(torch.from_numpy(mesh.vertices).cuda(),
                                    torch.from_numpy(mesh.triangles).cuda())
        n = 1_000_003
        lo, hi = shard_range(n, rank, world)
        segs, truth = rs.generate_segments_device(dmesh, hi - lo, 0.5, seed=7, first=lo)
        res = rs.run_batch(dmesh, segs, rs.EngineConfig(mode="count"))
        assert torch.equal(res.counts, truth.to(torch.int32))
        local = res.counts.cpu()
        sizes = [shard_range(n, r, world)[1] - shard_range(n, r, world)[0] for r in range(world)]
        pad = torch.zeros(max(sizes), dtype=torch.int32)
        pad[: local.shape[0]] = local
        bufs = [torch.zeros_like(pad) for _ in range(world)] if rank == 0 else None
        dist.gather(pad, gather_list=bufs, dst=0)
        out = torch.cat([b[:k] for b, k in zip(bufs, sizes)]).numpy() if rank == 0 else None
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_generated_shards_gather_to_rank0():
    """Two ranks (one GPU here) each generate and intersect their shard of a
    1M-segment batch; rank 0's gathered counts equal one rank generating the
    whole batch (shard invariance of the generator + sharded run_batch)."""
    import torch

    res = _spawn(_generated_worker, lambda q: (q,))
    mesh = rs.generate_scene(20_000, 0, 0.5, seed=2022).mesh
    dmesh = rs.Mesh.from_arrays(torch.from_numpy(mesh.vertices).cuda(), torch.from_numpy(mesh.triangles).cuda())
    segs, truth = rs.generate_segments_device(dmesh, 1_000_003, 0.5, seed=7)
    whole = rs.run_batch(dmesh, segs, rs.EngineConfig(mode="count")).counts.cpu().numpy()
    assert np.array_equal(res[0], whole)
    assert np.array_equal(whole, truth.cpu().numpy().astype(np.int32))
