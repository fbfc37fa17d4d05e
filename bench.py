#!/usr/bin/env python
"""Headline benchmark: Mrays/s of run_batch (boolean mode, 10M segments x
29,284-triangle terrain = BASELINE.json configs[1]) on N B200s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c2|c3|c4|c5] [--no-cpu-baseline]

One step = one full run_batch on device-resident inputs: BVH build over the
mesh (keys, sort, climb) + traversal/exact test of every segment + status
read-back (TraversalStackOverflow check), exactly what a caller of
`run_batch` gets.  Multi-GPU (torchrun, one rank per GPU): weak scaling, each
rank runs its own full 10M-segment batch against its own replica of the mesh;
no collective on the data path; value = all ranks' segments / max-over-ranks
time.  Rank 0 prints one JSON line.

`--impl reference` times the reference's own CPU implementation
(oracle/ref_engine.py over the reference's compiled _core kernel) on the
host's cores, same config/metric; rank 0 only.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

METRIC = "Mrays/sec (boolean mode, 10M rays x 30k tris) at 1/2/4/8 B200 vs host-CPU ref"
CONFIGS = {
    # name: (n_tri, n_rays, mode, layers, description)
    "c2": (29_284, 10_000_000, "boolean", 1, "boolean, 10M segments x 29,284-tri terrain (BASELINE configs[1])"),
    "c3": (29_284, 10_000_000, "barycentric", 1, "barycentric, 10M x 29,284 (configs[2])"),
    "c4": (29_284, 10_000_000, "count", 7, "count, 10M long segments x 7-layer 204,988 tris (configs[3])"),
    "c5": (2_000_000, 10_000_000, "boolean", 1, "boolean, 10M-segment shard x 2M tris (configs[4] per-GPU shard)"),
}
SEED = 2022


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def make_scene(cfg):
    import paper_2209_02878_b200 as rs

    n_tri, n_rays, _, layers, _ = CONFIGS[cfg]
    sc = rs.generate_scene(n_tri, n_rays, 0.5, seed=SEED)
    if layers > 1:
        sc = rs.layered_scene(sc, layers=layers)
    return sc


def measured_peaks():
    p = REPO / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "10"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append([time.perf_counter()] + parts)

    def wait_ready(self, timeout=5.0):
        t0 = time.perf_counter()
        while self.proc and not self.rows and time.perf_counter() - t0 < timeout:
            time.sleep(0.02)

    def mark(self):
        return time.perf_counter()

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self, t0=None, t1=None):
        rows = [r[1:] for r in self.rows if (t0 is None or r[0] >= t0) and (t1 is None or r[0] <= t1)]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[2 + k] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(rows[-1][1]) if rows[-1][1].isdigit() else None,
                "reasons": reasons, "samples": len(rows)}


def cpu_reference(cfg, steps, warmup, sc=None):
    """Reference CPU run_batch on this host; returns (Mrays/s, info)."""
    from oracle import ref_engine

    sc = sc or make_scene(cfg)
    mode = CONFIGS[cfg][2]
    V, T = sc.mesh.vertices, sc.mesh.triangles
    s, e = sc.segments.starts, sc.segments.ends
    workers = os.cpu_count() or 1
    # bounded sample: keep the whole leg within ~30 s of CPU time
    t0 = time.perf_counter()
    ref_engine.run_batch(V, T, s[:200_000], e[:200_000], mode, workers=workers)
    per_ray = (time.perf_counter() - t0) / 200_000
    n = s.shape[0]
    budget = 30.0 / max(1, steps + warmup)
    if per_ray * n > budget:
        n = max(100_000, int(budget / per_ray))
    s, e = s[:n], e[:n]
    for _ in range(warmup):
        ref_engine.run_batch(V, T, s, e, mode, workers=workers)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        ref_engine.run_batch(V, T, s, e, mode, workers=workers)
        times.append(time.perf_counter() - t0)
    best = min(times)
    info = {"cores": workers, "kind": ref_engine.kind(),
            "sample": f"first {n} of the {CONFIGS[cfg][1]} segments of config {cfg}, "
                      f"full mesh, best of {steps} run_batch calls (workers={workers})",
            "ms_per_step": 1e3 * float(np.mean(times))}
    try:
        model = [l for l in open("/proc/cpuinfo") if l.startswith("model name")][0].split(":")[1].strip()
        info["cpu"] = model
    except Exception:
        pass
    return n / best / 1e6, info


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cfg = args.config
    value, info = cpu_reference(cfg, args.steps, args.warmup)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "Mrays/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(info["ms_per_step"], 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32 boxes / f64 exact test",
        "data": "synthetic (generate_scene seed 2022)",
        "config": {"workload": CONFIGS[cfg][4], "mode": CONFIGS[cfg][2]},
        "cpu_baseline": {"value": round(value, 4), "unit": "Mrays/s", "cores": info["cores"],
                         "kind": info["kind"], "sample": info["sample"]},
        "e2e": {"value": round(value, 4), "unit": "Mrays/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--config", default="c2", choices=tuple(CONFIGS))
    ap.add_argument("--tree", default="auto")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--presort", action="store_true",
                    help="experiment: Morton-order the segments on the host before upload")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch
    import torch.distributed as dist

    import paper_2209_02878_b200 as rs
    from paper_2209_02878_b200 import _lib

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = args.config
    n_tri, n_rays, mode, layers, desc = CONFIGS[cfg]
    sc = make_scene(cfg)
    mesh_h, seg_h = sc.mesh, sc.segments
    if args.presort:
        seg_h, perm = rs.sort_segments_by_morton(seg_h)
        sc.expected_crossings = sc.expected_crossings[perm]
    dev = torch.device("cuda", local)
    mesh_d = rs.Mesh.from_arrays(torch.from_numpy(mesh_h.vertices).to(dev),
                                 torch.from_numpy(mesh_h.triangles).to(dev))
    seg_d = rs.SegmentBatch.from_arrays(torch.from_numpy(seg_h.starts).to(dev),
                                        torch.from_numpy(seg_h.ends).to(dev))
    n = seg_d.count
    config = rs.EngineConfig(mode=mode, tree=args.tree)
    kind = config.resolved_tree()
    out = {}
    if mode == "barycentric":
        out = {"ray": torch.empty(n, dtype=torch.int32, device=dev),
               "dist": torch.empty(n, dtype=torch.float32, device=dev),
               "tri": torch.empty(n, dtype=torch.int32, device=dev),
               "pt": torch.empty((n, 3), dtype=torch.float32, device=dev)}
    else:
        out = {"flags": torch.empty(n, dtype=torch.int32, device=dev)}
    lib = _lib.lib()
    # timed region: only the dominant kernel's CUDA events (phase events cost
    # ~40 us per step); the build/query split comes from a short instrumented
    # pass after the timed region
    timing_level = int(os.environ.get("RS_BENCH_TIMING", "2"))
    lib.rs_set_timing(timing_level)

    def step():
        return rs.run_device(mesh_d, seg_d, config, kind, out=out)

    for _ in range(args.warmup):
        res = step()
    # correctness gate on the benchmarked output: generated ground truth
    truth = sc.expected_crossings
    if os.environ.get("RS_BENCH_NOCHECK"):  # timing experiments on deliberately wrong builds only
        truth = None
    if truth is None:
        pass
    elif mode == "boolean":
        assert np.array_equal(res.crossing.cpu().numpy(), truth.astype(np.int32))
    elif mode == "count":
        assert np.array_equal(res.counts.cpu().numpy(), truth.astype(np.int32))
    else:
        assert np.array_equal(res.ray_index.cpu().numpy(), np.nonzero(truth)[0])

    build_ms, query_ms, hot_ms = [], [], []
    bms, qms, hms = C.c_float(), C.c_float(), C.c_float()
    stream = torch.cuda.current_stream()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = lib.rs_kernel_launches()
    with ClockSampler(local) as clocks:
        clocks.wait_ready()
        t_start = clocks.mark()
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(args.steps):
            step()
            if timing_level:
                lib.rs_last_timings(C.byref(bms), C.byref(qms), C.byref(hms))
                build_ms.append(bms.value)
                query_ms.append(qms.value)
                hot_ms.append(hms.value)
        ev1.record(stream)
        torch.cuda.synchronize()
        t_end = clocks.mark()
        time.sleep(0.05)
    launches = lib.rs_kernel_launches() - launches0
    hot_kernel = lib.rs_hot_kernel().decode()
    if timing_level != 1:
        # the build/query split: a few extra steps with the phase events on
        # (outside the timed region)
        lib.rs_set_timing(1)
        build_ms, query_ms = [], []
        for _ in range(5):
            step()
            lib.rs_last_timings(C.byref(bms), C.byref(qms), C.byref(hms))
            build_ms.append(bms.value)
            query_ms.append(qms.value)
            if not timing_level:
                hot_ms.append(hms.value)
        lib.rs_set_timing(0)
    stage_ms = None
    if os.environ.get("RS_BENCH_STAGES"):
        # diagnostics: per-stage marks on both streams (outside the timed region)
        lib.rs_set_timing(3)
        arr = (C.c_float * 16)()
        rows = []
        for _ in range(7):
            step()
            lib.rs_stage_times(arr, 16)
            rows.append(list(arr))
        lib.rs_set_timing(0)
        stage_ms = [round(float(np.median([r[k] for r in rows[2:]])), 4) for k in range(16)]
    if world > 1:
        dist.barrier()
    elapsed_ms = ev0.elapsed_time(ev1)
    t = torch.tensor([elapsed_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_ms = float(t.item())
    total_rays = n * world * args.steps
    value = total_rays / (max_ms / 1e3) / 1e6

    # e2e through the public API with host (pinned) buffers
    e2e = None
    if not args.no_e2e:
        pin = lambda a: torch.from_numpy(a).pin_memory().numpy()  # noqa: E731
        mesh_p = rs.Mesh.from_arrays(pin(mesh_h.vertices), pin(mesh_h.triangles))
        seg_p = rs.SegmentBatch.from_arrays(pin(seg_h.starts), pin(seg_h.ends))
        if os.environ.get("RS_E2E_CHUNK"):  # pipeline chunk experiments
            import dataclasses
            config = dataclasses.replace(config, chunk_rays=int(os.environ["RS_E2E_CHUNK"]))
        for _ in range(2):
            r = rs.run_batch(mesh_p, seg_p, config)
        ts = []
        for _ in range(max(3, args.steps // 4)):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = rs.run_batch(mesh_p, seg_p, config)
            ts.append(time.perf_counter() - t0)
        e2e_t = torch.tensor([float(np.mean(ts))], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(e2e_t, op=dist.ReduceOp.MAX)
        h2d = 24 * n + 12 * mesh_h.num_vertices + 12 * mesh_h.num_triangles
        d2h = 4 * n if mode != "barycentric" else 24 * r.num_crossing()
        e2e = {"value": round(n * world / e2e_t.item() / 1e6, 3), "unit": "Mrays/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": round(1e3 * e2e_t.item(), 3),
               "path": "run_batch(numpy pinned) -> rs_run_batch_host: chunked H2D/query/D2H"}

    # roofline of the dominant kernel (the traversal): SURVEY 8(d) compulsory
    # bytes per segment x segments per launch / its CUDA-event duration
    b_ray = 24 + (4 if mode != "barycentric" else 24 * 0.5)
    q_ms = float(np.mean(query_ms))
    h_ms = float(np.mean(hot_ms)) if hot_ms and min(hot_ms) > 0 else q_ms
    achieved = b_ray * n / (h_ms / 1e3) / 1e9
    peak, peak_kind = measured_peaks()
    traffic = None
    tf = REPO / "profiles" / f"traffic_{cfg}.json"
    if tf.exists():
        traffic = json.loads(tf.read_text()).get("dram_bytes_per_launch")
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "Mrays/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(max_ms / args.steps, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32 boxes / f64 exact test", "data": "synthetic (generate_scene seed 2022, "
        "same generator and draws as the reference)",
        "config": {"workload": desc, "mode": mode, "n_triangles": mesh_h.num_triangles,
                   "segments_per_gpu": n, "tree": kind, "l2": "inputs (240 MB) larger than L2",
                   "parallelism": f"ray shards x{world}, mesh/BVH replicated"},
        "phase_ms": {"build": round(float(np.mean(build_ms)), 4), "query": round(q_ms, 4),
                     "source": "traversal_kernel: CUDA events in the timed region; build/query: "
                               "5 instrumented steps after it",
                     "traversal_kernel": round(h_ms, 4)},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                     "kernel": hot_kernel, "peak_kind": peak_kind,
                     "algorithmic_bytes_per_segment": b_ray},
        "gpu_launches": int(launches),
        "clocks": clocks.summary(t_start, t_end + 0.02),
    }
    if stage_ms is not None:
        line["phase_ms"]["stages"] = stage_ms
    if e2e:
        line["e2e"] = e2e
    if os.environ.get("RS_DEBUG_STATUS"):
        st = (C.c_ulonglong * 8)()
        lib.rs_last_status(st)
        line["debug_status"] = dict(zip(["bad", "internal", "hits", "tile_counter", "visits", "mts",
                                         "cand_count", "pad"], [int(x) for x in st]))
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, info = cpu_reference(cfg, 2, 1, sc=sc)
        line["cpu_baseline"] = {"value": round(v, 4), "unit": "Mrays/s", "cores": info["cores"],
                                "kind": info["kind"], "sample": info["sample"]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
