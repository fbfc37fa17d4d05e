#!/usr/bin/env python
"""Headline benchmark: Mrays/s of run_batch on N B200s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c2|c3|c4|c5] [--scaling weak|strong] [--no-cpu-baseline]

Configs (BASELINE.json configs[1..4]; configs[0] is a parity-test case):
  c2  boolean, 10M segments x 29,284-tri terrain        (the headline, default)
  c3  barycentric, same inputs
  c4  count, 10M long segments x 7 stacked layers (204,988 tris)
  c5  boolean, 1B segments x 2M-tri terrain, sharded across the ranks; the
      segments are generated on each rank's GPU (rs_generate_segments) --
      24 GB would not come through PCIe from a numpy generator

One step = one full run_batch on device-resident inputs: BVH build over the
mesh (keys, sort, climb) + traversal/exact test of every segment (+ ordered
compaction for barycentric) + status read-back, i.e. exactly what a caller
of `run_batch` gets.  Inputs (240 MB per 10M segments) are larger than L2.

Multi-GPU (torchrun, one rank per GPU, mesh and BVH replicated, segments
sharded by contiguous ranges, no collective on the data path): c2-c4 scale
weakly by default (each rank its own 10M-segment batch; --scaling strong
splits the 10M), c5 strongly (the 1B job is split).  value = all ranks'
segments / max-over-ranks device time.  The result gather to rank 0 (NCCL)
is timed separately after the timed region and reported as "gather".

`--impl reference` times the reference's own CPU implementation (the
reference package's run_batch with its compiled Cython kernel, built from
/root/reference into oracle/_ref by oracle/Makefile) on all host cores, on
the same config, every step the full workload when that fits the time
budget (c2/c3: yes), else a stated prefix sample; rank 0 only.
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
SEED = 2022


class Cfg:
    def __init__(self, name, n_tri, n_rays, mode, layers, scaling, desc, units):
        self.name, self.n_tri, self.n_rays, self.mode = name, n_tri, n_rays, mode
        self.layers, self.scaling, self.desc = layers, scaling, desc
        # SURVEY.md 8(d) algorithmic units per segment (reference-tree counts):
        # B_ray compulsory HBM bytes, W32 FP32 lane-ops (12 x internal
        # visits), W64 FP64 ops (55 x exact tests)
        self.b_ray, self.w32, self.w64 = units


CONFIGS = {
    "c2": Cfg("c2", 29_284, 10_000_000, "boolean", 1, "weak",
              "boolean, 10M segments x 29,284-tri terrain (BASELINE configs[1])", (28, 404, 41)),
    "c3": Cfg("c3", 29_284, 10_000_000, "barycentric", 1, "weak",
              "barycentric, 10M x 29,284 (configs[2])", (36, 404, 55)),
    "c4": Cfg("c4", 29_284, 10_000_000, "count", 7, "weak",
              "count, 10M long segments x 7-layer 204,988 tris (configs[3])", (28, 881, 385)),
    "c5": Cfg("c5", 2_000_000, 1_000_000_000, "boolean", 1, "strong",
              "boolean, 1B segments x 2M-tri terrain, sharded across the GPUs (configs[4])",
              (28, 1939, 41)),
}


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def make_scene(cfg: Cfg, n_rays=None):
    import paper_2209_02878_b200 as rs

    sc = rs.generate_scene(cfg.n_tri, cfg.n_rays if n_rays is None else n_rays, 0.5, seed=SEED)
    if cfg.layers > 1:
        sc = rs.layered_scene(sc, layers=cfg.layers)
    return sc


def peaks():
    """HBM GB/s and FP32/FP64 op rates of this GPU.  HBM from the driver's
    MEASURED_PEAKS.json (burst copy); FP32/FP64 from the SM count x lanes x
    the measured max SM clock (B200: 128 FP32 lanes, 64 FP64 lanes per SM)."""
    p = REPO / "MEASURED_PEAKS.json"
    hbm, mhz, kind = 6650.0, 1965.0, "fallback (B200_PROFILING.md)"
    if p.exists():
        d = json.loads(p.read_text())
        hbm, mhz, kind = float(d["hbm_gbs"]), float(d.get("sm_max_mhz", mhz)), "measured"
    sms = 148
    try:
        import torch

        if torch.cuda.is_available():
            sms = torch.cuda.get_device_properties(0).multi_processor_count
    except Exception:
        pass
    return {"hbm_gbs": hbm, "fp32_tops": sms * 128 * mhz * 1e6 / 1e12,
            "fp64_tops": sms * 64 * mhz * 1e6 / 1e12, "kind": kind, "sms": sms, "mhz": mhz}


def roofline(cfg: Cfg, rays_per_s_kernel: float, rays_per_s_step: float, kernel: str,
             own: dict | None = None):
    """ceiling = min(HBM/B_ray, FP32/W32, FP64/W64); the
    binding resource is the label, `achieved`/`peak` are in its unit for the
    dominant kernel, and every resource's fraction is listed."""
    pk = peaks()
    ceilings = {"hbm": pk["hbm_gbs"] * 1e9 / cfg.b_ray,
                "fp32": pk["fp32_tops"] * 1e12 / cfg.w32,
                "fp64": pk["fp64_tops"] * 1e12 / cfg.w64}
    bound = min(ceilings, key=ceilings.get)
    per_unit = {"hbm": (cfg.b_ray / 1e9, pk["hbm_gbs"], "GB/s"),
                "fp32": (cfg.w32 / 1e12, pk["fp32_tops"], "Tlane-op/s"),
                "fp64": (cfg.w64 / 1e12, pk["fp64_tops"], "Tflop/s")}
    res = {}
    for r, (scale, peak, unit) in per_unit.items():
        a = rays_per_s_kernel * scale
        res[r] = {"achieved": round(a, 3), "peak": round(peak, 1), "unit": unit,
                  "frac": round(a / peak, 4)}
    scale, peak, unit = per_unit[bound]
    traffic = None
    tf = REPO / "profiles" / f"traffic_{cfg.name}.json"
    tinfo = None
    if tf.exists():
        tinfo = json.loads(tf.read_text())
        if tinfo.get("kernel") == kernel:
            traffic = tinfo.get("dram_bytes_per_launch")
    return {
        "bound": bound, "achieved": res[bound]["achieved"], "peak": res[bound]["peak"], "unit": unit,
        "frac": res[bound]["frac"], "traffic": traffic, "kernel": kernel,
        "ceiling_grays": round(ceilings[bound] / 1e9, 2),
        "kernel_grays": round(rays_per_s_kernel / 1e9, 3),
        "step_frac": round(rays_per_s_step / ceilings[bound], 4),
        "resources": res,
        "step_dram_bytes": tinfo.get("step_dram_bytes") if tinfo else None,
        "units": {"B_ray": cfg.b_ray, "W32": cfg.w32, "W64": cfg.w64,
                  "source": "SURVEY.md 8(d), reference-tree visit/test counts"},
        "peaks": pk["kind"] + "; FP32/FP64 = SMs x lanes x max SM clock",
        "traffic_source": tinfo.get("source") if tinfo else None,
        "own_tree": own_tree_roofline(cfg, pk, own["fast"], rays_per_s_kernel) if own else None,
        "reference_tree_units": own_tree_roofline(cfg, pk, own["reference"], rays_per_s_kernel)
        if own else None,
    }


def own_tree_roofline(cfg: Cfg, pk: dict, own: dict, rays_per_s_kernel: float) -> dict:
    """The same ceiling with this engine's own tree's work units (SURVEY
    8(d): "also report own-tree V_int/N_mt"): internal-node visits and exact
    tests per segment of the fast tree's per-segment walk (rs_query_stats on
    a sample), W32 = 12 V_int, W64 = 55 N_mt.  (The tile kernel does not walk
    per segment; these are the per-segment-walk units of the same tree.)"""
    v, m = own["internal_visits"] / own["n"], own["exact_tests"] / own["n"]
    w32, w64 = 12.0 * v, 55.0 * m
    ceil = {"hbm": pk["hbm_gbs"] * 1e9 / cfg.b_ray, "fp32": pk["fp32_tops"] * 1e12 / max(w32, 1e-9),
            "fp64": pk["fp64_tops"] * 1e12 / max(w64, 1e-9)}
    bound = min(ceil, key=ceil.get)
    return {"V_int": round(v, 3), "N_mt": round(m, 3), "W32": round(w32, 1), "W64": round(w64, 1),
            "bound": bound, "ceiling_grays": round(ceil[bound] / 1e9, 2),
            "frac": round(rays_per_s_kernel / ceil[bound], 4), "sample": own["n"]}


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


# --------------------------------------------------------------- reference --

def _ref_runner():
    """run_batch of the reference package itself (oracle/_ref/refpkg: the
    reference's Python sources + its _core.pyx compiled by oracle/Makefile),
    called through its public API; else the restated orchestration over the
    compiled kernel, else the C port."""
    refsrc = REPO / "oracle" / "_ref" / "refpkg" / "src"
    if (refsrc / "raysurf").is_dir():
        sys.path.insert(0, str(refsrc))
        import raysurf

        if "compiled" in raysurf.available_backends():
            def run(V, T, s, e, mode, workers):
                return raysurf.run_batch(raysurf.Mesh.from_arrays(V, T),
                                         raysurf.SegmentBatch.from_arrays(s, e),
                                         raysurf.EngineConfig(mode=mode, workers=workers,
                                                              backend="compiled"))
            return run, "reference", "raysurf.run_batch (reference package, compiled backend)"
    from oracle import ref_engine

    def run(V, T, s, e, mode, workers):
        return ref_engine.run_batch(V, T, s, e, mode, workers=workers)
    return run, ref_engine.kind(), "oracle/ref_engine.py over the reference kernel"


def cpu_inputs(cfg: Cfg, n_max: int, sc=None):
    """Host mesh + the first n_max segments of the config's batch."""
    if cfg.name == "c5":
        from oracle import gen_oracle
        import paper_2209_02878_b200 as rs

        mesh = sc.mesh if sc is not None else rs.generate_scene(cfg.n_tri, 0, 0.5, seed=SEED).mesh
        s, e, _ = gen_oracle.generate_segments(mesh.vertices, mesh.triangles, n_max, seed=SEED)
        return mesh.vertices, mesh.triangles, s, e
    sc = sc or make_scene(cfg)
    return (sc.mesh.vertices, sc.mesh.triangles, sc.segments.starts[:n_max], sc.segments.ends[:n_max])


def cpu_reference(cfg: Cfg, steps: int, warmup: int, budget_s: float, sc=None,
                  sample_cap: int = 10_000_000):
    """Time the reference on this host.  Every step runs the full config's
    batch when (steps + warmup) of them fit `budget_s`; otherwise a prefix of
    min(full, `sample_cap`) segments (c5: a 10M-segment shard of the 1B job,
    rows from the same generator as the GPU arm's), with fewer steps (>= 2)
    when even that overruns.  For a sample, the full config's rate is also
    extrapolated linearly from the reference's own phase timings (fixed
    build phases once + per-segment query cost x the full count).
    Returns (Mrays/s, info)."""
    run, kind, how = _ref_runner()
    workers = os.cpu_count() or 1
    n_full = cfg.n_rays
    probe_n = min(n_full, 1_000_000)
    V, T, s, e = cpu_inputs(cfg, probe_n, sc)
    t0 = time.perf_counter()
    run(V, T, s, e, cfg.mode, workers)
    t_probe = time.perf_counter() - t0
    # the probe's time counted as per-segment cost (its build included):
    # a conservative estimate of a step
    est = lambda k: t_probe * max(1.0, k / probe_n)  # noqa: E731
    n = n_full if est(n_full) * (steps + warmup) <= budget_s else min(n_full, sample_cap)
    if est(n) * (steps + warmup) > budget_s:
        steps = max(2, int(budget_s / est(n)) - warmup)
    if n != probe_n:
        V, T, s, e = cpu_inputs(cfg, n, sc)
    for _ in range(warmup):
        run(V, T, s, e, cfg.mode, workers)
    times, phases = [], []
    for _ in range(steps):
        t0 = time.perf_counter()
        r = run(V, T, s, e, cfg.mode, workers)
        times.append(time.perf_counter() - t0)
        phases.append(getattr(r, "timings", None) or {})
    k = int(np.argmin(times))
    best = times[k]
    info = {"cores": workers, "kind": kind, "n": n, "same_config": n == n_full, "steps": steps,
            "sample": (f"{'all' if n == n_full else 'first'} {n} of the {n_full} segments of config "
                       f"{cfg.name}, full mesh, best of {steps} run_batch calls (workers={workers}; {how})"),
            "ms_per_step": 1e3 * float(np.mean(times)), "ms_best": 1e3 * best,
            "phases_s": {p: round(v, 4) for p, v in phases[k].items()}}
    if n != n_full and "query" in phases[k]:
        per_seg = (phases[k]["query"] + phases[k].get("ray boxes", 0.0)) / n
        fixed = max(0.0, best - per_seg * n)
        info["extrapolated_full_config"] = {
            "value": round(n_full / (fixed + per_seg * n_full) / 1e6, 4), "unit": "Mrays/s",
            "how": f"fixed phases {fixed:.3f} s once + (query + ray boxes) {per_seg * 1e9:.1f} ns/segment "
                   f"x {n_full} segments, from the reference's ResultSet.timings of the best step"}
    try:
        model = [ln for ln in open("/proc/cpuinfo") if ln.startswith("model name")][0].split(":")[1].strip()
        info["cpu"] = model
    except Exception:
        pass
    return n / best / 1e6, info


def config_dict(cfg: Cfg, world: int, scaling: str, n_per_rank: int):
    return {"workload": cfg.desc, "mode": cfg.mode, "n_triangles": cfg.n_tri * cfg.layers,
            "segments_total": n_per_rank * world if scaling == "weak"
            else cfg.n_rays, "segments_per_gpu": n_per_rank,
            "l2": "inputs larger than L2 (24 B/segment)",
            "parallelism": f"segment shards x{world}, mesh/BVH replicated"}


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    value, info = cpu_reference(cfg, args.steps, args.warmup, budget_s=float(os.environ.get(
        "RS_REF_BUDGET_S", "240")))
    scaling = args.scaling or cfg.scaling
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "Mrays/s",
        "n_gpus": args.gpus, "steps": info["steps"], "warmup": args.warmup,
        "ms_per_step": round(info["ms_per_step"], 3), "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "f32 boxes / f64 exact test",
        "data": "synthetic (generate_scene seed 2022)",
        "config": config_dict(cfg, 1, scaling, info["n"]),
        "cpu_baseline": {"value": round(value, 4), "unit": "Mrays/s", "cores": info["cores"],
                         "kind": info["kind"], "sample": info["sample"],
                         "same_config": info["same_config"], "cpu": info.get("cpu"),
                         "phases_s": info["phases_s"],
                         "extrapolated_full_config": info.get("extrapolated_full_config")},
        "e2e": {"value": round(value, 4), "unit": "Mrays/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# -------------------------------------------------------------------- ours --

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--config", default="c2", choices=tuple(CONFIGS))
    ap.add_argument("--scaling", default=None, choices=("weak", "strong"))
    ap.add_argument("--rays", type=int, default=0, help="override the config's total segment count")
    ap.add_argument("--tree", default="auto")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.rays:
        CONFIGS[args.config].n_rays = args.rays
    if args.impl == "reference":
        return run_reference_arm(args)

    import torch
    import torch.distributed as dist

    import paper_2209_02878_b200 as rs
    from paper_2209_02878_b200 import _lib
    from paper_2209_02878_b200.parallel import shard_range

    rank, world, local = dist_env()
    # RS_BENCH_BACKEND=gloo: the multi-rank code path on a single GPU (ranks
    # share device local % device_count; collectives on CPU tensors) -- a
    # test of the N>1 logic, never a scaling measurement
    backend = os.environ.get("RS_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count()) if backend != "nccl" else local
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    cdev = torch.device("cuda", local) if backend == "nccl" else torch.device("cpu")
    cfg = CONFIGS[args.config]
    scaling = args.scaling or cfg.scaling
    mode = cfg.mode
    dev = torch.device("cuda", local)
    generated = cfg.name == "c5"
    sc = None
    if generated:
        mesh_h = rs.generate_scene(cfg.n_tri, 0, 0.5, seed=SEED).mesh
        lo, hi = shard_range(cfg.n_rays, rank, world) if scaling == "strong" else \
            (rank * cfg.n_rays, (rank + 1) * cfg.n_rays)
        mesh_d = rs.Mesh.from_arrays(torch.from_numpy(mesh_h.vertices).to(dev),
                                     torch.from_numpy(mesh_h.triangles).to(dev))
        seg_d, truth_d = rs.scene.generate_segments_device(mesh_d, hi - lo, 0.5, seed=SEED, first=lo,
                                                           device=dev)
    else:
        sc = make_scene(cfg)
        mesh_h, seg_h = sc.mesh, sc.segments
        lo, hi = shard_range(cfg.n_rays, rank, world) if scaling == "strong" else (0, cfg.n_rays)
        mesh_d = rs.Mesh.from_arrays(torch.from_numpy(mesh_h.vertices).to(dev),
                                     torch.from_numpy(mesh_h.triangles).to(dev))
        seg_d = rs.SegmentBatch.from_arrays(torch.from_numpy(seg_h.starts[lo:hi]).to(dev),
                                            torch.from_numpy(seg_h.ends[lo:hi]).to(dev))
        truth_d = torch.from_numpy(sc.expected_crossings[lo:hi]).to(dev)
    n = seg_d.count
    config = rs.EngineConfig(mode=mode, tree=args.tree)
    kind = config.resolved_tree()
    if mode == "barycentric":
        out = {"ray": torch.empty(n, dtype=torch.int32, device=dev),
               "dist": torch.empty(n, dtype=torch.float32, device=dev),
               "tri": torch.empty(n, dtype=torch.int32, device=dev),
               "pt": torch.empty((n, 3), dtype=torch.float32, device=dev)}
    else:
        out = {"flags": torch.empty(n, dtype=torch.int32, device=dev)}
    lib = _lib.lib()
    # timed region: the dominant kernel's CUDA events on every
    # `hot_every`-th step (timing level 2; the event nodes add ~10 us to a
    # step, phase events ~40 us), level 0 on the others; the build/query
    # split comes from a short instrumented pass after the timed region
    timing_level = int(os.environ.get("RS_BENCH_TIMING", "2"))
    hot_every = max(1, int(os.environ.get("RS_BENCH_HOT_EVERY", "10")))
    lib.rs_set_timing(timing_level)

    def step():
        return rs.run_device(mesh_d, seg_d, config, kind, out=out)

    for w in range(args.warmup):  # both graphs (with and without the kernel events) captured
        lib.rs_set_timing(timing_level if w % 2 == 0 else 0)
        res = step()
    # correctness gate on the benchmarked output: generated ground truth
    if not os.environ.get("RS_BENCH_NOCHECK"):  # timing experiments on deliberately wrong builds only
        if mode == "boolean":
            assert torch.equal(res.crossing, truth_d.to(torch.int32))
        elif mode == "count":
            assert torch.equal(res.counts, truth_d.to(torch.int32))
        else:
            assert torch.equal(res.ray_index.to(torch.int64),
                               torch.nonzero(truth_d).flatten())

    hot_ms = []
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
        for i in range(args.steps):
            sampled = timing_level and i % hot_every == 0
            lib.rs_set_timing(timing_level if sampled else 0)
            step()
            if sampled:
                lib.rs_last_timings(C.byref(bms), C.byref(qms), C.byref(hms))
                hot_ms.append(hms.value)
        ev1.record(stream)
        torch.cuda.synchronize()
        t_end = clocks.mark()
        time.sleep(0.05)
    launches = lib.rs_kernel_launches() - launches0
    hot_kernel = lib.rs_hot_kernel().decode()
    # the build/query split and the reference's phase keys: a few extra
    # steps with the phase events on (outside the timed region)
    lib.rs_set_timing(1)
    build_ms, query_ms, phases = [], [], []
    for _ in range(5):
        r = step()
        lib.rs_last_timings(C.byref(bms), C.byref(qms), C.byref(hms))
        build_ms.append(bms.value)
        query_ms.append(qms.value)
        phases.append(r.timings)
        if not timing_level:
            hot_ms.append(hms.value)
    lib.rs_set_timing(0)
    stage_ms = None
    if os.environ.get("RS_BENCH_STAGES"):
        # diagnostics: per-stage marks on both streams (outside the timed
        # region; include/raysurf_b200.h rs_stage_times lists the marks)
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
    t = torch.tensor([elapsed_ms], dtype=torch.float64, device=cdev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    max_ms = float(t.item())
    total_rays = n * world * args.steps
    value = total_rays / (max_ms / 1e3) / 1e6

    # result gather to rank 0 over NCCL (outside the timed region); shards
    # may differ by a row (strong scaling): padded to the longest
    gather = None
    if world > 1 and mode != "barycentric":
        sizes = torch.tensor([n], dtype=torch.int64, device=cdev)
        every = [torch.zeros_like(sizes) for _ in range(world)]
        dist.all_gather(every, sizes)
        m = int(max(int(x.item()) for x in every))
        flat = torch.zeros(m, dtype=torch.int32, device=cdev)
        flat[:n] = out["flags"].to(cdev)
        bufs = [torch.empty_like(flat) for _ in range(world)] if rank == 0 else None
        dist.gather(flat, gather_list=bufs, dst=0)
        dist.barrier()
        torch.cuda.synchronize()
        reps = 5
        g0 = time.perf_counter()
        ev_g0, ev_g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev_g0.record(stream)
        for _ in range(reps):
            dist.gather(flat, gather_list=bufs, dst=0)
        ev_g1.record(stream)
        torch.cuda.synchronize()
        g_ms = ev_g0.elapsed_time(ev_g1) / reps if backend == "nccl" else 1e3 * (time.perf_counter() - g0) / reps
        gt = torch.tensor([g_ms], dtype=torch.float64, device=cdev)
        dist.all_reduce(gt, op=dist.ReduceOp.MAX)
        gather = {"ms": round(float(gt.item()), 4), "bytes_to_rank0": 4 * m * (world - 1),
                  "how": f"dist.gather ({backend}) of every rank's int32 flags to rank 0, timed after "
                         "the timed region, max over ranks"}

    # e2e through the public API with host buffers (pinned, then pageable)
    e2e = None
    if not args.no_e2e:
        if generated:  # a 10M-segment sample of the generated batch, copied to the host
            m = min(n, 10_000_000)
            s_host, e_host = seg_d.starts[:m].cpu().numpy(), seg_d.ends[:m].cpu().numpy()
            e2e_note = f"sample: first {m} of this rank's {n} generated segments"
        else:
            m = n
            s_host, e_host = seg_h.starts[lo:hi], seg_h.ends[lo:hi]
            e2e_note = "the whole per-rank batch"
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
        mesh_p = rs.Mesh.from_arrays(pin(mesh_h.vertices), pin(mesh_h.triangles))
        seg_p = rs.SegmentBatch.from_arrays(pin(s_host), pin(e_host))
        seg_pg = rs.SegmentBatch.from_arrays(np.array(s_host), np.array(e_host))

        def e2e_time(mesh_x, seg_x, reps):
            for _ in range(2):
                r = rs.run_batch(mesh_x, seg_x, config)
            ts = []
            for _ in range(reps):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                r = rs.run_batch(mesh_x, seg_x, config)
                ts.append(time.perf_counter() - t0)
            tt = torch.tensor([float(np.median(ts))], dtype=torch.float64, device=cdev)
            if world > 1:
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            return tt.item(), r

        t_pin, r = e2e_time(mesh_p, seg_p, max(3, min(args.steps // 4, 25)))
        t_pg, _ = e2e_time(mesh_h, seg_pg, 7)
        h2d = 24 * m + 12 * mesh_h.num_vertices + 12 * mesh_h.num_triangles
        # boolean flags cross PCIe packed 32 per word (expanded to the int32
        # result on the host threads); count returns int32 counts
        d2h = (4 * ((m + 31) // 32) if mode == "boolean" else 4 * m) if mode != "barycentric" \
            else 24 * r.num_crossing()
        e2e = {"value": round(m * world / t_pin / 1e6, 3), "unit": "Mrays/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": round(1e3 * t_pin, 3),
               "pageable_value": round(m * world / t_pg / 1e6, 3),
               "pageable_ms_per_step": round(1e3 * t_pg, 3),
               "path": "run_batch(numpy, pinned) -> rs_run_batch_host: chunked H2D/query/D2H "
                       "(boolean flags as bits, expanded to int32 on the host); "
                       "pageable_*: the same call on plain numpy arrays",
               "segments": e2e_note}

    # per-segment work units on a sample (outside the timed region): this
    # engine's fast tree and, as a cross-check of SURVEY 8(d)'s figures, the
    # reference tree with the reference's traversal semantics
    own = None
    try:
        from paper_2209_02878_b200._backend import b200 as _b200

        m = min(n, 1_000_000)
        own = {}
        for kind_, ref_sem in (("fast", False), ("reference", True)):
            tree = _b200.DeviceTree(mesh_d, kind=kind_)
            st = tree.stats(seg_d.starts[:m], seg_d.ends[:m], mode, ref_semantics=ref_sem)
            tree.close()
            own[kind_] = dict(st, n=m)
    except Exception as exc:  # diagnostics only
        print(f"tree stats unavailable: {exc}", file=sys.stderr)
        own = None
    q_ms = float(np.mean(query_ms))
    h_ms = float(np.mean(hot_ms)) if hot_ms and min(hot_ms) > 0 else q_ms
    phase_keys = sorted({k for p in phases for k in p})
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "Mrays/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(max_ms / args.steps, 4),
        "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
        "dtype": "f32 boxes / f64 exact test",
        "data": ("synthetic: generate_scene(2M tris, seed 2022) mesh; segments generated on device "
                 "(rs_generate_segments: the reference generator's distribution, Philox keyed by "
                 "(seed, global row))") if generated else
                "synthetic (generate_scene seed 2022, same generator and draws as the reference)",
        "config": config_dict(cfg, world, scaling, n),
        "tree": kind,
        "phase_ms": {"build": round(float(np.mean(build_ms)), 4), "query": round(q_ms, 4),
                     "traversal_kernel": round(h_ms, 4),
                     "reference_phases": {k: round(1e3 * float(np.mean([p.get(k, 0.0) for p in phases])), 4)
                                          for k in phase_keys},
                     "source": f"traversal_kernel: CUDA events around it on every {hot_every}th step "
                               "of the timed region; the rest: 5 instrumented steps after it"},
        "roofline": roofline(cfg, n / (h_ms / 1e3), value * 1e6 / world, hot_kernel, own),
        "gpu_launches": int(launches),
        "clocks": clocks.summary(t_start, t_end + 0.02),
    }
    if stage_ms is not None:
        line["phase_ms"]["stages"] = stage_ms
    if os.environ.get("RS_DEBUG_STATUS"):
        st = (C.c_ulonglong * 8)()
        lib.rs_last_status(st)
        line["debug_status"] = dict(zip(["bad", "internal", "hits", "tile_counter", "visits", "mts",
                                         "cand_count", "dropped"], [int(x) for x in st]))
    if gather:
        line["gather"] = gather
    if e2e:
        line["e2e"] = e2e
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, info = cpu_reference(cfg, 2, 1, budget_s=30.0, sc=sc if not generated else None)
        line["cpu_baseline"] = {"value": round(v, 4), "unit": "Mrays/s", "cores": info["cores"],
                                "kind": info["kind"], "sample": info["sample"], "cpu": info.get("cpu"),
                                "extrapolated_full_config": info.get("extrapolated_full_config")}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
