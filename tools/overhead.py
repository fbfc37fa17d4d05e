"""Per-call host overhead of the device-resident run_batch: wall time per
call vs the GPU's busy time, for a tiny scene (GPU time ~0) and for C2.

    python tools/overhead.py [c2]
"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2209_02878_b200 as rs  # noqa: E402
from paper_2209_02878_b200 import _lib  # noqa: E402
from paper_2209_02878_b200.engine import EngineConfig, run_device  # noqa: E402


def measure(mesh_d, seg_d, n, label, reps=200):
    cfg = EngineConfig(mode="boolean")
    out = {"flags": torch.empty(n, dtype=torch.int32, device="cuda")}
    for _ in range(5):
        run_device(mesh_d, seg_d, cfg, "fast", out=out)
    torch.cuda.synchronize()
    lib = _lib.lib()
    # wall per call
    t0 = time.perf_counter()
    for _ in range(reps):
        run_device(mesh_d, seg_d, cfg, "fast", out=out)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / reps * 1e6
    # the C call alone (pointers prepared once)
    args = (rs.engine._ptr(mesh_d.vertices), mesh_d.num_vertices, rs.engine._ptr(mesh_d.triangles),
            mesh_d.num_triangles, rs.engine._ptr(seg_d.starts), rs.engine._ptr(seg_d.ends), n, 0, 1, 32, 64,
            rs.engine._ptr(out["flags"]), None, None, None, None)
    nh, bad = C.c_int64(0), C.c_int64(-1)
    s = rs.engine._stream()
    t0 = time.perf_counter()
    for _ in range(reps):
        lib.rs_run_batch_device(*args, C.byref(nh), C.byref(bad), s)
    torch.cuda.synchronize()
    capi = (time.perf_counter() - t0) / reps * 1e6
    if not hasattr(lib, "rs_stage_times"):
        print(f"{label}: wall/call {wall:.1f} us, C call {capi:.1f} us")
        return
    # GPU span of one call (trav end from the start mark) via the stage timing
    lib.rs_set_timing(3)
    arr = (C.c_float * 16)()
    rows = []
    for _ in range(12):
        lib.rs_run_batch_device(*args, C.byref(nh), C.byref(bad), s)
        lib.rs_stage_times(arr, 16)
        rows.append([x * 1e3 for x in arr])
    lib.rs_set_timing(0)
    med = [float(np.median([r[k] for r in rows[2:]])) for k in range(16)]
    names = {0: "prep", 1: "sort", 2: "climb", 4: "presets", 5: "sample", 6: "hist", 7: "scan",
             8: "scatter", 14: "trav0", 15: "trav1", 9: "status", 10: "frees", 11: "host launch",
             12: "host wait"}
    print(f"{label}: wall/call {wall:.1f} us, C call {capi:.1f} us; stages (us): " +
          ", ".join(f"{names[k]} {med[k]:.1f}" for k in sorted(names)))


def main():
    torch.cuda.init()
    sc = rs.generate_scene(2000, 20000, 0.5, seed=1)
    mesh_d, seg_d = rs.engine._to_device(sc.mesh, sc.segments)
    measure(mesh_d, seg_d, sc.segments.count, "tiny (2000 tris x 20k segs)", 500)
    if "c2" in sys.argv[1:]:
        sc = bench.make_scene("c2")
        mesh_d, seg_d = rs.engine._to_device(sc.mesh, sc.segments)
        measure(mesh_d, seg_d, sc.segments.count, "c2", 100)


if __name__ == "__main__":
    main()
