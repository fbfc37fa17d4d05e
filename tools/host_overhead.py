"""Host overhead of a device-resident run_batch call (C2): per-call wall of
back-to-back calls through run_device, through a bare ctypes call with
prepared arguments, and the device span of one graph replay."""
import ctypes as C
import sys
import time

sys.path.insert(0, ".")
import numpy as np
import torch

import paper_2209_02878_b200 as rs
from paper_2209_02878_b200 import _lib
from paper_2209_02878_b200.engine import _ptr, _stream

sc = rs.generate_scene(29_284, 10_000_000, 0.5, seed=2022)
d = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
mesh = rs.Mesh.from_arrays(d(sc.mesh.vertices), d(sc.mesh.triangles))
seg = rs.SegmentBatch.from_arrays(d(sc.segments.starts), d(sc.segments.ends))
cfg = rs.EngineConfig(mode="boolean")
out = {"flags": torch.empty(seg.count, dtype=torch.int32, device="cuda")}
lib = _lib.lib()
for lvl in (2, 0):
    lib.rs_set_timing(lvl)
    for _ in range(5):
        rs.run_device(mesh, seg, cfg, "fast", out=out)
    torch.cuda.synchronize()
    n = 200
    t0 = time.perf_counter()
    for _ in range(n):
        rs.run_device(mesh, seg, cfg, "fast", out=out)
    torch.cuda.synchronize()
    print(f"timing level {lvl}: run_device back-to-back {1e3 * (time.perf_counter() - t0) / n:.4f} ms/call")
    args = [_ptr(mesh.vertices), mesh.num_vertices, _ptr(mesh.triangles), mesh.num_triangles,
            _ptr(seg.starts), _ptr(seg.ends), seg.count, 0, 1, 32, 64, _ptr(out["flags"]), None, None,
            None, None]
    nh, bad = C.c_int64(0), C.c_int64(-1)
    s = _stream(0)
    f = lib.rs_run_batch_device
    t0 = time.perf_counter()
    for _ in range(n):
        f(*args, C.byref(nh), C.byref(bad), s)
    torch.cuda.synchronize()
    print(f"timing level {lvl}: bare ctypes back-to-back {1e3 * (time.perf_counter() - t0) / n:.4f} ms/call")
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    f(*args, C.byref(nh), C.byref(bad), s)
    ev1.record()
    torch.cuda.synchronize()
    print(f"timing level {lvl}: one call device span {ev0.elapsed_time(ev1):.4f} ms")
lib.rs_set_timing(3)
arr = (C.c_float * 16)()
for _ in range(5):
    rs.run_device(mesh, seg, cfg, "fast", out=out)
lib.rs_stage_times(arr, 16)
print("host graph launch ms", arr[11], "host wait ms", arr[12])
