"""End-to-end run_batch time (pinned numpy in/out) vs batch size on C2's
mesh: the slope is the per-segment (PCIe) cost, the intercept the fixed
per-call overhead."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2209_02878_b200 as rs  # noqa: E402

sc = rs.generate_scene(29_284, 10_000_000, 0.5, seed=2022)
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()  # noqa: E731
mesh = rs.Mesh.from_arrays(pin(sc.mesh.vertices), pin(sc.mesh.triangles))
out = {}
for n in (250_000, 1_000_000, 2_500_000, 5_000_000, 10_000_000):
    seg = rs.SegmentBatch.from_arrays(pin(sc.segments.starts[:n]), pin(sc.segments.ends[:n]))
    cfg = rs.EngineConfig(mode="boolean")
    for _ in range(2):
        rs.run_batch(mesh, seg, cfg)
    ts = []
    for _ in range(10):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rs.run_batch(mesh, seg, cfg)
        ts.append(time.perf_counter() - t0)
    out[n] = round(1e3 * float(np.median(ts)), 4)
ns = np.array(list(out), float)
ms = np.array(list(out.values()))
slope, icpt = np.polyfit(ns, ms, 1)
print(json.dumps({"ms": out, "ms_per_10M": round(slope * 1e7, 3), "intercept_ms": round(icpt, 3),
                  "h2d_GBs_implied": round(24e-9 / (slope * 1e-3), 1)}))
