"""Traversal statistics on the GPU: node visits / exact tests per segment for
each tree kind (the W32/W64 units of the roofline), plus per-kernel times."""
import json, sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2209_02878_b200 as rs
from paper_2209_02878_b200._backend import b200

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
n_tri = {"c2": 29284, "c5": 2_000_000}[cfg]
sc = rs.generate_scene(n_tri, 10_000_000, 0.5, seed=2022)
s = torch.from_numpy(sc.segments.starts).cuda(); e = torch.from_numpy(sc.segments.ends).cuda()
out = {}
for kind in ("fast", "reference"):
    dt = b200.DeviceTree(sc.mesh, kind=kind)
    info = dt.info()
    st = dt.stats(s, e, "boolean", ref_semantics=(kind == "reference"))
    out[kind] = {"height": info["height"], "visits_per_segment": st["internal_visits"] / s.shape[0],
                 "exact_tests_per_segment": st["exact_tests"] / s.shape[0]}
print(json.dumps(out))
