"""Where the C2 end-to-end call's time goes (diagnostics, run on the box).

    python tools/e2e_probe.py > profiles/round2/e2e_probe.json

Times, on pinned host buffers: a bare 240 MB H2D copy, a bare 40 MB D2H
copy, both at once on two streams (the PCIe floor of the e2e path), and
`run_batch` (boolean, C2) end to end with several `chunk_rays` settings
(0 = the engine's automatic 8 chunks + split tail).  Median of 5 each.
"""
from __future__ import annotations

import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2209_02878_b200 as rs  # noqa: E402


def pinned(a: np.ndarray) -> np.ndarray:
    t = torch.empty(a.shape, dtype=torch.from_numpy(a[:1]).dtype, pin_memory=True)
    t.numpy()[...] = a
    return t.numpy()


def med(f, reps=5):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    return round(float(np.median(ts)), 3)


def main():
    n = 10_000_000
    sc = rs.generate_scene(29_284, n, 0.5, seed=2022)
    s, e = pinned(sc.segments.starts), pinned(sc.segments.ends)
    mesh = rs.Mesh.from_arrays(pinned(sc.mesh.vertices), pinned(sc.mesh.triangles))
    segs = rs.SegmentBatch.from_arrays(s, e)
    out = {"n_rays": n, "h2d_bytes": 24 * n, "d2h_bytes": 4 * n}
    hs, he = torch.from_numpy(s), torch.from_numpy(e)
    ds, de = torch.empty_like(hs, device="cuda"), torch.empty_like(he, device="cuda")
    dflag = torch.zeros(n, dtype=torch.int32, device="cuda")
    hflag = torch.empty(n, dtype=torch.int32, pin_memory=True)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def h2d():
        with torch.cuda.stream(s1):
            ds.copy_(hs, non_blocking=True)
            de.copy_(he, non_blocking=True)
        s1.synchronize()

    def d2h():
        with torch.cuda.stream(s2):
            hflag.copy_(dflag, non_blocking=True)
        s2.synchronize()

    def both():
        with torch.cuda.stream(s1):
            ds.copy_(hs, non_blocking=True)
            de.copy_(he, non_blocking=True)
        with torch.cuda.stream(s2):
            hflag.copy_(dflag, non_blocking=True)
        s1.synchronize()
        s2.synchronize()

    for f in (h2d, d2h, both):
        f()
    out["h2d_ms"] = med(h2d)
    out["d2h_ms"] = med(d2h)
    out["h2d_plus_d2h_concurrent_ms"] = med(both)
    out["h2d_gbps"] = round(24 * n / out["h2d_ms"] / 1e6, 1)
    runs = {}
    for parts in (0, 4, 8, 12, 16, 24, 32):
        cfg = rs.EngineConfig(mode="boolean", chunk_rays=0 if parts == 0 else (n + parts - 1) // parts)
        r = rs.run_batch(mesh, segs, cfg)
        assert np.array_equal(r.crossing, sc.expected_crossings.astype(np.int32))
        runs[str(parts)] = med(lambda: rs.run_batch(mesh, segs, cfg))
    out["run_batch_ms_by_parts"] = runs
    print(json.dumps(out))


if __name__ == "__main__":
    main()
